"""Wall-clock vs device time of the certified 100k solve through the public entry point (the
bench's e2e leg): python tools/e2e_probe.py [N]"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_08170_b200 as f2m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
xy = f2m.generate_instance(n, 1).points_array()
xyp = torch.from_numpy(xy).pin_memory().numpy()
xo = torch.empty(n * 10 + 1, dtype=torch.float64).pin_memory().numpy()
lo = torch.empty(n, dtype=torch.float64).pin_memory().numpy()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for outs in (False, True):
    walls, tots = [], []
    for rep in range(20):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kw = dict(out_value=xo, out_duals=lo) if outs else {}
        r = f2m.full_solve_arrays(xyp, k=10, eps=1e-9, max_sweeps=200000, **kw)
        walls.append(time.perf_counter() - t0)
        tots.append(r["t_total"])
    print(" ".join(f"{w*1e3:.1f}" for w in walls))
    print(f"outs={outs}: wall {statistics.median(walls)*1e3:.3f} ms  t_total {statistics.median(tots)*1e3:.3f} ms "
          f"(knn {r['t_knn']*1e3:.3f} duals {r['t_duals']*1e3:.3f} extract {r['t_extract']*1e3:.3f})", flush=True)
