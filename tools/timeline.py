#!/usr/bin/env python
"""Device timeline of one certified 100k solve (CUPTI via torch.profiler; no kernel replay):
every kernel / memcpy / memset of our library in start order, with the idle gaps between them.

  python tools/timeline.py [N] > gpurun_out/timeline.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_2011_08170_b200 as f2m  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
xy = f2m.generate_instance(n, 1).points_array()
xyp = torch.from_numpy(xy).pin_memory().numpy()
xo = torch.empty(n * 10 + 1, dtype=torch.float64).pin_memory().numpy()
lo = torch.empty(n, dtype=torch.float64).pin_memory().numpy()


def solve():
    return f2m.full_solve_arrays(xyp, k=10, eps=1e-9, max_sweeps=200000, out_value=xo, out_duals=lo)


for _ in range(3):
    solve()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    r = solve()
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        evs.append((e.time_range.start, e.time_range.end, e.name))
evs.sort()
t0 = evs[0][0]
prev_end = t0
tot_gap = 0.0
by_name = {}
print(f"# n={n} t_total={r['t_total'] * 1e3:.3f} ms knn={r['t_knn'] * 1e3:.3f} duals={r['t_duals'] * 1e3:.3f} "
      f"extract={r['t_extract'] * 1e3:.3f}")
print(f"{'start_us':>10} {'dur_us':>9} {'gap_us':>8}  name")
for s, e, name in evs:
    gap = max(0.0, s - prev_end)
    tot_gap += gap
    by_name.setdefault(name[:70], [0, 0.0])
    by_name[name[:70]][0] += 1
    by_name[name[:70]][1] += e - s
    print(f"{s - t0:10.1f} {e - s:9.1f} {gap:8.1f}  {name[:90]}")
    prev_end = max(prev_end, e)
print(f"# device span {prev_end - t0:.1f} us, idle gaps {tot_gap:.1f} us, {len(evs)} device activities")
big = [e for e in evs if "sweep5" in e[2] or "allpairs_sweep" in e[2] or "gdp_sweep" in e[2]]
if big:
    s0, e0 = big[0][0], big[0][1]
    pre = sum(max(0.0, b[0] - a[1]) for a, b in zip(evs, evs[1:]) if b[0] <= s0)
    post = sum(max(0.0, b[0] - a[1]) for a, b in zip(evs, evs[1:]) if a[1] >= e0)
    print(f"# before sweep: {s0 - t0:.1f} us (idle {pre:.1f}); sweep {e0 - s0:.1f} us; after: {prev_end - e0:.1f} us "
          f"(idle {post:.1f})")
for name, (c, d) in sorted(by_name.items(), key=lambda x: -x[1][1])[:25]:
    print(f"# {d:9.1f} us  x{c:<4d} {name}")
