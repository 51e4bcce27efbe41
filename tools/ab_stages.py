"""A/B of the certified solve's stages across package builds (tools/build_variant.sh):
    python tools/ab_stages.py ROOT_A ROOT_B ... [--n 100000] [--reps 15]
Per build (own subprocess): median device times of k-NN + topology, duals, extraction + certificate
and the whole solve (f2m_full_solve_device, points resident in HBM)."""
import argparse
import json
import os
import subprocess
import sys

CHILD = r'''
import sys, json, statistics
sys.path.insert(0, %(root)r)
import torch
import paper_2011_08170_b200 as f2m
n = %(n)d
xy = torch.from_numpy(f2m.generate_instance(n, 1, 1000.0).points_array()).cuda()
dx = torch.empty(n * 10, dtype=torch.float64, device="cuda"); dl = torch.empty(n, dtype=torch.float64, device="cuda")
rs = []
for i in range(%(reps)d + 3):
    r = f2m.full_solve_device(n, xy.data_ptr(), False, 10, 1e-9, 200000, dx.data_ptr(), n * 10, dl.data_ptr())
    if i >= 3: rs.append(r)
med = lambda k: statistics.median(x[k] for x in rs) * 1e3
print(json.dumps({"root": %(root)r, "n": n, "knn_ms": med("t_knn"), "duals_ms": med("t_duals"),
                  "extract_ms": med("t_extract"), "total_ms": med("t_total"), "sweeps": rs[-1]["sweeps"]}))
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("roots", nargs="+")
    ap.add_argument("--n", type=int, default=100000)
    ap.add_argument("--reps", type=int, default=15)
    args = ap.parse_args()
    for r in args.roots:
        code = CHILD % dict(root=os.path.abspath(r), n=args.n, reps=args.reps)
        p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
        print(p.stdout.strip().splitlines()[-1] if p.returncode == 0 else f"{r} FAILED {p.stderr[-800:]}")


if __name__ == "__main__":
    main()
