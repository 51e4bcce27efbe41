"""Probe: the 2M-city instance on one B200 (BASELINE configs[4]).

  * a certified full solve (k-NN -> duals to eps 1e-9 -> extraction -> certificate) on one GPU:
    sweeps, time, objective, gap;
  * the partition the multi-rank resident engine would use at world W (W x (SMs-1) CTAs): is the
    per-CTA footprint still shared-memory resident?

Usage: python tools/probe_2m.py [--n 2000000] [--worlds 2,4,8] [--no-solve]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--worlds", default="2,4,8")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--max-sweeps", type=int, default=1_000_000)
    args = ap.parse_args()
    import torch

    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200 import _f2m

    inst = f2m.generate_instance(args.n, 1, 1000.0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for w in [int(x) for x in args.worlds.split(",") if x]:
        _f2m.set_sweep_partition(w * (sms - 1))
        try:
            g = f2m.build_knn_graph(inst, 10)
        finally:
            _f2m.set_sweep_partition(0)
        infos = [_f2m.sweep_multi_info(g, r, w) for r in range(w)]
        print(json.dumps({"probe": "partition", "n": args.n, "world": w, "g_total": infos[0]["g_total"],
                          "resident": infos[0]["resident"], "kernel_desc_hint": None,
                          "rows_per_rank": [i["end"] - i["begin"] for i in infos]}), flush=True)
        del g
    if not args.no_solve:
        g = f2m.build_knn_graph(inst, 10)
        for eps in (1e-9, 1e-10):
            f2m.solve_duals(g, eps=eps, max_sweeps=args.max_sweeps)  # warm-up
            t0 = time.perf_counter()
            st, rep = f2m.solve_duals(g, eps=eps, max_sweeps=args.max_sweeps)
            wall = time.perf_counter() - t0
            ms, sw = f2m.last_sweep_kernel()
            out = {"probe": "solve_duals", "n": args.n, "m": g.m, "eps": eps, "wall_s": wall,
                   "sweeps": rep["sweeps"], "converged": rep["converged"], "dual_value": rep["dual_value"],
                   "sweep_kernel_ms": ms, "us_per_sweep": 1e3 * ms / max(sw, 1), "kernel": f2m.last_sweep_kernel_desc()}
            for restarts in (5, 20):
                try:
                    t0 = time.perf_counter()
                    r = f2m.full_solve_graph(g, eps=eps, max_sweeps=args.max_sweeps, max_restarts=restarts)
                    out[f"full_r{restarts}"] = {"wall_s": time.perf_counter() - t0, "sweeps": r["sweeps"],
                                                "restarts": r["restarts"], "objective": r["objective"],
                                                "gap": r["gap"], "feasible": bool(r["feasible"])}
                    break
                except Exception as exc:  # noqa: BLE001
                    out[f"full_r{restarts}"] = {"wall_s": time.perf_counter() - t0,
                                                "error": f"{type(exc).__name__}: {exc}"[:300]}
            print(json.dumps(out), flush=True)

if __name__ == "__main__":
    main()
