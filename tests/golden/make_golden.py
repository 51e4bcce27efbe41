"""Generate the committed golden fixtures from the UNMODIFIED reference (oracle/_ref/f2m_dump).

Run here (where /root/reference exists):  python tests/golden/make_golden.py [names...] [--slow]

Each case runs the reference single-threaded through its own C++ API (oracle/ref_dump.cpp) and
stores: scalars (m, mean cost, sweep count, final max|delta|, dual value, objective, gap,
restarts) in <name>.json; SHA-256 digests of every array (edge list, lambda_0, lambda after N
sweeps, converged lambda, x) in the same JSON; and for small cases the arrays themselves in
<name>.npz. The GPU tests compare their outputs bit-for-bit against these (no /root/reference
access at test time).
"""
from __future__ import annotations

import hashlib
import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
DUMP = os.path.join(ROOT, "oracle", "_ref", "f2m_dump")

# name: (dump args, keep_arrays, slow)
CASES = {
    "u1k_s1": (["--synthetic", "1000", "1", "1000", "--k", "10", "--sweeps", "20"], True, False),
    "u1k_s2": (["--synthetic", "1000", "2", "1000", "--k", "10"], False, False),
    "u1k_s3": (["--synthetic", "1000", "3", "1000", "--k", "10"], False, False),
    "u1k_s4": (["--synthetic", "1000", "4", "1000", "--k", "10"], False, False),
    "u1k_s5": (["--synthetic", "1000", "5", "1000", "--k", "10"], False, False),
    # test_dual.cpp:144-161 thread-determinism configuration
    "u500_s21_b100_k6": (["--synthetic", "500", "21", "100", "--k", "6", "--sweeps", "25"], True, False),
    # acceptance criterion 6 (acceptance_main.cpp:199-234): 100 Jacobi sweeps, dual 68422.7
    "c6_u10k_s4242": (["--synthetic", "10000", "4242", "1000", "--k", "10", "--sweeps", "100",
                       "--no-solve"], False, False),
    "u10k_s1": (["--synthetic", "10000", "1", "1000", "--k", "10", "--sweeps", "5"], False, False),
    "u10k_s1_k20_rounded": (["--synthetic", "10000", "1", "1000", "--k", "20", "--rounded",
                             "--sweeps", "10", "--no-solve"], False, False),
    "u2k_s17_b300_k6_zero": (["--synthetic", "2000", "17", "300", "--k", "6", "--init", "zero",
                              "--sweeps", "30"], False, False),
    "u1k_s7_eta03": (["--synthetic", "1000", "7", "1000", "--k", "10", "--eta", "0.3",
                      "--sweeps", "15", "--no-solve"], False, False),
    # acceptance criterion 7 (acceptance_main.cpp:252-265) and the survey's 100k headline
    "c7_u100k_s31337_eps1e-8": (["--synthetic", "100000", "31337", "1000", "--k", "10", "--eps",
                                 "1e-8", "--max-sweeps", "200000", "--seed", "7", "--sweeps", "3"],
                                False, True),
    "u100k_s1": (["--synthetic", "100000", "1", "1000", "--k", "10", "--sweeps", "3"], False, True),
    # config 4 family: clustered instances from paper_2011_08170_b200.generate_clustered_instance
    # (the reference has no clustered generator; points are passed to it exactly)
    "clust20k_s1": (["--clustered", "20000", "1", "--k", "10", "--sweeps", "5"], False, True),
    "u200k_s1": (["--synthetic", "200000", "1", "1000", "--k", "10", "--max-sweeps", "200000",
                  "--full-only"], False, True),
    "clust200k_s1": (["--clustered", "200000", "1", "--k", "10", "--max-sweeps", "200000",
                      "--full-only"], False, True),
}
# bucketed == quadratic scan grid of test_graph.cpp:39-50 (rounded mode = heavy ties)
for _seed in (1, 2, 3):
    for _n in (30, 150, 700):
        for _k in (3, 6, 20):
            for _r in (False, True):
                CASES[f"knn_n{_n}_s{_seed}_k{_k}{'_r' if _r else ''}"] = (
                    ["--synthetic", str(_n), str(_seed), "100", "--k", str(_k), "--no-solve"]
                    + (["--rounded"] if _r else []), True, False)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _expand(args, d):
    """--clustered N SEED -> --points FILE written by the B200 package's host generator."""
    if "--clustered" not in args:
        return args
    i = args.index("--clustered")
    n, seed = int(args[i + 1]), int(args[i + 2])
    sys.path.insert(0, ROOT)
    import paper_2011_08170_b200 as f2m
    pts = f2m.generate_clustered_instance(n, seed).points_array()
    path = os.path.join(d, "in_points.f64")
    pts.astype(np.float64).tofile(path)
    return args[:i] + ["--points", path] + args[i + 3:]


def run_case(name: str, args, keep: bool) -> None:
    with tempfile.TemporaryDirectory() as d:
        subprocess.check_call([DUMP, d] + _expand(args, d))
        meta = json.load(open(os.path.join(d, "meta.json")))
        arrays = {}
        for fn, dt in (("eu.i32", np.int32), ("ev.i32", np.int32), ("ec.f64", np.float64),
                       ("lam0.f64", np.float64), ("lamN.f64", np.float64),
                       ("sweep_stats.f64", np.float64), ("lam_final.f64", np.float64),
                       ("x.f64", np.float64), ("x_full.f64", np.float64),
                       ("lam_full.f64", np.float64), ("points.f64", np.float64)):
            p = os.path.join(d, fn)
            if os.path.exists(p):
                arrays[fn.split(".")[0]] = np.fromfile(p, dtype=dt)
        meta["sha256"] = {k: sha(v) for k, v in arrays.items() if k != "points"}
        meta["sweep_stats"] = arrays["sweep_stats"].reshape(-1, 2).tolist()
        meta["args"] = args
        with open(os.path.join(HERE, name + ".json"), "w") as f:
            json.dump(meta, f, indent=1, sort_keys=True)
        if keep:
            np.savez_compressed(os.path.join(HERE, name + ".npz"),
                                **{k: v for k, v in arrays.items() if k != "points"})
        print(name, "m=", meta["m"], "sweeps=", meta.get("sweeps"), flush=True)


def main(argv):
    slow = "--slow" in argv
    names = [a for a in argv if not a.startswith("--")]
    if not os.path.exists(DUMP):
        subprocess.check_call(["make", "-C", os.path.join(ROOT, "oracle"), "ref"])
    for name, (args, keep, is_slow) in CASES.items():
        if names and name not in names:
            continue
        if is_slow and not slow and not names:
            continue
        run_case(name, args, keep)


if __name__ == "__main__":
    main(sys.argv[1:])
