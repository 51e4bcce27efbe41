"""CPU: pin the C restatement oracle (oracle/f2m_oracle.c) to the reference's golden vectors.

The fixtures were produced by the unmodified reference (tests/golden/make_golden.py over
oracle/_ref). If the oracle reproduces them bit-for-bit it can serve as the checker for the GPU
path on inputs the fixtures do not cover.
"""
import numpy as np
import pytest

from conftest import golden, golden_names, sha


def _xy(orc, args):
    i = args.index("--synthetic")
    return orc.generate_instance(int(args[i + 1]), int(args[i + 2]), float(args[i + 3]))


def _graph(orc, meta):
    a = meta["args"]
    xy = _xy(orc, a)
    n = xy.shape[0]
    k = max(3, min(int(a[a.index("--k") + 1]), n - 1))
    return orc.build_knn_graph(xy, k, "--rounded" in a)


@pytest.mark.parametrize("name", [n for n in golden_names() if n.startswith("knn_")])
def test_oracle_knn_and_scan_match_golden(orc, name):
    meta, arrays = golden(name)
    g = _graph(orc, meta)
    assert g.m == meta["m"]
    assert np.array_equal(g.eu, arrays["eu"]) and np.array_equal(g.ev, arrays["ev"])
    assert np.array_equal(g.cost, arrays["ec"])
    a = meta["args"]
    xy = _xy(orc, a)
    s = orc.knn_graph_scan(xy, max(3, min(int(a[a.index("--k") + 1]), xy.shape[0] - 1)), "--rounded" in a)
    assert np.array_equal(s.eu, g.eu) and np.array_equal(s.ev, g.ev) and np.array_equal(s.cost, g.cost)


CASES = ["u1k_s1", "u500_s21_b100_k6", "c6_u10k_s4242", "u2k_s17_b300_k6_zero", "u1k_s7_eta03",
         "u10k_s1_k20_rounded"]


@pytest.mark.parametrize("name", CASES)
def test_oracle_sweeps_match_golden(orc, name):
    meta, _ = golden(name)
    g = _graph(orc, meta)
    assert sha(g.eu) == meta["sha256"]["eu"] and sha(g.cost) == meta["sha256"]["ec"]
    assert g.mean_cost() == meta["mean_cost"]
    lam = orc.initial_state(g, init=meta["init"])
    assert sha(lam) == meta["sha256"]["lam0"]
    for mx_ref, dv_ref in meta["sweep_stats"]:
        mx, dv = orc.jacobi_sweep(g, lam, eta=meta["eta"])
        assert mx == mx_ref and dv == dv_ref
    assert sha(lam) == meta["sha256"]["lamN"]


def test_c6_dual_value(orc):
    meta, _ = golden("c6_u10k_s4242")
    assert meta["sweep_stats"][-1][1] == 68422.67083340639  # acceptance c6 golden


@pytest.mark.parametrize("name", ["u1k_s1", "u1k_s2", "u1k_s3", "u1k_s4", "u1k_s5", "u500_s21_b100_k6",
                                  "u2k_s17_b300_k6_zero", "u10k_s1"])
def test_oracle_solve_extract_full_match_golden(orc, name):
    meta, _ = golden(name)
    g = _graph(orc, meta)
    lam, rep = orc.solve_duals(g, eps=meta["eps"], init=meta["init"], max_sweeps=meta["max_sweeps"])
    assert rep["sweeps"] == meta["sweeps"] and rep["converged"] == bool(meta["converged"])
    assert rep["final_max_abs_delta"] == meta["final_max_abs_delta"]
    assert rep["dual_value"] == meta["dual_value"]
    assert sha(lam) == meta["sha256"]["lam_final"]
    if meta.get("extract_ok"):
        x, obj = orc.extract_primal(g, lam, max(1e-7, 10 * meta["eps"]) * g.mean_cost())
        assert sha(x) == meta["sha256"]["x"] and obj == meta["objective"]
        v = orc.verify(g, x, obj, lam)
        assert v["feasible"] == bool(meta["feasible"]) and v["gap"] == meta["gap"]
    if meta.get("full_ok") and meta["init"] == "local-midpoint":
        k = int(meta["args"][meta["args"].index("--k") + 1])
        fs = orc.full_solve_graph(g, k=k, eps=meta["eps"])
        assert fs["objective"] == meta["full_objective"] and fs["gap"] == meta["full_gap"]
        assert fs["restarts"] == meta["full_restarts"] and fs["sweeps"] == meta["full_sweeps"]
        assert sha(fs["value"]) == meta["sha256"]["x_full"]
        assert sha(fs["duals"]) == meta["sha256"]["lam_full"]


def test_golden_survey_numbers():
    """The fixtures reproduce the survey's measured reference numbers."""
    meta, _ = golden("u1k_s1")
    assert meta["m"] == 5794 and meta["sweeps"] == 1464
    assert meta["full_objective"] == 21633.006465552298
    meta, _ = golden("u10k_s1")
    assert meta["m"] == 57279 and meta["sweeps"] == 3165
    assert meta["full_objective"] == 68325.385827275997
    meta, _ = golden("c6_u10k_s4242")
    assert meta["m"] == 57093


def test_full_size_fixtures_if_present():
    import os
    from conftest import GOLDEN
    for name, m, sweeps in (("u100k_s1", 568737, 6359), ("c7_u100k_s31337_eps1e-8", 569454, 3751)):
        if not os.path.exists(os.path.join(GOLDEN, name + ".json")):
            pytest.skip(f"{name} fixture not generated")
        meta, _ = golden(name)
        assert meta["m"] == m and meta["sweeps"] == sweeps and meta["full_restarts"] == 0
