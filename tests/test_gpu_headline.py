"""GPU parity at the BASELINE headline configurations (BASELINE.json configs[2..3], the 200k
uniform instance the metric names, and acceptance c7).

Every fixture here is the unmodified reference's own full_solve (solve.cpp:101-106) at full size,
threads=1 (tests/golden/make_golden.py; the reference needed 263 s / 153 s / 1,553 s / 617 s of CPU
time to produce them). The GPU result must equal it bit for bit: sweep count, restarts, objective,
duality gap, SHA-256 of the edge values x and of the multipliers.
"""
import numpy as np
import pytest

from conftest import golden, sha

pytestmark = pytest.mark.gpu

HEADLINE = ["u100k_s1", "c7_u100k_s31337_eps1e-8", "u200k_s1", "clust200k_s1"]


def _instance(f2m, meta):
    a = meta["args"]
    if "--clustered" in a:
        i = a.index("--clustered")
        return f2m.generate_clustered_instance(int(a[i + 1]), int(a[i + 2]))
    i = a.index("--synthetic")
    return f2m.generate_instance(int(a[i + 1]), int(a[i + 2]), float(a[i + 3]))


def _kw(meta):
    a = meta["args"]
    return dict(k=int(a[a.index("--k") + 1]), eps=meta["eps"], max_sweeps=meta["max_sweeps"],
                seed=int(a[a.index("--seed") + 1]) if "--seed" in a else 0)


def _check(r, meta):
    assert r["restarts"] == meta["full_restarts"]
    assert r["sweeps"] == meta["full_sweeps"]
    assert r["objective"] == meta["full_objective"]
    assert r["gap"] == meta["full_gap"]
    assert bool(r["feasible"]) == bool(meta["full_feasible"])
    assert sha(np.asarray(r["value"])) == meta["sha256"]["x_full"]
    assert sha(np.asarray(r["duals"])) == meta["sha256"]["lam_full"]


@pytest.mark.parametrize("name", HEADLINE)
def test_headline_full_solve_bit_exact(f2m, name):
    """full_solve through the reference-named Python entry (bindings.cpp:155-182)."""
    meta, _ = golden(name)
    inst = _instance(f2m, meta)
    r = f2m.full_solve(inst, **_kw(meta))
    _check(r, meta)


@pytest.mark.parametrize("name", HEADLINE)
def test_headline_full_solve_c_abi_bit_exact(f2m, name):
    """The same solve through the C ABI with host buffers (f2m_full_solve: the bench's e2e path)."""
    meta, _ = golden(name)
    inst = _instance(f2m, meta)
    kw = _kw(meta)
    r = f2m.full_solve_arrays(inst.points_array(), k=kw["k"], eps=kw["eps"], max_sweeps=kw["max_sweeps"],
                              seed=kw["seed"])
    _check(r, meta)


@pytest.mark.parametrize("name", HEADLINE)
def test_headline_candidate_lists_bit_exact(f2m, name):
    meta, _ = golden(name)
    g = f2m.build_knn_graph(_instance(f2m, meta), _kw(meta)["k"])
    u, v, c = g.edge_arrays()
    assert g.m == meta["m"]
    assert sha(u) == meta["sha256"]["eu"] and sha(v) == meta["sha256"]["ev"] and sha(c) == meta["sha256"]["ec"]
    assert g.mean_cost() == meta["mean_cost"]


@pytest.mark.parametrize("name", HEADLINE)
def test_headline_solve_duals_bit_exact(f2m, name):
    """solve_duals alone (dual.cpp:210-246): sweeps, final max|delta|, dual value, lambda."""
    meta, _ = golden(name)
    kw = _kw(meta)
    g = f2m.build_knn_graph(_instance(f2m, meta), kw["k"])
    st, rep = f2m.solve_duals(g, eps=kw["eps"], max_sweeps=kw["max_sweeps"])
    assert rep["converged"] and rep["sweeps"] == meta["sweeps"]
    assert rep["final_max_abs_delta"] == meta["final_max_abs_delta"]
    assert rep["dual_value"] == meta["dual_value"]
    assert sha(np.asarray(st.lam)) == meta["sha256"]["lam_full"]


@pytest.mark.parametrize("world", [2, 4])
def test_clustered_200k_resident_ranks_bit_exact(world):
    """BASELINE configs[3] (clustered 200k) through the partition-resident multi-rank engine with
    in-process ranks: identical sweeps and multipliers to the reference's converged lambda."""
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_resident

    meta, _ = golden("clust200k_s1")
    inst = _instance(f2m, meta)
    lam, rep = solve_duals_resident(inst, 10, LocalComm(world), eps=meta["eps"], max_sweeps=meta["max_sweeps"])
    assert rep["converged"] and rep["sweeps"] == meta["sweeps"]
    assert sha(np.asarray(lam)) == meta["sha256"]["lam_full"]
