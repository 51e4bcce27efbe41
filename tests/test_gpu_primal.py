"""GPU parity: extraction + certificate (primal.cpp) and the pipeline (solve.cpp).

x must be identical, the objective bit-identical (sequential sum in edge order), the gap and
feasibility as the reference's; KATs from test_primal.cpp / test_solve.cpp.
"""
import numpy as np
import pytest

from conftest import golden, sha

pytestmark = pytest.mark.gpu


def _graph(f2m, name):
    meta, arrays = golden(name)
    a = meta["args"]
    i = a.index("--synthetic")
    inst = f2m.generate_instance(int(a[i + 1]), int(a[i + 2]), float(a[i + 3]))
    g = f2m.build_knn_graph(inst, int(a[a.index("--k") + 1]))
    return inst, g, meta, arrays


@pytest.mark.parametrize("name", ["u1k_s1", "u1k_s2", "u1k_s3", "u1k_s4", "u1k_s5", "u10k_s1",
                                  "u500_s21_b100_k6"])
def test_extract_and_verify_match_reference(f2m, name):
    inst, g, meta, arrays = _graph(f2m, name)
    st, rep = f2m.solve_duals(g, eps=meta["eps"], init=meta["init"])
    if not meta.get("extract_ok"):
        pytest.skip("reference extraction degenerate for this case")
    tol = max(1e-7, 10 * meta["eps"]) * g.mean_cost()
    sol = f2m.extract_primal(g, st, tol)
    x = np.array(sol.value)
    assert sha(x) == meta["sha256"]["x"]
    assert sol.objective == meta["objective"]
    ver = f2m.verify_solution(g, sol, st)
    assert ver["feasible"] == bool(meta["feasible"])
    assert ver["duality_gap"] == meta["gap"]


@pytest.mark.parametrize("name", ["u1k_s1", "u1k_s2", "u1k_s3", "u1k_s4", "u1k_s5", "u10k_s1",
                                  "u500_s21_b100_k6"])
def test_full_solve_matches_reference(f2m, name):
    inst, g, meta, _ = _graph(f2m, name)
    k = int(meta["args"][meta["args"].index("--k") + 1])
    r = f2m.full_solve(inst, k=k)
    assert r["restarts"] == meta["full_restarts"]
    assert r["sweeps"] == meta["full_sweeps"]
    assert r["objective"] == meta["full_objective"]
    assert r["gap"] == meta["full_gap"]
    assert sha(np.array(r["value"])) == meta["sha256"]["x_full"]
    assert sha(np.array(r["duals"])) == meta["sha256"]["lam_full"]


def test_full_solve_arrays_c_abi(f2m):
    inst, g, meta, _ = _graph(f2m, "u1k_s1")
    r = f2m.full_solve_arrays(inst.points_array(), k=10)
    assert r["objective"] == meta["full_objective"] and r["sweeps"] == meta["full_sweeps"]
    assert sha(r["value"]) == meta["sha256"]["x_full"]
    assert sha(r["duals"]) == meta["sha256"]["lam_full"]


def test_full_solve_arrays_caller_buffers(f2m):
    """Caller-owned (page-locked) result buffers: same bits, written in place, reused."""
    import torch
    inst, g, meta, _ = _graph(f2m, "u1k_s1")
    xb = torch.full((1000 * 10 + 1,), -1.0, dtype=torch.float64).pin_memory().numpy()
    lb = torch.full((1000,), -1.0, dtype=torch.float64).pin_memory().numpy()
    for _ in range(2):
        r = f2m.full_solve_arrays(inst.points_array(), k=10, out_value=xb, out_duals=lb)
        assert r["objective"] == meta["full_objective"]
        assert sha(r["value"]) == meta["sha256"]["x_full"]
        assert sha(r["duals"]) == meta["sha256"]["lam_full"]
        assert np.shares_memory(r["value"], xb) and np.shares_memory(r["duals"], lb)


def _sq(f2m):
    return f2m.Instance.from_points(np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float))


def test_classification_unit_square(f2m):
    # test_primal.cpp:36-53
    g = f2m.build_knn_graph(_sq(f2m), 3)
    lab = f2m.classify_edges(g, f2m.DualState([0.5] * 4), 1e-9)
    costs = [c for _, _, c in g.edges()]
    for e, c in enumerate(costs):
        assert (lab[e] == 1) == (c < 1.1)
        if c > 1.1:
            assert lab[e] == 2
    assert (f2m.classify_edges(g, f2m.DualState([0.0] * 4), 1e-9) == 2).all()
    with pytest.raises(ValueError):
        f2m.classify_edges(g, f2m.DualState([0.0] * 4), 0.0)


def test_zero_band_and_monotone_tol(f2m):
    # test_primal.cpp:55-74
    g = f2m.graph_from_edges(2, [0], [1], [1.0])
    assert f2m.classify_edges(g, f2m.DualState([0.5, 0.5 + 1e-12]), 1e-9)[0] == 1
    inst = f2m.generate_instance(40, 5, 10.0)
    g = f2m.build_knn_graph(inst, 5)
    lam = (np.random.default_rng(99).random(40) * 4.0).tolist()
    narrow = f2m.classify_edges(g, f2m.DualState(lam), 1e-6)
    wide = f2m.classify_edges(g, f2m.DualState(lam), 1e-1)
    assert (wide[narrow == 1] == 1).all()


def test_unit_square_extraction(f2m):
    # test_primal.cpp:76-91
    g = f2m.build_knn_graph(_sq(f2m), 3)
    st = f2m.DualState([0.5] * 4)
    sol = f2m.extract_primal(g, st, 1e-9)
    assert sol.objective == pytest.approx(4.0, rel=1e-15)
    for (u, v, c), x in zip(g.edges(), sol.value):
        assert x == (0.0 if c > 1.1 else 1.0)
    ver = f2m.verify_solution(g, sol, st)
    assert ver["feasible"] and ver["duality_gap"] == 0.0
    assert ver["violated_nodes"] == [] and ver["value_violations"] == []


def _prism(f2m):
    u, v, c = [], [], []
    for i in range(5):
        u += [i, 5 + i, i]
        v += [(i + 1) % 5, 5 + (i + 1) % 5, 5 + i]
        c += [2.0, 2.0, 1.9]
    return f2m.graph_from_edges(10, u, v, c)


def test_odd_zero_cycles_half_valued(f2m):
    # test_primal.cpp:93-120
    g = _prism(f2m)
    st = f2m.DualState([1.0] * 10)
    sol = f2m.extract_primal(g, st, 1e-9)
    halves = 0
    for (u, v, c), x in zip(g.edges(), sol.value):
        if c == 1.9:
            assert x == 1.0
        else:
            assert x == 0.5
            halves += 1
    assert halves == 10
    assert f2m.verify_solution(g, sol, st)["feasible"]


def test_c5_zero_component(f2m):
    # test_primal.cpp:122-131
    g = f2m.graph_from_edges(5, [0, 1, 2, 3, 0], [1, 2, 3, 4, 4], [1.0] * 5)
    assert f2m.solve_zero_component(g, [0, 1, 2, 3, 4], [1] * 5) == [0.5] * 5


def test_degenerate_cases(f2m):
    # test_primal.cpp:133-166
    g = f2m.graph_from_edges(25, list(range(25)), [(i + 1) % 25 for i in range(25)], [2.0] * 25)
    with pytest.raises(f2m.DegenerateExtraction, match="cap"):
        f2m.extract_primal(g, f2m.DualState([1.0] * 25), 1e-9)
    g = f2m.graph_from_edges(4, [0, 0, 0, 1, 1, 2], [1, 2, 3, 2, 3, 3], [1, 1, 1, 5, 5, 5])
    with pytest.raises(f2m.DegenerateExtraction, match="tight edges"):
        f2m.extract_primal(g, f2m.DualState([5.0, 0, 0, 0]), 1e-9)
    g = f2m.graph_from_edges(2, [0], [1], [1.0])
    with pytest.raises(f2m.DegenerateExtraction, match="no zero-band edge"):
        f2m.extract_primal(g, f2m.DualState([0.0, 0.0]), 1e-9)
    g = f2m.graph_from_edges(5, [0, 1, 2, 3, 1, 3], [1, 2, 3, 0, 4, 4], [2, 2, 2, 2, 1.9, 1.9])
    with pytest.raises(f2m.DegenerateExtraction, match="no feasible"):
        f2m.extract_primal(g, f2m.DualState([1.0] * 5), 1e-9)


def test_verification_reports_violations(f2m):
    # test_primal.cpp:168-194
    g = f2m.build_knn_graph(_sq(f2m), 3)
    st = f2m.DualState([0.5] * 4)
    sol = f2m.extract_primal(g, st, 1e-9)
    assert f2m.write_solution(g, sol, st).count("\n") == 5
    assert "objective 4 gap 0" in f2m.write_solution(g, sol, st)


@pytest.mark.parametrize("seed", range(0, 50, 7))
def test_small_complete_graphs_vs_brute_force(f2m, seed):
    # test_solve.cpp:24-43 / acceptance criterion 1
    n = 6 + seed % 5
    inst = f2m.generate_instance(n, seed, 100.0)
    r = f2m.full_solve(inst, k=n - 1, seed=seed)
    opt = f2m.brute_force_f2m(f2m.build_knn_graph(inst, n - 1), 45)["optimum"]
    assert r["feasible"]
    assert abs(r["objective"] - opt) <= 1e-6 * (1 + abs(opt))
    assert set(r["value"]) <= {0.0, 0.5, 1.0}


def test_small_complete_graphs_vs_reference(f2m, ref):
    for seed in range(40):
        n = 6 + seed % 5
        ours = f2m.full_solve(f2m.generate_instance(n, seed, 1000.0), k=64, seed=seed)
        theirs = ref.full_solve(ref.generate_instance(n, seed, 1000.0), k=64, seed=seed, threads=1)
        assert ours["objective"] == theirs["objective"]
        assert ours["value"] == theirs["value"]
        assert ours["restarts"] == theirs["restarts"] and ours["sweeps"] == theirs["sweeps"]
        assert ours["duals"] == theirs["duals"]


def test_tied_costs_restart_loop(f2m, ref):
    # test_solve.cpp:45-59: four co-circular points, all rounded costs 1 -> jitter restarts
    pts = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float)
    inst = f2m.Instance.from_points(pts, f2m.DistanceMode.EUC2D_ROUNDED)
    r = f2m.full_solve(inst, k=3)
    assert r["feasible"] and r["objective"] == pytest.approx(4.0, rel=1e-9) and r["restarts"] <= 5
    rinst = ref.parse_tsplib("DIMENSION: 4\nNODE_COORD_SECTION\n1 0 0\n2 1 0\n3 1 1\n4 0 1\nEOF\n")
    theirs = ref.full_solve(rinst, k=3, threads=1)
    assert r["restarts"] == theirs["restarts"] and r["value"] == theirs["value"]
    assert r["objective"] == theirs["objective"] and r["duals"] == theirs["duals"]


def test_coincident_points(f2m):
    # test_solve.cpp:61-70
    inst = f2m.Instance.from_points(np.full((4, 2), 3.0))
    r = f2m.full_solve(inst, k=3)
    assert r["feasible"] and r["objective"] == 0.0


def test_jitter_reproducible_and_single_pass(f2m):
    # test_solve.cpp:72-97
    inst = f2m.generate_instance(8, 3, 100.0)
    a = f2m.full_solve(inst, k=7, seed=17)
    b = f2m.full_solve(inst, k=7, seed=17)
    assert a == b
    inst = f2m.generate_instance(20, 4, 100.0)
    r = f2m.full_solve(inst, k=6, max_restarts=0)
    g = f2m.build_knn_graph(inst, 6)
    st, _ = f2m.solve_duals(g)
    direct = f2m.extract_primal(g, st, 1e-7 * g.mean_cost())
    assert r["value"] == direct.value and r["objective"] == direct.objective


def test_run_config_validation(f2m):
    sq = _sq(f2m)
    with pytest.raises(ValueError):
        f2m.full_solve(sq, k=2)
    with pytest.raises(ValueError):
        f2m.full_solve(sq, k=3, max_restarts=-1)


def test_smoke_surface_like_reference(f2m):
    # reference tests/python/test_smoke.py:34-108 through this package
    text = "NAME : square\nTYPE : TSP\nDIMENSION : 4\nEDGE_WEIGHT_TYPE : EUC_2D\nNODE_COORD_SECTION\n1 0 0\n2 1 0\n3 1 1\n4 0 1\nEOF"
    inst = f2m.parse_tsplib(text)
    inst.mode = f2m.DistanceMode.EUC2D_EXACT
    r = f2m.full_solve(inst, k=3)
    assert r["feasible"] and r["objective"] == pytest.approx(4.0, abs=1e-9) and abs(r["gap"]) <= 1e-9
    assert r["restarts"] == 0 and sorted(set(r["value"])) == [0.0, 1.0]
    inst = f2m.generate_instance(8, seed=3, box=100.0)
    g = f2m.build_knn_graph(inst, k=7)
    assert g.n == 8 and g.m == 28
    oracle = f2m.brute_force_f2m(g, max_edges=28)
    assert f2m.full_solve(inst, k=7)["objective"] == pytest.approx(oracle["optimum"], rel=1e-6)
    g = f2m.build_knn_graph(_sq(f2m), k=3)
    st, conv = f2m.solve_duals(g, mode="gauss-seidel")
    assert conv["converged"] and conv["dual_value"] == pytest.approx(4.0, abs=1e-6)
    sol = f2m.extract_primal(g, st, tol=1e-7 * g.mean_cost())
    v = f2m.verify_solution(g, sol, st)
    assert v["feasible"] and abs(v["duality_gap"]) <= 1e-9


def test_brute_force_oracle_kats(f2m):
    # test_oracle.cpp:60-97 (host enumerator = independent ground truth)
    tri = f2m.Instance.from_points(np.array([[0, 0], [3, 0], [0, 4]], float))
    g = f2m.graph_from_edges(3, [0, 0, 1], [1, 2, 2], [tri.distance(0, 1), tri.distance(0, 2), tri.distance(1, 2)])
    r = f2m.brute_force_f2m(g)
    assert r["optimum"] == pytest.approx(12.0, rel=1e-15) and r["value"] == [1.0, 1.0, 1.0]
    sq = f2m.build_knn_graph(_sq(f2m), 3)
    r = f2m.brute_force_f2m(sq)
    assert r["optimum"] == pytest.approx(4.0, rel=1e-15) and r["enumerated"] >= 1
    k5u, k5v = zip(*[(u, v) for u in range(5) for v in range(u + 1, 5)])
    assert f2m.brute_force_f2m(f2m.graph_from_edges(5, k5u, k5v, [1.0] * 10))["optimum"] == pytest.approx(5.0)
    g7 = f2m.build_knn_graph(f2m.generate_instance(7, 1, 10.0), 6)
    with pytest.raises(f2m.TooLarge):
        f2m.brute_force_f2m(g7)
    assert f2m.brute_force_f2m(g7, 21)["optimum"] > 0.0
    with pytest.raises(f2m.Infeasible):
        f2m.brute_force_f2m(f2m.graph_from_edges(2, [0], [1], [1.0]))
    with pytest.raises(f2m.Infeasible):
        f2m.brute_force_f2m(f2m.graph_from_edges(4, [0, 1, 2], [1, 2, 3], [1.0, 1.0, 1.0]))
