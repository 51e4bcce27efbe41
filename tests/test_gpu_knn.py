"""GPU parity: candidate graph (build_knn_graph, graph.cpp:169-240) — bit-exact edge lists.

Predicate = the reference's same_edges (tests/test_support.hpp:55-64): identical (u, v, cost)
sequence. Checked against golden fixtures from the unmodified reference and, for shapes the
fixtures do not cover, against the C restatement oracle (itself pinned to the fixtures).
"""
import numpy as np
import pytest

from conftest import golden, golden_names, sha

pytestmark = pytest.mark.gpu


def _inst(f2m, args):
    i = args.index("--synthetic")
    n, seed, box = int(args[i + 1]), int(args[i + 2]), float(args[i + 3])
    inst = f2m.generate_instance(n, seed, box)
    if "--rounded" in args:
        inst.mode = f2m.DistanceMode.EUC2D_ROUNDED
    k = int(args[args.index("--k") + 1])
    return inst, max(3, min(k, n - 1))


KNN_CASES = [n for n in golden_names() if n.startswith("knn_")] + [
    "u1k_s1", "u1k_s2", "c6_u10k_s4242", "u10k_s1", "u10k_s1_k20_rounded", "u500_s21_b100_k6",
    "u2k_s17_b300_k6_zero"]


@pytest.mark.parametrize("name", KNN_CASES)
def test_knn_matches_reference_golden(f2m, name):
    meta, _ = golden(name)
    inst, k = _inst(f2m, meta["args"])
    g = f2m.build_knn_graph(inst, k)
    u, v, c = g.edge_arrays()
    assert g.m == meta["m"]
    assert sha(u) == meta["sha256"]["eu"]
    assert sha(v) == meta["sha256"]["ev"]
    assert sha(c) == meta["sha256"]["ec"]
    assert g.mean_cost() == meta["mean_cost"]  # sequential sum, graph.cpp:47-49


def test_knn_edges_list_api(f2m):
    meta, arrays = golden("u1k_s1")
    inst, k = _inst(f2m, meta["args"])
    g = f2m.build_knn_graph(inst, k)
    edges = g.edges()
    assert [e[0] for e in edges] == arrays["eu"].tolist()
    assert [e[1] for e in edges] == arrays["ev"].tolist()
    assert [e[2] for e in edges] == arrays["ec"].tolist()


def _same_as_oracle(f2m, orc, xy, k, rounded):
    inst = f2m.Instance.from_points(np.asarray(xy, np.float64),
                                    f2m.DistanceMode.EUC2D_ROUNDED if rounded else f2m.DistanceMode.EUC2D_EXACT)
    g = f2m.build_knn_graph(inst, k)
    u, v, c = g.edge_arrays()
    o = orc.build_knn_graph(np.asarray(xy, np.float64), k, rounded)
    s = orc.knn_graph_scan(np.asarray(xy, np.float64), k, rounded)
    assert np.array_equal(o.eu, s.eu) and np.array_equal(o.cost, s.cost)
    assert np.array_equal(u, o.eu) and np.array_equal(v, o.ev) and np.array_equal(c, o.cost)
    return g


def test_elongated_point_set(f2m, orc):
    # test_graph.cpp:52-60: 200 points in a 1e6 x 1e-6 box
    rng = np.random.default_rng(55)
    xy = np.stack([rng.random(200) * 1e6, rng.random(200) * 1e-6], 1)
    _same_as_oracle(f2m, orc, xy, 4, False)


def test_clustered_and_coincident_points(f2m, orc):
    # test_graph.cpp:62-73: two tight clusters plus duplicates
    pts = []
    for i in range(12):
        pts.append((0.001 * i, 0.0))
        pts.append((500.0, 500.0 + 0.001 * (i % 3)))
    g = _same_as_oracle(f2m, orc, pts, 4, False)
    assert min(g.degrees()) >= 4


@pytest.mark.parametrize("n,k,rounded", [(2000, 6, False), (3000, 10, True), (1500, 20, False),
                                         (500, 33, False), (300, 40, True)])
def test_random_shapes_vs_oracle(f2m, orc, n, k, rounded):
    xy = orc.generate_instance(n, 1000 + n + k, 300.0)
    _same_as_oracle(f2m, orc, xy, k, rounded)


@pytest.mark.parametrize("k", list(range(3, 17)))
def test_every_candidate_count_vs_oracle(f2m, orc, k):
    """k = 3..12 run the register-resident k_knn_query_reg<K>, 13..16 the generic list; both
    must give the reference's lists, including (distance, id) tie-breaks on an integer grid."""
    xy = orc.generate_instance(1200, 77 + k, 500.0)
    _same_as_oracle(f2m, orc, xy, k, k % 2 == 0)
    xs, ys = np.meshgrid(np.arange(24.0), np.arange(17.0))
    _same_as_oracle(f2m, orc, np.stack([xs.ravel(), ys.ravel()], 1), k, False)


def test_clustered_generator_vs_oracle(f2m, orc):
    inst = f2m.generate_clustered_instance(20000, 5)
    xy = inst.points_array()
    _same_as_oracle(f2m, orc, xy, 10, False)


def test_integer_grid_heavy_ties(f2m, orc):
    xs, ys = np.meshgrid(np.arange(40.0), np.arange(30.0))
    xy = np.stack([xs.ravel(), ys.ravel()], 1)
    _same_as_oracle(f2m, orc, xy, 8, False)
    _same_as_oracle(f2m, orc, xy, 8, True)


def test_complete_graph_when_k_ge_n_minus_1(f2m):
    # test_graph.cpp:13-25
    sq = f2m.Instance.from_points(np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float))
    g = f2m.build_knn_graph(sq, 3)
    assert g.n == 4 and g.m == 6
    rep = f2m.validate_graph(g)
    assert rep["min_degree"] == 3 and rep["max_degree"] == 3
    inst = f2m.generate_instance(9, 5, 50.0)
    assert f2m.build_knn_graph(inst, 8).m == 36
    assert f2m.build_knn_graph(inst, 30).m == 36


def test_k20_degree(f2m):
    # test_graph.cpp:27-31
    g = f2m.build_knn_graph(f2m.generate_instance(50, 12, 200.0), 20)
    assert min(g.degrees()) >= 20


def test_argument_guards(f2m):
    # test_graph.cpp:33-37
    with pytest.raises(ValueError):
        f2m.build_knn_graph(f2m.generate_instance(10, 1), 2)
    with pytest.raises(ValueError):
        f2m.build_knn_graph(f2m.generate_instance(3, 1), 3)


def test_costs_match_distance_mode(f2m):
    # test_graph.cpp:75-82
    inst = f2m.generate_instance(60, 9, 10.0)
    inst.mode = f2m.DistanceMode.EUC2D_ROUNDED
    g = f2m.build_knn_graph(inst, 5)
    for u, v, c in g.edges():
        assert c == inst.distance(u, v)


def test_validate_graph_structural_defects(f2m):
    # test_graph.cpp:91-105
    tri = f2m.graph_from_edges(3, [0, 0, 1], [1, 2, 2], [3.0, 4.0, 5.0])
    with pytest.raises(RuntimeError, match="below 3"):
        f2m.validate_graph(tri)
    dup = f2m.graph_from_edges(4, [0, 1, 2, 0, 0, 1, 1], [1, 2, 3, 3, 2, 3, 2], [1.0] * 7)
    with pytest.raises(RuntimeError, match="duplicate"):
        f2m.validate_graph(dup)
    loop = f2m.graph_from_edges(4, [0, 1, 2, 0, 0, 1, 2], [1, 2, 3, 3, 2, 3, 2], [1.0] * 6 + [0.0])
    with pytest.raises(RuntimeError, match="self-loop"):
        f2m.validate_graph(loop)
    neg = f2m.graph_from_edges(4, [0, 0, 0, 1, 1, 2], [1, 2, 3, 2, 3, 3], [1, 1, -1, 1, 1, 1])
    with pytest.raises(RuntimeError, match="negative cost"):
        f2m.validate_graph(neg)


def test_from_edges_normalizes_and_indexes(f2m):
    # test_graph.cpp:117-131
    g = f2m.graph_from_edges(4, [3, 1, 2, 3, 2, 3], [0, 0, 1, 2, 0, 1], [2.0, 1.0, 4.0, 8.0, 16.0, 32.0])
    assert g.edges()[0][:2] == (0, 1)
    assert list(g.degrees()) == [3, 3, 3, 3]
    assert g.mean_cost() == pytest.approx((1 + 2 + 4 + 8 + 16 + 32) / 6.0)
    with pytest.raises(IndexError):
        f2m.graph_from_edges(2, [0], [2], [1.0])


def test_write_lp_structure(f2m):
    # test_solve.cpp:100-137 / acceptance criterion 9
    sq = f2m.Instance.from_points(np.array([[0, 0], [1, 0], [1, 1], [0, 1]], float))
    g = f2m.build_knn_graph(sq, 3)
    text = f2m.write_lp(g)
    assert text == f2m.write_lp(g)
    assert text.startswith("Minimize")
    assert "deg_3: x_0_3 + x_1_3 + x_2_3 = 2" in text
    assert text.count("= 2") == 4 and text.count("0 <= x_") == 6
