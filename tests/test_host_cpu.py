"""CPU: host-side API (instance format, generators, config errors), the C-ABI library's exports,
and the oracle against the live reference when oracle/_ref is built.
"""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT

SQUARE = "\n".join(["NAME : square", "TYPE : TSP", "DIMENSION : 4", "EDGE_WEIGHT_TYPE : EUC_2D",
                    "NODE_COORD_SECTION", "1 0 0", "2 1 0", "3 1 1", "4 0 1", "EOF"])


def test_parse_and_distance(f2m):
    # reference tests/python/test_smoke.py:34-42
    inst = f2m.parse_tsplib(SQUARE)
    assert len(inst) == 4 and inst.name == "square"
    assert inst.mode == f2m.DistanceMode.EUC2D_ROUNDED
    assert inst.distance(0, 1) == 1.0 and inst.distance(0, 2) == 1.0
    inst.mode = f2m.DistanceMode.EUC2D_EXACT
    assert inst.distance(0, 2) == pytest.approx(math.sqrt(2.0), abs=1e-15)
    with pytest.raises(IndexError):
        inst.distance(0, 4)


@pytest.mark.parametrize("text,msg", [
    ("DIMENSION : 3\n", "NODE_COORD_SECTION"),
    ("NODE_COORD_SECTION\n1 0 0\n", "before DIMENSION"),
    ("DIMENSION : x\n", "not an integer"),
    ("DIMENSION : 0\n", "positive"),
    ("DIMENSION : 2\nEDGE_WEIGHT_TYPE : GEO\n", "EUC_2D"),
    ("DIMENSION : 2\nNODE_COORD_SECTION\n1 0 0\n3 1 1\n", "out of range"),
    ("DIMENSION : 2\nNODE_COORD_SECTION\n1 0 0\n1 1 1\n", "duplicate"),
    ("DIMENSION : 2\nNODE_COORD_SECTION\n1 0 0\n", "missing coordinate"),
    ("NAME : x\n", "missing DIMENSION"),
])
def test_parse_errors(f2m, text, msg):
    with pytest.raises(ValueError, match=msg):
        f2m.parse_tsplib(text)


def test_round_trip_and_fixture(f2m):
    inst = f2m.generate_instance(17, seed=5, box=250.0)
    back = f2m.parse_tsplib(f2m.serialize_tsplib(inst))
    assert back.points == inst.points
    with pytest.raises(ValueError):
        f2m.load_tsplib("/nonexistent/file.tsp")


def test_generate_instance_matches_oracle_and_reference(f2m, orc):
    for n, seed, box in ((1, 0, 1.0), (1000, 1, 1000.0), (777, 123456789, 3.5)):
        ours = f2m.generate_instance(n, seed, box).points_array()
        assert np.array_equal(ours, orc.generate_instance(n, seed, box))
    with pytest.raises(ValueError):
        f2m.generate_instance(0, 1)
    with pytest.raises(ValueError):
        f2m.generate_instance(5, 1, 0.0)


def test_generate_instance_matches_live_reference(f2m, ref):
    for n, seed in ((100, 3), (5000, 99)):
        assert f2m.generate_instance(n, seed).points == ref.generate_instance(n, seed).points


def test_clustered_generator_deterministic(f2m):
    a = f2m.generate_clustered_instance(5000, 1).points_array()
    b = f2m.generate_clustered_instance(5000, 1).points_array()
    assert np.array_equal(a, b) and a.shape == (5000, 2)
    assert f2m.generate_clustered_instance(5000, 2).points_array()[0, 0] != a[0, 0]


def test_instance_from_points(f2m):
    xy = np.array([[0.0, 1.0], [2.0, 3.0]])
    inst = f2m.Instance.from_points(xy, name="two")
    assert inst.name == "two" and inst.mode == f2m.DistanceMode.EUC2D_EXACT
    assert np.array_equal(inst.points_array(), xy)
    with pytest.raises(ValueError):
        f2m.Instance.from_points(np.zeros((3, 3)))


def test_exception_hierarchy(f2m):
    assert issubclass(f2m.ParseError, ValueError) and issubclass(f2m.TooLarge, ValueError)
    for e in (f2m.DegenerateExtraction, f2m.Infeasible, f2m.SolveFailed, f2m.DeviceError):
        assert issubclass(e, RuntimeError)


def test_no_silent_cpu_fallback(f2m):
    """Without a CUDA device every compute call fails loudly (there is no CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    inst = f2m.generate_instance(50, 1)
    with pytest.raises(f2m.DeviceError):
        f2m.build_knn_graph(inst, 5)
    with pytest.raises(f2m.DeviceError):
        f2m.full_solve(inst, k=5)


def test_full_solve_arrays_rejects_bad_output_buffers(f2m):
    """Caller-owned result buffers are checked before any device work (size, dtype, layout)."""
    import numpy as np
    xy = f2m.generate_instance(50, 1).points_array()
    with pytest.raises(ValueError, match="out_value"):
        f2m.full_solve_arrays(xy, k=5, out_value=np.zeros(10))
    with pytest.raises(ValueError, match="out_value"):
        f2m.full_solve_arrays(xy, k=5, out_value=np.zeros(251, dtype=np.float32))
    with pytest.raises(ValueError, match="out_duals"):
        f2m.full_solve_arrays(xy, k=5, out_value=np.zeros(251), out_duals=np.zeros(100)[::2])


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "f2m_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(f2m_[a-z0-9_]+)\s*\(", text)))


def test_c_abi_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2011_08170_b200", "libf2m_gpu.so"))
    syms = _declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_c_abi_host_only_calls():
    """Calls that need no device: config validation and error reporting."""
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2011_08170_b200", "libf2m_gpu.so"))

    class Cfg(ctypes.Structure):
        _fields_ = [("b", ctypes.c_int), ("eta", ctypes.c_double), ("eps", ctypes.c_double),
                    ("max_sweeps", ctypes.c_int), ("mode", ctypes.c_int), ("update", ctypes.c_int),
                    ("init", ctypes.c_int), ("threads", ctypes.c_int), ("num_gpus", ctypes.c_int)]
    lib.f2m_last_error.restype = ctypes.c_char_p
    assert lib.f2m_engine_config_validate(ctypes.byref(Cfg(2, 0.5, 1e-9, 100, 0, 0, 0, 0))) == 0
    assert lib.f2m_engine_config_validate(ctypes.byref(Cfg(2, 0.0, 1e-9, 100, 0, 0, 0, 0))) == 1
    assert b"eta" in lib.f2m_last_error()
    assert lib.f2m_engine_config_validate(ctypes.byref(Cfg(9, 0.5, 1e-9, 100, 0, 0, 0, 0))) == 1
    assert lib.f2m_engine_config_validate(ctypes.byref(Cfg(2, 0.5, 1e-9, 100, 0, 0, 0, 0, 8))) == 0
    assert lib.f2m_engine_config_validate(ctypes.byref(Cfg(2, 0.5, 1e-9, 100, 0, 0, 0, 0, -1))) == 1
    assert b"num_gpus" in lib.f2m_last_error()


def test_oracle_vs_live_reference_small(orc, ref):
    """The C restatement against the reference's own Python binding on fresh random inputs."""
    rng = np.random.default_rng(1)
    for trial in range(6):
        n = int(rng.integers(20, 400))
        seed = int(rng.integers(0, 1 << 30))
        k = int(rng.integers(3, 12))
        rinst = ref.generate_instance(n, seed, 100.0)
        rounded = trial % 2 == 1
        if rounded:
            rinst.mode = ref.DistanceMode.EUC2D_ROUNDED
        rg = ref.build_knn_graph(rinst, k, threads=1)
        og = orc.build_knn_graph(orc.generate_instance(n, seed, 100.0), k, rounded)
        assert [tuple(e) for e in rg.edges()] == list(zip(og.eu.tolist(), og.ev.tolist(), og.cost.tolist()))
        st, rep = ref.solve_duals(rg, threads=1, max_sweeps=500)
        lam, orep = orc.solve_duals(og, max_sweeps=500)
        assert rep["sweeps"] == orep["sweeps"] and rep["dual_value"] == orep["dual_value"]
        assert st.lam == lam.tolist()
