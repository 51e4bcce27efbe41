"""Single-process multi-GPU solve through the C ABI (EngineConfig::num_gpus, csrc/gpu/multi.cu).

A C++ caller of solve_duals (dual.hpp:79-81) / full_solve reaches several GPUs by setting
num_gpus: the graph is replicated and partitioned across the devices and one persistent sweep
kernel per device exchanges halo multipliers through peer memory. The result must be
bit-identical to the one-GPU solve (and so to the reference). The GPU box has one B200, so the
ranks share it here (f2m_set_gpu_list([0, 0, ...]): each rank gets its own slice of the SMs and
its own rings, the stores go through the same peer-pointer tables) — the code path a multi-GPU
node runs, minus the NVLink hop.
"""
import numpy as np
import pytest

from conftest import golden, sha

pytestmark = pytest.mark.gpu


@pytest.fixture
def shared_gpu(f2m):
    def use(world):
        f2m._f2m.set_gpu_list([0] * world)
    yield use
    f2m._f2m.set_gpu_list([])


@pytest.mark.parametrize("world", [2, 3, 4])
def test_solve_duals_num_gpus_bit_exact_10k(f2m, shared_gpu, world):
    shared_gpu(world)
    g = f2m.build_knn_graph(f2m.generate_instance(10000, 3), 10)
    st1, rep1 = f2m.solve_duals(g, max_sweeps=50000)
    stm, repm = f2m.solve_duals(g, max_sweeps=50000, num_gpus=world)
    info = f2m._f2m.multi_gpu_info(g)
    assert info["world"] == world
    assert "multi-rank" in f2m.last_sweep_kernel_desc()
    assert repm["converged"] and repm["sweeps"] == rep1["sweeps"]
    assert repm["final_max_abs_delta"] == rep1["final_max_abs_delta"]
    assert repm["dual_value"] == rep1["dual_value"]
    assert np.array_equal(np.asarray(stm.lam), np.asarray(st1.lam))


def test_full_solve_num_gpus_matches_reference_golden_100k(f2m, shared_gpu):
    """The headline instance (BASELINE configs[2]) certified through full_solve_graph with the
    sweeps on 2 ranks: x, lambda, objective, gap and sweeps equal the reference's own run."""
    shared_gpu(2)
    meta, _ = golden("u100k_s1")
    g = f2m.build_knn_graph(f2m.generate_instance(100000, 1), 10)
    r = f2m.full_solve_graph(g, k=10, eps=meta["eps"], max_sweeps=meta["max_sweeps"], num_gpus=2)
    assert r["sweeps"] == meta["full_sweeps"] and r["restarts"] == meta["full_restarts"]
    assert r["objective"] == meta["full_objective"] and r["gap"] == meta["full_gap"]
    assert sha(np.asarray(r["value"])) == meta["sha256"]["x_full"]
    assert sha(np.asarray(r["duals"])) == meta["sha256"]["lam_full"]


def test_num_gpus_fixed_sweeps_2m_world8(f2m, shared_gpu):
    """BASELINE configs[4] shape: 2M cities over 8 ranks (1,176 partition CTAs would be the
    8-GPU layout; sharing one GPU each rank gets 17), 64 fixed sweeps, bit-exact against the
    one-GPU kernel."""
    shared_gpu(8)
    g = f2m.build_knn_graph(f2m.generate_instance(2_000_000, 1), 10)
    st1, rep1 = f2m.solve_duals(g, eps=1e-300, max_sweeps=64)
    stm, repm = f2m.solve_duals(g, eps=1e-300, max_sweeps=64, num_gpus=8)
    assert rep1["sweeps"] == repm["sweeps"] == 64 and not repm["converged"]
    assert repm["final_max_abs_delta"] == rep1["final_max_abs_delta"]
    assert np.array_equal(np.asarray(stm.lam), np.asarray(st1.lam))


def test_num_gpus_clamped_to_slices(f2m, shared_gpu):
    """A 60-node graph has two 32-node slices: num_gpus=4 runs on 2 ranks, same result."""
    shared_gpu(4)
    g = f2m.build_knn_graph(f2m.generate_instance(60, 5), 8)
    st1, rep1 = f2m.solve_duals(g, max_sweeps=20000)
    stm, repm = f2m.solve_duals(g, max_sweeps=20000, num_gpus=4)
    assert f2m._f2m.multi_gpu_info(g)["world"] == 2
    assert repm["sweeps"] == rep1["sweeps"]
    assert np.array_equal(np.asarray(stm.lam), np.asarray(st1.lam))


def test_num_gpus_beyond_visible_devices_is_an_argument_error(f2m):
    import torch

    f2m._f2m.set_gpu_list([])
    g = f2m.build_knn_graph(f2m.generate_instance(2000, 1), 10)
    with pytest.raises(ValueError, match="num_gpus"):
        f2m.solve_duals(g, num_gpus=torch.cuda.device_count() + 1)


def test_num_gpus_explicit_initial_state(f2m, shared_gpu):
    """solve_duals(initial=...) with num_gpus: lambda_0 crosses to the replicas' order."""
    shared_gpu(2)
    g = f2m.build_knn_graph(f2m.generate_instance(5000, 11), 10)
    st0 = f2m.make_initial_state(g)
    lam0 = np.asarray(st0.lam) * 0.5
    init = f2m.DualState(list(lam0))
    st1, rep1 = f2m.solve_duals(g, max_sweeps=30000, initial=init)
    stm, repm = f2m.solve_duals(g, max_sweeps=30000, initial=f2m.DualState(list(lam0)), num_gpus=2)
    assert repm["sweeps"] == rep1["sweeps"]
    assert np.array_equal(np.asarray(stm.lam), np.asarray(st1.lam))
