"""generate_instance (instance.cpp:143-157) on the device: bit-identical to the reference's host
SplitMix64 stream (the host C++ restatement is itself pinned to the live reference in
tests/test_host_cpu.py)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,seed,box", [(1, 0, 1.0), (7, 3, 100.0), (1000, 1, 1000.0), (100_000, 1, 1000.0),
                                        (2_000_000, 1, 1000.0), (4097, 2**63 + 5, 0.5)])
def test_device_generator_bit_exact(f2m, n, seed, box):
    import torch

    d = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    f2m._f2m.generate_instance_device(n, seed, box, d.data_ptr(), torch.cuda.current_stream().cuda_stream)
    host = f2m.generate_instance(n, seed, box).points_array().reshape(-1)
    assert np.array_equal(d.cpu().numpy().view(np.uint64), host.view(np.uint64))


def test_device_generator_feeds_the_device_pipeline(f2m):
    """Points generated in HBM go straight into full_solve_device: same result as the host path."""
    import torch

    n = 20000
    d = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    f2m._f2m.generate_instance_device(n, 5, 1000.0, d.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dx = torch.empty(n * 10, dtype=torch.float64, device="cuda")
    dl = torch.empty(n, dtype=torch.float64, device="cuda")
    r = f2m.full_solve_device(n, d.data_ptr(), False, 10, 1e-9, 200000, dx.data_ptr(), n * 10, dl.data_ptr())
    h = f2m.full_solve_arrays(f2m.generate_instance(n, 5, 1000.0).points_array(), k=10, max_sweeps=200000)
    assert r["sweeps"] == h["sweeps"] and r["objective"] == h["objective"]
    assert np.array_equal(dl.cpu().numpy(), np.asarray(h["duals"]))


def test_device_generator_rejects_bad_arguments(f2m):
    with pytest.raises(ValueError):
        f2m._f2m.generate_instance_device(0, 1, 1.0, 0, 0)
    with pytest.raises(ValueError):
        f2m._f2m.generate_instance_device(5, 1, -1.0, 0, 0)
