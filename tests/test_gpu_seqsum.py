"""GPU parity: the exact parallel evaluation of sequential fp64 sums (csrc/gpu/seqsum.cu).

The reference accumulates the objective (primal.cpp:226-230), the dual-objective chunk sums
(dual.cpp:96-109) and mean_cost (graph.cpp:47-49) left to right in one fp64 chain. f2m_seq_sums
must return that chain's value bit for bit, for every input; the checker is numpy's cumulative
sum (a plain left-to-right loop) from +0.0. Inputs are chosen to hit every route of the walk:
binade crossings, exact ties (t/ulp = k + 1/2), sign changes, cancellation, zeros / -0.0,
subnormals, non-finite terms, ragged segments.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _seq(v, seg_len):
    k = len(v)
    if seg_len <= 0 or seg_len > k:
        seg_len = max(k, 1)
    out = []
    with np.errstate(invalid="ignore", over="ignore"):
        for lo in range(0, k, seg_len):
            out.append(np.cumsum(np.concatenate([[0.0], v[lo:lo + seg_len]]))[-1])
    return np.array(out, dtype=np.float64)


def _gpu(f2m_mod, v, seg_len):
    import torch
    k = len(v)
    d = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    nseg = 0 if k == 0 else (k + (seg_len if 0 < seg_len <= k else k) - 1) // (seg_len if 0 < seg_len <= k else k)
    out = torch.full((max(nseg, 1),), -12345.0, dtype=torch.float64, device="cuda")
    f2m_mod._f2m.seq_sums(d.data_ptr(), k, seg_len, out.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out.cpu().numpy()[:nseg]


def _same(a, b):
    assert a.shape == b.shape
    nan = np.isnan(a) & np.isnan(b)
    ok = (a.view(np.int64) == b.view(np.int64)) | nan
    assert ok.all(), f"{int((~ok).sum())} of {len(a)} segments differ; first: " \
                     f"{a[~ok][:3]!r} vs {b[~ok][:3]!r}"


def _cases():
    r = np.random.default_rng(7)
    yield "uniform_pos", r.uniform(0, 1000, 100_003)
    yield "costs_sqrt", np.sqrt(r.uniform(0, 2e6, 568_737))
    yield "products_half", np.sqrt(r.uniform(0, 2e6, 300_000)) * r.choice([0.0, 0.0, 0.0, 0.5, 1.0], 300_000)
    yield "mixed_sign", r.normal(0, 100, 200_000)
    yield "all_negative", -r.exponential(3.0, 150_000)
    yield "integers", r.integers(0, 1000, 250_000).astype(np.float64)
    yield "half_integers", r.integers(0, 2000, 250_000).astype(np.float64) * 0.5
    yield "lognormal_wide", r.lognormal(0, 12, 120_000) * r.choice([-1.0, 1.0], 120_000)
    # ties: once acc >= 2^52, adding 0.5 / 1.5 lands exactly half-way between doubles
    yield "ties_2p52", np.concatenate([[2.0 ** 52], np.full(5000, 0.5), np.full(5000, 1.5), r.uniform(0, 4, 5000)])
    yield "ties_2p53", np.concatenate([[2.0 ** 53], np.ones(9000), np.full(3000, 3.0)])
    yield "cancellation", np.concatenate([r.normal(0, 1e6, 50_000), -r.normal(0, 1e6, 50_000)])
    yield "zeros_then_values", np.concatenate([np.zeros(10_000), -np.zeros(300), r.uniform(0, 1, 20_000)])
    yield "neg_zeros", -np.zeros(5000)
    yield "tiny_subnormal", r.uniform(0, 1, 50_000) * 5e-324 * 1000
    yield "with_inf", np.concatenate([r.uniform(0, 1, 3000), [np.inf], r.uniform(0, 1, 3000)])
    yield "with_nan", np.concatenate([r.uniform(0, 1, 3000), [np.nan], r.uniform(0, 1, 3000)])
    yield "inf_minus_inf", np.array([1.0, np.inf, 2.0, -np.inf, 3.0])
    yield "huge", r.uniform(0, 1, 20_000) * 1e300
    yield "growing", np.arange(1, 70_001, dtype=np.float64) ** 1.5


@pytest.mark.parametrize("seg_len", [0, 2048, 8192, 1000, 1])
def test_seq_sums_bit_exact(f2m, seg_len):
    for name, v in _cases():
        if seg_len == 1 and len(v) > 30_000:
            v = v[:30_000]
        got = _gpu(f2m, v, seg_len)
        _same(got, _seq(v, seg_len))


@pytest.mark.parametrize("k", [1, 2, 31, 127, 128, 129, 4095, 4096, 4097, 131_073])
def test_seq_sums_ragged_sizes(f2m, k):
    r = np.random.default_rng(k)
    for v in (r.uniform(0, 10, k), r.normal(0, 1, k), np.sqrt(r.uniform(0, 1e6, k))):
        for seg_len in (0, 128, 2048):
            _same(_gpu(f2m, v, seg_len), _seq(v, seg_len))


def test_seq_sums_empty(f2m):
    assert _gpu(f2m, np.zeros(0), 0).shape == (0,)


def test_seq_sums_random_fuzz(f2m):
    """Many short mixed inputs (a few seconds): random magnitudes, signs, zeros and ties."""
    r = np.random.default_rng(2024)
    for _ in range(60):
        k = int(r.integers(1, 20_000))
        scale = 10.0 ** r.uniform(-8, 8, k)
        v = r.uniform(-1, 1, k) * scale
        v[r.random(k) < 0.2] = 0.0
        if r.random() < 0.5:
            v = np.abs(v)
        if r.random() < 0.3:  # quantised values: frequent exact ties
            v = np.round(v * 4) / 4
        seg_len = int(r.choice([0, 64, 2048, 8192, int(r.integers(1, 5000))]))
        _same(_gpu(f2m, v, seg_len), _seq(v, seg_len))
