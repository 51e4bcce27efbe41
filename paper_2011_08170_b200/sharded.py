"""Node-sharded multi-GPU GDP solve.

One process per GPU (torchrun). Every rank holds the same candidate graph (built by the same
deterministic kernels), owns a contiguous range of the graph's spatial node order
(``Shard.info()``: positions ``[rank*stride, (rank+1)*stride)``), and per Jacobi sweep

1. runs ``k_shard_sweep`` on its rows, reading the full multiplier vector of the previous sweep
   and writing its own ``stride`` entries (``f2m_shard_sweep``, one kernel launch);
2. all-gathers the shards with NCCL over NVLink (``all_gather_into_tensor``) into the next full
   vector — concatenation in rank order is position order by construction;
3. records its shard's max |delta| (IEEE bits, atomic max on the device).

Convergence (max |delta| <= eps*mean_cost, dual.cpp:235) needs the global max of every sweep, but
not before the next sweep starts: the per-sweep maxima of a chunk of sweeps are all-reduced (MAX)
in one collective and read back once per chunk. The full vector of every sweep of the chunk stays
in a ring, so the multipliers of the first converged sweep are returned exactly — the sharded
solve is bit-identical to the one-GPU solve (a Jacobi sweep freezes lambda for the whole sweep,
dual.cpp:129-167), which tests/test_sharded.py checks on the GPU (in-process shards) and with the
gloo backend on CPU (two processes).

``run_sharded_jacobi`` is the collective schedule; it is independent of how a shard sweeps, so the
CPU tests drive it with a numpy restatement while the product path drives it with the CUDA kernel.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np
import torch


class TorchDistComm:
    """Collectives over torch.distributed (NCCL on GPUs, gloo on CPU): one shard per process."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_gather(self, out_full: torch.Tensor, shards: Sequence[torch.Tensor]) -> None:
        (shard,) = shards
        self.dist.all_gather_into_tensor(out_full, shard, group=self.group)

    def all_reduce_max(self, parts: Sequence[torch.Tensor]) -> torch.Tensor:
        (t,) = parts
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t


class LocalComm:
    """All shards in this process (simulated ranks on one device): the all-gather is the ordered
    concatenation, the all-reduce an element-wise max. Same schedule as TorchDistComm."""

    def __init__(self, world: int):
        self.rank = 0
        self.world = world

    def all_gather(self, out_full: torch.Tensor, shards: Sequence[torch.Tensor]) -> None:
        torch.cat(list(shards), out=out_full)

    def all_reduce_max(self, parts: Sequence[torch.Tensor]) -> torch.Tensor:
        out = parts[0].clone()
        for p in parts[1:]:
            torch.maximum(out, p, out=out)
        return out


@dataclass
class ShardedResult:
    lam_full: torch.Tensor          # multipliers after the last kept sweep (position order, padded)
    sweeps: int
    converged: bool
    final_max_abs_delta: float
    record: List[float] = field(default_factory=list)  # global max |delta| of every sweep


def _bits_to_double(bits: torch.Tensor) -> np.ndarray:
    return bits.detach().to("cpu").numpy().astype(np.int64).view(np.float64)


class ShardedJacobi:
    """Collective schedule of the sharded Jacobi solve (solve_duals' loop, dual.cpp:227-239).

    sweep_fns[i](lam_full, out_shard, max_bits) performs one sweep of local shard i (out_shard has
    `stride` entries; max_bits is a 0-d int64 tensor receiving max |delta| bits) on the CURRENT
    stream. Full vectors are world*stride long, in position order. On CUDA the steady-state chunk
    (sweep kernels + all-gathers + the max all-reduce of the chunk's maxima) is captured once in a
    CUDA graph and replayed, so there is no per-sweep host work; the object keeps the graph, so
    repeated runs (benchmarks, jitter restarts) pay the capture once."""

    def __init__(self, sweep_fns, comm, stride: int, device, chunk: int = 32, cuda_graph: bool = True):
        self.fns = list(sweep_fns)
        self.comm = comm
        self.stride = stride
        self.chunk = max(1, int(chunk))
        self.dev = torch.device(device)
        nfull = stride * comm.world
        self.ring = torch.empty((self.chunk, nfull), dtype=torch.float64, device=self.dev)
        self.outs = [torch.empty(stride, dtype=torch.float64, device=self.dev) for _ in self.fns]
        self.bits = [torch.zeros(self.chunk, dtype=torch.int64, device=self.dev) for _ in self.fns]
        self.use_graph = cuda_graph and self.dev.type == "cuda" and self.chunk >= 2
        self.graph = None
        self.gmax_static = None

    def _eager(self, prev, s, c):
        for b in self.bits:
            b.zero_()
        for j in range(c):
            for fn, out, b in zip(self.fns, self.outs, self.bits):
                fn(prev, out, b[j])
            slot = self.ring[(s + j) % self.chunk]
            self.comm.all_gather(slot, self.outs)
            prev = slot
        return _bits_to_double(self.comm.all_reduce_max([b[:c] for b in self.bits]))

    def _steady(self):
        # chunk-aligned steady state: sweep j reads slot j-1 (slot chunk-1 for j = 0, the previous
        # chunk's last sweep) and writes slot j — the same work every chunk
        if self.graph is None:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                for b in self.bits:
                    b.zero_()
                for j in range(self.chunk):
                    src = self.ring[(j - 1) % self.chunk]
                    for fn, out, b in zip(self.fns, self.outs, self.bits):
                        fn(src, out, b[j])
                    self.comm.all_gather(self.ring[j], self.outs)
                self.gmax_static = self.comm.all_reduce_max(list(self.bits))
        self.graph.replay()
        return _bits_to_double(self.gmax_static)

    def run(self, lam0_full: torch.Tensor, threshold: float, max_sweeps: int) -> ShardedResult:
        """Sweeps from lam0_full until max|delta| <= threshold (threshold < 0: exactly max_sweeps)."""
        chunk = self.chunk
        assert lam0_full.numel() == self.ring.shape[1]
        prev = lam0_full
        record: List[float] = []
        s = 0
        while s < max_sweeps:
            c = min(chunk, max_sweeps - s)
            if self.use_graph and s > 0 and c == chunk:
                gmax = self._steady()
            else:
                gmax = self._eager(prev, s, c)
            prev = self.ring[(s + c - 1) % chunk]
            for j in range(c):
                g = float(gmax[j])
                record.append(g)
                k = s + j
                if threshold >= 0.0 and g <= threshold:
                    return ShardedResult(self.ring[k % chunk].clone(), k + 1, True, g, record)
            s += c
        lam = self.ring[(s - 1) % chunk].clone() if s > 0 else lam0_full.clone()
        return ShardedResult(lam, s, False, record[-1] if record else math.inf, record)


def run_sharded_jacobi(sweep_fns, comm, stride: int, lam0_full: torch.Tensor, threshold: float,
                       max_sweeps: int, chunk: int = 32, cuda_graph: bool = True) -> ShardedResult:
    """One-shot ShardedJacobi(...).run(...)."""
    return ShardedJacobi(sweep_fns, comm, stride, lam0_full.device, chunk, cuda_graph).run(
        lam0_full, threshold, max_sweeps)


def solve_duals_sharded(graph, comm=None, eps: float = 1e-9, max_sweeps: int = 20000, b: int = 2,
                        eta: float = 0.5, update: str = "midpoint", init: str = "local-midpoint",
                        chunk: int = 32, threshold: Optional[float] = None):
    """solve_duals (dual.cpp:210-246) across ranks on CUDA devices.

    comm: TorchDistComm() inside an initialised NCCL process group (one GPU per rank), or
    LocalComm(world) to run `world` shards in this process on the current device. Returns
    (lambda in node-id order as numpy, report dict) on every rank."""
    from . import _f2m

    if comm is None:
        comm = TorchDistComm()
    dev = torch.device("cuda", torch.cuda.current_device())
    ranks = [comm.rank] if isinstance(comm, TorchDistComm) else list(range(comm.world))
    shards = [_f2m.shard_create(graph, r, comm.world, b, eta, update) for r in ranks]
    info = shards[0].info()
    n, stride = info["n"], info["stride"]
    stream = torch.cuda.current_stream(dev)
    lam0 = torch.zeros(stride * comm.world, dtype=torch.float64, device=dev)
    if n > 0:
        _f2m.initial_state_positions(graph, lam0.data_ptr(), b, init, stream.cuda_stream)
    if threshold is None:
        threshold = eps * graph.mean_cost()  # dual.cpp:221 (host fp64 product, no FMA)

    def make_fn(sh):
        def fn(lam_full, out, bits):
            sh.sweep(lam_full.data_ptr(), out.data_ptr(), bits.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
        return fn

    res = run_sharded_jacobi([make_fn(sh) for sh in shards], comm, stride, lam0, threshold, max_sweeps, chunk)
    ids = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    if n > 0:
        _f2m.positions_to_ids(graph, res.lam_full.data_ptr(), ids.data_ptr(), stream.cuda_stream)
    lam = ids[:n].cpu().numpy()
    report = {"converged": res.converged, "sweeps": res.sweeps, "final_max_abs_delta": res.final_max_abs_delta,
              "record": res.record, "world": comm.world, "stride": stride}
    return lam, report
