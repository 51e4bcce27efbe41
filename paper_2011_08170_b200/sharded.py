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

    def all_to_all(self, recvs: Sequence[torch.Tensor], sends: Sequence[torch.Tensor],
                   recv_counts: Sequence[Sequence[int]], send_counts: Sequence[Sequence[int]]) -> None:
        (recv,), (send,) = recvs, sends
        self.dist.all_to_all_single(recv, send, output_split_sizes=list(recv_counts[0]),
                                    input_split_sizes=list(send_counts[0]), group=self.group)


class LocalComm:
    """All shards in this process (simulated ranks on one device): the all-gather is the ordered
    concatenation, the all-reduce an element-wise max. Same schedule as TorchDistComm.

    Test-only for the persistent engines (ShardedP2P, ShardedResident): their in-process ranks are
    `world` cooperative launches on separate streams of ONE device that spin-wait on each other,
    and CUDA guarantees co-residency only inside one grid, not across grids. They run concurrently
    on an otherwise idle device (the SMs are split between them) and every poll has a 20 s watchdog
    that aborts instead of hanging; production multi-GPU runs one rank per device (TorchDistComm
    across processes, or DeviceComm in one process)."""

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

    def all_to_all(self, recvs, sends, recv_counts, send_counts) -> None:
        # shard r's chunk for shard q sits at offset sum(send_counts[r][:q]) of sends[r]
        for r in range(self.world):
            off = 0
            for q in range(self.world):
                cnt = recv_counts[r][q]
                if cnt:
                    src_off = sum(send_counts[q][:r])
                    recvs[r][off:off + cnt].copy_(sends[q][src_off:src_off + cnt])
                off += cnt


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


@dataclass
class HaloPlan:
    """Halo exchange plan of one rank: which positions it receives from / sends to every rank.
    Every rank derives all plans from the same (replicated) graph, so sends and receives match."""
    recv_pos: np.ndarray      # int32, positions this rank reads from other ranks, grouped by owner
    recv_counts: List[int]    # per owner rank
    send_pos: np.ndarray      # int32, own positions other ranks read, grouped by reader
    send_counts: List[int]    # per reader rank


def halo_plans(n: int, world: int, stride: int, pos_u: np.ndarray, pos_v: np.ndarray) -> List[HaloPlan]:
    """From the edge endpoints in position space: rank r reads position p of rank q != r iff p is
    a neighbour of a row r owns. The plan of every rank, in O(m log m)."""
    pos_u = np.asarray(pos_u, np.int64)
    pos_v = np.asarray(pos_v, np.int64)
    ou, ov = pos_u // stride, pos_v // stride
    cross = ou != ov
    reader = np.concatenate([ou[cross], ov[cross]])
    pos = np.concatenate([pos_v[cross], pos_u[cross]])
    key = np.unique(reader * (stride * world) + pos)  # sorted by (reader, position)
    reader, pos = key // (stride * world), key % (stride * world)
    owner = pos // stride
    plans = []
    for r in range(world):
        sel = reader == r
        rp, ro = pos[sel], owner[sel]  # sorted by position => grouped by owner (contiguous ranges)
        recv_counts = np.bincount(ro, minlength=world).astype(int).tolist()
        sel2 = owner == r
        sp, sr = pos[sel2], reader[sel2]  # sorted by (reader, position)
        send_counts = np.bincount(sr, minlength=world).astype(int).tolist()
        plans.append(HaloPlan(rp.astype(np.int32), recv_counts, sp.astype(np.int32), send_counts))
    return plans


class ShardedJacobiHalo:
    """Collective schedule with a halo exchange instead of the all-gather: per sweep every rank
    sweeps its rows into its own copy of the multiplier vector, packs the values other ranks read,
    exchanges them with one all-to-all (NCCL sends/receives between spatially adjacent ranks only;
    ~2 % of the multipliers at 2M cities over 8 ranks) and unpacks what it reads. The vector of
    every sweep of a chunk stays in a per-rank ring; the multipliers of the stopping sweep are
    all-gathered once at the end. Bit-identical to ShardedJacobi and to one GPU.

    sweep_fns[i](lam_local_in, out_shard_view, max_bits) as in ShardedJacobi; pack(src, idx, dst,
    count) / unpack(src, idx, dst, count) move values on the current stream (idx: device int32)."""

    def __init__(self, sweep_fns, comm, stride: int, plans: Sequence[HaloPlan], ranks: Sequence[int], device,
                 pack: Callable, unpack: Callable, chunk: int = 32, cuda_graph: bool = True):
        self.fns = list(sweep_fns)
        self.comm = comm
        self.stride = stride
        self.ranks = list(ranks)
        self.chunk = max(1, int(chunk))
        self.dev = torch.device(device)
        self.pack, self.unpack = pack, unpack
        nfull = stride * comm.world
        self.rings = [torch.empty((self.chunk, nfull), dtype=torch.float64, device=self.dev) for _ in self.fns]
        self.bits = [torch.zeros(self.chunk, dtype=torch.int64, device=self.dev) for _ in self.fns]
        self.plans = [plans[r] for r in self.ranks]
        self.all_recv_counts = [plans[r].recv_counts for r in self.ranks]
        self.all_send_counts = [plans[r].send_counts for r in self.ranks]
        self.recv_idx = [torch.from_numpy(pl.recv_pos).to(self.dev) for pl in self.plans]
        self.send_idx = [torch.from_numpy(pl.send_pos).to(self.dev) for pl in self.plans]
        self.recvbuf = [torch.empty(len(pl.recv_pos), dtype=torch.float64, device=self.dev) for pl in self.plans]
        self.sendbuf = [torch.empty(len(pl.send_pos), dtype=torch.float64, device=self.dev) for pl in self.plans]
        self.use_graph = cuda_graph and self.dev.type == "cuda" and self.chunk >= 2
        self.graph = None
        self.gmax_static = None

    def _sweep(self, srcs, j):
        for i, (fn, ring, b) in enumerate(zip(self.fns, self.rings, self.bits)):
            r = self.ranks[i]
            fn(srcs[i], ring[j][r * self.stride:(r + 1) * self.stride], b[j])
            self.pack(ring[j], self.send_idx[i], self.sendbuf[i], len(self.plans[i].send_pos))
        self.comm.all_to_all(self.recvbuf, self.sendbuf, self.all_recv_counts, self.all_send_counts)
        for i, ring in enumerate(self.rings):
            self.unpack(self.recvbuf[i], self.recv_idx[i], ring[j], len(self.plans[i].recv_pos))

    def _eager(self, srcs, s, c):
        for b in self.bits:
            b.zero_()
        for j in range(c):
            slot = (s + j) % self.chunk
            self._sweep(srcs if j == 0 else [ring[(s + j - 1) % self.chunk] for ring in self.rings], slot)
        return _bits_to_double(self.comm.all_reduce_max([b[:c] for b in self.bits]))

    def _steady(self):
        if self.graph is None:
            self.graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(self.graph):
                for b in self.bits:
                    b.zero_()
                for j in range(self.chunk):
                    self._sweep([ring[(j - 1) % self.chunk] for ring in self.rings], j)
                self.gmax_static = self.comm.all_reduce_max(list(self.bits))
        self.graph.replay()
        return _bits_to_double(self.gmax_static)

    def run(self, lam0_local: Sequence[torch.Tensor], threshold: float, max_sweeps: int):
        """Returns (sweeps, converged, final max, record, slot) — the ring slot holding the
        stopping sweep's vectors (None: the initial vectors)."""
        chunk = self.chunk
        srcs = list(lam0_local)
        record: List[float] = []
        s = 0
        while s < max_sweeps:
            c = min(chunk, max_sweeps - s)
            if self.use_graph and s > 0 and c == chunk:
                gmax = self._steady()
            else:
                gmax = self._eager(srcs, s, c)
            srcs = [ring[(s + c - 1) % chunk] for ring in self.rings]
            for j in range(c):
                g = float(gmax[j])
                record.append(g)
                if threshold >= 0.0 and g <= threshold:
                    return s + j + 1, True, g, record, (s + j) % chunk
            s += c
        return s, False, (record[-1] if record else math.inf), record, ((s - 1) % chunk if s > 0 else None)


def run_sharded_jacobi(sweep_fns, comm, stride: int, lam0_full: torch.Tensor, threshold: float,
                       max_sweeps: int, chunk: int = 32, cuda_graph: bool = True) -> ShardedResult:
    """One-shot ShardedJacobi(...).run(...)."""
    return ShardedJacobi(sweep_fns, comm, stride, lam0_full.device, chunk, cuda_graph).run(
        lam0_full, threshold, max_sweeps)


def solve_duals_sharded(graph, comm=None, eps: float = 1e-9, max_sweeps: int = 20000, b: int = 2,
                        eta: float = 0.5, update: str = "midpoint", init: str = "local-midpoint",
                        chunk: int = 32, threshold: Optional[float] = None, exchange: str = "halo"):
    """solve_duals (dual.cpp:210-246) across ranks on CUDA devices.

    comm: TorchDistComm() inside an initialised NCCL process group (one GPU per rank), or
    LocalComm(world) to run `world` shards in this process on the current device.
    exchange: "halo" (all-to-all of the values other ranks read, default), "allgather" (the
    whole vector every sweep) or "p2p" (one persistent kernel per rank for all sweeps, halo
    multipliers and sweep maxima stored straight into the peers' memory; see _solve_duals_p2p). Returns (lambda in node-id order as numpy, report dict) on every
    rank."""
    if exchange == "halo":
        return _solve_duals_halo(graph, comm, eps, max_sweeps, b, eta, update, init, chunk, threshold)
    if exchange == "p2p":
        return _solve_duals_p2p(graph, comm, eps, max_sweeps, b, eta, update, init, threshold)
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


def make_halo_schedule(graph, comm, b: int = 2, eta: float = 0.5, update: str = "midpoint",
                       init: str = "local-midpoint", chunk: int = 32):
    """The halo-exchange schedule of `graph` on this process's shards (one for TorchDistComm,
    all for LocalComm) plus the initial multipliers; used by the solve and by the benchmarks."""
    from . import _f2m

    dev = torch.device("cuda", torch.cuda.current_device())
    ranks = [comm.rank] if isinstance(comm, TorchDistComm) else list(range(comm.world))
    shards = [_f2m.shard_create(graph, r, comm.world, b, eta, update) for r in ranks]
    info = shards[0].info()
    n, stride = info["n"], info["stride"]
    lam0 = torch.zeros(stride * comm.world, dtype=torch.float64, device=dev)
    if n > 0:
        _f2m.initial_state_positions(graph, lam0.data_ptr(), b, init, torch.cuda.current_stream(dev).cuda_stream)
    pos = graph.positions()
    u, v, _ = graph.edge_arrays()
    plans = halo_plans(n, comm.world, stride, pos[u], pos[v])

    def cur():
        return torch.cuda.current_stream(dev).cuda_stream

    def make_fn(sh):
        def fn(lam_in, out, bits):
            sh.sweep(lam_in.data_ptr(), out.data_ptr(), bits.data_ptr(), cur())
        return fn

    def pack(src, idx, dst, count):
        if count:
            _f2m.gather_f64(src.data_ptr(), idx.data_ptr(), dst.data_ptr(), count, cur())

    def unpack(src, idx, dst, count):
        if count:
            _f2m.scatter_f64(src.data_ptr(), idx.data_ptr(), dst.data_ptr(), count, cur())

    sched = ShardedJacobiHalo([make_fn(sh) for sh in shards], comm, stride, plans, ranks, dev, pack, unpack, chunk)
    sched.shards = shards  # keep the handles alive with the schedule
    meta = {"n": n, "stride": stride, "ranks": ranks, "plans": plans,
            "halo_values_per_sweep": int(sum(len(p.recv_pos) for p in plans))}
    return sched, lam0, meta


def _solve_duals_halo(graph, comm, eps, max_sweeps, b, eta, update, init, chunk, threshold):
    from . import _f2m

    if comm is None:
        comm = TorchDistComm()
    dev = torch.device("cuda", torch.cuda.current_device())
    sched, lam0, meta = make_halo_schedule(graph, comm, b, eta, update, init, chunk)
    n, stride, ranks = meta["n"], meta["stride"], meta["ranks"]
    nfull = stride * comm.world
    if threshold is None:
        threshold = eps * graph.mean_cost()  # dual.cpp:221 (host fp64 product, no FMA)
    sweeps, converged, fmax, record, slot = sched.run([lam0] * len(ranks), threshold, max_sweeps)
    # the stopping sweep's multipliers: every rank's own range of its ring slot
    if slot is None:
        full = lam0
    else:
        full = torch.empty(nfull, dtype=torch.float64, device=dev)
        views = [sched.rings[i][slot][r * stride:(r + 1) * stride].contiguous() for i, r in enumerate(ranks)]
        comm.all_gather(full, views)
    ids = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    if n > 0:
        _f2m.positions_to_ids(graph, full.data_ptr(), ids.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    lam = ids[:n].cpu().numpy()
    report = {"converged": converged, "sweeps": sweeps, "final_max_abs_delta": fmax, "record": record,
              "world": comm.world, "stride": stride, "exchange": "halo",
              "halo_values_per_sweep": meta["halo_values_per_sweep"]}
    return lam, report


def p2p_plan_arrays(plans: Sequence[HaloPlan], rank: int):
    """Flat send / receive lists of `rank` for the fused peer-memory solve: recv_pos (positions
    this rank reads, grouped by owner), and per value it sends: own position, reader rank and the
    index of that value in the reader's receive list (both sides sort by position)."""
    world = len(plans)
    recv_pos = plans[rank].recv_pos.astype(np.int32)
    send_pos, send_peer, send_dst = [], [], []
    off = 0
    for r in range(world):
        cnt = plans[rank].send_counts[r]
        if cnt:
            seg = plans[rank].send_pos[off:off + cnt]
            base = int(sum(plans[r].recv_counts[:rank]))  # owner `rank`'s segment in r's receive list
            assert plans[r].recv_counts[rank] == cnt
            send_pos.append(seg)
            send_peer.append(np.full(cnt, r, np.int32))
            send_dst.append(base + np.arange(cnt, dtype=np.int32))
        off += cnt
    cat = (lambda xs: np.concatenate(xs).astype(np.int32)) if send_pos else (lambda xs: np.zeros(0, np.int32))
    return recv_pos, cat(send_pos), cat(send_peer), cat(send_dst)


class ShardedP2P:
    """Fused peer-memory solve (SURVEY §8(e) "faster fused variant"): every rank launches ONE
    persistent kernel (f2m_p2p_launch) that runs all sweeps of its rows; halo multipliers and
    sweep maxima are stored straight into the other ranks' receive buffers / boards (NVLink peer
    memory from torch symmetric memory across processes; plain device memory for LocalComm ranks,
    which run concurrently on one GPU, each on its own stream). Bit-identical to one GPU.

    Build once per graph; run(lam0_full, threshold, max_sweeps) -> (lam_full in position order,
    result dict) may be called repeatedly (buffers are re-zeroed and ranks re-synchronised)."""

    def __init__(self, graph, comm, b: int = 2, eta: float = 0.5, update: str = "midpoint", ctas: int = 0):
        from . import _f2m

        self._f2m = _f2m
        self.comm = comm
        self.dev = torch.device("cuda", torch.cuda.current_device())
        dev = self.dev
        self.world = world = comm.world
        self.local = local = not isinstance(comm, TorchDistComm)
        self.ranks = ranks = list(range(world)) if local else [comm.rank]
        self.shards = {r: _f2m.shard_create(graph, r, world, b, eta, update) for r in ranks}
        info = next(iter(self.shards.values())).info()
        self.n, self.stride = n, stride = info["n"], info["stride"]
        pos = graph.positions()
        u, v, _ = graph.edge_arrays()
        plans = halo_plans(n, world, stride, pos[u], pos[v])
        nrecv = [len(p.recv_pos) for p in plans]
        self.halo_values = int(sum(nrecv))
        recv_words = 2 * 2 * max(max(nrecv), 1)  # 2 parities x LL pair (2 words) per value
        board_words = 4 * world * 2
        if local:
            self.recv_bufs = {r: torch.zeros(recv_words, dtype=torch.int64, device=dev) for r in ranks}
            self.boards = {r: torch.zeros(board_words, dtype=torch.int64, device=dev) for r in ranks}
            recv_ptrs = [self.recv_bufs[r].data_ptr() for r in range(world)]
            board_ptrs = [self.boards[r].data_ptr() for r in range(world)]
        else:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem

            group = comm.group if comm.group is not None else dist.group.WORLD
            rb = symm_mem.empty(recv_words, dtype=torch.int64, device=dev)
            bd = symm_mem.empty(board_words, dtype=torch.int64, device=dev)
            self._handles = (symm_mem.rendezvous(rb, group), symm_mem.rendezvous(bd, group))
            self.recv_bufs, self.boards = {comm.rank: rb}, {comm.rank: bd}
            recv_ptrs, board_ptrs = list(self._handles[0].buffer_ptrs), list(self._handles[1].buffer_ptrs)
        self.peer_recv = torch.tensor(recv_ptrs, dtype=torch.int64, device=dev)
        self.peer_board = torch.tensor(board_ptrs, dtype=torch.int64, device=dev)
        self.peer_nrecv = torch.tensor(nrecv, dtype=torch.int64, device=dev)
        # every local rank's grid co-resident: the device's CTA capacity split between them
        self.ctas = ctas or max(1, _f2m.p2p_max_ctas(b) // len(ranks))
        self.per = {}
        for r in ranks:
            rp, sp, speer, sdst = p2p_plan_arrays(plans, r)
            t = lambda x: torch.from_numpy(np.ascontiguousarray(x if len(x) else np.zeros(1, np.int32))).to(dev)  # noqa: E731
            self.per[r] = dict(rp=t(rp), nr=len(rp), sp=t(sp), speer=t(speer), sdst=t(sdst), ns=len(sp),
                               a=torch.empty(stride * world, dtype=torch.float64, device=dev),
                               b=torch.empty(stride * world, dtype=torch.float64, device=dev),
                               ctl=torch.zeros(_f2m.p2p_ctl_bytes() // 8 + 1, dtype=torch.int64, device=dev),
                               stream=torch.cuda.Stream(dev))

    def launch(self, lam0_full: torch.Tensor, threshold: float, max_sweeps: int, ev_start=None, ev_end=None) -> None:
        """Zero the exchange buffers, synchronise the ranks, launch every local rank's kernel
        (optionally bracketed by CUDA events on the current stream)."""
        for r in self.ranks:
            self.recv_bufs[r].zero_()
            self.boards[r].zero_()
            self.per[r]["a"].copy_(lam0_full)
        torch.cuda.synchronize(self.dev)  # buffers zeroed before any rank publishes
        if not self.local:
            import torch.distributed as dist
            dist.barrier(group=self.comm.group)
        cur = torch.cuda.current_stream(self.dev)
        if ev_start is not None:
            ev_start.record(cur)
        for r in self.ranks:
            q = self.per[r]
            q["stream"].wait_stream(cur)
            self.shards[r].p2p_launch(q["rp"].data_ptr(), q["nr"], self.recv_bufs[r].data_ptr(), q["sp"].data_ptr(),
                                      q["speer"].data_ptr(), q["sdst"].data_ptr(), q["ns"], self.peer_recv.data_ptr(),
                                      self.peer_nrecv.data_ptr(), self.boards[r].data_ptr(),
                                      self.peer_board.data_ptr(), q["a"].data_ptr(), q["b"].data_ptr(),
                                      float(threshold), int(max_sweeps), self.ctas, q["ctl"].data_ptr(),
                                      q["stream"].cuda_stream)
        for r in self.ranks:
            cur.wait_stream(self.per[r]["stream"])
        if ev_end is not None:
            ev_end.record(cur)

    def collect(self):
        """After launch() completed: (lam_full in position order, result dict), on every rank."""
        n, stride, world = self.n, self.stride, self.world
        lam_full = torch.zeros(stride * world, dtype=torch.float64, device=self.dev)
        res = None
        for r in self.ranks:
            res_r = self._f2m.p2p_result(self.per[r]["ctl"].data_ptr())
            assert res is None or (res_r["sweeps"], res_r["converged"]) == (res["sweeps"], res["converged"])
            res = res_r
            out = self.per[r]["b"] if res_r["out_buffer"] else self.per[r]["a"]
            lo, hi = r * stride, min((r + 1) * stride, n)
            lam_full[lo:hi] = out[lo:hi]
        if not self.local:  # every rank holds its own rows: assemble the full vector
            mine = lam_full[self.comm.rank * stride:(self.comm.rank + 1) * stride].clone()
            self.comm.all_gather(lam_full, [mine])
        return lam_full, res

    def run(self, lam0_full: torch.Tensor, threshold: float, max_sweeps: int):
        self.launch(lam0_full, threshold, max_sweeps)
        torch.cuda.synchronize(self.dev)
        return self.collect()


def _solve_duals_p2p(graph, comm, eps, max_sweeps, b, eta, update, init, threshold):
    from . import _f2m

    if comm is None:
        comm = TorchDistComm()
    dev = torch.device("cuda", torch.cuda.current_device())
    sched = ShardedP2P(graph, comm, b, eta, update)
    n, stride, world = sched.n, sched.stride, sched.world
    if threshold is None:
        threshold = eps * graph.mean_cost()  # dual.cpp:221 (host fp64 product, no FMA)
    lam0 = torch.zeros(stride * world, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev).cuda_stream
    if n > 0:
        _f2m.initial_state_positions(graph, lam0.data_ptr(), b, init, stream)
    if max_sweeps > 0 and n > 0:
        lam_full, res = sched.run(lam0, threshold, max_sweeps)
    else:
        lam_full, res = lam0, {"converged": False, "sweeps": 0, "final_max_abs_delta": float("inf")}
    ids = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    if n > 0:
        _f2m.positions_to_ids(graph, lam_full.data_ptr(), ids.data_ptr(), stream)
    report = {"converged": res["converged"], "sweeps": res["sweeps"],
              "final_max_abs_delta": res["final_max_abs_delta"], "world": world, "stride": stride,
              "exchange": "p2p", "halo_values": sched.halo_values}
    return ids[:n].cpu().numpy(), report


def gather_ranges(comm, vec: torch.Tensor, lo: int, hi: int, width: int) -> None:
    """Every rank owns the contiguous range vec[lo:hi] (ranges of different lengths, at most
    `width`); afterwards every rank's `vec` holds all ranks' ranges. One padded all-gather over
    comm's group: each rank contributes [lo, hi, values..., padding]."""
    mine = torch.zeros(width + 2, dtype=vec.dtype, device=vec.device)
    mine[0], mine[1] = float(lo), float(hi)
    mine[2:2 + hi - lo] = vec[lo:hi]
    allv = torch.empty((comm.world, width + 2), dtype=vec.dtype, device=vec.device)
    comm.all_gather(allv.view(-1), [mine])
    for q in range(comm.world):
        a, z = int(allv[q, 0].item()), int(allv[q, 1].item())
        vec[a:z] = allv[q, 2:2 + z - a]


class ShardedResident:
    """The one-GPU partition-resident sweep kernel (k_gdp_sweep5) spread over ranks: the graph is
    built once per rank with world x Gp partition CTAs (f2m_set_sweep_partition), rank r runs CTAs
    [r*Gp, (r+1)*Gp) plus its own convergence master, and every boundary multiplier and CTA sweep
    max is stored into every rank's LL / max ring (NVLink peer memory via torch symmetric memory;
    plain device memory for LocalComm ranks, which then run concurrently on one GPU). No barrier,
    host work or collective per sweep; bit-identical to one GPU.

    ShardedResident(inst, k, comm).run(threshold, max_sweeps) -> (lambda in node-id order, report).

    In-process ranks (LocalComm) run `world` cooperative launches on separate streams of ONE GPU
    that spin on each other's LL words. CUDA guarantees co-residency only inside one cooperative
    grid, so this form is a test configuration: it relies on the launches running concurrently
    (they fit: world x (Gp + 1) CTAs <= SMs) and the 20 s in-kernel watchdog turns a serialised
    schedule into an error instead of a hang. Production multi-GPU runs one process per GPU
    (TorchDistComm) or one host thread over several GPUs (EngineConfig::num_gpus, multi.cu)."""

    def __init__(self, inst, k: int, comm, b: int = 2, eta: float = 0.5, update: str = "midpoint",
                 init: str = "local-midpoint", ctas_per_rank: int = 0):
        import paper_2011_08170_b200 as f2m
        from . import _f2m

        self._f2m = _f2m
        self.comm = comm
        nslices = -(-int(inst.points_array().shape[0]) // 32)
        if nslices < comm.world:
            raise ValueError(f"ShardedResident: {nslices} 32-row slices cannot be split over {comm.world} ranks "
                             f"(every rank needs at least one partition CTA); use fewer ranks")
        self.b, self.eta, self.update = b, eta, update
        self.dev = dev = torch.device("cuda", torch.cuda.current_device())
        self.world = world = comm.world
        self.local = local = not isinstance(comm, TorchDistComm)
        self.ranks = list(range(world)) if local else [comm.rank]
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        # one SM per rank's master; in-process ranks share this device's SMs
        gp = ctas_per_rank or (max(1, (sms - world) // world) if local else sms - 1)
        gp = max(1, min(gp, nslices // world))  # every partition CTA needs at least one 32-row slice
        _f2m.set_sweep_partition(world * gp)
        try:
            self.graph = f2m.build_knn_graph(inst, k)
        finally:
            _f2m.set_sweep_partition(0)
        g = self.graph
        self.n = n = g.n
        self.info = {r: _f2m.sweep_multi_info(g, r, world) for r in self.ranks}
        i0 = next(iter(self.info.values()))
        self.g_total = i0["g_total"]
        self.resident = bool(i0["resident"])
        self._words = (int(i0["ll_words"]), int(i0["cmax_words"]))
        self.connected = False
        if local:
            self.connect()
        self.lam0 = torch.zeros(max(n, 1), dtype=torch.float64, device=dev)
        if n > 0:
            _f2m.initial_state_positions(g, self.lam0.data_ptr(), b, init, torch.cuda.current_stream(dev).cuda_stream)
        self.rings = {r: torch.empty((8, max(n, 1)), dtype=torch.float64, device=dev) for r in self.ranks}
        self.ctl = {r: torch.zeros(_f2m.sweep_multi_ctl_bytes() // 8 + 1, dtype=torch.int64, device=dev)
                    for r in self.ranks}
        self.streams = {r: torch.cuda.Stream(dev) for r in self.ranks}

    def connect(self) -> None:
        """Allocate the LL / max rings and exchange their addresses. Across processes this is a
        collective (torch symmetric-memory rendezvous over comm's group): every rank must reach
        it, so callers that can fail per rank agree first (bench.py `_agree`); everything before
        it in __init__ is rank-local."""
        if self.connected:
            return
        dev, world = self.dev, self.world
        llw, cmw = self._words
        if self.local:
            self.ll = {r: torch.zeros(llw, dtype=torch.int64, device=dev) for r in self.ranks}
            self.cmax = {r: torch.zeros(cmw, dtype=torch.int64, device=dev) for r in self.ranks}
            ll_ptrs = [self.ll[r].data_ptr() for r in range(world)]
            cm_ptrs = [self.cmax[r].data_ptr() for r in range(world)]
        else:
            import torch.distributed as dist
            import torch.distributed._symmetric_memory as symm_mem

            group = self.comm.group if self.comm.group is not None else dist.group.WORLD
            lb = symm_mem.empty(llw, dtype=torch.int64, device=dev)
            cb = symm_mem.empty(cmw, dtype=torch.int64, device=dev)
            self._handles = (symm_mem.rendezvous(lb, group), symm_mem.rendezvous(cb, group))
            self.ll, self.cmax = {self.comm.rank: lb}, {self.comm.rank: cb}
            ll_ptrs, cm_ptrs = list(self._handles[0].buffer_ptrs), list(self._handles[1].buffer_ptrs)
        self.ll_peers = torch.tensor(ll_ptrs, dtype=torch.int64, device=dev)
        self.cmax_peers = torch.tensor(cm_ptrs, dtype=torch.int64, device=dev)
        self.connected = True

    def launch(self, threshold: float, max_sweeps: int, ev_start=None, ev_end=None) -> None:
        self.connect()
        for r in self.ranks:
            self.ll[r].zero_()
            self.cmax[r].zero_()
            self.rings[r][0].copy_(self.lam0)
        torch.cuda.synchronize(self.dev)  # rings zeroed on every rank before any rank publishes
        if not self.local:
            import torch.distributed as dist
            dist.barrier(group=self.comm.group)
        cur = torch.cuda.current_stream(self.dev)
        if ev_start is not None:
            ev_start.record(cur)
        for r in self.ranks:
            st = self.streams[r]
            st.wait_stream(cur)
            self._f2m.sweep_multi_launch(self.graph, self.b, self.eta, self.update, r, self.world,
                                         self.rings[r].data_ptr(), self.ll[r].data_ptr(), self.ll_peers.data_ptr(),
                                         self.cmax[r].data_ptr(), self.cmax_peers.data_ptr(), float(threshold),
                                         int(max_sweeps), self.ctl[r].data_ptr(), st.cuda_stream)
        for r in self.ranks:
            cur.wait_stream(self.streams[r])
        if ev_end is not None:
            ev_end.record(cur)

    def collect_local(self):
        """This process's ranks' results (no collective): (lambda in position order with this
        process's ranges filled, result dict). Raises on a watchdog abort."""
        n = self.n
        lam_pos = torch.zeros(max(n, 1), dtype=torch.float64, device=self.dev)
        res = None
        for r in self.ranks:
            rr = self._f2m.sweep_multi_result(self.ctl[r].data_ptr())
            assert res is None or (rr["sweeps"], rr["converged"]) == (res["sweeps"], res["converged"])
            res = rr
            lo, hi = self.info[r]["begin"], self.info[r]["end"]
            lam_pos[lo:hi] = self.rings[r][rr["out_buffer"]][lo:hi]
        return lam_pos, res

    def gather(self, lam_pos):
        """Every rank's owned range into every rank's vector (collective across processes)."""
        if not self.local:  # ranks own contiguous position ranges of different lengths: pad, gather
            if not hasattr(self, "_width"):  # the longest rank range (identical topology on every rank)
                spans = [self._f2m.sweep_multi_info(self.graph, q, self.world) for q in range(self.world)]
                self._width = max(1, max(x["end"] - x["begin"] for x in spans))
            lo, hi = self.info[self.comm.rank]["begin"], self.info[self.comm.rank]["end"]
            gather_ranges(self.comm, lam_pos, lo, hi, self._width)
        return lam_pos

    def collect(self):
        lam_pos, res = self.collect_local()
        return self.gather(lam_pos), res

    def to_ids(self, lam_pos):
        """Position-order multipliers -> node-id order (host numpy array)."""
        ids = torch.empty(max(self.n, 1), dtype=torch.float64, device=self.dev)
        if self.n > 0:
            self._f2m.positions_to_ids(self.graph, lam_pos.data_ptr(), ids.data_ptr(),
                                       torch.cuda.current_stream(self.dev).cuda_stream)
        return ids[:self.n].cpu().numpy()

    def peer_bytes_per_sweep(self):
        """Peer-memory (NVLink) bytes each rank stores into other ranks per sweep: LL words of the
        boundary multipliers other ranks read + the CTA maxima, 16 B each (max over ranks)."""
        return max(self._f2m.sweep_multi_traffic(self.graph, q, self.world)["bytes_per_sweep"]
                   for q in range(self.world))

    def run(self, threshold: float, max_sweeps: int):
        self.launch(threshold, max_sweeps)
        torch.cuda.synchronize(self.dev)
        lam_pos, res = self.collect()
        report = {"converged": res["converged"], "sweeps": res["sweeps"],
                  "final_max_abs_delta": res["final_max_abs_delta"], "world": self.world, "g_total": self.g_total,
                  "exchange": "resident"}
        return self.to_ids(lam_pos), report


def solve_duals_resident(inst, k: int, comm=None, eps: float = 1e-9, max_sweeps: int = 20000, **kw):
    """solve_duals (dual.cpp:210-246) of build_knn_graph(inst, k) with the multi-GPU
    partition-resident sweep kernel (ShardedResident). Returns (lambda, report) on every rank."""
    if comm is None:
        comm = TorchDistComm()
    eng = ShardedResident(inst, k, comm, **kw)
    threshold = eps * eng.graph.mean_cost()  # dual.cpp:221 (host fp64 product, no FMA)
    return eng.run(threshold, max_sweeps)
