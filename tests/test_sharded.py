"""Node-sharded multi-GPU GDP: the sharded solve must be bit-identical to the
single-process solve for every world size.

CPU (world 2, gloo, two processes): the collective schedules of paper_2011_08170_b200/sharded.py
(all-gather: run_sharded_jacobi; halo exchange: ShardedJacobiHalo) driven by a numpy restatement
of a shard's Jacobi rows, against the C oracle's solve_duals (pinned to the reference's golden
vectors).
GPU: the CUDA shard kernel + the same schedule with in-process shards (LocalComm, worlds 1..8) and
through torch.distributed/NCCL (world 1), against the persistent one-GPU solver.
"""
import os
import socket

import numpy as np
import pytest
import torch

from oracle import oracle as orc  # checker only


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _shard_rows(g, begin, end):
    """Padded incident lists of nodes [begin, end): neighbour ids and costs (+inf padding)."""
    deg = np.zeros(g.n, np.int64)
    np.add.at(deg, g.eu, 1)
    np.add.at(deg, g.ev, 1)
    rows = end - begin
    width = int(deg[begin:end].max()) if rows else 1
    nb = np.repeat(np.arange(begin, end)[:, None], width, axis=1)
    cost = np.full((rows, width), np.inf)
    fill = np.zeros(rows, np.int64)
    for u, v, c in zip(g.eu, g.ev, g.cost):
        for a, b in ((u, v), (v, u)):
            if begin <= a < end:
                r = a - begin
                nb[r, fill[r]] = b
                cost[r, fill[r]] = c
                fill[r] += 1
    return nb, cost


def _numpy_sweep(nb, cost, begin, end, b=2, eta=0.5):
    """One Jacobi sweep of rows [begin, end) in the reference's arithmetic (dual.cpp:33-68,
    140-161): values (c - l_v) - l_u, the b-th and (b+1)-th smallest, midpoint update."""
    def fn(lam_full, out, bits):
        lam = lam_full.numpy()
        lv = lam[begin:end]
        val = (cost - lv[:, None]) - lam[nb]
        s = np.sort(val, axis=1)
        d = 0.5 * (s[:, b - 1] + s[:, b])
        o = out.numpy()
        o[:] = 0.0
        o[: end - begin] = lv + eta * d
        m = np.max(np.abs(d)) if len(d) else 0.0
        mb = np.array([m], np.float64).view(np.int64)[0]
        bits.copy_(torch.maximum(bits, torch.tensor(mb, dtype=torch.int64)))
    return fn


def _gloo_worker(rank, world, port, n, seed, eps, max_sweeps, out_path):
    import torch.distributed as dist

    from paper_2011_08170_b200.sharded import TorchDistComm, run_sharded_jacobi

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = orc.build_knn_graph(orc.generate_instance(n, seed), 10)
        stride = (g.n + world - 1) // world
        begin, end = min(g.n, rank * stride), min(g.n, (rank + 1) * stride)
        nb, cost = _shard_rows(g, begin, end)
        lam0 = torch.zeros(stride * world, dtype=torch.float64)
        lam0[: g.n] = torch.from_numpy(orc.initial_state(g))
        res = run_sharded_jacobi([_numpy_sweep(nb, cost, begin, end)], TorchDistComm(), stride, lam0,
                                 eps * g.mean_cost(), max_sweeps, chunk=7)
        if rank == 0:
            np.savez(out_path, lam=res.lam_full[: g.n].numpy(), sweeps=res.sweeps, conv=res.converged,
                     fmax=res.final_max_abs_delta, record=np.array(res.record))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("max_sweeps", [20000, 37])
def test_gloo_world2_matches_oracle(tmp_path, max_sweeps):
    import torch.multiprocessing as mp

    n, seed, eps = 1000, 3, 1e-9
    out = str(tmp_path / "res.npz")
    mp.spawn(_gloo_worker, args=(2, _free_port(), n, seed, eps, max_sweeps, out), nprocs=2, join=True)
    r = np.load(out)
    g = orc.build_knn_graph(orc.generate_instance(n, seed), 10)
    lam, rep = orc.solve_duals(g, eps=eps, max_sweeps=max_sweeps)
    assert int(r["sweeps"]) == rep["sweeps"]
    assert bool(r["conv"]) == rep["converged"]
    assert float(r["fmax"]) == rep["final_max_abs_delta"]
    assert np.array_equal(r["lam"], lam)
    assert len(r["record"]) >= rep["sweeps"]


def test_schedule_chunk_boundaries():
    """Converging exactly at a chunk boundary and mid-chunk returns that sweep's vector."""
    from paper_2011_08170_b200.sharded import LocalComm, run_sharded_jacobi

    g = orc.build_knn_graph(orc.generate_instance(300, 5), 10)
    lam_ref, rep = orc.solve_duals(g, eps=1e-9)
    for world in (1, 3):
        stride = (g.n + world - 1) // world
        fns = []
        for r in range(world):
            b, e = min(g.n, r * stride), min(g.n, (r + 1) * stride)
            nb, cost = _shard_rows(g, b, e)
            fns.append(_numpy_sweep(nb, cost, b, e))
        for chunk in (1, 2, rep["sweeps"], rep["sweeps"] - 1, 64):
            lam0 = torch.zeros(stride * world, dtype=torch.float64)
            lam0[: g.n] = torch.from_numpy(orc.initial_state(g))
            res = run_sharded_jacobi(fns, LocalComm(world), stride, lam0, 1e-9 * g.mean_cost(), 20000, chunk)
            assert res.sweeps == rep["sweeps"] and res.converged
            assert np.array_equal(res.lam_full[: g.n].numpy(), lam_ref)


# ----------------------------------------------------------------------------------- GPU
def _gpu_graph(n, seed):
    import paper_2011_08170_b200 as f2m

    return f2m.build_knn_graph(f2m.generate_instance(n, seed), 10)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_local_shards_match_single_gpu(world):
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_sharded

    g = _gpu_graph(10000, 1)
    st, rep = f2m.solve_duals(g)
    lam, srep = solve_duals_sharded(g, LocalComm(world), chunk=16, exchange="allgather")
    assert srep["sweeps"] == rep["sweeps"] == 3165
    assert srep["converged"] and rep["converged"]
    assert srep["final_max_abs_delta"] == rep["final_max_abs_delta"]
    assert np.array_equal(lam, np.asarray(st.lam))


@pytest.mark.gpu
def test_local_shards_truncated_matches_jacobi_sweeps():
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_sharded

    g = _gpu_graph(5000, 2)
    st = f2m.make_initial_state(g)
    rec, _ = f2m.jacobi_sweeps(g, st, 45)
    lam, srep = solve_duals_sharded(g, LocalComm(4), max_sweeps=45, chunk=8, threshold=-1.0)
    assert srep["sweeps"] == 45 and not srep["converged"]
    assert np.array_equal(lam, np.asarray(st.lam))
    assert np.array_equal(np.asarray(srep["record"]), np.asarray(rec))


@pytest.mark.gpu
def test_nccl_world1_matches_single_gpu():
    import torch.distributed as dist

    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import TorchDistComm, solve_duals_sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = _gpu_graph(3000, 4)
        st, rep = f2m.solve_duals(g)
        lam, srep = solve_duals_sharded(g, TorchDistComm(), chunk=32, exchange="allgather")
        assert srep["sweeps"] == rep["sweeps"]
        assert np.array_equal(lam, np.asarray(st.lam))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ halo exchange
def _halo_gloo_worker(rank, world, port, n, seed, eps, out_path):
    import torch.distributed as dist

    from paper_2011_08170_b200.sharded import ShardedJacobiHalo, TorchDistComm, halo_plans

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = orc.build_knn_graph(orc.generate_instance(n, seed), 10)
        stride = (g.n + world - 1) // world
        begin, end = min(g.n, rank * stride), min(g.n, (rank + 1) * stride)
        nb, cost = _shard_rows(g, begin, end)
        plans = halo_plans(g.n, world, stride, g.eu, g.ev)  # positions == ids on the CPU
        lam0 = torch.zeros(stride * world, dtype=torch.float64)
        lam0[: g.n] = torch.from_numpy(orc.initial_state(g))

        def pack(src, idx, dst, count):
            dst.copy_(src[idx.long()])

        def unpack(src, idx, dst, count):
            dst[idx.long()] = src

        sched = ShardedJacobiHalo([_numpy_sweep(nb, cost, begin, end)], TorchDistComm(), stride, plans, [rank],
                                  "cpu", pack, unpack, chunk=5)
        sweeps, conv, fmax, record, slot = sched.run([lam0], eps * g.mean_cost(), 20000)
        full = torch.empty(stride * world, dtype=torch.float64)
        dist.all_gather_into_tensor(full, sched.rings[0][slot][rank * stride:(rank + 1) * stride].contiguous())
        if rank == 0:
            np.savez(out_path, lam=full[: g.n].numpy(), sweeps=sweeps, conv=conv, fmax=fmax,
                     halo=sum(len(p.recv_pos) for p in plans))
    finally:
        dist.destroy_process_group()


def test_halo_plans_match_neighbourhoods():
    from paper_2011_08170_b200.sharded import halo_plans

    g = orc.build_knn_graph(orc.generate_instance(500, 8), 10)
    world = 4
    stride = (g.n + world - 1) // world
    plans = halo_plans(g.n, world, stride, g.eu, g.ev)
    for r in range(world):
        b, e = r * stride, min(g.n, (r + 1) * stride)
        need = set()
        for u, v in zip(g.eu, g.ev):
            if b <= u < e and not b <= v < e:
                need.add(int(v))
            if b <= v < e and not b <= u < e:
                need.add(int(u))
        assert plans[r].recv_pos.tolist() == sorted(need)
        for q in range(world):
            assert plans[r].send_counts[q] == plans[q].recv_counts[r]


def test_gloo_world2_halo_matches_oracle(tmp_path):
    import torch.multiprocessing as mp

    n, seed, eps = 1000, 3, 1e-9
    out = str(tmp_path / "res.npz")
    mp.spawn(_halo_gloo_worker, args=(2, _free_port(), n, seed, eps, out), nprocs=2, join=True)
    r = np.load(out)
    g = orc.build_knn_graph(orc.generate_instance(n, seed), 10)
    lam, rep = orc.solve_duals(g, eps=eps)
    assert int(r["sweeps"]) == rep["sweeps"] and bool(r["conv"])
    assert float(r["fmax"]) == rep["final_max_abs_delta"]
    assert np.array_equal(r["lam"], lam)
    assert 0 < int(r["halo"]) < n


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_local_shards_halo_match_single_gpu(world):
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_sharded

    g = _gpu_graph(10000, 1)
    st, rep = f2m.solve_duals(g)
    lam, srep = solve_duals_sharded(g, LocalComm(world), chunk=16, exchange="halo")
    assert srep["sweeps"] == rep["sweeps"] == 3165
    assert srep["final_max_abs_delta"] == rep["final_max_abs_delta"]
    assert np.array_equal(lam, np.asarray(st.lam))


@pytest.mark.gpu
def test_nccl_world1_halo_matches_single_gpu():
    import torch.distributed as dist

    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import TorchDistComm, solve_duals_sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = _gpu_graph(3000, 4)
        st, rep = f2m.solve_duals(g)
        lam, srep = solve_duals_sharded(g, TorchDistComm(), chunk=32, exchange="halo")
        assert srep["sweeps"] == rep["sweeps"]
        assert np.array_equal(lam, np.asarray(st.lam))
    finally:
        dist.destroy_process_group()


# ------------------------------------------------------------------ fused peer-memory solve
def test_p2p_plan_arrays_match_receive_lists():
    """Every value a rank sends lands at the index its reader expects for that position."""
    from paper_2011_08170_b200.sharded import halo_plans, p2p_plan_arrays

    rng = np.random.default_rng(5)
    n, world = 3000, 5
    stride = -(-n // world)
    u = rng.integers(0, n, 20000)
    v = (u + rng.integers(1, 200, 20000)) % n
    plans = halo_plans(n, world, stride, u, v)
    recv = [p2p_plan_arrays(plans, r)[0] for r in range(world)]
    for q in range(world):
        _, sp, speer, sdst = p2p_plan_arrays(plans, q)
        assert np.all(sp // stride == q)  # only own positions are sent
        for pos, r, d in zip(sp, speer, sdst):
            assert recv[r][d] == pos
    assert sum(len(p2p_plan_arrays(plans, q)[1]) for q in range(world)) == sum(len(x) for x in recv)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_local_shards_p2p_match_single_gpu(world):
    """world concurrent persistent kernels on one GPU exchanging through device memory."""
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_sharded

    g = _gpu_graph(10000, 1)
    st, rep = f2m.solve_duals(g)
    lam, srep = solve_duals_sharded(g, LocalComm(world), exchange="p2p")
    assert srep["sweeps"] == rep["sweeps"] == 3165
    assert srep["converged"] and rep["converged"]
    assert srep["final_max_abs_delta"] == rep["final_max_abs_delta"]
    assert np.array_equal(lam, np.asarray(st.lam))


@pytest.mark.gpu
def test_local_shards_p2p_truncated_and_fixed_count():
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_sharded

    g = _gpu_graph(5000, 2)
    st = f2m.make_initial_state(g)
    f2m.jacobi_sweeps(g, st, 45)
    lam, srep = solve_duals_sharded(g, LocalComm(4), max_sweeps=45, threshold=-1.0, exchange="p2p")
    assert srep["sweeps"] == 45 and not srep["converged"]
    assert np.array_equal(lam, np.asarray(st.lam))


@pytest.mark.gpu
def test_nccl_world1_p2p_matches_single_gpu():
    """The multi-process path (torch symmetric memory for the peer buffers) at world 1."""
    import torch.distributed as dist

    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import TorchDistComm, solve_duals_sharded

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        g = _gpu_graph(3000, 4)
        st, rep = f2m.solve_duals(g)
        lam, srep = solve_duals_sharded(g, TorchDistComm(), exchange="p2p")
        assert srep["sweeps"] == rep["sweeps"]
        assert np.array_equal(lam, np.asarray(st.lam))
    finally:
        dist.destroy_process_group()


def test_p2p_plan_arrays_degenerate_worlds():
    """World 1 (nothing crosses) and a rank that owns no row of any cross edge."""
    from paper_2011_08170_b200.sharded import halo_plans, p2p_plan_arrays

    u = np.array([0, 1, 2, 3], np.int64)
    v = np.array([1, 2, 3, 0], np.int64)
    plans = halo_plans(4, 1, 4, u, v)
    rp, sp, speer, sdst = p2p_plan_arrays(plans, 0)
    assert len(rp) == len(sp) == len(speer) == len(sdst) == 0
    # world 3 over 6 positions, edges only inside rank 0 and between ranks 1 and 2
    u = np.array([0, 2, 3], np.int64)
    v = np.array([1, 4, 5], np.int64)
    plans = halo_plans(6, 3, 2, u, v)
    rp0, sp0, _, _ = p2p_plan_arrays(plans, 0)
    assert len(rp0) == 0 and len(sp0) == 0
    rp1, sp1, speer1, sdst1 = p2p_plan_arrays(plans, 1)
    rp2, sp2, speer2, sdst2 = p2p_plan_arrays(plans, 2)
    assert sorted(rp1.tolist()) == [4, 5] and sorted(rp2.tolist()) == [2, 3]
    for sp, speer, sdst in ((sp1, speer1, sdst1), (sp2, speer2, sdst2)):
        for pos, r, d in zip(sp, speer, sdst):
            assert [rp1, rp2][r - 1][d] == pos


# ------------------------------------------------------------------ multi-GPU partition-resident kernel
@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 4])
def test_local_resident_ranks_match_single_gpu(world):
    """world concurrent launches of the partition-resident sweep kernel on one GPU, each running
    its share of a world x Gp partition and storing LL / max rings into every rank's copy."""
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_resident

    inst = f2m.generate_instance(10000, 1, 1000.0)
    g = f2m.build_knn_graph(inst, 10)
    st, rep = f2m.solve_duals(g)
    lam, srep = solve_duals_resident(inst, 10, LocalComm(world))
    assert srep["sweeps"] == rep["sweeps"] == 3165 and srep["converged"]
    assert srep["final_max_abs_delta"] == rep["final_max_abs_delta"]
    assert np.array_equal(lam, np.asarray(st.lam))


@pytest.mark.gpu
def test_local_resident_ranks_small_graph():
    """A graph with fewer 32-row slices than SMs: the per-rank partition shrinks to fit."""
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, solve_duals_resident

    inst = f2m.generate_instance(1000, 3, 1000.0)
    st, rep = f2m.solve_duals(f2m.build_knn_graph(inst, 10))
    lam, srep = solve_duals_resident(inst, 10, LocalComm(4))
    assert srep["sweeps"] == rep["sweeps"] and srep["g_total"] <= 32
    assert np.array_equal(lam, np.asarray(st.lam))


@pytest.mark.gpu
def test_local_resident_ranks_100k_and_truncated():
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, ShardedResident

    inst = f2m.generate_instance(100000, 1, 1000.0)
    g = f2m.build_knn_graph(inst, 10)
    st, rep = f2m.solve_duals(g, max_sweeps=200000)
    eng = ShardedResident(inst, 10, LocalComm(2))
    lam, srep = eng.run(1e-9 * eng.graph.mean_cost(), 200000)
    assert srep["sweeps"] == rep["sweeps"] == 6359
    assert np.array_equal(lam, np.asarray(st.lam))
    st2 = f2m.make_initial_state(g)
    f2m.jacobi_sweeps(g, st2, 57)
    lam2, srep2 = eng.run(-1.0, 57)
    assert srep2["sweeps"] == 57 and not srep2["converged"]
    assert np.array_equal(lam2, np.asarray(st2.lam))


@pytest.mark.gpu
def test_local_resident_8_ranks_2m_fixed_sweeps():
    """BASELINE configs[4]'s shape through the torch-driven engine: 2M cities over 8 in-process
    ranks (8 x 17 partition CTAs sharing the one GPU, streaming form), 64 fixed sweeps,
    bit-exact against the one-GPU kernel's multipliers."""
    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import LocalComm, ShardedResident

    inst = f2m.generate_instance(2_000_000, 1, 1000.0)
    g = f2m.build_knn_graph(inst, 10)
    st = f2m.make_initial_state(g)
    f2m.jacobi_sweeps(g, st, 64)
    del g
    eng = ShardedResident(inst, 10, LocalComm(8))
    lam, srep = eng.run(-1.0, 64)
    assert srep["sweeps"] == 64 and not srep["converged"] and srep["world"] == 8
    assert np.array_equal(lam, np.asarray(st.lam))


@pytest.mark.gpu
def test_nccl_world1_resident_matches_single_gpu():
    import torch.distributed as dist

    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import TorchDistComm, solve_duals_resident

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        inst = f2m.generate_instance(3000, 4, 1000.0)
        st, rep = f2m.solve_duals(f2m.build_knn_graph(inst, 10))
        lam, srep = solve_duals_resident(inst, 10, TorchDistComm())
        assert srep["sweeps"] == rep["sweeps"]
        assert np.array_equal(lam, np.asarray(st.lam))
    finally:
        dist.destroy_process_group()


def _gather_ranges_worker(rank, world, port, out_path):
    import torch.distributed as dist

    from paper_2011_08170_b200.sharded import TorchDistComm, gather_ranges

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # a subgroup of ranks {1, 2}: the gather must run over the subgroup only (rank 0 never joins)
        sub = dist.new_group([1, 2])
        if rank in (1, 2):
            comm = TorchDistComm(group=sub)
            n = 11
            spans = [(0, 7), (7, 11)]  # ragged ranges, width 7
            lo, hi = spans[comm.rank]
            vec = torch.full((n,), -1.0, dtype=torch.float64)
            vec[lo:hi] = torch.arange(lo, hi, dtype=torch.float64) * 10 + comm.rank
            gather_ranges(comm, vec, lo, hi, 7)
            np.save(f"{out_path}.{rank}.npy", vec.numpy())
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_gloo_gather_ranges_subgroup(tmp_path):
    """ShardedResident.collect's padded gather of ragged rank ranges, over a process subgroup
    (world 3, group {1, 2}): every member ends with all ranges."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "g")
    mp.spawn(_gather_ranges_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    want = np.array([i * 10 + (0 if i < 7 else 1) for i in range(11)], np.float64)
    for r in (1, 2):
        assert np.array_equal(np.load(f"{out}.{r}.npy"), want)


def _agree_worker(rank, world, port, out_path):
    import sys

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        import bench

        # a leg whose setup fails on rank 1 only: every rank must see "not ok" and skip together,
        # and the next collective (the barrier) must still complete on all ranks
        first = bench._agree(rank != 1)
        second = bench._agree(True)
        dist.barrier()
        np.save(f"{out_path}.{rank}.npy", np.array([first, second]))
    finally:
        dist.destroy_process_group()


def test_gloo_bench_agreement_skips_together(tmp_path):
    """bench.py's cross-rank agreement before every multi-rank leg's collectives (world 3, gloo):
    one failing rank makes all ranks skip the leg instead of leaving the others blocked."""
    import torch.multiprocessing as mp

    out = str(tmp_path / "a")
    mp.spawn(_agree_worker, args=(3, _free_port(), out), nprocs=3, join=True)
    for r in range(3):
        assert np.load(f"{out}.{r}.npy").tolist() == [False, True]
