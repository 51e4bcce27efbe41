#!/usr/bin/env python
"""Node-sharded GDP sweep throughput: per-sweep time of the sharded schedule
(CUDA shard kernel + NCCL all-gather of lambda + chunked max all-reduce).

  python tools/bench_sharded.py --n 2000000 --sweeps 200              # 1 GPU (NCCL world 1)
  torchrun --nproc-per-node 8 --master-addr 127.0.0.1 tools/bench_sharded.py --n 2000000
  python tools/bench_sharded.py --n 200000 --local 4                  # 4 simulated shards, 1 GPU

Runs exactly --sweeps Jacobi sweeps (threshold -1) after --warmup, timed with CUDA events on the
launching stream, max over ranks; prints one JSON line on rank 0. With --solve it instead runs
the convergent solve and checks sweeps/lambda against the persistent one-GPU kernel (rank 0).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2_000_000)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--clustered", action="store_true")
    ap.add_argument("--sweeps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--chunk", type=int, default=32)
    ap.add_argument("--local", type=int, default=0, help="simulate this many shards in one process")
    ap.add_argument("--solve", action="store_true")
    ap.add_argument("--exchange", default="halo", choices=["halo", "allgather", "p2p", "resident"])
    args = ap.parse_args()

    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    import torch.distributed as dist

    import paper_2011_08170_b200 as f2m
    from paper_2011_08170_b200.sharded import (LocalComm, ShardedJacobi, ShardedP2P, ShardedResident,
                                               TorchDistComm, make_halo_schedule, solve_duals_sharded)
    from paper_2011_08170_b200 import _f2m

    f2m.set_device(local)
    if args.local:
        comm = LocalComm(args.local)
    else:
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29533")
        dist.init_process_group("nccl", rank=rank, world_size=ws, device_id=torch.device("cuda", local))
        comm = TorchDistComm()
    gen = f2m.generate_clustered_instance if args.clustered else f2m.generate_instance
    if args.exchange == "resident":  # the partition-resident kernel across ranks (fixed sweep count)
        dev = torch.device("cuda", local)
        eng = ShardedResident(gen(args.n, args.seed), 10, comm)
        eng.run(-1.0, max(args.warmup, 2))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        eng.launch(-1.0, args.sweeps, e0, e1)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if not args.local:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        per = ms * 1e3 / args.sweeps
        line = {"n": args.n, "m": eng.graph.m, "world": comm.world, "exchange": "resident", "sweeps": args.sweeps,
                "us_per_sweep": per, "gdp_iterations_per_s": 1e6 / per, "g_total": eng.g_total,
                "algorithmic_GBps": eng.graph.sweep_bytes() / (per * 1e-6) / 1e9,
                "kernel": f2m.last_sweep_kernel_desc()}
        if rank == 0:
            print(json.dumps(line), flush=True)
        if not args.local:
            dist.destroy_process_group()
        return
    t0 = time.perf_counter()
    g = f2m.build_knn_graph(gen(args.n, args.seed), 10)
    t_graph = time.perf_counter() - t0
    dev = torch.device("cuda", local)
    line = {"n": args.n, "m": g.m, "world": comm.world, "clustered": args.clustered, "t_graph_s": t_graph}
    if args.solve:
        t0 = time.perf_counter()
        lam, rep = solve_duals_sharded(g, comm, chunk=args.chunk, max_sweeps=200000, exchange=args.exchange)
        torch.cuda.synchronize()
        line.update(solve_s=time.perf_counter() - t0, sweeps=rep["sweeps"], converged=rep["converged"])
        if rank == 0:
            st, r1 = f2m.solve_duals(g, max_sweeps=200000)
            line.update(one_gpu_sweeps=r1["sweeps"], bit_identical=bool((lam == st.lam).all()))
    elif args.exchange == "p2p":  # one persistent kernel per rank for all sweeps (fixed count)
        stream = torch.cuda.current_stream(dev)
        sched = ShardedP2P(g, comm)
        lam0 = torch.zeros(sched.stride * comm.world, dtype=torch.float64, device=dev)
        _f2m.initial_state_positions(g, lam0.data_ptr(), 2, "local-midpoint", stream.cuda_stream)
        sched.run(lam0, -1.0, max(args.warmup, 2))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sched.launch(lam0, -1.0, args.sweeps, e0, e1)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if not args.local:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        per = ms * 1e3 / args.sweeps
        line.update(sweeps=args.sweeps, us_per_sweep=per, gdp_iterations_per_s=1e6 / per,
                    algorithmic_GBps=g.sweep_bytes() / (per * 1e-6) / 1e9, exchange="p2p",
                    halo_values_per_sweep=sched.halo_values, ctas_per_rank=sched.ctas)
        if rank == 0:
            print(json.dumps(line), flush=True)
        if not args.local:
            dist.destroy_process_group()
        return
    elif args.exchange == "halo":
        stream = torch.cuda.current_stream(dev)
        sched, lam0, meta = make_halo_schedule(g, comm, chunk=args.chunk)
        lam0s = [lam0] * len(meta["ranks"])
        run = lambda k: sched.run(lam0s, -1.0, k)  # noqa: E731
        run(max(args.warmup, 2 * args.chunk))
        line["halo_values_per_sweep"] = meta["halo_values_per_sweep"]
    else:
        ranks = [comm.rank] if isinstance(comm, TorchDistComm) else list(range(comm.world))
        shards = [_f2m.shard_create(g, r, comm.world) for r in ranks]
        stride = shards[0].info()["stride"]
        lam0 = torch.zeros(stride * comm.world, dtype=torch.float64, device=dev)
        stream = torch.cuda.current_stream(dev)
        _f2m.initial_state_positions(g, lam0.data_ptr(), 2, "local-midpoint", stream.cuda_stream)

        def fn_of(sh):  # launches on the CURRENT stream (the capture stream inside a CUDA graph)
            return lambda lf, out, bits: sh.sweep(lf.data_ptr(), out.data_ptr(), bits.data_ptr(),
                                                  torch.cuda.current_stream(dev).cuda_stream)

        fns = [fn_of(sh) for sh in shards]
        sched = ShardedJacobi(fns, comm, stride, dev, args.chunk)
        run = lambda k: sched.run(lam0, -1.0, k)  # noqa: E731
        run(max(args.warmup, 2 * args.chunk))  # eager chunk + graph capture + replay
    if not args.solve:
        torch.cuda.synchronize()
        if not args.local:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run(args.sweeps)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if not args.local:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        per = ms * 1e3 / args.sweeps
        bytes_per_sweep = g.sweep_bytes()
        line.update(sweeps=args.sweeps, us_per_sweep=per, gdp_iterations_per_s=1e6 / per,
                    algorithmic_GBps=bytes_per_sweep / (per * 1e-6) / 1e9, chunk=args.chunk,
                    exchange=args.exchange)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if not args.local:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
