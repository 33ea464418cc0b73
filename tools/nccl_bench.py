#!/usr/bin/env python
"""NCCL microbenchmark for the slab decomposition's two collectives:
  * the halo: ncclSend/ncclRecv of one g-plane block to each ring neighbour, posted in the
    library's order (mhd_halo_plan), at the configs' message sizes — 2 planes x 9 fields x n^2
    doubles: 37.7 MB at n = 512 (configs[3]), 151 MB at n = 1024 (configs[4]), 9.4 MB at 256;
  * the dt reduction: an allreduce(max) of 16 bytes (two uint64 patterns).
Times by CUDA events on the communication stream, max over ranks; rank 0 prints one JSON line.

  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 tools/nccl_bench.py
  (--backend gloo runs the same schedule on CPU tensors, for checking the script without GPUs)
"""
import argparse
import json
import os
import time

import torch
import torch.distributed as dist


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--sizes", type=int, nargs="*", default=[256, 512, 1024])
    ap.add_argument("--ghost", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    gpu = args.backend == "nccl"
    if gpu:
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
        dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
    else:
        dist.init_process_group("gloo")
    dev = torch.device("cuda") if gpu else torch.device("cpu")
    up, down = (rank + 1) % world, (rank - 1) % world

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        if gpu:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            e0.record()
            for _ in range(args.iters):
                fn()
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.iters
        else:
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(args.iters):
                fn()
            ms = (time.perf_counter() - t0) * 1e3 / args.iters
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    out = {"world": world, "backend": args.backend, "halo": [], "allreduce_16B": None}
    for n in args.sizes:
        count = args.ghost * 9 * n * n
        bufs = [torch.zeros(count, dtype=torch.float64, device=dev) for _ in range(4)]

        def halo():
            # send top -> up, recv bottom <- down, send bottom -> down, recv top <- up (mhd_halo_plan)
            ops = [dist.P2POp(dist.isend, bufs[0], up), dist.P2POp(dist.irecv, bufs[1], down),
                   dist.P2POp(dist.isend, bufs[2], down), dist.P2POp(dist.irecv, bufs[3], up)]
            for r in dist.batch_isend_irecv(ops):
                r.wait()
        if world > 1:
            ms = timed(halo)
            mb = count * 8 / 1e6
            out["halo"].append({"n": n, "message_MB": mb, "ms": ms, "GBps_per_direction": 2 * mb / 1e3 / (ms * 1e-3)})
    red = torch.zeros(2, dtype=torch.int64, device=dev)
    out["allreduce_16B"] = {"us": timed(lambda: dist.all_reduce(red, op=dist.ReduceOp.MAX)) * 1e3}
    if rank == 0:
        print(json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
