#!/usr/bin/env python
"""Kernel timeline of a few steps (nsys is not in this image): torch.profiler's CUPTI activity
trace records every kernel and copy of the process — libmhd's stage / dt kernels, NCCL's kernels,
the halo copies — with start/end timestamps and streams.  Writes a Chrome trace (chrome://tracing
or Perfetto) and one JSON line with, per RK stage, the interior launch, the halo transfer and the
boundary launches and how much of the halo ran under the interior launch.

  MHD_NCCL_SELF=1 python tools/timeline.py --out profiles/r02_timeline_nccl_self.json
      one periodic rank, the z halo through NCCL (send/recv to itself) on the comm stream
  python tools/timeline.py --slabs 4 --out ...   in-process slabs (device-copy halo)
  python -m torch.distributed.run --nproc-per-node 8 --master-addr 127.0.0.1 tools/timeline.py --size 1024 \
      --out timeline.json      NCCL ranks: the global n^3 box in z slabs, one trace per rank
      (timeline.rank<r>.json) with the NCCL send/recv kernels beside the interior launches
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def intervals(trace):
    ev = [e for e in trace.get("traceEvents", []) if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
    out = []
    for e in ev:
        out.append({"name": e["name"], "cat": e["cat"], "ts": float(e["ts"]), "end": float(e["ts"]) + float(e["dur"]),
                    "stream": e.get("args", {}).get("stream")})
    return sorted(out, key=lambda e: e["ts"])


def overlap(a, b):
    return max(0.0, min(a["end"], b["end"]) - max(a["ts"], b["ts"]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", "--n", dest="n", type=int, default=256)  # (--n is torchrun's under torchrun)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--slabs", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out/timeline.json")
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    from paper_2510_24175_b200 import inputs as I
    from paper_2510_24175_b200 import mhd
    p = I.orszag_tang_3d(args.n)
    world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
    if world > 1:  # NCCL ranks (torchrun): the global n^3 box split into z slabs, one trace per rank
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", rank))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [mhd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        solver = mhd.Solver(p, rank=rank, nranks=world, device=local, nccl_id=obj[0],
                            stream=torch.cuda.current_stream())
        z0, nz = solver.offset[2], solver.extent[2]
        U0 = I.workload_ic("ot3d", p, z0, z0 + nz)
        root, ext = os.path.splitext(args.out)
        args.out = f"{root}.rank{rank}{ext}"
    elif args.slabs > 1:
        U0 = I.workload_ic("ot3d", p, 0, p.n[2])
        solver = mhd.SolverGroup(p, args.slabs)
        solver.slabs[0].set_stream(torch.cuda.current_stream())
    else:
        U0 = I.workload_ic("ot3d", p, 0, p.n[2])
        solver = mhd.Solver(p, stream=torch.cuda.current_stream())
    solver.set_state(U0)
    solver.run(2)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        solver.run(args.steps)
        torch.cuda.synchronize()
    os.makedirs(os.path.dirname(os.path.abspath(args.out)), exist_ok=True)
    prof.export_chrome_trace(args.out)
    trace = json.load(open(args.out))
    iv = intervals(trace)
    stages = [e for e in iv if "k_stage" in e["name"]]
    halo = [e for e in iv if "nccl" in e["name"].lower() or e["cat"] == "gpu_memcpy"]
    barriers = [e["end"] - e["ts"] for e in iv if "k_push_barrier" in e["name"]]  # (MHD_HALO_PUSH)
    summary = {"n": args.n, "slabs": args.slabs, "ranks": world, "rank": rank, "steps": args.steps,
               "nccl_self": os.environ.get("MHD_NCCL_SELF") == "1",
               "stage_launches": len(stages), "halo_events": len(halo),
               "kernels": sorted({e["name"][:60] for e in iv}), "stages": [],
               "push_barrier_us": barriers}
    # per stage: the long (interior) launch and the halo events that ran beside it
    for s in stages:
        if s["end"] - s["ts"] < 0.25 * max(x["end"] - x["ts"] for x in stages):
            continue  # a boundary launch
        h = [e for e in halo if e["end"] > s["ts"] - 50 and e["ts"] < s["end"]]
        tot = sum(e["end"] - e["ts"] for e in h)
        ov = sum(overlap(e, s) for e in h)
        summary["stages"].append({"interior_us": s["end"] - s["ts"], "halo_us": tot,
                                  "halo_under_interior_frac": ov / tot if tot > 0 else None,
                                  "halo": [(e["name"][:40], round(e["end"] - e["ts"], 1), e["stream"]) for e in h]})
    print(json.dumps(summary), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
