#!/usr/bin/env python
"""NCCL slab parity (tests/test_gpu_parity.py::test_nccl_two_ranks_bitwise): under torchrun with
N ranks, one GPU each, every case runs the real multi-rank path of libmhd — NCCL send/recv halo
on the comm stream overlapped with the interior launch, ncclAllReduce for dt, counters and bad
cells (mhd_api.cu fused_stage / whole_fill_ghosts / reduce_and_read) — and each rank compares its
slab with the same problem run as one domain on its own GPU: dt log and state bitwise, global
counters equal.  The "-push" cases run the halo push instead (MHD_HALO_PUSH=1: boundary planes
stored by the stage epilogue into the neighbours' NCCL symmetric windows, an LSA barrier per
stage).  Rank 0 writes the results as JSON (--out).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/nccl_parity.py --out r.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def cases(I, world):
    nz = 8 * world
    ot = I.orszag_tang_3d(32).replace(n=(40, 21, nz), hi=(1.0, 1.0, nz / 32.0))
    yield "ot3d-plm-rk2", ot, I.with_noise(I.orszag_tang_3d_ic(ot), ot)
    w = ot.replace(limiter=I.WENOZ, stepper=I.RK3)
    yield "ot3d-wenoz-rk3", w, I.with_noise(I.orszag_tang_3d_ic(w), w)
    c = I.ct_problem(I.orszag_tang_3d(16).replace(n=(16, 16, nz), hi=(1.0, 1.0, nz / 16.0)))
    yield "ot3d-ct-rk2", c, np.ascontiguousarray(I.orszag_tang_3d_ic(c.replace(ct=0, glm=1))[:8])
    b = I.blast_3d(16, cubes=world)
    yield "blast-weak", b, I.blast_3d_ic(b)
    o = ot.replace(bc=(I.PERIODIC, I.PERIODIC, I.OUTFLOW))
    yield "ot3d-outflow-z", o, I.with_noise(I.orszag_tang_3d_ic(o), o)
    # the halo push over NCCL symmetric windows (MHD_HALO_PUSH=1; fused stages only)
    yield "ot3d-plm-rk2-push", ot, I.with_noise(I.orszag_tang_3d_ic(ot), ot)
    r3 = ot.replace(stepper=I.RK3)
    yield "ot3d-plm-rk3-push", r3, I.with_noise(I.orszag_tang_3d_ic(r3), r3)
    yield "blast-weak-push", b, I.blast_3d_ic(b)
    yield "ot3d-outflow-z-push", o, I.with_noise(I.orszag_tang_3d_ic(o), o)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=4)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2510_24175_b200 import inputs as I
    from paper_2510_24175_b200 import mhd

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    res = []
    for name, p, U0 in cases(I, world):
        s1 = mhd.Solver(p, device=local)
        s1.set_state(np.ascontiguousarray(U0))
        log1 = s1.run(args.steps)
        U1, d1 = s1.get_state(), s1.diag()
        s1.destroy()
        obj = [mhd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        push = name.endswith("-push")
        if push:
            os.environ["MHD_HALO_PUSH"] = "1"
        try:
            s = mhd.Solver(p, rank=rank, nranks=world, device=local, nccl_id=obj[0])
        finally:
            os.environ.pop("MHD_HALO_PUSH", None)
        z0, nz = s.offset[2], s.extent[2]
        pushed = s.halo_push
        s.set_state(np.ascontiguousarray(U0[:, z0:z0 + nz]))
        logP = s.run(args.steps)
        UP, dP = s.get_state(), s.diag()
        s.destroy()
        ok = bool(np.array_equal(log1, logP) and np.array_equal(U1[:, z0:z0 + nz], UP) and
                  all(d1[k] == dP[k] for k in ("p_floors", "plm_fallbacks", "hlld_to_hll")))
        flag = torch.tensor([1 if ok else 0], device="cuda")
        dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        res.append({"case": name, "bitwise": bool(flag.item()), "global": list(p.n), "ranks": world,
                    "steps": args.steps, **({"halo_push_active": pushed} if push else {})})
    if rank == 0:
        line = json.dumps({"cases": res})
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(line)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
