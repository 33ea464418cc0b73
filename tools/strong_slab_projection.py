#!/usr/bin/env python
"""Per-GPU step time of the strong-scaling run (BASELINE configs[4]: Orszag-Tang 1024^3 split into
N z slabs), measured on ONE GPU: one rank's slab, 1024 x 1024 x 1024/N, run through the slab
schedule with the rank as its own periodic z neighbour (MHD_NCCL_SELF=1: one-rank NCCL
communicator; the halo by ncclSend/ncclRecv beside the interior launch, or with --halo push by
the stage epilogue into the NCCL symmetric window + an LSA barrier per stage).  Compared with
the whole 1024^3 on one GPU it projects the compute side of the strong-scaling efficiency,
E(N) ~ T(1) / (N T_slab(N)); what it leaves out is the NVLink transfer itself (2 x g planes per
neighbour per stage, overlapped with the stage) and the cross-GPU latency of the dt allreduce and
the barrier.  One JSON line per N.

  python tools/strong_slab_projection.py --N 1 2 4 8 [--halo push] [--steps 4] [--scheme wenoz-rk3]
(the split WENO-Z stage keeps the exchange: it waits for the halo, then runs its five launches;
WENO-Z + RK3 at 1024^3 needs N >= 4 to fit — three state arrays and the split scratch — so
--N 4 8 reports the efficiency relative to N = 4)
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=1024)
    ap.add_argument("--N", type=int, nargs="*", default=[1, 2, 4, 8])
    ap.add_argument("--halo", default="exchange", choices=["exchange", "push"])
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--scheme", default="plm-rk2", choices=["plm-rk2", "wenoz-rk3"],
                    help="wenoz-rk3: the paper's strong-scaling scheme (split WENO-Z stage, GLM, SSP-RK3)")
    args = ap.parse_args()
    import torch
    from paper_2510_24175_b200 import inputs as I
    from paper_2510_24175_b200 import mhd
    n = args.size
    base = None
    for N in args.N:
        nz = n // N
        p = I.orszag_tang_3d(n).replace(n=(n, n, nz), hi=(1.0, 1.0, nz / n))
        if args.scheme == "wenoz-rk3":
            p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
        env = {}
        if N > 1:  # the slab schedule (a one-slab run keeps the plain whole-domain path)
            env["MHD_NCCL_SELF"] = "1"
            if args.halo == "push":
                env["MHD_HALO_PUSH"] = "1"
        os.environ.update(env)
        try:
            s = mhd.Solver(p, stream=torch.cuda.current_stream())
        finally:
            for k in env:
                os.environ.pop(k, None)
        s.set_state(I.workload_ic("ot3d", p, 0, nz))
        s.run(2)
        s.profile_enable(True, capacity=12 * args.steps + 8)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s.run(args.steps)
        e1.record()
        torch.cuda.synchronize()
        pr = s.profile_read_stages()
        line = {"global": [n, n, n], "N": N, "slab": [n, n, nz], "halo": args.halo if N > 1 else None,
                "halo_push_active": s.halo_push, "steps": args.steps,
                "ms_per_step": e0.elapsed_time(e1) / args.steps,
                "scheme": args.scheme,
                "stage_ms_per_step": (pr["stage1"][0] + pr["stage2"][0] + pr["stage3"][0]) / args.steps,
                "dt_ms_per_step": pr["dt"][0] / args.steps,
                "halo_exposed_ms_per_step": pr["halo_exposed"][0] / args.steps}
        if base is None:  # the first N listed is the reference (1 where the whole box fits one GPU)
            base = (N, line["ms_per_step"])
        key = "projected_E" if base[0] == 1 else f"projected_E_rel_to_N{base[0]}"
        line[key] = base[0] * base[1] / (N * line["ms_per_step"])
        print(json.dumps(line), flush=True)
        s.destroy()
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
