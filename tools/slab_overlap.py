#!/usr/bin/env python
"""Exposed halo time of the slab schedule on ONE GPU (no nsys in this image): P in-process z slabs
(MHD_TRANSPORT_LOCAL) run exactly the NCCL ranks' stage schedule — interior launch on the compute
stream while the halo runs on each slab's comm stream (device copies here), then the boundary
launches — and mhd_profile_read_stages reports, per stage, the compute stream's wait for the halo
after the interior (class 4).  Prints one JSON line per P.  Under torchrun, bench.py reports the
same quantity for the NCCL transport ("halo_exposed_ms_per_step").

  python tools/slab_overlap.py --n 256 --P 2 4 8
  MHD_HALO_PUSH=1 python tools/slab_overlap.py ...   the halo pushed by each stage's epilogue
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=256)
    ap.add_argument("--P", type=int, nargs="*", default=[2, 4, 8])
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    import torch
    from paper_2510_24175_b200 import inputs as I
    from paper_2510_24175_b200 import mhd
    p = I.orszag_tang_3d(args.n)
    U0 = I.workload_ic("ot3d", p, 0, p.n[2])
    s1 = mhd.Solver(p, stream=torch.cuda.current_stream())  # P = 1 reference: one slab, no halo
    s1.set_state(U0)
    s1.run(2)
    s1.profile_enable(True, capacity=args.steps * 5 + 8)
    s1.run(args.steps)
    pr = s1.profile_read_stages()
    print(json.dumps({"n": args.n, "P": 1, "steps": args.steps,
                      "stage_ms_per_step_sum_over_slabs": (pr["stage1"][0] + pr["stage2"][0]) / args.steps,
                      "halo_exposed_ms_per_step_sum_over_slabs": 0.0}), flush=True)
    s1.destroy()
    for P in args.P:
        g = mhd.SolverGroup(p, P)
        g.slabs[0].set_stream(torch.cuda.current_stream())  # the group runs on slab 0's stream
        g.set_state(U0)
        g.run(2)
        for s in g.slabs:
            s.profile_enable(True, capacity=args.steps * 5 + 8)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.run(args.steps)
        e1.record()
        torch.cuda.synchronize()
        profs = [s.profile_read_stages() for s in g.slabs]
        halo = sum(pr["halo_exposed"][0] for pr in profs)
        stages = sum(pr["stage1"][0] + pr["stage2"][0] for pr in profs)
        print(json.dumps({"n": args.n, "P": P, "steps": args.steps, "ms_per_step": e0.elapsed_time(e1) / args.steps,
                          "stage_ms_per_step_sum_over_slabs": stages / args.steps,
                          "halo_exposed_ms_per_step_sum_over_slabs": halo / args.steps,
                          "halo_exposed_share_of_stage_time": halo / max(stages, 1e-9),
                          "halo_push": g.slabs[0].halo_push,
                          "transport": ("in-process halo push from the stage epilogue (MHD_HALO_PUSH=1)"
                                        if g.slabs[0].halo_push else
                                        "in-process device copies (MHD_TRANSPORT_LOCAL)") + ", one GPU"}), flush=True)
        g.destroy()


if __name__ == "__main__":
    main()
