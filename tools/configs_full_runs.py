#!/usr/bin/env python
"""Full runs of the small BASELINE configs on the GPU and on the CPU oracle side by side
(SURVEY.md §8(d).9): configs[0] Brio-Wu 512 cells to t = 0.1 and configs[1] OT-2D 512^2 to
t = 0.5, plus a few steps of configs[2] (OT-3D 256^3) on the oracle.  Reports zone-updates/s on
the GPU (the native loop mhd_run, device time by CUDA events) and on the host cores (all threads,
OMP_PROC_BIND=close; and one thread), the speed-up, and whether the two dt logs and final
states are bitwise equal.  One JSON line per config.

  python tools/configs_full_runs.py [--skip-1thread]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-1thread", action="store_true")
    args = ap.parse_args()
    import torch
    import oracle
    from paper_2510_24175_b200 import inputs as I
    from paper_2510_24175_b200 import mhd
    cases = [("configs[0] Brio-Wu 512, PLM-MC + HLL, RK2, to t = 0.1", I.brio_wu(512), None, 0.1),
             ("configs[1] OT-2D 512^2, PLM-MC + HLLD + GLM, RK2, to t = 0.5", I.orszag_tang_2d(512), None, 0.5),
             ("configs[2] OT-3D 256^3, PLM-MC + HLLD + GLM, RK2, 3 steps", I.orszag_tang_3d(256), 3, 0.0)]
    for name, p, nsteps, t_end in cases:
        if p.n[2] > 1:
            U0 = I.workload_ic("ot3d", p, 0, p.n[2])
        elif p.n[1] > 1:
            U0 = I.orszag_tang_2d_ic(p)
        else:
            U0 = I.brio_wu_ic(p)
        steps_cap = nsteps or 1_000_000
        # GPU: the native loop, device time
        s = mhd.Solver(p, stream=torch.cuda.current_stream())
        s.set_state(np.ascontiguousarray(U0))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        log_g = s.run(steps_cap, t_end)
        e1.record()
        torch.cuda.synchronize()
        gms = e0.elapsed_time(e1)
        Ug = s.get_state()
        s.destroy()
        zu = p.cells * len(log_g)
        # CPU oracle, all threads
        o = oracle.Oracle(p, U0)
        t0 = time.perf_counter()
        log_o = o.run(steps_cap, t_end)
        el = time.perf_counter() - t0
        cores = oracle.num_threads()
        line = {"config": name, "cells": p.cells, "steps": len(log_g), "zone_updates": zu,
                "gpu": {"ms": gms, "zone_updates_per_s": zu / (gms * 1e-3), "timing": "CUDA events around mhd_run"},
                "cpu_oracle": {"s": el, "zone_updates_per_s": zu / el, "threads": cores,
                               "omp": {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES")}},
                "bitwise_equal": bool(np.array_equal(log_g, log_o) and np.array_equal(Ug, o.U))}
        if not args.skip_1thread:
            n1 = min(len(log_o), max(1, int(len(log_o) * min(1.0, 20.0 / max(el * cores, 1e-9)))))
            oracle.set_num_threads(1)
            o1 = oracle.Oracle(p, U0)
            t0 = time.perf_counter()
            o1.run(n1, 0.0)
            el1 = time.perf_counter() - t0
            oracle.set_num_threads(cores)
            line["cpu_oracle"]["one_thread_zone_updates_per_s"] = p.cells * n1 / el1
            line["cpu_oracle"]["one_thread_steps"] = n1
        line["gpu_over_cpu"] = line["gpu"]["zone_updates_per_s"] / line["cpu_oracle"]["zone_updates_per_s"]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
