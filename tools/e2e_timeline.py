#!/usr/bin/env python
"""Copy/kernel timeline of the end-to-end loop bench.py times for its `e2e` number (pinned host
state in, step, pinned host state out, every step) through torch.profiler's CUPTI trace: per copy
its duration and achieved GB/s, the overlap of the two directions, and the gaps between them —
where the e2e step time goes beyond the PCIe copies themselves.  One JSON line.

  python tools/e2e_timeline.py [--size 512] [--workload blast3d] [--steps 3]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--size", type=int, default=512)
    ap.add_argument("--workload", default="blast3d")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--trace", default=None)
    args = ap.parse_args()
    import torch
    from torch.profiler import ProfilerActivity, profile
    import bench
    from paper_2510_24175_b200 import mhd
    p = bench.build_problem(args.workload, 1, args.size, "plm-rk2", "weak")
    U0 = bench.build_ic(args.workload, p, 0, p.n[2])
    s = mhd.Solver(p, stream=torch.cuda.current_stream())
    Uh = torch.from_numpy(U0).pin_memory()
    Uo = torch.empty_like(Uh).pin_memory()
    s.set_state(U0)
    s.set_state_async(Uh)
    s.step(s.compute_dt())
    s.get_state_async(Uo)
    s.io_join()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        e0.record()
        for _ in range(args.steps):
            s.set_state_async(Uh)
            s.step(s.compute_dt())
            s.get_state_async(Uo)
        s.io_join()
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    path = args.trace or "/tmp/e2e_trace.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X"]
    gpu = sorted([e for e in ev if e.get("cat") in ("kernel", "gpu_memcpy")], key=lambda e: e["ts"])
    t0 = gpu[0]["ts"] if gpu else 0.0
    h2d = [e for e in gpu if e["cat"] == "gpu_memcpy" and "HtoD" in e["name"]]
    d2h = [e for e in gpu if e["cat"] == "gpu_memcpy" and "DtoH" in e["name"] and e["dur"] > 1000]
    nbytes = Uh.numel() * 8

    def span(e):
        return (e["ts"] - t0) / 1e3, (e["ts"] + e["dur"] - t0) / 1e3

    def ov(a, b):
        return max(0.0, min(a[1], b[1]) - max(a[0], b[0]))
    hs, ds = [span(e) for e in h2d if e["dur"] > 1000], [span(e) for e in d2h]
    both = sum(ov(a, b) for a in hs for b in ds)
    kern = [e for e in gpu if e["cat"] == "kernel"]
    out = {"workload": args.workload, "size": args.size, "steps": args.steps, "ms_per_step": ms / args.steps,
           "bytes_per_copy": nbytes,
           "h2d_ms": [round(b - a, 2) for a, b in hs], "d2h_ms": [round(b - a, 2) for a, b in ds],
           "h2d_gbps": [round(nbytes / ((b - a) * 1e6), 1) for a, b in hs],
           "d2h_gbps": [round(nbytes / ((b - a) * 1e6), 1) for a, b in ds],
           "h2d_spans_ms": [(round(a, 1), round(b, 1)) for a, b in hs],
           "d2h_spans_ms": [(round(a, 1), round(b, 1)) for a, b in ds],
           "both_directions_overlap_ms": round(both, 1),
           "kernel_ms_total": round(sum(e["dur"] for e in kern) / 1e3, 1),
           "kernels": sorted({e["name"][:50] for e in kern})}
    print(json.dumps(out), flush=True)
    s.destroy()


if __name__ == "__main__":
    main()
