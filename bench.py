#!/usr/bin/env python
"""bench.py — zone-updates/s of the fp64 3D ideal-MHD Godunov step on B200 (BASELINE.json metric).

Workload: BASELINE configs[2], 3D Orszag-Tang 256^3 periodic, PLM-MC + HLLD + GLM,
SSP-RK2, CFL 0.4 — the single-GPU roofline run — per GPU.  With N GPUs the job is weak-scaled:
a 256 x 256 x (256 N) periodic box (z extent N), one 256^3 z-slab per rank, halo exchange by NCCL
send/recv and the dt reduction by ncclAllReduce(max) inside the library.

A step is one user-loop iteration: dt = mhd_compute_dt() (k_dt + 16-byte read-back) then
mhd_step(dt) (z ghost planes + 2 fused stage kernels).  A zone-update is one interior cell
advanced one full step (R25).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mhd|reference]

--impl reference times the CPU oracle (the reference arm of this tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "zone-updates/sec (fp64 3D ideal MHD) at 1/2/4/8 B200; HBM GB/s fraction"
UNIT = "zone-updates/s"
NV = 9
# algorithmic HBM bytes of one fused stage launch per interior cell:
# stage 1 reads U^n, writes U*; stage 2 reads U*, reads U^n, writes U^n+1  -> 144 + 216 = 360 B/zu
STAGE_BYTES_PER_CELL = {1: 2 * NV * 8, 2: 3 * NV * 8}
# algorithmic fp64 operations (+ - * / sqrt, each counted once) of one interior cell in one RK
# stage, 3D PLM-MC + HLLD(F* path) + GLM, no redundant work:
# cons2prim 19 + 3 x PLM-MC 81 + 3 x face solve 243 + update 81 (+ 19 for the RK2 average in stage 2)
FLOPS_CELL_STAGE = {1: 19 + 3 * 81 + 3 * 243 + 81, 2: 19 + 3 * 81 + 3 * 243 + 81 + 19}
# WENO-Z: 71 ops per field and side -> 1278 per cell-direction; RK3 weights 27 per stage
_WZ = 19 + 3 * 1278 + 3 * 243 + 81
FLOPS_PER_LAUNCH_AVG = {"plm-rk2": (FLOPS_CELL_STAGE[1] + FLOPS_CELL_STAGE[2]) / 2.0,
                        "wenoz-rk3": (_WZ + (_WZ + 27) + (_WZ + 28)) / 3.0}
BYTES_PER_LAUNCH_AVG = {"plm-rk2": (2 * NV * 8 + 3 * NV * 8) / 2.0, "wenoz-rk3": (2 * NV * 8 + 3 * NV * 8 * 2) / 3.0}
# CT stages are five launches (prim, 3 face passes, update); their roofline is not the fused kernel's
FLOPS_PER_LAUNCH_AVG.update({"ct-plm-rk2": None, "ct-wenoz-rk3": None})
BYTES_PER_LAUNCH_AVG.update({"ct-plm-rk2": None, "ct-wenoz-rk3": None})
N_SM, FP64_LANES_PER_SM = 148, 64


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """SM clocks, power and clock-event (throttle) reasons during the timed region
    (B200_PROFILING.md's clocks line).  NVML polled every 20 ms from a thread (the timed region is
    ~0.1 s, shorter than nvidia-smi's start-up), one sample taken on entry and one on exit;
    falls back to `nvidia-smi -lms 200` without NVML."""

    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int, period: float = 0.02):
        self.index, self.period = index, period
        self.rows = []  # (sm_mhz, max_mhz, power_w, {reasons})
        self.proc = None
        self.nv = None
        self.stop = threading.Event()

    def _nvml_sample(self):
        nv, h = self.nv, self.h
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        pw = nv.nvmlDeviceGetPowerUsage(h) / 1000.0
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        masks = (nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap)
        self.rows.append((float(sm), float(mx), pw, {n for n, m in zip(self.NAMES, masks) if bits & m}))

    def _nvml_loop(self):
        while not self.stop.is_set():
            try:
                self._nvml_sample()
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv, self.h = pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._nvml_sample()
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nv = None
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._smi_read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def _smi_read(self):
        for line in self.proc.stdout:
            p = [x.strip() for x in line.split(",")]
            if len(p) >= 7:
                num = lambda x: float(x) if x.replace(".", "").isdigit() else None
                self.rows.append((num(p[0]), num(p[1]), num(p[2]),
                                  {n for i, n in enumerate(self.NAMES) if p[3 + i].lower() == "active"}))

    def __exit__(self, *exc):
        if self.nv is not None:
            self.stop.set()
            self.t.join(timeout=1)
            try:
                self._nvml_sample()
            except Exception:
                pass
        elif self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [r[0] for r in self.rows if r[0] is not None]
        mx = [r[1] for r in self.rows if r[1] is not None]
        pw = [r[2] for r in self.rows if r[2] is not None]
        reasons = sorted(set().union(*(r[3] for r in self.rows)))
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "power_w_max": max(pw) if pw else None,
                "source": "nvml" if self.nv is not None else "nvidia-smi"}


SCHEMES = {
    "plm-rk2": "PLM-MC + HLLD + GLM, SSP-RK2, CFL 0.4",
    "wenoz-rk3": "WENOZ + HLLD + GLM, SSP-RK3, CFL 0.4",
    "ct-plm-rk2": "PLM-MC + HLLD + constrained transport, SSP-RK2, CFL 0.4",
    "ct-wenoz-rk3": "WENOZ + HLLD + constrained transport, SSP-RK3, CFL 0.4",
}
WORKLOADS = {
    "ot3d": "3D Orszag-Tang (BASELINE configs[2] at 256^3, configs[4] at 1024^3)",
    "blast3d": "3D MHD blast, one blast per GPU cube (BASELINE configs[3], 512^3 per GPU)",
    "cpa3d": "3D circularly polarised Alfven wave along the diagonal (SURVEY §8(f) row 1)",
}


def build_problem(workload: str, n_gpus: int, n: int, scheme: str = "plm-rk2"):
    """per-GPU n^3 cube; with N GPUs the box is n x n x (n N) with z extent N (weak scaling)"""
    from paper_2510_24175_b200 import inputs as I
    if workload == "ot3d":
        p = I.orszag_tang_3d(n, nz=n * n_gpus, z_extent=float(n_gpus))
    elif workload == "blast3d":
        p = I.blast_3d(n, cubes=n_gpus)
    elif workload == "cpa3d":
        p = I.cpa_3d(n).replace(n=(n, n, n * n_gpus), hi=(1.0, 1.0, float(n_gpus)))
    else:
        raise ValueError(workload)
    if scheme.endswith("wenoz-rk3"):
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
    if scheme.startswith("ct-"):
        p = I.ct_problem(p)
    return p


def build_ic(workload: str, p, z0: int, z1: int):
    from paper_2510_24175_b200 import inputs as I
    return I.workload_ic(workload, p, z0, z1)


def cpu_info():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        model = [l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")]
        return model[0] if model else "unknown"
    except Exception:
        return "unknown"


def oracle_sample(workload: str, n: int, nz_s: int, steps: int, warmup: int, scheme: str = "plm-rk2"):
    """The CPU oracle, as it stands, on a bounded sample of the workload: the first nz_s planes of
    the n^3 initial condition as a periodic n x n x nz_s slab (same per-cell work)."""
    import oracle
    full = build_problem(workload, 1, n, scheme)
    dz = (full.hi[2] - full.lo[2]) / full.n[2]
    p = full.replace(n=(n, n, nz_s), hi=(full.hi[0], full.hi[1], full.lo[2] + nz_s * dz))
    U = build_ic(workload, full, 0, nz_s)
    o = oracle.Oracle(p, U)
    for _ in range(warmup):
        dt, ch = o.compute_dt()
        o.step(dt, ch)
    t0 = time.perf_counter()
    for _ in range(steps):
        dt, ch = o.compute_dt()
        o.step(dt, ch)
    el = time.perf_counter() - t0
    return p.cells * steps / el, el, oracle.num_threads(), p


def run_reference(args, rank, world):
    if rank != 0:
        return
    n = args.n
    nz_s = max(4, min(n, (256 ** 3 // 4) // (n * n)))  # ~4.2 M cells per step
    v, el, cores, p = oracle_sample(args.workload, n, nz_s, args.steps, args.warmup, args.scheme)
    sample = (f"CPU oracle (oracle/mhd_oracle.c, gcc -O2 -ffp-contract=off, OpenMP {cores} threads), "
              f"{args.steps} timed steps after {args.warmup} warm-up of a {n}x{n}x{nz_s} periodic slab of the "
              f"{n}^3 {args.workload} IC ({nz_s}/{n} of the workload's planes per step)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.workload}_{n}^3_per_gpu", "cells_per_step": p.cells, "sample": f"{n}x{n}x{nz_s}",
                       "parallelism": "host cores"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu": cpu_info()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mhd", choices=["mhd", "reference"])
    ap.add_argument("--n", type=int, default=256, help="cells per axis per GPU (configs[2]: 256)")
    ap.add_argument("--workload", default="ot3d", choices=sorted(WORKLOADS))
    ap.add_argument("--scheme", default="plm-rk2", choices=sorted(SCHEMES),
                    help="plm-rk2: the north star's PLM-MC + HLLD + GLM + SSP-RK2 (default); wenoz-rk3: the "
                         "paper's strong-scaling WENOZ + HLLD + GLM + SSP-RK3 (PAPER.md:270); ct-wenoz-rk3: its "
                         "weak-scaling WENOZ + HLLD + CT + SSP-RK3 (PAPER.md:179, one GPU)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-planes", type=int, default=256, help="cpu_baseline sample: planes of the grid")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "mhd" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2510_24175_b200 import inputs as I
    from paper_2510_24175_b200 import mhd

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    p = build_problem(args.workload, world, args.n, args.scheme)
    nz_loc = p.n[2] // world
    nccl_id = None
    if world > 1:
        obj = [mhd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    s = mhd.Solver(p, rank=rank, nranks=world, device=local_rank, nccl_id=nccl_id)
    stream = torch.cuda.current_stream()
    s.set_stream(stream)
    U0 = build_ic(args.workload, p, rank * nz_loc, (rank + 1) * nz_loc)
    if U0.nbytes <= 8 << 30:
        s.set_state(torch.from_numpy(U0).cuda())
    else:  # 1024^3: host copy-in (the library stages through its second array: no third array)
        s.set_state(U0)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        s.step(s.compute_dt())
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the library's stream = torch's current stream)
    nst = 3 if p.stepper else 2
    s.profile_enable(True, capacity=args.steps * (nst + 1) + 8)  # one event pair per stage and per dt pass
    with ClockSampler(local_rank) as clk:
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        s.run(args.steps)  # mhd_run: the native compute_dt / step loop
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
    ms = e0.elapsed_time(e1)
    prof = s.profile_read()
    s.profile_enable(False)
    ms_max = max_over_ranks(ms)
    cells = p.cells
    value = cells * args.steps / (ms_max * 1e-3)
    diag = s.diag()

    # ---- roofline of the dominant kernel (fused stage kernel, ~97% of the step)
    pk, pk_kind = peaks()
    stage_ms, stage_n = prof["stage"]
    dt_ms, dt_n = prof["dt"]
    cells_loc = p.cells // world
    stage_avg_s = stage_ms * 1e-3 / max(stage_n, 1)
    ct = args.scheme.startswith("ct-")
    flops_launch = cells_loc * (FLOPS_PER_LAUNCH_AVG[args.scheme] or FLOPS_PER_LAUNCH_AVG["plm-rk2"])
    bytes_launch = cells_loc * (BYTES_PER_LAUNCH_AVG[args.scheme] or BYTES_PER_LAUNCH_AVG["plm-rk2"])
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    fp64_peak = N_SM * FP64_LANES_PER_SM * sm_mhz * 1e6 / 1e12  # TFLOP/s, 1 op per lane per clock (no FMA)
    achieved = flops_launch / stage_avg_s / 1e12
    ncu = {}  # the committed one-launch ncu capture of this scheme's stage kernel (tools/refresh_profiles.sh)
    summ = "ncu_stage_summary.json" if args.scheme == "plm-rk2" else f"ncu_stage_summary_{args.scheme}.json"
    try:
        with open(os.path.join(ROOT, "profiles", summ)) as f:
            ncu = json.load(f)
        if args.n != 256 or args.workload != "ot3d":
            ncu = {}  # captured on the default workload only
    except Exception:
        pass
    roof = {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
            "traffic": ncu.get("dram_bytes_per_launch"),
            "kernel": "k_stage (fused cons2prim + PLM + GLM + HLL/HLLD + flux divergence + RK2 update)",
            "peak_kind": f"derived: {N_SM} SM x {FP64_LANES_PER_SM} FP64 lanes x {sm_mhz:.0f} MHz (recipe has no FMA)",
            "flops_per_cell_stage_avg": FLOPS_PER_LAUNCH_AVG[args.scheme], "algorithmic_flops_per_launch": flops_launch,
            "stage_ms_per_launch": stage_avg_s * 1e3, "stage_launches": stage_n,
            "stage_share_of_step": stage_ms / max(ms, 1e-9), "dt_ms_per_launch": dt_ms / max(dt_n, 1),
            "hbm": {"achieved": bytes_launch / stage_avg_s / 1e9, "peak": pk.get("hbm_gbs"), "unit": "GB/s",
                    "frac": bytes_launch / stage_avg_s / 1e9 / pk.get("hbm_gbs", 6537.3), "peak_kind": pk_kind,
                    "algorithmic_bytes_per_launch": bytes_launch},
            "ncu": ncu or None}
    if args.scheme != "plm-rk2":  # 3D GLM WENO-Z: the split stage (mhd_split.cu); ncu: its x-face kernel
        roof["kernel"] = ("split WENO-Z stage (k_sp_prim + k_sp_face_x + k_sp_face_m<1> + k_sp_face_m<2> + "
                          "k_sp_update; stage_ms and achieved are per 5-launch stage)")
        roof["traffic"] = None
    if ct:  # the timed unit is a 5-launch stage, not the fused kernel: report the stage time only
        roof = {"bound": "alu", "achieved": None, "peak": fp64_peak, "unit": "TFLOP/s", "frac": None,
                "traffic": None, "kernel": "CT stage (k_ct_prim + 3 x k_ct_face + k_ct_update)",
                "stage_ms_per_launch": stage_avg_s * 1e3, "stage_launches": stage_n,
                "stage_share_of_step": stage_ms / max(ms, 1e-9)}

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if not args.no_e2e and U0.nbytes <= 8 << 30:
        Uh = torch.from_numpy(U0).pin_memory()
        Uo = torch.empty_like(Uh).pin_memory()
        ke = max(1, args.steps)
        s.set_state_async(Uh)  # warm-up: the staging arrays and copy streams are created on first use
        s.step(s.compute_dt())
        s.get_state_async(Uo)
        s.io_join()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(ke):  # the pipelined public API: step n's copies overlap its neighbours' kernels
            s.set_state_async(Uh)
            s.step(s.compute_dt())
            s.get_state_async(Uo)
        s.io_join()  # the stream waits for the last download before f1
        f1.record(stream)
        torch.cuda.synchronize()
        barrier()
        ems = max_over_ranks(f0.elapsed_time(f1))
        e2e = {"value": cells * ke / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": Uh.numel() * 8,
               "d2h_bytes_per_step": Uo.numel() * 8, "steps": ke,
               "what": "per step: mhd_set_state_async(pinned host U) + mhd_compute_dt + mhd_step + "
                       "mhd_get_state_async(pinned host); mhd_io_join before the stop event"}

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        nz_s = min(args.cpu_planes, args.n, max(4, (256 ** 3) // (args.n * args.n)))
        v, el, cores, pp = oracle_sample(args.workload, args.n, nz_s, 1, 0, args.scheme)
        cpu = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_info(),
               "sample": f"1 step (compute_dt + RK2 step) of a {args.n}x{args.n}x{nz_s} periodic slab of the "
                         f"{args.n}^3 {args.workload} IC, {el:.1f} s on {cores} OpenMP threads"}

    s.destroy()
    # kernels per step: k_dt + the dt read-back store, and per RK stage the fused k_stage, or five
    # launches for CT and for the 3D GLM WENO-Z
    # split stage (mhd_split.cu; MHD_FUSED_WENOZ=1 selects the fused kernel)
    split = (p.limiter == I.WENOZ and p.n[2] > 1 and not p.ct and os.environ.get("MHD_FUSED_WENOZ") != "1")
    # with slabs the fused stage is three launches (interior, then the two boundary ranges)
    launches_per_stage = 5 if (p.ct or split) else (3 if world > 1 else 1)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": f"{args.workload}_{args.n}^3_per_gpu ({WORKLOADS[args.workload]}; global {p.n[0]}x{p.n[1]}x{p.n[2]})",
                           "scheme": SCHEMES[args.scheme], "cells": cells,
                           "parallelism": f"z-slab x{world}", "l2": "inputs larger than L2 (2 x 1.27 GB arrays per GPU)"},
                "roofline": roof, "clocks": clk.summary(), "gpu_launches": args.steps * (2 + (3 if p.stepper else 2) * launches_per_stage),
                "e2e": e2e, "cpu_baseline": cpu, "diag": diag,
                "lib": mhd.version()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
