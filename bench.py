#!/usr/bin/env python
"""bench.py — zone-updates/s of the fp64 3D ideal-MHD Godunov step on B200 (BASELINE.json metric).

Scaling modes (one process per GPU under torchrun, z slabs, NCCL halo exchange
and ncclAllReduce(max) for dt inside the library):
  --scaling weak   (default) BASELINE configs[3]: 3D MHD blast, 512^3 per GPU, one blast per
                   unit cube along z — the global box is 512 x 512 x 512N.  At N = 1 this is a
                   single-GPU 512^3 run of the same fused kernel.
  --scaling strong BASELINE configs[4]: 3D Orszag-Tang 1024^3 (the north star's scaling target),
                   split into N z slabs of 1024/N planes.
--workload / --size (alias --n) override the problem (e.g. --workload ot3d --size 256: configs[2], the
256^3 single-GPU roofline run; with --scaling weak the size is per GPU, with strong it is global).
Scheme (both modes): PLM-MC + HLLD + GLM, SSP-RK2, CFL 0.4 (--scheme for the paper's others).

A step is one user-loop iteration: dt = mhd_compute_dt() (k_dt + a 72-byte read-back) then
mhd_step(dt) (z ghost planes / halo + 2 fused stage kernels).  A zone-update is one interior cell
advanced one full step (R25).  The parallel efficiency E(N) = value(N) / (N value(1))
is computed from the per-N lines by the driver (tools/scaling_report.py does the same here).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--scaling weak|strong] [--impl mhd|reference]

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
# Algorithmic work of one stage launch per interior cell, per RK stage.
# HBM bytes: stage 1 reads U^n, writes U* (144 B); RK2 stage 2 reads U*, U^n, writes U^n+1 (216 B);
# RK3 stages 2 and 3 read U_in, U^n and write U_out (216 B) -> 360 B per RK2 zone-update.
# fp64 ops (+ - * / sqrt, each counted once, 3D PLM-MC + HLLD (F* path) + GLM, no redundant work):
# cons2prim 19 + 3 x PLM-MC 81 + 3 x face solve 243 + update 81 (+ 19 for the RK2 average in
# stage 2; the RK3 weights: 27 in stage 2, 28 in stage 3).  WENO-Z: 71 ops per field and side
# -> 1278 per cell-direction.
_PLM = 19 + 3 * 81 + 3 * 243 + 81
_WZ = 19 + 3 * 1278 + 3 * 243 + 81
FLOPS_PER_STAGE = {"plm-rk2": (_PLM, _PLM + 19), "wenoz-rk3": (_WZ, _WZ + 27, _WZ + 28),
                   "ct-plm-rk2": None, "ct-wenoz-rk3": None}  # (CT: five launches, no single-kernel roofline)
BYTES_PER_STAGE = {"plm-rk2": (2 * NV * 8, 3 * NV * 8), "wenoz-rk3": (2 * NV * 8, 3 * NV * 8, 3 * NV * 8),
                   "ct-plm-rk2": None, "ct-wenoz-rk3": None}
KERNELS = {"plm-rk2": "k_stage (fused cons2prim + PLM + GLM + HLL/HLLD + flux divergence + RK2 update)",
           "wenoz-rk3": "split WENO-Z stage (k_sp_prim + k_sp_face_x + k_sp_face_m<1> + k_sp_face_m<2> + k_sp_update; "
                        "times are per 5-launch stage)",
           "ct-plm-rk2": "CT stage (k_ct_prim + 3 x k_ct_face + k_ct_update)",
           "ct-wenoz-rk3": "CT stage (k_ct_prim + 3 x k_ct_face + k_ct_update)"}
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

    def _nvml_handle(self, nv):
        """the NVML handle of CUDA device `index` (by UUID: CUDA_VISIBLE_DEVICES may renumber)"""
        try:
            import torch
            u = str(torch.cuda.get_device_properties(self.index).uuid)
            return nv.nvmlDeviceGetHandleByUUID(u if u.startswith("GPU-") else "GPU-" + u)
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

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
            self.nv, self.h = pynvml, self._nvml_handle(pynvml)
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


# the two scaling modes' default problems (BASELINE.json configs[3] and configs[4])
SCALING = {"weak": ("blast3d", 512, "BASELINE configs[3]: 3D MHD blast, 512^3 per GPU (weak scaling)"),
           "strong": ("ot3d", 1024, "BASELINE configs[4]: 3D Orszag-Tang 1024^3 split over the GPUs (strong scaling)")}


def build_problem(workload: str, n_gpus: int, n: int, scheme: str = "plm-rk2", scaling: str = "weak"):
    """weak: a per-GPU n^3 cube, the box n x n x (n N) with z extent N; strong: the global n^3
    box, split into N z slabs of n/N planes by the library"""
    from paper_2510_24175_b200 import inputs as I
    if scaling == "strong":
        if n % n_gpus or n // n_gpus < 4:
            raise ValueError(f"strong scaling: {n} planes do not split into {n_gpus} slabs of >= 4")
        n_gpus_box = 1
    else:
        n_gpus_box = n_gpus
    p = _problem(I, workload, n_gpus_box, n)
    if scheme.endswith("wenoz-rk3"):
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
    if scheme.startswith("ct-"):
        p = I.ct_problem(p)
    return p


def slab_plan(p, world: int):
    """(global shape, [(rank, z0, z1)]) — the z planes each rank owns (mhd_local_box's rule)"""
    nz = p.n[2] // world
    return tuple(p.n), [(r, r * nz, (r + 1) * nz) for r in range(world)]


def _problem(I, workload, n_gpus, n):
    if workload == "ot3d":
        p = I.orszag_tang_3d(n, nz=n * n_gpus, z_extent=float(n_gpus))
    elif workload == "blast3d":
        p = I.blast_3d(n, cubes=n_gpus)
    elif workload == "cpa3d":
        p = I.cpa_3d(n).replace(n=(n, n, n * n_gpus), hi=(1.0, 1.0, float(n_gpus)))
    else:
        raise ValueError(workload)
    return p


def build_ic(workload: str, p, z0: int, z1: int):
    from paper_2510_24175_b200 import inputs as I
    return I.workload_ic(workload, p, z0, z1)


def cpu_topology():
    """(model name, sockets, cores per socket, threads per core) from lscpu"""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        kv = {l.split(":", 1)[0].strip(): l.split(":", 1)[1].strip() for l in out.splitlines() if ":" in l}
        return (kv.get("Model name", "unknown"), int(kv.get("Socket(s)", "0") or 0),
                int(kv.get("Core(s) per socket", "0") or 0), int(kv.get("Thread(s) per core", "0") or 0))
    except Exception:
        return ("unknown", 0, 0, 0)


def oracle_slab(workload: str, p, nz_s: int):
    """a bounded sample of the workload for the CPU oracle: nz_s planes around the middle of the
    first GPU's z range as a periodic n x n x nz_s box (same per-cell work; blast: through the
    blast)"""
    z0 = max(0, min(p.n[0], p.n[2]) // 2 - nz_s // 2)  # the middle of the first cube (weak) or of the box
    dz = (p.hi[2] - p.lo[2]) / p.n[2]
    ps = p.replace(n=(p.n[0], p.n[1], nz_s), lo=(p.lo[0], p.lo[1], p.lo[2] + z0 * dz),
                   hi=(p.hi[0], p.hi[1], p.lo[2] + (z0 + nz_s) * dz))
    return ps, build_ic(workload, p, z0, z0 + nz_s)


def oracle_rate(ps, U, steps: int, warmup: int, threads: int = 0):
    """zone-updates/s of the CPU oracle (as it stands) on (ps, U): `steps` timed compute_dt + step
    after `warmup`; threads = 0 keeps the OpenMP default (all host cores)"""
    import oracle
    n0 = oracle.num_threads()
    if threads:
        oracle.set_num_threads(threads)
    try:
        o = oracle.Oracle(ps, U)
        for _ in range(warmup):
            dt, ch = o.compute_dt()
            o.step(dt, ch)
        t0 = time.perf_counter()
        for _ in range(steps):
            dt, ch = o.compute_dt()
            o.step(dt, ch)
        el = time.perf_counter() - t0
        return ps.cells * steps / el, el, oracle.num_threads()
    finally:
        oracle.set_num_threads(n0)


def cpu_baseline(workload: str, p, scheme: str, steps: int = 12):
    """the oracle on all host cores (OMP_PROC_BIND=close, OMP_PLACES=cores) on
    a ~4 M-cell slab of the workload, `steps` steps, and on one core on a 1/8 slab; ~10-20 s"""
    model, sockets, cps, tpc = cpu_topology()
    n2 = p.n[0] * p.n[1]
    nz_all = max(4, min(p.n[2], (4 << 20) // n2))
    ps, U = oracle_slab(workload, p, nz_all)
    v_all, el_all, cores = oracle_rate(ps, U, steps, 0)
    nz_one = max(4, nz_all // 8)
    ps1, U1 = oracle_slab(workload, p, nz_one)
    v_one, el_one, _ = oracle_rate(ps1, U1, 1, 0, threads=1)
    return {"value": v_all, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": model, "sockets": sockets,
            "cores_per_socket": cps, "threads_per_core": tpc,
            "omp": {k: os.environ.get(k) for k in ("OMP_PROC_BIND", "OMP_PLACES")},
            "per_core_value": v_one, "speedup_all_cores": v_all / v_one,
            "sample": (f"CPU oracle (oracle/mhd_oracle.c, gcc -O2 -ffp-contract=off, OpenMP): {steps} steps "
                       f"(compute_dt + {'RK3' if p.stepper else 'RK2'} step) of a {ps.n[0]}x{ps.n[1]}x{ps.n[2]} periodic "
                       f"slab of the {workload} IC on {cores} threads ({el_all:.1f} s); per core: 1 step of a "
                       f"{ps1.n[0]}x{ps1.n[1]}x{ps1.n[2]} slab on 1 thread ({el_one:.1f} s)")}


def resolve(args):
    """the workload, n and config label of the arm (scaling-mode defaults, --workload/--n overrides)"""
    wl, n, label = SCALING[args.scaling]
    if args.workload is not None or args.n is not None:
        wl = args.workload or wl
        n = args.n or (256 if wl != "blast3d" else 512)
        label = (f"{wl} {n}^3 {'per GPU (weak scaling)' if args.scaling == 'weak' else 'global (strong scaling)'}"
                 + (" — BASELINE configs[2], the single-GPU roofline run" if (wl, n) == ("ot3d", 256) else "")
                 + (" — BASELINE configs[3]" if (wl, n, args.scaling) == ("blast3d", 512, "weak") else "")
                 + (" — BASELINE configs[4]" if (wl, n, args.scaling) == ("ot3d", 1024, "strong") else ""))
    return wl, n, label


def run_reference(args, rank, world):
    if rank != 0:
        return
    wl, n, label = resolve(args)
    p = build_problem(wl, world, n, args.scheme, args.scaling)
    n2 = p.n[0] * p.n[1]
    nz_s = max(4, min(p.n[2], (4 << 20) // n2))  # ~4.2 M cells per step
    ps, U = oracle_slab(wl, p, nz_s)
    v, el, cores = oracle_rate(ps, U, args.steps, args.warmup)
    model, sockets, cps, tpc = cpu_topology()
    sample = (f"CPU oracle (oracle/mhd_oracle.c, gcc -O2 -ffp-contract=off, OpenMP {cores} threads, "
              f"OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')}), {args.steps} timed steps after {args.warmup} "
              f"warm-up of a {ps.n[0]}x{ps.n[1]}x{ps.n[2]} periodic slab of the workload's IC "
              f"({ps.cells / p.cells * world:.4f} of one GPU's cells per step)")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": label, "global": list(p.n), "cells_per_step": ps.cells,
                       "sample": f"{ps.n[0]}x{ps.n[1]}x{ps.n[2]}", "parallelism": "host cores"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu": model, "sockets": sockets, "cores_per_socket": cps, "threads_per_core": tpc},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def load_ncu(scheme: str, wl: str, n: int, scaling: str):
    """the committed one-launch ncu captures of this scheme's stage kernel on this workload
    (tools/refresh_profiles.sh): {"stage1": {...}, "stage2": {...}} or {}"""
    for name in (f"ncu_stage_{scheme}_{wl}{n}.json",):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return json.load(f)
        except Exception:
            pass
    return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mhd", choices=["mhd", "reference"])
    ap.add_argument("--scaling", default="weak", choices=sorted(SCALING),
                    help="weak: configs[3] blast 512^3 per GPU (default); strong: configs[4] OT 1024^3 split over N")
    ap.add_argument("--size", "--n", dest="n", type=int, default=None,
                    help="cells per axis (weak: per GPU; strong: global); under torchrun use --size "
                         "(torchrun's own parser takes --n for --nnodes)")
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--scheme", default="plm-rk2", choices=sorted(SCHEMES),
                    help="plm-rk2: the north star's PLM-MC + HLLD + GLM + SSP-RK2 (default); wenoz-rk3: the "
                         "paper's strong-scaling WENOZ + HLLD + GLM + SSP-RK3 (PAPER.md:270); ct-wenoz-rk3: its "
                         "weak-scaling WENOZ + HLLD + CT + SSP-RK3 (PAPER.md:179)")
    ap.add_argument("--halo", default="exchange", choices=["exchange", "push"],
                    help="z slabs: exchange = NCCL send/recv overlapped with the interior launch (default); "
                         "push = each stage's epilogue stores its boundary planes into the neighbours' NCCL "
                         "symmetric windows, one launch + an LSA barrier per stage (MHD_HALO_PUSH, DESIGN.md §8)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.halo == "push":
        os.environ["MHD_HALO_PUSH"] = "1"
    args.warmup = max(args.warmup, 3) if args.impl == "mhd" else args.warmup
    # the oracle's OpenMP threads stay on their cores (read when libgomp initialises)
    os.environ.setdefault("OMP_PROC_BIND", "close")
    os.environ.setdefault("OMP_PLACES", "cores")

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
    wl, n, label = resolve(args)
    p = build_problem(wl, world, n, args.scheme, args.scaling)
    _, plan = slab_plan(p, world)
    _, z0, z1 = plan[rank]
    nccl_id = None
    if world > 1:
        obj = [mhd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    s = mhd.Solver(p, rank=rank, nranks=world, device=local_rank, nccl_id=nccl_id)
    push = s.halo_push  # (set up, and agreed over the ranks, by mhd_create)
    assert s.offset[2] == z0 and s.extent[2] == z1 - z0
    stream = torch.cuda.current_stream()
    s.set_stream(stream)
    U0 = build_ic(wl, p, z0, z1)
    small = U0.nbytes <= 16 << 30
    if small:
        s.set_state(torch.from_numpy(U0).cuda())
    else:  # 1024^3 on few GPUs: host copy-in (the library stages through its second array)
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
    # one event pair per stage and per dt pass, and per stage one for the exposed halo wait (slabs)
    s.profile_enable(True, capacity=args.steps * (2 * nst + 1) + 8)
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
    prof = s.profile_read_stages()
    s.profile_enable(False)
    ms_max = max_over_ranks(ms)
    cells = p.cells
    value = cells * args.steps / (ms_max * 1e-3)
    diag = s.diag()

    # ---- roofline of the dominant kernel (the fused stage kernel, ~96% of the step), per stage
    pk, pk_kind = peaks()
    cells_loc = p.cells // world
    ct = args.scheme.startswith("ct-")
    sm_mhz = pk.get("sm_max_mhz", 1965.0)
    fp64_peak = N_SM * FP64_LANES_PER_SM * sm_mhz * 1e6 / 1e12  # TFLOP/s, 1 op per lane per clock (no FMA)
    hbm_peak = pk.get("hbm_gbs", 6537.3)
    stage_ms = sum(prof[f"stage{i}"][0] for i in (1, 2, 3))
    stage_n = sum(prof[f"stage{i}"][1] for i in (1, 2, 3))
    stage_avg_s = stage_ms * 1e-3 / max(stage_n, 1)
    ncu = load_ncu(args.scheme, wl, n, args.scaling) if world == 1 else {}
    per_stage = []
    for i in range(1, nst + 1):
        t_ms, cnt = prof[f"stage{i}"]
        t_s = t_ms * 1e-3 / max(cnt, 1)
        fl = FLOPS_PER_STAGE[args.scheme][i - 1] if FLOPS_PER_STAGE.get(args.scheme) else None
        by = BYTES_PER_STAGE[args.scheme][i - 1] if BYTES_PER_STAGE.get(args.scheme) else None
        cap = ncu.get(f"stage{i}") or {}
        per_stage.append({"stage": i, "ms_per_launch": t_s * 1e3, "launches": cnt,
                          "algorithmic_flops_per_cell": fl, "algorithmic_bytes_per_cell": by,
                          "achieved_tflops": fl * cells_loc / t_s / 1e12 if fl and cnt else None,
                          "achieved_hbm_gbs": by * cells_loc / t_s / 1e9 if by and cnt else None,
                          "ncu_dram_bytes_per_cell": cap.get("dram_bytes_per_cell"),
                          "ncu_fp64_pipe_active_pct": cap.get("fp64_pipe_active_pct")})
    fl_avg = (sum(FLOPS_PER_STAGE[args.scheme]) / nst) if FLOPS_PER_STAGE.get(args.scheme) else None
    by_avg = (sum(BYTES_PER_STAGE[args.scheme]) / nst) if BYTES_PER_STAGE.get(args.scheme) else None
    caps = [ncu.get(f"stage{i}") for i in range(1, nst + 1)]
    traffic = (sum(c["dram_bytes_per_launch"] for c in caps) / nst) if all(caps) else None
    achieved = fl_avg * cells_loc / stage_avg_s / 1e12 if fl_avg else None
    roof = {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
            "frac": achieved / fp64_peak if achieved else None, "traffic": traffic,
            "kernel": KERNELS[args.scheme],
            "peak_kind": f"derived: {N_SM} SM x {FP64_LANES_PER_SM} FP64 lanes x {sm_mhz:.0f} MHz (the recipe has no FMA; "
                         "measured DADD rate 99.7% of it, profiles/r01_probe_fp64.jsonl)",
            "units": "achieved = algorithmic fp64 ops per launch (per-cell count of DESIGN.md §7 x the launch's cells, "
                     "averaged over the RK stages) / mean stage time by CUDA events; traffic = ncu dram bytes per launch, "
                     "averaged over the same stages (one capture of each stage)",
            "algorithmic_flops_per_launch": fl_avg * cells_loc if fl_avg else None,
            "algorithmic_bytes_per_launch": by_avg * cells_loc if by_avg else None,
            "cells_per_launch": cells_loc, "stage_ms_per_launch": stage_avg_s * 1e3, "stage_launches": stage_n,
            "stage_share_of_step": stage_ms / max(ms, 1e-9),
            "dt_ms_per_launch": prof["dt"][0] / max(prof["dt"][1], 1),
            "halo_exposed_ms_per_step": prof["halo_exposed"][0] / args.steps,
            "fp64_pipe_active_pct": (sum(c["fp64_pipe_active_pct"] for c in caps) / nst) if all(caps) else None,
            "per_stage": per_stage,
            "hbm": {"achieved": by_avg * cells_loc / stage_avg_s / 1e9 if by_avg else None, "peak": hbm_peak,
                    "unit": "GB/s", "frac": by_avg * cells_loc / stage_avg_s / 1e9 / hbm_peak if by_avg else None,
                    "peak_kind": pk_kind},
            "ncu": ncu or None}

    # ---- e2e through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    e2e_note = "--no-e2e" if args.no_e2e else None
    if not args.no_e2e and small:
        # two pinned host copies of the state per rank on the node must fit in 80% of the free host RAM
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = None
        need = 2 * U0.nbytes * int(os.environ.get("LOCAL_WORLD_SIZE", world))
        if avail is not None and need > 0.8 * avail:
            small = False
            e2e_note = f"not measured: {need / 1e9:.0f} GB of pinned host buffers exceed 80% of the free host RAM"
    if not args.no_e2e and small:
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
               "what": "per step and rank: mhd_set_state_async(pinned host U) + mhd_compute_dt + mhd_step + "
                       "mhd_get_state_async(pinned host); mhd_io_join before the stop event"}
        del Uh, Uo
    s.destroy()

    # ---- CPU oracle baseline (rank 0, N = 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(wl, p, args.scheme)

    # kernels per step: k_dt + the dt read-back store, and per RK stage the fused k_stage (three
    # launches with slabs: interior and the two boundary ranges), or five launches for CT and for
    # the 3D GLM WENO-Z split stage (mhd_split.cu; MHD_FUSED_WENOZ=1 selects the fused kernel)
    split = (p.limiter == I.WENOZ and p.n[2] > 1 and not p.ct and os.environ.get("MHD_FUSED_WENOZ") != "1")
    # (halo push: the stage's launches and the LSA barrier kernel)
    slabs = world > 1 or os.environ.get("MHD_NCCL_SELF") == "1"  # (one-rank NCCL slab: the slab schedule)
    launches_per_stage = (5 + push) if (p.ct or split) else (2 if push else 3 if slabs else 1)
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
                "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": label, "problem": WORKLOADS[wl], "global": list(p.n),
                           "per_gpu": [p.n[0], p.n[1], p.n[2] // world], "scheme": SCHEMES[args.scheme],
                           "cells": cells, "parallelism": f"z-slab x{world}",
                           "halo": ("push (stage epilogue -> NCCL symmetric windows)" if push else
                                    "exchange (NCCL send/recv beside the interior launch)") if world > 1 else None,
                           "l2": f"inputs larger than L2 (2 x {U0.nbytes / 1e9:.2f} GB state arrays per GPU)"},
                "roofline": roof, "clocks": clk.summary(),
                "gpu_launches": args.steps * (2 + nst * launches_per_stage),
                "e2e": e2e, "cpu_baseline": cpu, "diag": diag, "lib": mhd.version()}
        if e2e is None:
            line["e2e_note"] = e2e_note or "not measured: the per-rank state exceeds 16 GiB (two pinned host copies)"
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
