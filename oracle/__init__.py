"""TEST INFRASTRUCTURE ONLY — the CPU oracle of the fp64 ideal-MHD Godunov step.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2510_24175_b200``) never imports it and shares no code with it.

Thin ctypes binding over ``oracle/liboracle.so`` (plain C, ``mhd_oracle.c``),
which follows DESIGN.md §3 step by step.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mhd_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# R-ARITH: no implicit FMA contraction, no fast-math, no FTZ.
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (called by __graft_entry__.build())."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "mhd_oracle.h"))):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


class Config(C.Structure):
    _fields_ = [("n", C.c_int64 * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3),
                ("bc_lo", C.c_int32 * 3), ("bc_hi", C.c_int32 * 3), ("gamma", C.c_double),
                ("cfl", C.c_double), ("limiter", C.c_int32), ("riemann", C.c_int32),
                ("glm", C.c_int32), ("stepper", C.c_int32), ("glm_alpha", C.c_double),
                ("p_floor", C.c_double), ("ct", C.c_int32), ("pad2_", C.c_int32)]


class Counters(C.Structure):
    _fields_ = [("p_floors", C.c_int64), ("plm_fallbacks", C.c_int64), ("hlld_to_hll", C.c_int64),
                ("first_bad_cell", C.c_int64), ("bad_stage", C.c_int32), ("pad_", C.c_int32)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k in
                ("p_floors", "plm_fallbacks", "hlld_to_hll", "first_bad_cell", "bad_stage")}


_lib = None
_D = C.POINTER(C.c_double)


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_LIB)
        L.orc_counters_reset.argtypes = [C.POINTER(Counters)]
        L.orc_cons2prim.argtypes = [C.POINTER(Config), _D, _D]
        L.orc_cons2prim.restype = C.c_int
        L.orc_total_energy.argtypes = [C.c_double, _D]
        L.orc_total_energy.restype = C.c_double
        L.orc_fast_speed.argtypes = [C.c_double] * 6
        L.orc_fast_speed.restype = C.c_double
        L.orc_limited_slope.argtypes = [C.c_int32, C.c_double, C.c_double]
        L.orc_limited_slope.restype = C.c_double
        L.orc_ct_divb.argtypes = [C.POINTER(Config), _D, _D]
        L.orc_ct_divb.restype = C.c_int
        L.orc_wenoz.argtypes = [C.c_double] * 5
        L.orc_wenoz.restype = C.c_double
        L.orc_face_flux.argtypes = [C.POINTER(Config), _D, _D, C.c_double, _D]
        L.orc_face_flux.restype = C.c_int
        L.orc_face_flux_batch.argtypes = [C.POINTER(Config), _D, _D, C.c_int64, C.c_double, _D]
        L.orc_face_flux_batch.restype = C.c_int64
        L.orc_hlld_fan.argtypes = [C.POINTER(Config), _D, _D, C.c_double, _D]
        L.orc_hlld_fan.restype = None
        L.orc_compute_dt.argtypes = [C.POINTER(Config), _D, _D, _D, C.POINTER(Counters)]
        L.orc_compute_dt.restype = C.c_int
        L.orc_step.argtypes = [C.POINTER(Config), _D, C.c_double, C.c_double, C.POINTER(Counters)]
        L.orc_step.restype = C.c_int
        L.orc_stage.argtypes = [C.POINTER(Config), _D, _D, C.c_double, C.c_double, C.POINTER(Counters)]
        L.orc_stage.restype = C.c_int
        L.orc_run.argtypes = [C.POINTER(Config), _D, C.c_int64, C.c_double, _D, C.POINTER(C.c_int64),
                              C.POINTER(Counters)]
        L.orc_run.restype = C.c_int
        L.orc_num_threads.restype = C.c_int
        L.orc_set_num_threads.argtypes = [C.c_int]
        _lib = L
    return _lib


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


def make_config(problem) -> Config:
    """Build the C config from an ``inputs.Problem`` (or any object with the same fields)."""
    c = Config()
    for d in range(3):
        c.n[d] = int(problem.n[d])
        c.lo[d] = float(problem.lo[d])
        c.hi[d] = float(problem.hi[d])
        c.bc_lo[d] = int(problem.bc[d])
        c.bc_hi[d] = int(problem.bc[d])
    c.gamma = float(problem.gamma)
    c.cfl = float(problem.cfl)
    c.limiter = int(problem.limiter)
    c.riemann = int(problem.riemann)
    c.glm = int(problem.glm)
    c.stepper = int(getattr(problem, "stepper", 0))
    c.glm_alpha = float(problem.glm_alpha)
    c.p_floor = float(problem.p_floor)
    c.ct = int(getattr(problem, "ct", 0))
    return c


class OracleError(RuntimeError):
    def __init__(self, rc, counters):
        super().__init__(f"oracle rc={rc} counters={counters.as_dict()}")
        self.rc = rc
        self.counters = counters


class Oracle:
    """Stateful convenience wrapper: holds U (interior, [nvar][nz][ny][nx]) and counters."""

    def __init__(self, problem, U: np.ndarray):
        self.cfg = make_config(problem)
        self.U = np.ascontiguousarray(U, dtype=np.float64).copy()
        self.cnt = Counters()
        lib().orc_counters_reset(C.byref(self.cnt))
        self.t = 0.0
        self.steps = 0

    def compute_dt(self):
        dt, ch = C.c_double(), C.c_double()
        rc = lib().orc_compute_dt(C.byref(self.cfg), _ptr(self.U), C.byref(dt), C.byref(ch), C.byref(self.cnt))
        if rc:
            raise OracleError(rc, self.cnt)
        return dt.value, ch.value

    def step(self, dt, ch):
        rc = lib().orc_step(C.byref(self.cfg), _ptr(self.U), dt, ch, C.byref(self.cnt))
        if rc:
            raise OracleError(rc, self.cnt)
        self.t += dt
        self.steps += 1

    def run(self, nsteps: int, t_end: float = 0.0):
        """c.14 driver; returns the dt log (np.float64 array)."""
        log = np.zeros(max(nsteps, 1), dtype=np.float64)
        done = C.c_int64()
        rc = lib().orc_run(C.byref(self.cfg), _ptr(self.U), nsteps, t_end, _ptr(log), C.byref(done),
                           C.byref(self.cnt))
        if rc:
            raise OracleError(rc, self.cnt)
        self.steps += done.value
        self.t += float(log[:done.value].sum()) if done.value else 0.0
        return log[:done.value].copy()

    def counters(self):
        return self.cnt.as_dict()


def cons2prim(problem, U):
    cfg = make_config(problem)
    U = np.ascontiguousarray(U, dtype=np.float64)
    V = np.zeros_like(U)
    fl = lib().orc_cons2prim(C.byref(cfg), _ptr(U), _ptr(V))
    return V, fl


def total_energy(gamma, V):
    V = np.ascontiguousarray(V, dtype=np.float64)
    return lib().orc_total_energy(gamma, _ptr(V))


def fast_speed(gamma, rho, p, bn, bt1, bt2):
    return lib().orc_fast_speed(gamma, rho, p, bn, bt1, bt2)


def ct_divb(problem, U):
    """discrete div b of a CT state (face fields 5..7), per interior cell [nz][ny][nx]."""
    cfg = make_config(problem)
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros(U.shape[1:], dtype=np.float64)
    rc = lib().orc_ct_divb(C.byref(cfg), _ptr(U), _ptr(out))
    if rc:
        raise OracleError(rc, Counters())
    return out


def wenoz(a, b, c, d, e):
    return lib().orc_wenoz(a, b, c, d, e)


def limited_slope(limiter, dm, dp):
    return lib().orc_limited_slope(limiter, dm, dp)


def face_flux(problem, VL, VR, ch):
    """Batched face flux in the normal frame; VL, VR: [n][nvar]. Returns (F, n_hll_fallbacks)."""
    cfg = make_config(problem)
    VL = np.ascontiguousarray(VL, dtype=np.float64)
    VR = np.ascontiguousarray(VR, dtype=np.float64)
    if VL.ndim == 1:
        VL, VR = VL[None], VR[None]
    F = np.zeros_like(VL)
    nfb = lib().orc_face_flux_batch(C.byref(cfg), _ptr(VL), _ptr(VR), VL.shape[0], ch, _ptr(F))
    return F, int(nfb)


def hlld_fan(problem, VL, VR, ch):
    """Test-only: the HLLD wave fan of one face pair (normal frame).  Returns a dict with the
    speeds SL, SsL, SM, SsR, SR, pts, the branch `flag` (0 fan, 1 SM guard, 2 wave-ordering
    guard, 3 supersonic), the R6 flags degL / degR and the states UL, UsL, UssL, UssR, UsR, UR
    and fluxes FL, FR (8 components each)."""
    cfg = make_config(problem)
    VL = np.ascontiguousarray(VL, dtype=np.float64)
    VR = np.ascontiguousarray(VR, dtype=np.float64)
    out = np.zeros(73, dtype=np.float64)
    lib().orc_hlld_fan(C.byref(cfg), _ptr(VL), _ptr(VR), ch, _ptr(out))
    d = dict(zip(("SL", "SsL", "SM", "SsR", "SR", "pts"), out[:6]))
    d["flag"], d["degL"], d["degR"] = int(out[6]), bool(out[7]), bool(out[8])
    A = out[9:].reshape(8, 8)
    for j, k in enumerate(("UL", "UsL", "UssL", "UssR", "UsR", "UR", "FL", "FR")):
        d[k] = A[j].copy()
    return d


def compute_dt(problem, U):
    """c.13 on a contiguous interior U without copying it (for full-size states): (dt, ch)."""
    cfg = make_config(problem)
    assert U.flags.c_contiguous and U.dtype == np.float64
    dt, ch = C.c_double(), C.c_double()
    cnt = Counters()
    lib().orc_counters_reset(C.byref(cnt))
    rc = lib().orc_compute_dt(C.byref(cfg), _ptr(U), C.byref(dt), C.byref(ch), C.byref(cnt))
    if rc:
        raise OracleError(rc, cnt)
    return dt.value, ch.value


def stage(problem, U, dt, ch):
    cfg = make_config(problem)
    U = np.ascontiguousarray(U, dtype=np.float64)
    out = np.zeros_like(U)
    cnt = Counters()
    lib().orc_counters_reset(C.byref(cnt))
    rc = lib().orc_stage(C.byref(cfg), _ptr(U), _ptr(out), dt, ch, C.byref(cnt))
    if rc:
        raise OracleError(rc, cnt)
    return out, cnt.as_dict()


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(int(n))
