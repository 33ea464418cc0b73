"""Thin ctypes binding of libmhd (include/mhd.h) — argument marshalling only.

Every step of the hot path runs in the CUDA kernels of ``csrc/``; this module only converts
Python/numpy/torch arguments into the C ABI.  There is no CPU fallback: if ``libmhd.so`` is
missing or no CUDA device is visible the calls raise.

Names follow the ABI: ``create`` / ``set_state`` / ``compute_dt`` / ``step`` / ``get_state`` /
``destroy`` (BASELINE.json north star).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from . import inputs as _inputs

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MHD_LIB") or os.path.join(_HERE, "libmhd.so")  # MHD_LIB: A/B builds

MHD_OK, MHD_E_ARG, MHD_E_STATE, MHD_E_CUDA, MHD_E_NCCL, MHD_E_NOMEM, MHD_E_UNPHYSICAL = range(7)
_NAMES = {0: "MHD_OK", 1: "MHD_E_ARG", 2: "MHD_E_STATE", 3: "MHD_E_CUDA", 4: "MHD_E_NCCL", 5: "MHD_E_NOMEM",
          6: "MHD_E_UNPHYSICAL"}

# every symbol include/mhd.h declares (checked by the CPU test suite)
EXPORTS = ("mhd_nccl_get_unique_id", "mhd_create", "mhd_set_stream", "mhd_local_box", "mhd_device_bytes",
           "mhd_set_state", "mhd_get_state", "mhd_compute_dt", "mhd_step", "mhd_get_diag", "mhd_last_error",
           "mhd_destroy", "mhd_debug_face_flux", "mhd_profile_enable", "mhd_profile_read", "mhd_version",
           "mhd_group_compute_dt", "mhd_group_step", "mhd_halo_plan", "mhd_debug_fast_ops",
           "mhd_get_state_box", "mhd_set_state_async", "mhd_get_state_async", "mhd_io_join",
           "mhd_workspace_bytes", "mhd_bind_workspace", "mhd_run", "mhd_profile_read_stages",
           "mhd_halo_push")
TRANSPORT_NCCL, TRANSPORT_LOCAL = 0, 1


class Grid(C.Structure):
    _fields_ = [("n", C.c_int64 * 3), ("lo", C.c_double * 3), ("hi", C.c_double * 3)]


class BC(C.Structure):
    _fields_ = [("lo", C.c_int32 * 3), ("hi", C.c_int32 * 3)]


class Scheme(C.Structure):
    _fields_ = [("limiter", C.c_int32), ("riemann", C.c_int32), ("glm", C.c_int32), ("stepper", C.c_int32),
                ("glm_alpha", C.c_double), ("p_floor", C.c_double), ("ct", C.c_int32), ("reserved", C.c_int32)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("nranks", C.c_int32), ("device", C.c_int32), ("transport", C.c_int32),
                ("nccl_id", C.c_uint8 * 128)]


class Diag(C.Structure):
    _fields_ = [("steps", C.c_int64), ("p_floors", C.c_int64), ("plm_fallbacks", C.c_int64),
                ("hlld_to_hll", C.c_int64), ("first_bad_cell", C.c_int64), ("bad_stage", C.c_int32),
                ("reserved", C.c_int32)]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_ if k != "reserved"}


class MhdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def load() -> C.CDLL:
    """Load libmhd.so (built in-tree by ``build.py``).  Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libmhd.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = C.CDLL(LIB_PATH)
    P = C.c_void_p
    L.mhd_nccl_get_unique_id.argtypes = [C.POINTER(C.c_uint8)]
    L.mhd_create.argtypes = [C.POINTER(Grid), C.c_double, C.c_double, C.POINTER(BC), C.POINTER(Scheme),
                             C.POINTER(Dist), C.POINTER(P)]
    L.mhd_set_stream.argtypes = [P, P]
    L.mhd_local_box.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.mhd_device_bytes.argtypes = [P, C.POINTER(C.c_size_t)]
    L.mhd_set_state.argtypes = [P, P, C.c_int32]
    L.mhd_get_state.argtypes = [P, P, C.c_int32]
    if hasattr(L, "mhd_get_state_box"):  # (absent from older builds used in A/B runs)
        L.mhd_get_state_box.argtypes = [P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), P, C.c_int32]
    if hasattr(L, "mhd_run"):
        L.mhd_run.argtypes = [P, C.c_int64, C.c_double, P, C.POINTER(C.c_int64)]
    if hasattr(L, "mhd_bind_workspace"):
        L.mhd_workspace_bytes.argtypes = [P, C.POINTER(C.c_size_t)]
        L.mhd_bind_workspace.argtypes = [P, P, C.c_size_t]
    if hasattr(L, "mhd_io_join"):
        L.mhd_set_state_async.argtypes = [P, P]
        L.mhd_get_state_async.argtypes = [P, P]
        L.mhd_io_join.argtypes = [P]
    L.mhd_compute_dt.argtypes = [P, C.POINTER(C.c_double)]
    L.mhd_step.argtypes = [P, C.c_double]
    L.mhd_get_diag.argtypes = [P, C.POINTER(Diag)]
    L.mhd_last_error.argtypes = [P]
    L.mhd_last_error.restype = C.c_char_p
    L.mhd_destroy.argtypes = [P]
    L.mhd_destroy.restype = None
    L.mhd_debug_face_flux.argtypes = [P, P, P, C.c_int64, C.c_double, P, C.POINTER(C.c_int64)]
    L.mhd_version.restype = C.c_char_p
    if hasattr(L, "mhd_debug_fast_ops"):  # (absent from older builds used in A/B runs)
        L.mhd_debug_fast_ops.argtypes = [P, P, C.c_int64, P, P]
    L.mhd_profile_enable.argtypes = [P, C.c_int32]
    L.mhd_profile_read.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    L.mhd_profile_read_stages.argtypes = [P, C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    if hasattr(L, "mhd_halo_push"):  # (older A/B builds lack it)
        L.mhd_halo_push.argtypes = [P]
    L.mhd_group_compute_dt.argtypes = [C.POINTER(P), C.c_int32, C.POINTER(C.c_double)]
    L.mhd_group_step.argtypes = [C.POINTER(P), C.c_int32, C.c_double]
    L.mhd_halo_plan.argtypes = [C.c_int32, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_int32)]
    _lib = L
    return L


def version() -> str:
    return load().mhd_version().decode()


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = load().mhd_nccl_get_unique_id(buf)
    if rc:
        raise MhdError(rc, "ncclGetUniqueId failed")
    return bytes(buf)


def halo_plan(rank: int, nranks: int, nz_glob: int, z_periodic: bool = True, ghost: int = 2):
    """The 4 transfers of one RK stage for a z slab: rows (peer, 0 send / 1 recv, first storage
    plane, planes) in posting order (pure host logic of libmhd, usable without a GPU)."""
    buf = (C.c_int32 * 16)()
    rc = load().mhd_halo_plan(rank, nranks, nz_glob, 1 if z_periodic else 0, ghost, buf)
    if rc:
        raise MhdError(rc, "mhd_halo_plan")
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(4)]


def debug_fast_ops(a, b):
    """Test-only: (out [n][8], ok [n]) of mhd_debug_fast_ops for CUDA float64 tensors a, b."""
    import torch
    L = load()
    out = torch.empty((a.shape[0], 8), dtype=torch.float64, device=a.device)
    ok = torch.empty(a.shape[0], dtype=torch.int32, device=a.device)
    rc = L.mhd_debug_fast_ops(C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr()), a.shape[0],
                              C.c_void_p(out.data_ptr()), C.c_void_p(ok.data_ptr()))
    if rc != 0:
        raise MhdError(rc, "mhd_debug_fast_ops failed")
    return out, ok


def _ptr_of(U):
    """(pointer, on_device, nbytes) of a numpy array or a torch tensor (CPU or CUDA)."""
    if isinstance(U, np.ndarray):
        if U.dtype != np.float64 or not U.flags["C_CONTIGUOUS"]:
            raise ValueError("state must be a C-contiguous float64 array")
        return U.ctypes.data, 0, U.nbytes
    import torch
    if not isinstance(U, torch.Tensor):
        raise TypeError("state must be a numpy array or a torch tensor")
    if U.dtype != torch.float64 or not U.is_contiguous():
        raise ValueError("state must be a contiguous float64 tensor")
    return U.data_ptr(), 1 if U.is_cuda else 0, U.numel() * 8


class Solver:
    """One libmhd context: the state of this rank's slab on one GPU."""

    def __init__(self, problem: "_inputs.Problem", rank: int = 0, nranks: int = 1, device: int = -1,
                 nccl_id: Optional[bytes] = None, stream=None, transport: int = TRANSPORT_NCCL):
        L = load()
        self.problem = problem
        g = Grid()
        bc = BC()
        for d in range(3):
            g.n[d] = int(problem.n[d])
            g.lo[d] = float(problem.lo[d])
            g.hi[d] = float(problem.hi[d])
            bc.lo[d] = int(problem.bc[d])
            bc.hi[d] = int(problem.bc[d])
        sc = Scheme(int(problem.limiter), int(problem.riemann), int(problem.glm), int(getattr(problem, "stepper", 0)),
                    float(problem.glm_alpha), float(problem.p_floor), int(getattr(problem, "ct", 0)), 0)
        dist = None
        if nranks > 1 or device >= 0:
            dist = Dist(rank, nranks, device, transport)
            if nccl_id is not None:
                C.memmove(dist.nccl_id, nccl_id, 128)
        h = C.c_void_p()
        rc = L.mhd_create(C.byref(g), float(problem.gamma), float(problem.cfl), C.byref(bc), C.byref(sc),
                          C.byref(dist) if dist is not None else None, C.byref(h))
        if rc:
            raise MhdError(rc, "mhd_create failed")
        self._h = h
        self._L = L
        off, ext = (C.c_int64 * 3)(), (C.c_int64 * 3)()
        L.mhd_local_box(h, off, ext)
        self.offset = tuple(off)
        self.extent = tuple(ext)
        self.nvar = problem.nvar
        self.local_shape = (self.nvar, ext[2], ext[1], ext[0])
        if stream is not None:
            self.set_stream(stream)

    # --- ABI calls -------------------------------------------------------------------------
    def _check(self, rc):
        if rc:
            raise MhdError(rc, self._L.mhd_last_error(self._h).decode())

    def set_stream(self, stream) -> None:
        """stream: a torch.cuda.Stream, an int handle or None (library's own stream)."""
        handle = getattr(stream, "cuda_stream", stream)
        self._check(self._L.mhd_set_stream(self._h, C.c_void_p(handle)))

    def set_state(self, U) -> None:
        p, dev, nbytes = _ptr_of(U)
        if nbytes != int(np.prod(self.local_shape)) * 8:
            raise ValueError(f"state must have shape {self.local_shape}")
        self._check(self._L.mhd_set_state(self._h, C.c_void_p(p), dev))

    def get_state(self, out=None):
        if out is None:
            out = np.empty(self.local_shape, dtype=np.float64)
        p, dev, nbytes = _ptr_of(out)
        if nbytes != int(np.prod(self.local_shape)) * 8:
            raise ValueError(f"output must have shape {self.local_shape}")
        self._check(self._L.mhd_get_state(self._h, C.c_void_p(p), dev))
        return out

    def workspace_bytes(self) -> int:
        b = C.c_size_t()
        self._check(self._L.mhd_workspace_bytes(self._h, C.byref(b)))
        return b.value

    def bind_workspace(self, buf) -> None:
        """Move the state arrays into a caller-owned CUDA tensor (>= workspace_bytes() bytes);
        keep `buf` alive while the solver lives.  Clears the state."""
        nbytes = buf.numel() * buf.element_size()
        self._check(self._L.mhd_bind_workspace(self._h, C.c_void_p(buf.data_ptr()), nbytes))
        self._workspace = buf

    def _host_ptr(self, U):
        p, dev, nbytes = _ptr_of(U)
        if dev or nbytes != int(np.prod(self.local_shape)) * 8:
            raise ValueError(f"need a host buffer of shape {self.local_shape}")
        return p

    def set_state_async(self, U) -> None:
        """Start the upload of U (pinned host memory: torch.Tensor.pin_memory()); it becomes the
        state at the next compute_dt / step / get_state*.  Keep U alive and unchanged until io_join."""
        self._check(self._L.mhd_set_state_async(self._h, C.c_void_p(self._host_ptr(U))))

    def get_state_async(self, out) -> None:
        """Start the download of the current state into `out` (pinned host); complete after
        io_join() and a synchronisation of the stream."""
        self._check(self._L.mhd_get_state_async(self._h, C.c_void_p(self._host_ptr(out))))

    def io_join(self) -> None:
        self._check(self._L.mhd_io_join(self._h))

    def get_state_box(self, off, ext) -> np.ndarray:
        """State of the global cell box [off, off+ext) (x, y, z) as [nvar][ez][ey][ex] (host)."""
        out = np.empty((self.problem.nvar, ext[2], ext[1], ext[0]), dtype=np.float64)
        o, e = (C.c_int64 * 3)(*off), (C.c_int64 * 3)(*ext)
        self._check(self._L.mhd_get_state_box(self._h, o, e, C.c_void_p(out.ctypes.data), 0))
        return out

    def compute_dt(self) -> float:
        dt = C.c_double()
        self._check(self._L.mhd_compute_dt(self._h, C.byref(dt)))
        return dt.value

    def step(self, dt: float) -> None:
        self._check(self._L.mhd_step(self._h, float(dt)))

    def diag(self) -> dict:
        d = Diag()
        self._check(self._L.mhd_get_diag(self._h, C.byref(d)))
        return d.as_dict()

    def device_bytes(self) -> int:
        b = C.c_size_t()
        self._check(self._L.mhd_device_bytes(self._h, C.byref(b)))
        return b.value

    def debug_face_flux(self, VL, VR, ch: float):
        """VL, VR: CUDA float64 tensors [n][nvar] (normal frame). Returns (F, n_hll)."""
        import torch
        F = torch.empty_like(VL)
        nh = C.c_int64()
        self._check(self._L.mhd_debug_face_flux(self._h, C.c_void_p(VL.data_ptr()), C.c_void_p(VR.data_ptr()),
                                                VL.shape[0], float(ch), C.c_void_p(F.data_ptr()), C.byref(nh)))
        return F, nh.value

    def profile_enable(self, on: bool = True, capacity: int = 0) -> None:
        """capacity: timed units (RK stages + dt passes) to make room for (0: the default 1024)."""
        self._check(self._L.mhd_profile_enable(self._h, (capacity if capacity > 1 else 1) if on else 0))

    def profile_read(self):
        """{'stage': (ms, stages), 'dt': (ms, passes)} since profile_enable (one event pair per RK
        stage, whatever its launch count, and per dt pass)."""
        ms, n = (C.c_double * 2)(), (C.c_int64 * 2)()
        self._check(self._L.mhd_profile_read(self._h, ms, n))
        return {"stage": (ms[0], n[0]), "dt": (ms[1], n[1])}

    def profile_read_stages(self):
        """{'dt': (ms, passes), 'stage1': (ms, stages), 'stage2': ..., 'stage3': ..., 'halo_exposed':
        (ms, waits)} since profile_enable."""
        ms, n = (C.c_double * 5)(), (C.c_int64 * 5)()
        self._check(self._L.mhd_profile_read_stages(self._h, ms, n))
        return {"dt": (ms[0], n[0]), "stage1": (ms[1], n[1]), "stage2": (ms[2], n[2]), "stage3": (ms[3], n[3]),
                "halo_exposed": (ms[4], n[4])}

    @property
    def halo_push(self) -> bool:
        """True if this context's stages push their boundary planes to the z neighbours
        (MHD_HALO_PUSH=1 at creation, include/mhd.h mhd_halo_push)."""
        return hasattr(self._L, "mhd_halo_push") and self._L.mhd_halo_push(self._h) == 1

    def destroy(self) -> None:
        if getattr(self, "_h", None):
            self._L.mhd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    # --- harness (DESIGN.md §3 c.14 driver loop) ---------------------------------------------
    def run(self, nsteps: int, t_end: float = 0.0):
        """mhd_run: the compute_dt/step loop in native code; with t_end > 0 the last dt is
        clamped.  Returns the dt log."""
        log = np.zeros(max(int(nsteps), 1), dtype=np.float64)
        done = C.c_int64()
        self._check(self._L.mhd_run(self._h, int(nsteps), float(t_end), C.c_void_p(log.ctypes.data), C.byref(done)))
        return log[:done.value].copy()


class SolverGroup:
    """nranks z slabs of one problem in this process on one device (MHD_TRANSPORT_LOCAL): the
    decomposition of the multi-GPU path (slab plan, halo planes, counters, dt reduction) with
    device copies in place of NCCL.  Used to check decomposition invariance on one GPU."""

    def __init__(self, problem: "_inputs.Problem", nranks: int):
        self.problem = problem
        self.slabs = [Solver(problem, rank=r, nranks=nranks, transport=TRANSPORT_LOCAL) for r in range(nranks)]
        self._arr = (C.c_void_p * nranks)(*[s._h.value for s in self.slabs])
        self._L = load()

    def _check(self, rc):
        if rc:
            msgs = "; ".join(self._L.mhd_last_error(s._h).decode() for s in self.slabs)
            raise MhdError(rc, msgs)

    def set_state(self, U):
        """U: the global interior state [nvar][nz][ny][nx] (numpy)."""
        for s in self.slabs:
            z0, nz = s.offset[2], s.extent[2]
            s.set_state(np.ascontiguousarray(U[:, z0:z0 + nz]))

    def get_state(self):
        return np.concatenate([s.get_state() for s in self.slabs], axis=1)

    def compute_dt(self) -> float:
        dt = C.c_double()
        self._check(self._L.mhd_group_compute_dt(self._arr, len(self.slabs), C.byref(dt)))
        return dt.value

    def step(self, dt: float) -> None:
        self._check(self._L.mhd_group_step(self._arr, len(self.slabs), float(dt)))

    def run(self, nsteps: int, t_end: float = 0.0):
        log, t = [], 0.0
        while len(log) < nsteps and (t_end <= 0.0 or t < t_end):
            dt = self.compute_dt()
            if t_end > 0.0 and t + dt > t_end:
                dt = t_end - t
            self.step(dt)
            log.append(dt)
            t = t + dt
        return np.array(log, dtype=np.float64)

    def diag(self) -> dict:
        ds = [s.diag() for s in self.slabs]
        out = {k: sum(d[k] for d in ds) for k in ("p_floors", "plm_fallbacks", "hlld_to_hll")}
        out["steps"] = ds[0]["steps"]
        return out

    def destroy(self):
        # rank 0 owns the group's stream: free it last
        for s in reversed(self.slabs):
            s.destroy()
