"""Seeded, synthetic input generators shared by the oracle side and the CUDA side.

This module holds problem descriptions and initial conditions only — none of the
method's arithmetic (no reconstruction, Riemann solver, update or timestep).  The
only formula here is the definition of total energy used to *state* an initial
condition in conservative variables, E = p/(gamma-1) + rho|v|^2/2 + |B|^2/2
(Heaviside-Lorentz units, R3), evaluated once in numpy.

Problems follow DESIGN.md §4 (the input recipe):
  * Sod (gamma 1.4) and Brio-Wu (gamma 2) shock tubes            — BASELINE configs[0]
  * 2D Orszag-Tang, PLUTO normalisation on [0,1]^2               — configs[1]
  * 3D Orszag-Tang with z-modulation eps = 0.2                    — configs[2], [4]
  * 3D MHD blast, one blast per unit cube along z                 — configs[3]
  * linear Alfven wave and circularly polarised Alfven wave (CPA) — convergence pins
  * random physical face-state pairs (seeded)                    — Riemann-solver parity

The paper names the 3D Orszag-Tang and CPA problems (§4.2) but
defers their parameters to another paper; the parameters here are the readings
R20-R23 of DESIGN.md.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Tuple

import numpy as np

PERIODIC, OUTFLOW = 0, 1
RK2, RK3 = 0, 1
MINMOD, MC, WENOZ = 0, 1, 2
HLL, HLLD = 0, 1


@dataclasses.dataclass
class Problem:
    name: str
    n: Tuple[int, int, int]
    lo: Tuple[float, float, float] = (0.0, 0.0, 0.0)
    hi: Tuple[float, float, float] = (1.0, 1.0, 1.0)
    bc: Tuple[int, int, int] = (PERIODIC, PERIODIC, PERIODIC)
    gamma: float = 5.0 / 3.0
    cfl: float = 0.4
    limiter: int = MC
    riemann: int = HLLD
    glm: int = 1
    glm_alpha: float = 0.1
    p_floor: float = 1e-12
    t_end: float = 0.0
    stepper: int = 0  # 0 SSP-RK2 (north star), 1 SSP-RK3 (the paper's RK3)
    ct: int = 0       # 1 constrained transport: fields 5..7 face-centred, glm 0

    @property
    def nvar(self) -> int:
        return 8 + (1 if self.glm else 0)

    @property
    def shape(self):
        """interior array shape [nvar][nz][ny][nx]"""
        return (self.nvar, self.n[2], self.n[1], self.n[0])

    @property
    def cells(self) -> int:
        return int(self.n[0]) * int(self.n[1]) * int(self.n[2])

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


def centres(p: Problem, d: int) -> np.ndarray:
    """cell-centre coordinates along axis d (harness only, never the solver; DESIGN.md R-GRID)."""
    dx = (p.hi[d] - p.lo[d]) / p.n[d]
    return p.lo[d] + (np.arange(p.n[d], dtype=np.float64) + 0.5) * dx


def mesh(p: Problem):
    x, y, z = centres(p, 0), centres(p, 1), centres(p, 2)
    Z, Y, X = np.meshgrid(z, y, x, indexing="ij")
    return X, Y, Z


def prim_to_cons_ic(p: Problem, rho, vx, vy, vz, pr, bx, by, bz, psi=None) -> np.ndarray:
    """State an IC in conservative variables (R3 energy definition)."""
    shape = (p.n[2], p.n[1], p.n[0])
    f = [np.broadcast_to(np.asarray(a, dtype=np.float64), shape) for a in (rho, vx, vy, vz, pr, bx, by, bz)]
    rho, vx, vy, vz, pr, bx, by, bz = f
    U = np.empty(p.shape, dtype=np.float64)
    U[0] = rho
    U[1] = rho * vx
    U[2] = rho * vy
    U[3] = rho * vz
    U[4] = pr / (p.gamma - 1.0) + 0.5 * rho * (vx * vx + vy * vy + vz * vz) + 0.5 * (bx * bx + by * by + bz * bz)
    U[5] = bx
    U[6] = by
    U[7] = bz
    if p.glm:
        U[8] = 0.0 if psi is None else np.broadcast_to(psi, shape)
    return U


# ----------------------------------------------------------------------------------------------
# problem definitions
# ----------------------------------------------------------------------------------------------
def sod(n=512, riemann=HLLD, limiter=MC) -> Problem:
    return Problem("sod", (n, 1, 1), bc=(OUTFLOW, OUTFLOW, OUTFLOW), gamma=1.4, riemann=riemann, limiter=limiter,
                   glm=0, t_end=0.2)


def sod_ic(p: Problem) -> np.ndarray:
    X, _, _ = mesh(p)
    left = X < 0.5
    return prim_to_cons_ic(p, np.where(left, 1.0, 0.125), 0, 0, 0, np.where(left, 1.0, 0.1), 0, 0, 0)


def brio_wu(n=512, riemann=HLL, limiter=MC) -> Problem:
    """BASELINE configs[0]: Brio-Wu, 512 cells, PLM+HLL, RK2, CFL 0.4, t=0.1."""
    return Problem("brio_wu", (n, 1, 1), bc=(OUTFLOW, OUTFLOW, OUTFLOW), gamma=2.0, riemann=riemann,
                   limiter=limiter, glm=0, t_end=0.1)


def brio_wu_ic(p: Problem) -> np.ndarray:
    X, _, _ = mesh(p)
    left = X < 0.5
    return prim_to_cons_ic(p, np.where(left, 1.0, 0.125), 0, 0, 0, np.where(left, 1.0, 0.1), 0.75,
                           np.where(left, 1.0, -1.0), 0)


def orszag_tang_2d(n=512, glm=1, limiter=MC, riemann=HLLD) -> Problem:
    """BASELINE configs[1]: PLUTO normalisation on [0,1]^2 (R20)."""
    return Problem("ot2d", (n, n, 1), gamma=5.0 / 3.0, glm=glm, limiter=limiter, riemann=riemann, t_end=0.5)


def orszag_tang_2d_ic(p: Problem) -> np.ndarray:
    X, Y, _ = mesh(p)
    tp = 2.0 * math.pi
    return prim_to_cons_ic(p, 25.0 / 9.0, -np.sin(tp * Y), np.sin(tp * X), 0.0, 5.0 / 3.0, -np.sin(tp * Y),
                           np.sin(2.0 * tp * X), 0.0)


def orszag_tang_3d(n=256, nz=None, z_extent=1.0, limiter=MC, riemann=HLLD) -> Problem:
    """BASELINE configs[2] (256^3) and [4] (1024^3); z-modulated extension, eps = 0.2 (R21)."""
    nz = n if nz is None else nz
    return Problem("ot3d", (n, n, nz), hi=(1.0, 1.0, z_extent), gamma=5.0 / 3.0, limiter=limiter, riemann=riemann,
                   glm=1, t_end=0.5)


def orszag_tang_3d_ic(p: Problem, eps: float = 0.2, z_range=None) -> np.ndarray:
    """z_range=(k0, k1) builds only global planes k0..k1-1 (one rank's slab)."""
    sub = p
    if z_range is not None:
        k0, k1 = z_range
        dz = (p.hi[2] - p.lo[2]) / p.n[2]
        sub = p.replace(n=(p.n[0], p.n[1], k1 - k0), lo=(p.lo[0], p.lo[1], p.lo[2] + k0 * dz),
                        hi=(p.hi[0], p.hi[1], p.lo[2] + k1 * dz))
    X, Y, Z = mesh(sub)
    tp = 2.0 * math.pi
    a = 1.0 + eps * np.sin(tp * Z)
    return prim_to_cons_ic(sub, 25.0 / 9.0, -a * np.sin(tp * Y), a * np.sin(tp * X), eps * np.sin(tp * Z), 5.0 / 3.0,
                           -np.sin(tp * Y), np.sin(2.0 * tp * X), 0.0)


def blast_3d(n=512, cubes=1, limiter=MC) -> Problem:
    """BASELINE configs[3]: one blast per unit cube along z (R22)."""
    return Problem("blast3d", (n, n, n * cubes), hi=(1.0, 1.0, float(cubes)), gamma=5.0 / 3.0, limiter=limiter,
                   riemann=HLLD, glm=1, t_end=0.2)


def blast_3d_ic(p: Problem, z_range=None) -> np.ndarray:
    sub = p
    if z_range is not None:
        k0, k1 = z_range
        dz = (p.hi[2] - p.lo[2]) / p.n[2]
        sub = p.replace(n=(p.n[0], p.n[1], k1 - k0), lo=(p.lo[0], p.lo[1], p.lo[2] + k0 * dz),
                        hi=(p.hi[0], p.hi[1], p.lo[2] + k1 * dz))
    X, Y, Z = mesh(sub)
    zc = np.floor(Z) + 0.5
    r2 = (X - 0.5) ** 2 + (Y - 0.5) ** 2 + (Z - zc) ** 2
    pr = np.where(r2 < 0.01, 10.0, 0.1)
    b = 1.0 / math.sqrt(2.0)
    return prim_to_cons_ic(sub, 1.0, 0.0, 0.0, 0.0, pr, b, b, 0.0)


def linear_alfven(n=64, limiter=MC) -> Problem:
    return Problem("alfven_linear", (n, 1, 1), gamma=5.0 / 3.0, limiter=limiter, riemann=HLLD, glm=0, t_end=1.0)


def linear_alfven_ic(p: Problem, amp: float = 1e-6) -> np.ndarray:
    X, _, _ = mesh(p)
    s = amp * np.sin(2.0 * math.pi * X)
    return prim_to_cons_ic(p, 1.0, 0.0, -s, 0.0, 0.6, 1.0, s, 0.0)


def cpa_1d(n=64, limiter=MC, riemann=HLLD) -> Problem:
    return Problem("cpa1d", (n, 1, 1), gamma=5.0 / 3.0, limiter=limiter, riemann=riemann, glm=0, t_end=1.0)


def cpa_1d_ic(p: Problem, amp: float = 0.1) -> np.ndarray:
    """circularly polarised Alfven wave along x: v_perp = -B_perp (rho=1, B_par=1), moves at +v_A = 1."""
    X, _, _ = mesh(p)
    ph = 2.0 * math.pi * X
    by, bz = amp * np.sin(ph), amp * np.cos(ph)
    return prim_to_cons_ic(p, 1.0, 0.0, -by, -bz, 0.1, 1.0, by, bz)


def cpa_2d(n=64, limiter=MC) -> Problem:
    """CPA propagating along the diagonal of [0, sqrt5] x [0, sqrt5/2]... simplified: along (1,1) of [0,1]^2."""
    return Problem("cpa2d", (n, n, 1), gamma=5.0 / 3.0, limiter=limiter, riemann=HLLD, glm=1, t_end=1.0)


def cpa_2d_ic(p: Problem, amp: float = 0.1) -> np.ndarray:
    """wave vector k = 2pi(1,1): wavelength 1/sqrt2 along the diagonal; v_A = 1 so one period is t = 1/sqrt2."""
    X, Y, _ = mesh(p)
    s2 = 1.0 / math.sqrt(2.0)
    ph = 2.0 * math.pi * (X + Y)
    par = np.array([s2, s2, 0.0])
    t1 = np.array([-s2, s2, 0.0])
    t2 = np.array([0.0, 0.0, 1.0])
    bp1, bp2 = amp * np.sin(ph), amp * np.cos(ph)
    B = [par[c] + bp1 * t1[c] + bp2 * t2[c] for c in range(3)]
    V = [-(bp1 * t1[c] + bp2 * t2[c]) for c in range(3)]
    return prim_to_cons_ic(p, 1.0, V[0], V[1], V[2], 0.1, B[0], B[1], B[2])


def cpa_3d(n=64, limiter=MC, riemann=HLLD) -> Problem:
    """3D circularly polarised Alfven wave (the paper's second gPLUTO benchmark, PAPER.md:176-181
    §4.2; parameters deferred there, reading R23 / SPEC.md:140): rho = 1, p = 0.1, B_par = 1,
    amplitude 0.1, propagating along the box diagonal n = (1,1,1)/sqrt3 of the periodic unit cube
    (wave vector 2pi(1,1,1): one wavelength 1/sqrt3 per axis period); v_A = 1, so the exact
    solution returns to the initial condition after one period t = 1/sqrt3."""
    return Problem("cpa3d", (n, n, n), gamma=5.0 / 3.0, limiter=limiter, riemann=riemann, glm=1,
                   t_end=1.0 / math.sqrt(3.0))


def cpa_3d_fields(p: Problem, t: float = 0.0, amp: float = 0.1, z_range=None):
    """primitive fields (rho, v, p, B) of the exact 3D CPA solution at time t (cell centres)."""
    sub = p
    if z_range is not None:
        k0, k1 = z_range
        dz = (p.hi[2] - p.lo[2]) / p.n[2]
        sub = p.replace(n=(p.n[0], p.n[1], k1 - k0), lo=(p.lo[0], p.lo[1], p.lo[2] + k0 * dz),
                        hi=(p.hi[0], p.hi[1], p.lo[2] + k1 * dz))
    X, Y, Z = mesh(sub)
    s3 = math.sqrt(3.0)
    n = np.array([1.0, 1.0, 1.0]) / s3
    t1 = np.array([1.0, -1.0, 0.0]) / math.sqrt(2.0)
    t2 = np.array([1.0, 1.0, -2.0]) / math.sqrt(6.0)
    ph = 2.0 * math.pi * ((X + Y + Z) - s3 * t)  # phase moves at v_A = 1 along n
    b1, b2 = amp * np.sin(ph), amp * np.cos(ph)
    B = [n[c] + b1 * t1[c] + b2 * t2[c] for c in range(3)]
    V = [-(b1 * t1[c] + b2 * t2[c]) for c in range(3)]  # v_perp = -B_perp/sqrt(rho): moves along +n
    return 1.0, V, 0.1, B


def cpa_3d_ic(p: Problem, z_range=None) -> np.ndarray:
    rho, V, pr, B = cpa_3d_fields(p, 0.0, z_range=z_range)
    sub = p if z_range is None else p.replace(n=(p.n[0], p.n[1], z_range[1] - z_range[0]))
    return prim_to_cons_ic(sub, rho, V[0], V[1], V[2], pr, B[0], B[1], B[2])


def ct_problem(p: Problem) -> Problem:
    """the same problem with constrained transport instead of GLM (3D periodic only)"""
    return p.replace(ct=1, glm=0)


def _edge_coords(p: Problem, stag):
    """meshgrid of cell centres shifted by -1/2 cell along the axes in stag (edge / face centres)"""
    cs = []
    for d in range(3):
        dx = (p.hi[d] - p.lo[d]) / p.n[d]
        c = p.lo[d] + (np.arange(p.n[d], dtype=np.float64) + (0.0 if d in stag else 0.5)) * dx
        cs.append(c)
    Z, Y, X = np.meshgrid(cs[2], cs[1], cs[0], indexing="ij")
    return X, Y, Z


def ct_faces_from_potential(p: Problem, A_fn, b0=(0.0, 0.0, 0.0)) -> np.ndarray:
    """face-centred field b = curl A from the edge-centred vector potential A_fn(X, Y, Z) -> (Ax, Ay, Az)
    (discretely divergence-free to rounding), plus a uniform field b0.  Returns [3][nz][ny][nx]:
    b_x at x-face i-1/2, b_y at y-face j-1/2, b_z at z-face k-1/2 of cell (i,j,k)."""
    dx = [(p.hi[d] - p.lo[d]) / p.n[d] for d in range(3)]
    Ax = A_fn(*_edge_coords(p, (1, 2)))[0]  # at (x_i, y_{j-1/2}, z_{k-1/2})
    Ay = A_fn(*_edge_coords(p, (0, 2)))[1]  # at (x_{i-1/2}, y_j, z_{k-1/2})
    Az = A_fn(*_edge_coords(p, (0, 1)))[2]  # at (x_{i-1/2}, y_{j-1/2}, z_k)
    up = lambda a, ax: np.roll(a, -1, axis=ax)  # value at index + 1 (periodic); axes: 0 z, 1 y, 2 x
    bx = (up(Az, 1) - Az) / dx[1] - (up(Ay, 0) - Ay) / dx[2] + b0[0]
    by = (up(Ax, 0) - Ax) / dx[2] - (up(Az, 2) - Az) / dx[0] + b0[1]
    bz = (up(Ay, 2) - Ay) / dx[0] - (up(Ax, 1) - Ax) / dx[1] + b0[2]
    return np.stack([bx, by, bz])


def ct_state(p: Problem, rho, V, pr, bface) -> np.ndarray:
    """CT conservative state: rho, m, E with the cell-centred B = face average, and the face fields."""
    bc = [0.5 * (bface[0] + np.roll(bface[0], -1, axis=2)), 0.5 * (bface[1] + np.roll(bface[1], -1, axis=1)),
          0.5 * (bface[2] + np.roll(bface[2], -1, axis=0))]
    U = prim_to_cons_ic(p, rho, V[0], V[1], V[2], pr, bc[0], bc[1], bc[2])
    U[5:8] = bface
    return U


def cpa_3d_ct_ic(p: Problem, amp: float = 0.1) -> np.ndarray:
    """3D CPA with face-centred b = B_par n + curl A_w, A_w = (amp/|k|)(sin phi t1 + cos phi t2)
    (curl A_w = amp (sin phi t1 + cos phi t2) for phi = k.x, k = 2pi(1,1,1))."""
    s3 = math.sqrt(3.0)
    n = np.array([1.0, 1.0, 1.0]) / s3
    t1 = np.array([1.0, -1.0, 0.0]) / math.sqrt(2.0)
    t2 = np.array([1.0, 1.0, -2.0]) / math.sqrt(6.0)
    kabs = 2.0 * math.pi * s3

    def A(X, Y, Z):
        ph = 2.0 * math.pi * (X + Y + Z)
        return [(amp / kabs) * (np.sin(ph) * t1[c] + np.cos(ph) * t2[c]) for c in range(3)]
    bface = ct_faces_from_potential(p, A, b0=tuple(n))
    rho, V, pr, _ = cpa_3d_fields(p, 0.0, amp)
    return ct_state(p, rho, V, pr, bface)


def with_noise(U: np.ndarray, p: Problem, amp: float = 1e-3, seed: int = 2510) -> np.ndarray:
    """'OT + noise' stress IC: multiplies rho and E by (1 + amp*U(-1,1)), seeded."""
    rng = np.random.default_rng(seed)
    U = U.copy()
    U[0] *= 1.0 + amp * rng.uniform(-1.0, 1.0, size=U[0].shape)
    U[4] *= 1.0 + amp * rng.uniform(-1.0, 1.0, size=U[4].shape)
    return U


def random_face_states(n: int, seed: int, glm: bool = True, jump: float = None):
    """Random physical primitive pairs in the normal frame:
    rho, p log-uniform in [1e-2, 1e2]; v, B uniform in [-2, 2]; psi uniform in [-0.1, 0.1].
    With ``jump`` the right state is the left one perturbed by a relative factor up to ``jump``
    (neighbour-like pairs)."""
    rng = np.random.default_rng(seed)
    nvar = 9 if glm else 8

    def draw(m):
        V = np.empty((m, nvar))
        V[:, 0] = 10.0 ** rng.uniform(-2, 2, m)
        V[:, 1:4] = rng.uniform(-2, 2, (m, 3))
        V[:, 4] = 10.0 ** rng.uniform(-2, 2, m)
        V[:, 5:8] = rng.uniform(-2, 2, (m, 3))
        if glm:
            V[:, 8] = rng.uniform(-0.1, 0.1, m)
        return V

    VL = draw(n)
    if jump is None:
        VR = draw(n)
    else:
        VR = VL * (1.0 + jump * rng.uniform(-1, 1, VL.shape))
    return VL, VR


# ----------------------------------------------------------------------------------------------
# BASELINE.json configs
# ----------------------------------------------------------------------------------------------
CONFIGS = {
    "brio_wu_512": (lambda: brio_wu(512), brio_wu_ic),
    "ot2d_512": (lambda: orszag_tang_2d(512), orszag_tang_2d_ic),
    "ot3d_256": (lambda: orszag_tang_3d(256), orszag_tang_3d_ic),
    "blast3d_512": (lambda: blast_3d(512), blast_3d_ic),
    "ot3d_1024": (lambda: orszag_tang_3d(1024), orszag_tang_3d_ic),
    "cpa3d_256": (lambda: cpa_3d(256), cpa_3d_ic),
}


def workload_ic(workload: str, p: Problem, z0: int = 0, z1: int = -1, chunk: int = 64) -> np.ndarray:
    """Initial condition of global planes [z0, z1) of a bench workload ("ot3d", "blast3d",
    "cpa3d"), generated in z chunks into one array (keeps the host peak near the array size
    for 1024^3)."""
    z1 = p.n[2] if z1 < 0 else z1
    if p.ct and workload == "cpa3d":  # face fields from the edge vector potential (whole grid)
        assert (z0, z1) == (0, p.n[2])
        return cpa_3d_ct_ic(p)
    fn = {"ot3d": orszag_tang_3d_ic, "blast3d": blast_3d_ic, "cpa3d": cpa_3d_ic}[workload]
    pg = p.replace(ct=0, glm=1) if p.ct else p  # OT and blast fields are face-exact: CT takes fields 0..7
    U = np.empty((p.nvar, z1 - z0, p.n[1], p.n[0]), dtype=np.float64)
    for a in range(z0, z1, chunk):
        b = min(z1, a + chunk)
        U[:, a - z0:b - z0] = fn(pg, z_range=(a, b))[:p.nvar]
    return U
