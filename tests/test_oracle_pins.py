"""Pins of the CPU oracle's building blocks against closed forms, textbook special cases and
properties fixed by the mathematics (table "what pins each part"; SURVEY.md
§8(c).18).  Nothing here retypes the oracle's own association order: the expected values come
from textbook formulas, worked examples, brute force or exact invariants.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2510_24175_b200 import inputs as I


# ---------------------------------------------------------------------------------------------
# textbook helpers (independent of the oracle)
# ---------------------------------------------------------------------------------------------
def phys_flux_textbook(V, gamma):
    """ideal-MHD x-flux of primitive V=(rho,u,v,w,p,Bx,By,Bz) (e.g. Miyoshi & Kusano 2005 eq. 2-3)."""
    r, u, v, w, p, bx, by, bz = V[:8]
    B2 = bx * bx + by * by + bz * bz
    pt = p + B2 / 2
    E = p / (gamma - 1) + r * (u * u + v * v + w * w) / 2 + B2 / 2
    vb = u * bx + v * by + w * bz
    return np.array([r * u, r * u * u + pt - bx * bx, r * u * v - bx * by, r * u * w - bx * bz,
                     (E + pt) * u - bx * vb, 0.0, by * u - bx * v, bz * u - bx * w])


def cf_textbook(gamma, r, p, bn, bt1, bt2):
    a2 = gamma * p / r
    b2 = (bn * bn + bt1 * bt1 + bt2 * bt2) / r
    return math.sqrt(0.5 * (a2 + b2 + math.sqrt((a2 + b2) ** 2 - 4 * a2 * bn * bn / r)))


def hllc_toro(VL, VR, gamma):
    """HLLC for Euler (Toro ch. 10.4) with the same outer speed estimates as the oracle's reading
    R4 (Miyoshi-Kusano eq. 67) so that HLLD(B=0) must reduce to it (M&K 2005 §4)."""
    def state(V):
        r, u, v, w, p = V[:5]
        E = p / (gamma - 1) + 0.5 * r * (u * u + v * v + w * w)
        U = np.array([r, r * u, r * v, r * w, E])
        F = np.array([r * u, r * u * u + p, r * u * v, r * u * w, (E + p) * u])
        return U, F, math.sqrt(gamma * p / r)
    UL, FL, cL = state(VL)
    UR, FR, cR = state(VR)
    SL = min(VL[1], VR[1]) - max(cL, cR)
    SR = max(VL[1], VR[1]) + max(cL, cR)
    if SL > 0:
        return FL
    if SR < 0:
        return FR
    rL, uL, pL = VL[0], VL[1], VL[4]
    rR, uR, pR = VR[0], VR[1], VR[4]
    Ss = (pR - pL + rL * uL * (SL - uL) - rR * uR * (SR - uR)) / (rL * (SL - uL) - rR * (SR - uR))

    def ustar(U, V, S):
        r, u, v, w, p = V[:5]
        fac = r * (S - u) / (S - Ss)
        E = U[4]
        return fac * np.array([1.0, Ss, v, w, E / r + (Ss - u) * (Ss + p / (r * (S - u)))])
    if Ss >= 0:
        return FL + SL * (ustar(UL, VL, SL) - UL)
    return FR + SR * (ustar(UR, VR, SR) - UR)


def prob(glm=1, riemann=I.HLLD, gamma=5.0 / 3.0, limiter=I.MC):
    return I.Problem("unit", (8, 1, 1), gamma=gamma, glm=glm, riemann=riemann, limiter=limiter)


# ---------------------------------------------------------------------------------------------
# c.3 / c.4 conservative <-> primitive
# ---------------------------------------------------------------------------------------------
def test_energy_worked_examples():
    # rho=1, v=0, p=1, B=0, gamma=5/3 -> E = 1.5
    # (gamma-1 = 2/3 is not representable: the bar is 2 ulp, SPEC.md:55 asks 1e-13)
    assert abs(oracle.total_energy(5 / 3, np.array([1, 0, 0, 0, 1, 0, 0, 0.0])) - 1.5) <= 2 * np.finfo(float).eps * 1.5
    # rho=1, v=(1,0,0), p=0.6, B=(0.5,0,0) -> E = 0.6/(2/3) + 0.5 + 0.125 = 1.525
    E = oracle.total_energy(5 / 3, np.array([1, 1, 0, 0, 0.6, 0.5, 0, 0.0]))
    assert abs(E - 1.525) <= 2 * np.finfo(float).eps * 1.525


def test_cons2prim_worked_example_and_roundtrip():
    p = prob(glm=0)
    V, fl = oracle.cons2prim(p, np.array([1, 1, 0, 0, 1.525, 0.5, 0, 0.0]))
    assert fl == 0
    assert np.allclose(V, [1, 1, 0, 0, 0.6, 0.5, 0, 0], rtol=0, atol=4e-16)
    rng = np.random.default_rng(7)
    pg = prob(glm=1)
    for _ in range(500):
        Vt = np.concatenate([[10 ** rng.uniform(-2, 2)], rng.uniform(-2, 2, 3), [10 ** rng.uniform(-2, 2)],
                             rng.uniform(-2, 2, 3), rng.uniform(-0.1, 0.1, 1)])
        U = I.prim_to_cons_ic(I.Problem("c", (1, 1, 1), gamma=pg.gamma), *Vt[:8], psi=Vt[8])[:, 0, 0, 0]
        V, fl = oracle.cons2prim(pg, U)
        assert fl == 0
        scale = np.abs(Vt).max()
        # pressure recovery loses digits when p << kinetic+magnetic energy (SPEC.md:55 1e-13 bar
        # is relative to the state's energy scale)
        tol = 1e-13 * np.maximum(np.abs(Vt), 1.0)
        tol[4] = 1e-13 * max(U[4], 1.0) * (pg.gamma - 1)
        assert np.all(np.abs(V - Vt) <= tol + 1e-15 * scale), (Vt, V)


def test_pressure_floor_counted():
    p = prob(glm=0)
    U = np.array([1.0, 0, 0, 0, 0.5 * 1.0, 1.0, 0, 0])  # E = 0.5 = magnetic energy -> p = 0
    V, fl = oracle.cons2prim(p, U)
    assert fl == 1 and V[4] == p.p_floor


# ---------------------------------------------------------------------------------------------
# c.4 fast speed
# ---------------------------------------------------------------------------------------------
def test_fast_speed_special_cases():
    g = 5 / 3
    # B = 0: sound speed (1 ulp: two correctly-rounded sqrt of an exact square-root form)
    for r, p in [(1.0, 1.0), (0.125, 0.1), (3.7, 0.02)]:
        c = oracle.fast_speed(g, r, p, 0, 0, 0)
        assert abs(c - math.sqrt(g * p / r)) <= 2 * np.finfo(float).eps * c
    # B_t = 0: c_f = max(a, |b_n|)
    for r, p, bn in [(1.0, 1.0, 0.3), (1.0, 0.1, 2.0), (2.0, 0.5, -1.5)]:
        c = oracle.fast_speed(g, r, p, bn, 0, 0)
        ref = max(math.sqrt(g * p / r), abs(bn) / math.sqrt(r))
        assert abs(c - ref) <= 4 * np.finfo(float).eps * ref
    # general: textbook form
    rng = np.random.default_rng(3)
    for _ in range(1000):
        r, p = 10 ** rng.uniform(-2, 2, 2)
        b = rng.uniform(-2, 2, 3)
        c = oracle.fast_speed(g, r, p, *b)
        assert abs(c - cf_textbook(g, r, p, *b)) <= 1e-13 * c


# ---------------------------------------------------------------------------------------------
# c.5 limiters: truth table, constants, linear data, TVD bound
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("dm,dp,mm,mc", [
    (1.0, 2.0, 1.0, 1.5), (2.0, 1.0, 1.0, 1.5), (1.0, 5.0, 1.0, 2.0), (-1.0, -5.0, -1.0, -2.0),
    (-3.0, -1.0, -1.0, -2.0), (1.0, -1.0, 0.0, 0.0), (-1.0, 1.0, 0.0, 0.0), (0.0, 3.0, 0.0, 0.0),
    (3.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0), (0.25, 0.25, 0.25, 0.25), (-0.5, -0.5, -0.5, -0.5)])
def test_limiter_truth_table(dm, dp, mm, mc):
    assert oracle.limited_slope(0, dm, dp) == mm
    assert oracle.limited_slope(1, dm, dp) == mc


def test_limiter_tvd_random():
    rng = np.random.default_rng(11)
    for lim in (0, 1):
        for _ in range(2000):
            a, b, c = rng.normal(size=3)
            s = oracle.limited_slope(lim, b - a, c - b)
            for face in (b + 0.5 * s, b - 0.5 * s):
                assert min(a, b, c) - 1e-15 <= face <= max(a, b, c) + 1e-15


# ---------------------------------------------------------------------------------------------
# c.6-c.10 Riemann fluxes
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("riemann", [I.HLL, I.HLLD])
def test_flux_consistency(riemann):
    """F(V,V) = physical flux; psi/Bn entries from the GLM pre-solve."""
    p = prob(glm=1, riemann=riemann)
    VL, _ = I.random_face_states(400, seed=5)
    F, nfb = oracle.face_flux(p, VL, VL, ch=2.0)
    assert nfb == 0
    for q in range(len(VL)):
        ref = phys_flux_textbook(VL[q], p.gamma)
        scale = np.abs(ref).max() + 1.0
        assert np.all(np.abs(F[q, [0, 1, 2, 3, 4, 6, 7]] - ref[[0, 1, 2, 3, 4, 6, 7]]) <= 1e-12 * scale)
        assert F[q, 5] == VL[q, 8]                     # psi_m = psi
        assert F[q, 8] == 4.0 * VL[q, 5]               # ch^2 * Bm = ch^2 * Bn


@pytest.mark.parametrize("riemann", [I.HLL, I.HLLD])
def test_flux_upwind_limits(riemann):
    """supersonic to the right -> F = physical F(VL); to the left -> F(VR)."""
    p = prob(glm=0, riemann=riemann)
    VL, VR = I.random_face_states(200, seed=8, glm=False)
    VL[:, 5] = VR[:, 5]  # common Bn (1D, no GLM)
    for sgn in (+1, -1):
        a, b = VL.copy(), VR.copy()
        a[:, 1] = sgn * 500.0
        b[:, 1] = sgn * 500.0
        F, _ = oracle.face_flux(p, a, b, 1.0)
        Fs, _ = oracle.face_flux(p, a if sgn > 0 else b, a if sgn > 0 else b, 1.0)
        assert np.array_equal(F, Fs)
        for q in range(len(a)):
            ref = phys_flux_textbook(a[q] if sgn > 0 else b[q], p.gamma)
            assert np.allclose(F[q], ref, rtol=1e-13, atol=1e-12 * np.abs(ref).max())


def test_hlld_stationary_contact_exact():
    """HLLD resolves an isolated stationary contact exactly: mass and energy flux 0 (M&K 2005 §3);
    HLL smears it (non-zero mass flux) — this makes the pin discriminating."""
    g = 5 / 3
    for bn in (0.0, 0.7):
        VL = np.array([1.0, 0, 0, 0, 1.0, bn, 0.4, -0.3])
        VR = np.array([5.0, 0, 0, 0, 1.0, bn, 0.4, -0.3])
        Fd, _ = oracle.face_flux(prob(glm=0, riemann=I.HLLD, gamma=g), VL, VR, 1.0)
        Fh, _ = oracle.face_flux(prob(glm=0, riemann=I.HLL, gamma=g), VL, VR, 1.0)
        assert abs(Fd[0, 0]) <= 1e-14 and abs(Fd[0, 4]) <= 1e-14
        assert abs(Fh[0, 0]) > 1e-2


def test_hlld_stationary_rotational_discontinuity_exact():
    """An isolated stationary rotational (Alfven) discontinuity — rho, p, vn = Bn/sqrt(rho), |Bt|
    continuous and [vt] = [Bt]/sqrt(rho) (Rankine-Hugoniot) — is resolved exactly by HLLD
    (M&K 2005 §3): the numerical flux equals the physical flux of either side."""
    g = 5 / 3
    rng = np.random.default_rng(21)
    for _ in range(50):
        r, p = 10 ** rng.uniform(-1, 1, 2)
        bn = rng.uniform(0.5, 2.0)
        bmag = rng.uniform(0.2, 2.0)
        th1, th2 = rng.uniform(0, 2 * math.pi, 2)
        btL = bmag * np.array([math.cos(th1), math.sin(th1)])
        btR = bmag * np.array([math.cos(th2), math.sin(th2)])
        vn = bn / math.sqrt(r)
        vtL = rng.uniform(-1, 1, 2)
        vtR = vtL + (btR - btL) / math.sqrt(r)
        VL = np.array([r, vn, *vtL, p, bn, *btL])
        VR = np.array([r, vn, *vtR, p, bn, *btR])
        FL, FR = phys_flux_textbook(VL, g), phys_flux_textbook(VR, g)
        assert np.allclose(FL, FR, rtol=0, atol=1e-12 * (np.abs(FL).max() + 1))  # the test case is an RD
        F, nfb = oracle.face_flux(prob(glm=0, riemann=I.HLLD, gamma=g), VL, VR, 1.0)
        assert nfb == 0
        assert np.allclose(F[0], FL, rtol=0, atol=1e-11 * (np.abs(FL).max() + 1))
        Fh, _ = oracle.face_flux(prob(glm=0, riemann=I.HLL, gamma=g), VL, VR, 1.0)
        assert not np.allclose(Fh[0], FL, rtol=0, atol=1e-6)


def test_hlld_reduces_to_hllc_without_field():
    """B = 0: HLLD = HLLC (M&K 2005 §4) against an independent Toro HLLC."""
    for gamma in (1.4, 5 / 3):
        p = prob(glm=0, riemann=I.HLLD, gamma=gamma)
        VL, VR = I.random_face_states(2000, seed=13, glm=False)
        VL[:, 5:8] = 0.0
        VR[:, 5:8] = 0.0
        F, nfb = oracle.face_flux(p, VL, VR, 1.0)
        assert nfb == 0
        for q in range(len(VL)):
            ref = hllc_toro(VL[q], VR[q], gamma)
            scale = np.abs(ref).max() + 1e-300
            got = F[q, :5]
            assert np.all(np.abs(got - ref) <= 1e-12 * scale), (q, got, ref)
            assert F[q, 5:].tolist() == [0.0, 0.0, 0.0]


def test_hll_flux_integral_consistency():
    """HLL: F = (SR FL - SL FR + SL SR (UR-UL))/(SR-SL) is the flux whose single intermediate state is
    the integral average of the Riemann fan (Harten-Lax-van Leer 1983).  Pin it by the identity
    SR*U_hll - F = SR*UR - FR with U_hll = (SR UR - SL UL - (FR-FL))/(SR-SL), evaluated with textbook
    fluxes and the textbook fast speed."""
    g = 5 / 3
    p = prob(glm=0, riemann=I.HLL, gamma=g)
    VL, VR = I.random_face_states(300, seed=17, glm=False)
    VR[:, 5] = VL[:, 5]
    F, _ = oracle.face_flux(p, VL, VR, 1.0)
    for q in range(len(VL)):
        cl = cf_textbook(g, VL[q, 0], VL[q, 4], *VL[q, 5:8])
        cr = cf_textbook(g, VR[q, 0], VR[q, 4], *VR[q, 5:8])
        SL = min(VL[q, 1], VR[q, 1]) - max(cl, cr)
        SR = max(VL[q, 1], VR[q, 1]) + max(cl, cr)
        if SL > 0 or SR < 0:
            continue

        def U(V):
            r, u, v, w, pr, bx, by, bz = V
            return np.array([r, r * u, r * v, r * w, pr / (g - 1) + r * (u * u + v * v + w * w) / 2 +
                             (bx * bx + by * by + bz * bz) / 2, bx, by, bz])
        FL, FR = phys_flux_textbook(VL[q], g), phys_flux_textbook(VR[q], g)
        Uh = (SR * U(VR[q]) - SL * U(VL[q]) - (FR - FL)) / (SR - SL)
        lhs = SR * Uh - F[q, :8]
        rhs = SR * U(VR[q]) - FR
        scale = np.abs(rhs).max() + np.abs(SR * Uh).max()
        assert np.all(np.abs(lhs - rhs) <= 1e-12 * scale)


def test_glm_interface_solution():
    """c.6: the GLM subsystem (d_t Bn + d_x psi = 0, d_t psi + ch^2 d_x Bn = 0) is linear with
    characteristic speeds +-ch; its exact Riemann solution at the interface is
    Bm = (BL+BR)/2 - (psiR-psiL)/(2ch), psim = (psiL+psiR)/2 - ch (BR-BL)/2 (Dedner et al. 2002 eq. 41).
    Pin: the interface state is constant along both characteristics, psi +- ch*B is carried unchanged."""
    p = prob(glm=1)
    VL, VR = I.random_face_states(500, seed=19)
    ch = 1.7
    F, _ = oracle.face_flux(p, VL, VR, ch)
    Bm = F[:, 8] / (ch * ch)
    psim = F[:, 5]
    # right-going characteristic w+ = psi + ch*B comes from the left, w- = psi - ch*B from the right
    assert np.allclose(psim + ch * Bm, VL[:, 8] + ch * VL[:, 5], rtol=0, atol=1e-12)
    assert np.allclose(psim - ch * Bm, VR[:, 8] - ch * VR[:, 5], rtol=0, atol=1e-12)


def test_frame_rotation_invariance_bitwise():
    """R8: permuting vector components is exact, so the y- and z-direction fluxes of the stage
    operator equal the x-direction flux with components permuted, bitwise.  Checked on a full
    stage: Brio-Wu along x vs along y vs along z."""
    px = I.brio_wu(64)
    U = I.brio_wu_ic(px)
    out_x, cx = oracle.stage(px, U, 1e-3, 1.0)
    for d in (1, 2):
        n = [1, 1, 1]
        n[d] = 64
        pd = px.replace(n=tuple(n))
        Ud = np.empty((8,) + tuple(reversed(n)))
        for f in range(8):
            src = f
            if 1 <= f <= 3:
                src = 1 + (f - 1 - d) % 3
            if 5 <= f <= 7:
                src = 5 + (f - 5 - d) % 3
            Ud[f] = U[src].reshape(tuple(reversed(n)))
        out_d, cd = oracle.stage(pd, Ud, 1e-3, 1.0)
        for f in range(8):
            src = f
            if 1 <= f <= 3:
                src = 1 + (f - 1 - d) % 3
            if 5 <= f <= 7:
                src = 5 + (f - 5 - d) % 3
            assert np.array_equal(out_d[f].ravel(), out_x[src].ravel()), (d, f)
        assert cd == cx


# ---------------------------------------------------------------------------------------------
# WENO-Z reconstruction (§8(f) row 3; Borges et al. 2008, reading R31)
# ---------------------------------------------------------------------------------------------
def test_wenoz_constants_and_quadratics():
    for c in (1.0, 1.3, -2.7e-3, 5e4):
        assert abs(oracle.wenoz(c, c, c, c, c) - c) <= 4 * np.finfo(float).eps * abs(c)
    # cell averages of a quadratic: all three candidate stencils are exact, so the face value
    # is exact whatever the nonlinear weights (f = x^2 on unit cells: avg_i = i^2 + 1/12)
    rng = np.random.default_rng(3)
    for _ in range(200):
        a2, a1, a0, h = rng.normal(size=3).tolist() + [10 ** rng.uniform(-3, 0)]
        def avg(i):  # average of a0 + a1 x + a2 x^2 over [(i-1/2)h, (i+1/2)h]
            return a0 + a1 * i * h + a2 * (i * i * h * h + h * h / 12.0)
        exact = a0 + a1 * 0.5 * h + a2 * 0.25 * h * h
        got = oracle.wenoz(avg(-2), avg(-1), avg(0), avg(1), avg(2))
        scale = abs(a0) + abs(a1) + abs(a2)
        assert abs(got - exact) <= 1e-13 * scale


def test_wenoz_essentially_non_oscillatory():
    """a jump across the face: the upwind smooth stencil dominates (weights of the stencils that
    cross the jump vanish like eps^2/beta^2), so no overshoot."""
    assert abs(oracle.wenoz(0.0, 0.0, 0.0, 1.0, 1.0)) < 1e-30
    assert abs(oracle.wenoz(1.0, 1.0, 0.0, 0.0, 0.0)) < 1e-30
    rng = np.random.default_rng(5)
    for _ in range(500):
        lo, hi = sorted(rng.normal(size=2))
        v = [lo, lo, lo, hi, hi]
        q = oracle.wenoz(*v)
        assert lo - 1e-12 <= q <= lo + 1e-6 * (hi - lo) + 1e-12


def test_wenoz_fifth_order_on_smooth_data():
    """on smooth data the WENO-Z weights approach the linear weights fast enough that the
    reconstruction error of cell averages of sin falls at >= 4th order (5th for linear weights)."""
    errs = []
    for h in (0.1, 0.05, 0.025):
        def avg(i):  # average of sin over [(i-1/2)h + x0, (i+1/2)h + x0]
            x0 = 0.3
            return (math.cos(x0 + (i - 0.5) * h) - math.cos(x0 + (i + 0.5) * h)) / h
        got = oracle.wenoz(avg(-2), avg(-1), avg(0), avg(1), avg(2))
        errs.append(abs(got - math.sin(0.3 + 0.5 * h)))
    orders = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert min(orders) >= 4.0, (errs, orders)
