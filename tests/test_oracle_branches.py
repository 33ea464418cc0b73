"""Pins of the oracle's rare branches — -m "not gpu".

Each branch is pinned against something other than the oracle's own arithmetic:
  * R6  (HLLD degeneracy, Miyoshi & Kusano 2005 §4 "the degenerate case"):
        a tangential-velocity jump with B_t = 0 and c_A > a (fast = Alfven speed, so
        rho (S - v_n)(S - S_M) - B_n^2 = 0): the exact MHD solution is two Alfven waves with the
        closed-form middle state v_t = mean, B_t = sgn(B_n) sqrt(rho) dv_t / 2 — the HLLD flux
        must be the physical flux of that state (a wrong or missing degeneracy branch gives NaN
        or another state).
  * R7  (SM outside (SL, SR), and the wave-ordering guard S*L < SL or S*R > SR): the returned
        flux is the textbook HLL flux (Harten, Lax & van Leer 1983 with the M&K eq. 67 speeds),
        re-derived here from the textbook fast speed and physical flux; *when* the guard fires
        is checked against an independent transcription of M&K eqs. 38, 43, 51.
  * HLLD star states: the integral (HLL) consistency of the four intermediate states,
        sum_k (S_k+1 - S_k) U_k = SR UR - SL UL - (FR - FL) (Harten-Lax-van Leer), the
        Rankine-Hugoniot conditions across the outer waves S_a U*_a - F*_a = S_a U_a - F_a with
        F*_a the MHD flux of U*_a at normal velocity S_M and total pressure p_t* (the HLLD
        ansatz, M&K eqs. 31-36), and the jump conditions across the Alfven and contact waves
        (rho and v_n = S_M continuous across S*; v_t, B_t continuous across S_M).
  * R17 (reconstruction positivity fallback): on rough 1D data where WENO-Z gives rho+ or p-
        <= 0, one oracle stage equals bitwise the composition of independently pinned pieces
        (cons2prim, WENO-Z, the face flux) with those cells reconstructed at first order, the
        counter equals the number of such cells, and the fallback is what keeps the density
        positive where the unguarded reconstruction would not.
"""
import math

import numpy as np
import pytest

import oracle
from paper_2510_24175_b200 import inputs as I

from test_oracle_pins import cf_textbook, phys_flux_textbook


def prob(glm=0, riemann=I.HLLD, gamma=5.0 / 3.0, limiter=I.MC, n=8):
    return I.Problem("unit", (n, 1, 1), gamma=gamma, glm=glm, riemann=riemann, limiter=limiter)


def cons_textbook(V, gamma):
    r, u, v, w, p, bx, by, bz = V[:8]
    E = p / (gamma - 1) + r * (u * u + v * v + w * w) / 2 + (bx * bx + by * by + bz * bz) / 2
    return np.array([r, r * u, r * v, r * w, E, bx, by, bz])


def hll_textbook(VL, VR, gamma):
    """HLL flux with the Miyoshi-Kusano eq. 67 outer speeds, from textbook pieces."""
    cL = cf_textbook(gamma, VL[0], VL[4], VL[5], VL[6], VL[7])
    cR = cf_textbook(gamma, VR[0], VR[4], VR[5], VR[6], VR[7])
    SL = min(VL[1], VR[1]) - max(cL, cR)
    SR = max(VL[1], VR[1]) + max(cL, cR)
    FL, FR = phys_flux_textbook(VL, gamma), phys_flux_textbook(VR, gamma)
    if SL > 0:
        return FL
    if SR < 0:
        return FR
    UL, UR = cons_textbook(VL, gamma), cons_textbook(VR, gamma)
    return (SR * FL - SL * FR + SL * SR * (UR - UL)) / (SR - SL)


def mk_speeds_textbook(VL, VR, gamma):
    """M&K 2005 eqs. 38 (S_M), 43 (rho*), 51 (S*) and 67 (SL, SR), written from the paper's
    formulas in plain form."""
    cL = cf_textbook(gamma, VL[0], VL[4], VL[5], VL[6], VL[7])
    cR = cf_textbook(gamma, VR[0], VR[4], VR[5], VR[6], VR[7])
    SL = min(VL[1], VR[1]) - max(cL, cR)
    SR = max(VL[1], VR[1]) + max(cL, cR)
    B = VL[5]
    ptL = VL[4] + (VL[5] ** 2 + VL[6] ** 2 + VL[7] ** 2) / 2
    ptR = VR[4] + (VR[5] ** 2 + VR[6] ** 2 + VR[7] ** 2) / 2
    SM = ((SR - VR[1]) * VR[0] * VR[1] - (SL - VL[1]) * VL[0] * VL[1] - ptR + ptL) / (
        (SR - VR[1]) * VR[0] - (SL - VL[1]) * VL[0])
    rsL = VL[0] * (SL - VL[1]) / (SL - SM)
    rsR = VR[0] * (SR - VR[1]) / (SR - SM)
    SsL = SM - abs(B) / math.sqrt(rsL) if rsL > 0 else -math.inf
    SsR = SM + abs(B) / math.sqrt(rsR) if rsR > 0 else math.inf
    return SL, SsL, SM, SsR, SR


def rel_err(a, b):
    scale = max(np.abs(b).max(), 1e-300)
    return np.abs(np.asarray(a) - np.asarray(b)).max() / scale


# ---------------------------------------------------------------------------------------------
# R6: degenerate star states
# ---------------------------------------------------------------------------------------------
def test_r6_degenerate_alfven_split_of_tangential_jump():
    """B_t = 0 on both sides, c_A > a, equal rho, p, v_n; only v_t jumps, by eps.  To first order
    in eps the exact solution is two Alfven waves at v_n -+ c_A around the middle state
    (rho, v_n, mean v_t, p, B_n, sgn(B_n) sqrt(rho) (v_tR - v_tL)/2) (linearised ideal MHD: the
    Alfven eigenvectors dB_t = -+ sgn(B_n) sqrt(rho) dv_t); the nonlinear corrections (the
    magnetic pressure of the new B_t) are O(eps^2).  The HLLD flux — whose star states are the
    degenerate ones here — must equal the physical flux of that middle state to O(eps^2) while
    the flux itself changes at O(eps): a missing degeneracy branch gives NaN (1/0), a wrong one
    (e.g. v*_t = 0 or B*_t from the regular formulas at d = 0) an O(1) or O(eps) error."""
    p = prob()
    g = p.gamma
    rng = np.random.default_rng(6)
    checked = 0
    for _ in range(400):
        rho = 10 ** rng.uniform(-1, 1)
        pr = 10 ** rng.uniform(-3, -1)
        B = rng.choice([-1.0, 1.0]) * rng.uniform(1.0, 3.0)
        vn = rng.uniform(-0.5, 0.5)
        assert B * B / rho > g * pr / rho  # c_A > a: c_f = c_A, the degenerate case
        vt = rng.uniform(-1, 1, 2)
        dir_ = rng.uniform(-1, 1, 2)
        cA = abs(B) / math.sqrt(rho)
        if not (vn - cA < 0.0 < vn + cA):
            continue
        errs = []
        for eps in (1e-3, 1e-4):
            VL = np.array([rho, vn, *vt, pr, B, 0.0, 0.0])
            VR = VL.copy()
            VR[2:4] = vt + eps * dir_
            fan = oracle.hlld_fan(p, VL, VR, 1.0)
            assert fan["degL"] and fan["degR"], fan
            if fan["flag"] != 0:  # S*_a == S_a up to rounding: the ordering guard may take HLL (R7)
                break
            # the degenerate star states carry no tangential jump
            # (v*_t = v_t exactly; rho* = rho up to the rounding of m / (S - S_M))
            for Us, U in ((fan["UsL"], fan["UL"]), (fan["UsR"], fan["UR"])):
                assert np.all(Us[6:8] == 0.0) and abs(Us[0] / U[0] - 1.0) <= 1e-14
                assert np.abs(Us[2:4] / Us[0] - U[2:4] / U[0]).max() <= 1e-14 * (1 + np.abs(U[2:4] / U[0]).max())
            sg = math.copysign(1.0, B)
            mid = np.array([rho, vn, 0.5 * (VL[2] + VR[2]), 0.5 * (VL[3] + VR[3]), pr, B,
                            sg * math.sqrt(rho) * (VR[2] - VL[2]) / 2, sg * math.sqrt(rho) * (VR[3] - VL[3]) / 2])
            F, nfb = oracle.face_flux(p, VL, VR, 1.0)
            assert nfb == 0 and np.all(np.isfinite(F))
            Fmid = phys_flux_textbook(mid, g)
            change = np.abs(Fmid - phys_flux_textbook(VL, g)).max()
            err = np.abs(F[0] - Fmid).max()
            scale = np.abs(Fmid).max() + 1.0
            assert change > 0.1 * eps * abs(dir_).max() * min(1.0, abs(B))  # the flux does move at O(eps)
            assert err <= 5.0 * eps * eps * scale, (eps, err, F[0], Fmid)
            errs.append(err)
        else:
            checked += 1
    assert checked >= 60, checked
def test_r6_uniform_degenerate_state_is_consistent():
    """F(V, V) = physical F(V) at the degenerate point itself (no NaN from 1/d)."""
    p = prob()
    rng = np.random.default_rng(61)
    for _ in range(200):
        rho = 10 ** rng.uniform(-1, 1)
        V = np.array([rho, rng.uniform(-0.5, 0.5), *rng.uniform(-1, 1, 2), 10 ** rng.uniform(-3, -1),
                      rng.choice([-1.0, 1.0]) * rng.uniform(1, 3), 0.0, 0.0])
        fan = oracle.hlld_fan(p, V, V, 1.0)
        assert fan["flag"] == 3 or (fan["degL"] and fan["degR"])  # (3: supersonic, no fan)
        F, _ = oracle.face_flux(p, V, V, 1.0)
        assert rel_err(F[0], phys_flux_textbook(V, p.gamma)) <= 1e-13


# ---------------------------------------------------------------------------------------------
# R7: HLL fallbacks
# ---------------------------------------------------------------------------------------------
def _strong_pairs(rng, n):
    for _ in range(n):
        def st():
            return np.array([10 ** rng.uniform(-4, 4), rng.uniform(-20, 20), rng.uniform(-5, 5), rng.uniform(-5, 5),
                             10 ** rng.uniform(-4, 4), 0.0, rng.uniform(-5, 5), rng.uniform(-5, 5)])
        VL, VR = st(), st()
        VL[5] = VR[5] = rng.uniform(-5, 5)
        yield VL, VR


def test_r7_wave_ordering_guard_returns_textbook_hll():
    p = prob()
    g = p.gamma
    rng = np.random.default_rng(7)
    hits = agree = 0
    for VL, VR in _strong_pairs(rng, 60000):
        fan = oracle.hlld_fan(p, VL, VR, 1.0)
        F, nfb = oracle.face_flux(p, VL, VR, 1.0)
        assert nfb == (1 if fan["flag"] in (1, 2) else 0)
        SL, SsL, SM, SsR, SR = mk_speeds_textbook(VL, VR, g)
        scale = max(abs(SL), abs(SR))
        if fan["flag"] != 3:
            margin = min(SsL - SL, SR - SsR)
            # the guard fires exactly when the textbook ordering is violated (away from ties)
            if abs(margin) > 1e-9 * scale:
                assert (fan["flag"] == 2) == (margin < 0), (fan["flag"], margin)
                agree += 1
        if fan["flag"] == 2:
            hits += 1
            assert rel_err(F[0], hll_textbook(VL, VR, g)) <= 1e-12
    assert hits >= 40 and agree > 50000, (hits, agree)


def test_r7_sm_guard_returns_textbook_hll():
    """SM outside (SL, SR): with |v_n| = 1e17 colliding and a density ratio >= 1e20, S_M rounds
    onto SL; the flux is the HLL flux and the fallback is counted."""
    p = prob()
    for rr in (1e20, 1e25, 1e30):
        VL = np.array([1.0, 1e17, 0.3, -0.2, 1.0, 0.5, 0.4, 0.1])
        VR = np.array([rr, -1e17, 0.1, 0.2, 1.0, 0.5, -0.3, 0.2])
        fan = oracle.hlld_fan(p, VL, VR, 1.0)
        assert fan["flag"] == 1 and not (fan["SL"] < fan["SM"] < fan["SR"])
        F, nfb = oracle.face_flux(p, VL, VR, 1.0)
        assert nfb == 1
        assert rel_err(F[0], hll_textbook(VL, VR, p.gamma)) <= 1e-12


# ---------------------------------------------------------------------------------------------
# HLLD intermediate states: consistency and jump conditions
# ---------------------------------------------------------------------------------------------
def _fan_pairs(rng, n):
    for _ in range(n):
        VL = np.array([10 ** rng.uniform(-1, 1), rng.uniform(-1, 1), *rng.uniform(-1, 1, 2), 10 ** rng.uniform(-1, 1),
                       0.0, *rng.uniform(-2, 2, 2)])
        VR = np.array([10 ** rng.uniform(-1, 1), rng.uniform(-1, 1), *rng.uniform(-1, 1, 2), 10 ** rng.uniform(-1, 1),
                       0.0, *rng.uniform(-2, 2, 2)])
        VL[5] = VR[5] = rng.uniform(-2, 2)
        yield VL, VR


def test_hlld_integral_consistency_and_jump_conditions():
    p = prob()
    g = p.gamma
    rng = np.random.default_rng(18)
    n = 0
    for VL, VR in _fan_pairs(rng, 3000):
        f = oracle.hlld_fan(p, VL, VR, 1.0)
        if f["flag"] != 0:
            continue
        n += 1
        SL, SsL, SM, SsR, SR = f["SL"], f["SsL"], f["SM"], f["SsR"], f["SR"]
        UL, UsL, UssL, UssR, UsR, UR, FL, FR = (f[k] for k in ("UL", "UsL", "UssL", "UssR", "UsR", "UR", "FL", "FR"))
        # the side states and fluxes are the textbook ones
        assert rel_err(UL, cons_textbook(VL, g)) <= 1e-14 and rel_err(FL, phys_flux_textbook(VL, g)) <= 1e-14
        assert rel_err(UR, cons_textbook(VR, g)) <= 1e-14 and rel_err(FR, phys_flux_textbook(VR, g)) <= 1e-14
        # integral consistency (the fan averages to the HLL state)
        lhs = (SsL - SL) * UsL + (SM - SsL) * UssL + (SsR - SM) * UssR + (SR - SsR) * UsR
        rhs = SR * UR - SL * UL - (FR - FL)
        scale = np.abs(SR * UR).max() + np.abs(SL * UL).max() + np.abs(FR).max() + np.abs(FL).max()
        assert np.abs(lhs - rhs).max() <= 1e-12 * scale, (lhs, rhs)
        # Rankine-Hugoniot across the outer waves (M&K 2005 eqs. 31-36): the star state, with
        # normal velocity S_M and the total pressure p_t* of the HLLD ansatz, has the MHD flux
        # F(U*; p_t*) with F(U*) - F(U) = S (U* - U)
        pts = f["pts"]
        for S, U, F, Us in ((SL, UL, FL, UsL), (SR, UR, FR, UsR)):
            r = Us[0]
            v = Us[1:4] / r
            b = Us[5:8]
            Fs = np.array([r * v[0], r * v[0] * v[0] + pts - b[0] * b[0], r * v[0] * v[1] - b[0] * b[1],
                           r * v[0] * v[2] - b[0] * b[2], (Us[4] + pts) * v[0] - b[0] * (v @ b), 0.0,
                           b[1] * v[0] - b[0] * v[1], b[2] * v[0] - b[0] * v[2]])
            jump = Fs - F - S * (Us - U)
            sc = np.abs(F).max() + abs(S) * (np.abs(Us).max() + np.abs(U).max())
            assert np.abs(jump).max() <= 1e-12 * sc, jump
        # across the Alfven waves rho and v_n = SM; across the contact v_t and B_t continuous
        assert UssL[0] == UsL[0] and UssR[0] == UsR[0]
        assert np.array_equal(UssL[5:8], UssR[5:8])
        assert abs(UssL[2] / UssL[0] - UssR[2] / UssR[0]) <= 1e-12 * (1 + abs(UssL[2] / UssL[0]))
        assert abs(UsL[1] / UsL[0] - SM) <= 1e-12 * (1 + abs(SM)) and abs(UsR[1] / UsR[0] - SM) <= 1e-12 * (1 + abs(SM))
        # the face flux is the flux of the region containing x/t = 0, built from these states
        F0, _ = oracle.face_flux(p, VL, VR, 1.0)
        FsL, FsR = FL + SL * (UsL - UL), FR + SR * (UsR - UR)
        if SsL >= 0:
            Fr = FsL
        elif SM >= 0:
            Fr = FsL + SsL * (UssL - UsL)
        elif SsR >= 0:
            Fr = FsR + SsR * (UssR - UsR)
        else:
            Fr = FsR
        assert rel_err(F0[0], Fr) <= 1e-13
    assert n > 2000


# ---------------------------------------------------------------------------------------------
# R17: reconstruction positivity fallback (WENO-Z)
# ---------------------------------------------------------------------------------------------
def _rough_1d(n, seed):
    rng = np.random.default_rng(seed)
    rho = 10 ** rng.uniform(-3, 1, n)
    pr = 10 ** rng.uniform(-3, 0, n)
    v = rng.uniform(-0.2, 0.2, (3, n))
    B = np.stack([np.full(n, 0.7), rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n)])
    return rho, v, pr, B


def test_r17_wenoz_positivity_fallback_first_order():
    n = 24
    p = I.Problem("rough", (n, 1, 1), gamma=5.0 / 3.0, glm=0, riemann=I.HLLD, limiter=I.WENOZ)
    rho, v, pr, B = _rough_1d(n, 17)
    U = I.prim_to_cons_ic(p, rho[None, None], v[0][None, None], v[1][None, None], v[2][None, None],
                          pr[None, None], B[0][None, None], B[1][None, None], B[2][None, None])
    dt, ch = 1e-4, 1.0
    S, cnt = oracle.stage(p, U, dt, ch)
    # the same stage from pinned pieces: cons2prim, WENO-Z, face flux (x is the normal frame)
    Vc = np.stack([oracle.cons2prim(p, U[:, 0, 0, i])[0] for i in range(n)], axis=1)  # [nvar][n]
    qp, qm = np.zeros_like(Vc), np.zeros_like(Vc)
    fallback = np.zeros(n, dtype=bool)
    unguarded_bad = 0
    for i in range(n):
        w = [Vc[:, (i + o) % n] for o in (-2, -1, 0, 1, 2)]
        for f in range(8):
            qp[f, i] = oracle.wenoz(w[0][f], w[1][f], w[2][f], w[3][f], w[4][f])
            qm[f, i] = oracle.wenoz(w[4][f], w[3][f], w[2][f], w[1][f], w[0][f])
        if not (qp[0, i] > 0 and qm[0, i] > 0 and qp[4, i] > 0 and qm[4, i] > 0):
            fallback[i] = True
            unguarded_bad += 1
            qp[:, i] = qm[:, i] = Vc[:, i]
    assert fallback.sum() >= 3, fallback.sum()  # the data really exercise the branch
    assert cnt["plm_fallbacks"] == int(fallback.sum())
    Ff = np.zeros((8, n + 1))
    for i in range(n + 1):  # face i - 1/2
        F, _ = oracle.face_flux(p, qp[:, (i - 1) % n], qm[:, i % n], ch)
        Ff[:, i] = F[0]
    lam = dt / (1.0 / n)
    Uc = U[:, 0, 0, :]
    ref = Uc - lam * (Ff[:, 1:] - Ff[:, :-1])
    assert np.array_equal(S[:, 0, 0, :], ref)
    # without the fallback some face state would carry a non-positive density or pressure
    assert unguarded_bad == fallback.sum() > 0


@pytest.mark.parametrize("side", ["rho_plus", "p_minus"])
def test_r17_each_condition_triggers(side):
    """Both sides and both variables of the R17 condition matter: a cell where only rho+ (or only
    p-) is non-positive is reconstructed at first order."""
    rng = np.random.default_rng(170)
    while True:
        v = 10 ** rng.uniform(-3, 1, 5)
        a, b = oracle.wenoz(*v), oracle.wenoz(*v[::-1])
        if side == "rho_plus" and a <= 0 < b:
            break
        if side == "p_minus" and b <= 0 < a:
            break
    n = 12
    p = I.Problem("one", (n, 1, 1), gamma=5.0 / 3.0, glm=0, riemann=I.HLLD, limiter=I.WENOZ)
    rho = np.ones(n)
    pr = np.ones(n)
    sl = [(4 + o) % n for o in range(5)]
    if side == "rho_plus":
        rho[sl] = v
    else:
        pr[sl] = v
    z = np.zeros((1, 1, n))
    U = I.prim_to_cons_ic(p, rho[None, None], z, z, z, pr[None, None], z + 0.5, z, z)
    _, cnt = oracle.stage(p, U, 1e-5, 1.0)
    expect, only = 0, 0
    for i in range(n):
        wr = [rho[(i + o) % n] for o in (-2, -1, 0, 1, 2)]
        wp = [pr[(i + o) % n] for o in (-2, -1, 0, 1, 2)]
        c = [oracle.wenoz(*wr) <= 0, oracle.wenoz(*wr[::-1]) <= 0, oracle.wenoz(*wp) <= 0, oracle.wenoz(*wp[::-1]) <= 0]
        expect += any(c)
        only += c == ([True, False, False, False] if side == "rho_plus" else [False, False, False, True])
    assert only >= 1 and cnt["plm_fallbacks"] == expect
