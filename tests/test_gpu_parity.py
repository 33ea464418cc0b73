"""GPU parity: the CUDA path (through the C ABI, libmhd.so) against the independent CPU oracle on
identical seeded inputs.  Bar (BASELINE.json north star): per-field relative L-inf <= 1e-12 and an
exactly equal dt sequence; the recipe is designed for bitwise equality, so the
tests also report/require equal counters.  Sizes span several 32 x 8 tiles and ragged tails."""
import math
import os

import numpy as np
import pytest

import oracle
from paper_2510_24175_b200 import inputs as I

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def mhd():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from paper_2510_24175_b200 import mhd as M
    M.load()
    return M


def rel_linf(a, b):
    """per-field max|a-b| / max|b| (R24)."""
    out = []
    for f in range(a.shape[0]):
        scale = max(np.abs(b[f]).max(), 1e-300)
        out.append(np.abs(a[f] - b[f]).max() / scale)
    return np.array(out)


def run_both(mhd, p, U0, nsteps, t_end=0.0):
    o = oracle.Oracle(p, U0)
    log_o = o.run(nsteps, t_end)
    s = mhd.Solver(p)
    s.set_state(np.ascontiguousarray(U0))
    log_g = s.run(nsteps, t_end)
    Ug = s.get_state()
    dg = s.diag()
    s.destroy()
    return o, log_o, Ug, log_g, dg


def assert_parity(o, log_o, Ug, log_g, dg, exact_counters=True):
    assert len(log_o) == len(log_g)
    assert np.array_equal(log_o, log_g), "dt sequences differ"
    err = rel_linf(Ug, o.U)
    assert np.all(err <= TOL), err
    co = o.counters()
    if exact_counters:
        for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
            assert co[k] == dg[k], (k, co[k], dg[k])
    return err


# ---------------------------------------------------------------------------------------------
# face solve
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("riemann", [I.HLL, I.HLLD])
@pytest.mark.parametrize("glm", [0, 1])
@pytest.mark.parametrize("jump", [None, 0.5, 0.05])
def test_face_flux_bitwise(mhd, riemann, glm, jump):
    import torch
    p = I.Problem("ff", (8, 1, 1), riemann=riemann, glm=glm)
    VL, VR = I.random_face_states(20000, seed=101 + (0 if jump is None else int(jump * 100)), glm=bool(glm),
                                  jump=jump)
    if not glm:
        VR[:, 5] = VL[:, 5]
    ch = 3.3
    Fo, nfo = oracle.face_flux(p, VL, VR, ch)
    s = mhd.Solver(p)
    Fg, nfg = s.debug_face_flux(torch.from_numpy(VL).cuda(), torch.from_numpy(VR).cuda(), ch)
    s.destroy()
    Fg = Fg.cpu().numpy()
    assert nfo == nfg
    assert np.array_equal(Fo, Fg), np.abs(Fo - Fg).max()


def _fast_ops_inputs(n=1 << 21, seed=7):
    rng = np.random.default_rng(seed)
    m = n // 4
    wide = lambda: rng.choice([-1.0, 1.0], m) * 10.0 ** rng.uniform(-320, 308, m)
    mid = lambda: rng.choice([-1.0, 1.0], m) * 10.0 ** rng.uniform(-6, 6, m)
    bits = lambda: rng.integers(0, 2**64, m, dtype=np.uint64, endpoint=False).view(np.float64)
    special = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                        1.7976931348623157e308, 1.0, -1.0, 2.0, 0.5, 1.0 - 2**-53, 1.0 + 2**-52, 3.0,
                        np.nextafter(2.0, 0.0), 1e-300, 1e300, 4.0e-310], dtype=np.float64)
    sa, sb = np.meshgrid(special, special)
    # operands of the face solve: positive, O(1) to O(1e6), plus the all-ones mantissas
    pos = 10.0 ** rng.uniform(-4, 6, m)
    ones = (np.uint64(0x3FFFFFFFFFFFFFFF) - rng.integers(0, 1 << 12, m).astype(np.uint64)).view(np.float64)
    a = np.concatenate([wide(), mid(), bits(), pos, sa.ravel(), ones])
    b = np.concatenate([wide(), mid(), bits(), ones, sb.ravel(), pos])
    return a, b


def test_fast_div_sqrt_bitwise(mhd):
    """The branch-free reciprocal / division / square-root sequences of the face solve equal the
    IEEE operators bitwise wherever their range test passes, and the device IEEE operators equal
    numpy's (correctly rounded) results."""
    import torch
    a, b = _fast_ops_inputs()
    out, ok = mhd.debug_fast_ops(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda())
    out, ok = out.cpu().numpy(), ok.cpu().numpy()
    with np.errstate(all="ignore"):
        ref = [1.0 / b, a / b, np.sqrt(a), np.abs(a) / b]
    b_normal_pos = (b >= 2.2250738585072014e-308) & np.isfinite(b)
    for j in range(4):
        fast, ieee = out[:, 2 * j], out[:, 2 * j + 1]
        both_nan = np.isnan(ieee) & np.isnan(ref[j])
        assert np.array_equal(ieee.view(np.uint64)[~both_nan], ref[j].view(np.uint64)[~both_nan]), j
        sel = (ok >> j) & 1 == 1
        if j == 3:  # |a| / b is defined for positive normal b (a checked square root)
            sel &= b_normal_pos
            assert np.all(sel[(a == 0) & b_normal_pos])  # zero numerators stay on the fast path
        assert np.array_equal(fast[sel].view(np.uint64), ieee[sel].view(np.uint64)), j
    # the range tests reject only rare operands: every positive O(1e-4..1e6) one passes
    n4 = (1 << 21) // 4
    pos = slice(3 * n4, 4 * n4)
    assert np.all(ok[pos] == 15), np.unique(ok[pos], return_counts=True)


@pytest.mark.parametrize("limiter,stepper", [(I.MC, I.RK2), (I.WENOZ, I.RK3)])
def test_exact_resolve_path_parity(mhd, limiter, stepper):
    """Faces whose branch-free operators fail a range test are re-solved with the IEEE operators
    (k_stage's out-of-line exact path).  Here the lower half in z is at rest with gamma p = Bx^2,
    B = (1, 0, 0): on its x faces the fast-speed discriminant is exactly 0 and sqrt(0) is outside
    the fast range, so every such face takes the exact path; the upper half is a moving state.
    The run must still equal the oracle bitwise."""
    p = I.Problem("exact_path", (16, 16, 32), gamma=2.0, limiter=limiter, stepper=stepper)
    X, Y, Z = I.mesh(p)
    tp = 2.0 * math.pi
    low = Z < 0.5
    rho = np.where(low, 1.0 + 0.3 * np.sin(tp * X) * np.cos(tp * Y), 1.0)
    vx = np.where(low, 0.0, -0.5 * np.sin(tp * Y))
    vy = np.where(low, 0.0, 0.5 * np.sin(tp * X))
    vz = np.where(low, 0.0, 0.05 * np.sin(tp * Z))
    by = np.where(low, 0.0, 0.3 * np.sin(tp * X))
    bz = np.where(low, 0.0, 0.2 * np.cos(tp * Y))
    U0 = I.prim_to_cons_ic(p, rho, vx, vy, vz, 0.5, 1.0, by, bz)
    # the premise: in the lower half p = (gamma-1)((E - ke) - me) = 0.5 exactly, so gamma p = Bx^2
    # and the discriminant (a2 - b2)^2 + 4 a2 bt2 of every x face there is exactly 0
    pr = (p.gamma - 1.0) * ((U0[4] - 0.0) - 0.5 * ((U0[5] * U0[5] + U0[6] * U0[6]) + U0[7] * U0[7]))
    assert np.all(pr[low] == 0.5) and np.all(p.gamma * pr[low] == U0[5][low] ** 2)
    res = run_both(mhd, p, U0, 6)
    assert_parity(*res)


# ---------------------------------------------------------------------------------------------
# whole runs
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("riemann,limiter", [(I.HLL, I.MC), (I.HLLD, I.MC), (I.HLL, I.MINMOD)])
def test_brio_wu_full_run(mhd, riemann, limiter):
    """BASELINE configs[0]: Brio-Wu 512, PLM+HLL, RK2, CFL 0.4, to t = 0.1 (full run)."""
    p = I.brio_wu(512, riemann=riemann, limiter=limiter)
    res = run_both(mhd, p, I.brio_wu_ic(p), 100000, p.t_end)
    assert_parity(*res)
    assert 480 < len(res[1]) < 500


def test_sod_outflow(mhd):
    p = I.sod(300)
    assert_parity(*run_both(mhd, p, I.sod_ic(p), 100000, p.t_end))


def test_1d_glm(mhd):
    p = I.brio_wu(200).replace(glm=1)
    assert_parity(*run_both(mhd, p, I.brio_wu_ic(p), 150))


@pytest.mark.parametrize("n", [(64, 64), (50, 37)])
def test_ot2d(mhd, n):
    p = I.orszag_tang_2d(64).replace(n=(n[0], n[1], 1))
    assert_parity(*run_both(mhd, p, I.orszag_tang_2d_ic(p), 120))


@pytest.mark.slow
def test_ot2d_512_config_to_t05(mhd):
    """BASELINE configs[1] (2D Orszag-Tang 512^2, PLM+HLLD+GLM, to t = 0.5): the full run equal
    to the oracle's element by element with the same dt sequence; it conserves mass, momentum,
    energy and B to round-off (periodic) and keeps the point symmetry of the vortex (scalars
    even, vectors odd about the centre)."""
    p = I.orszag_tang_2d(512)
    U0 = I.orszag_tang_2d_ic(p)
    s = mhd.Solver(p)
    s.set_state(np.ascontiguousarray(U0))
    log = s.run(100000, 0.5)
    U = s.get_state()
    s.destroy()
    # the whole run (2886 steps, the last one clamped to t = 0.5) against the oracle: dt log and
    # final state bitwise (the oracle's OpenMP spans the (z, y) loops: ~2 min on 16 host cores)
    o = oracle.Oracle(p, U0)
    log_o = o.run(100000, 0.5)
    assert np.array_equal(log, log_o) and np.array_equal(U, o.U)
    assert abs(float(np.sum(log)) - 0.5) <= 1e-12 and len(log) > 1000
    for f in range(8):
        scale = np.abs(U0[f]).sum()
        assert abs(U[f].sum() - U0[f].sum()) <= 1e-11 * scale, f
    rot = lambda a: a[:, ::-1, ::-1]
    for f, sgn in ((0, 1), (4, 1), (1, -1), (2, -1), (5, -1), (6, -1)):
        assert np.abs(U[f] - sgn * rot(U[f])).max() <= 1e-8 * np.abs(U[f]).max(), f
    assert np.abs(U[3]).max() == 0 and np.abs(U[7]).max() == 0


@pytest.mark.parametrize("limiter,riemann", [(I.MC, I.HLLD), (I.MINMOD, I.HLLD), (I.MC, I.HLL)])
def test_ot3d_small(mhd, limiter, riemann):
    p = I.orszag_tang_3d(32, limiter=limiter, riemann=riemann)
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    assert_parity(*run_both(mhd, p, U0, 15))


def test_ot3d_ragged(mhd):
    """ragged tiles in x (40 = 32 + 8) and y (21 = 2*8 + 5) and a z extent that is not a chunk multiple."""
    p = I.orszag_tang_3d(32).replace(n=(40, 21, 19), hi=(1.25, 0.65625, 0.59375))
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    assert_parity(*run_both(mhd, p, U0, 10))


def test_blast3d_small(mhd):
    p = I.blast_3d(32)
    assert_parity(*run_both(mhd, p, I.blast_3d_ic(p), 20))


def test_3d_outflow_shock_tube_along_z(mhd):
    """Brio-Wu along z inside a 3D box with outflow on every face: exercises the z outflow ghost
    planes and the z frame (z, x, y) of the face solve."""
    n = 48
    p = I.Problem("bwz", (8, 8, n), bc=(I.OUTFLOW,) * 3, gamma=2.0, glm=1, riemann=I.HLLD)
    pz = I.brio_wu(n).replace(glm=1)
    U1 = I.brio_wu_ic(pz)[:, 0, 0, :]  # [nv][n] along x
    U = np.zeros(p.shape)
    for f in range(9):
        src = f
        if 1 <= f <= 3:
            src = 1 + (f - 1 - 2) % 3
        if 5 <= f <= 7:
            src = 5 + (f - 5 - 2) % 3
        U[f] = U1[src][:, None, None]
    assert_parity(*run_both(mhd, p, U, 40))


# ---------------------------------------------------------------------------------------------
# API behaviour
# ---------------------------------------------------------------------------------------------
def test_state_roundtrip_host_and_device(mhd):
    import torch
    p = I.orszag_tang_3d(16)
    U = I.with_noise(I.orszag_tang_3d_ic(p), p)
    s = mhd.Solver(p)
    s.set_state(U)
    assert np.array_equal(s.get_state(), U)
    Ud = torch.from_numpy(U).cuda()
    s.set_state(Ud)
    out = torch.empty_like(Ud)
    s.get_state(out)
    assert torch.equal(out, Ud)
    s.destroy()


@pytest.mark.parametrize("scheme", ["plm_rk2", "wenoz_rk3", "ct"])
def test_bind_workspace_torch_memory(mhd, scheme):
    """The state arrays re-homed into a torch-allocated CUDA buffer give the same run bitwise."""
    import torch
    from test_oracle_scheme import _random_ct_state
    p = I.orszag_tang_3d(16).replace(n=(24, 20, 16))
    if scheme == "wenoz_rk3":
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
    if scheme == "ct":
        p = p.replace(ct=1, glm=0)
        U0 = _random_ct_state(p)
    else:
        U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    ref = mhd.Solver(p)
    ref.set_state(U0)
    log_r = ref.run(4)
    want = ref.get_state()
    ref.destroy()
    s = mhd.Solver(p)
    nb = s.workspace_bytes()
    buf = torch.empty(nb + 256, dtype=torch.uint8, device="cuda")
    with pytest.raises(mhd.MhdError):
        s.bind_workspace(buf[: nb - 256])  # too short
    s.bind_workspace(buf)
    s.set_state(U0)
    log = s.run(4)
    assert np.array_equal(log, log_r) and np.array_equal(s.get_state(), want)
    s.destroy()
    del buf


def _harsh_state(limiter, seed, p_lo, vmax, rho_lo):
    """Random cells (log-uniform density and pressure, uniform velocity and field): pressure
    floors, reconstruction fallbacks and HLLD -> HLL fallbacks all occur."""
    p = I.orszag_tang_3d(32, limiter=limiter).replace(n=(32, 24, 20), hi=(1.0, 0.75, 0.625))
    rng = np.random.default_rng(seed)
    sh = (p.n[2], p.n[1], p.n[0])
    rho = 10.0 ** rng.uniform(rho_lo, 1, sh)
    pr = 10.0 ** rng.uniform(p_lo, -2, sh)
    v = rng.uniform(-vmax, vmax, (3,) + sh)
    B = rng.uniform(-2, 2, (3,) + sh)
    return p, I.prim_to_cons_ic(p, rho, v[0], v[1], v[2], pr, B[0], B[1], B[2])


@pytest.mark.parametrize("case", ["plm_rk2", "wenoz_rk3_split", "wenoz_rk3_fused"])
def test_rare_event_counters_parity(mhd, case):
    """The rare events the owner-rule counters record (pressure floors, reconstruction
    positivity fallbacks, HLLD -> HLL fallbacks) occur, and the GPU counts equal the oracle's."""
    if case == "plm_rk2":
        p, U0 = _harsh_state(I.MC, 0, -13, 3.0, -2)
        n, need = 3, ("p_floors", "hlld_to_hll")  # (PLM is positivity preserving here)
    else:
        p, U0 = _harsh_state(I.WENOZ, 0, -13, 0.3, -1)
        p = p.replace(stepper=I.RK3)
        n, need = 2, ("p_floors", "plm_fallbacks", "hlld_to_hll")
    if case == "wenoz_rk3_fused":
        os.environ["MHD_FUSED_WENOZ"] = "1"
    try:
        res = run_both(mhd, p, U0, n)
    finally:
        os.environ.pop("MHD_FUSED_WENOZ", None)
    assert_parity(*res)
    co = res[0].counters()
    assert all(co[k] > 0 for k in need), co


@pytest.mark.parametrize("limiter,P", [(I.MC, 2), (I.MC, 4), (I.WENOZ, 2), (I.WENOZ, 4)])
def test_rare_event_counters_slab_group(mhd, limiter, P):
    """Owner rule across slab boundaries: with rare events on every slab, P slabs count exactly
    what one domain counts (and produce the same bits)."""
    if limiter == I.MC:
        p, U0 = _harsh_state(I.MC, 1, -13, 3.0, -2)
    else:
        p, U0 = _harsh_state(I.WENOZ, 1, -13, 0.3, -1)
        p = p.replace(stepper=I.RK3)
    s = mhd.Solver(p)
    s.set_state(np.ascontiguousarray(U0))
    log1 = s.run(2)
    U1, d1 = s.get_state(), s.diag()
    s.destroy()
    g = mhd.SolverGroup(p, P)
    g.set_state(U0)
    logP = g.run(2)
    UP, dP = g.get_state(), g.diag()
    g.destroy()
    assert np.array_equal(log1, logP) and np.array_equal(U1, UP)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dP[k], (k, d1[k], dP[k])
    assert d1["p_floors"] > 0 and d1["hlld_to_hll"] > 0


def test_unphysical_detection_matches_oracle(mhd):
    """A run that turns unphysical: the GPU reports the same first bad cell and stage as the
    oracle (lowest global linear index, atomicMin)."""
    p, U0 = _harsh_state(I.WENOZ, 0, -13, 3.0, -2)
    p = p.replace(stepper=I.RK3)
    o = oracle.Oracle(p, U0)
    with pytest.raises(oracle.OracleError) as ei:
        o.run(3)
    want = ei.value.counters.as_dict()
    s = mhd.Solver(p)
    s.set_state(np.ascontiguousarray(U0))
    with pytest.raises(mhd.MhdError):
        s.run(3)
    d = s.diag()
    s.destroy()
    assert (d["first_bad_cell"], d["bad_stage"]) == (want["first_bad_cell"], want["bad_stage"]), (d, want)


@pytest.mark.parametrize("scheme", ["plm_rk2", "wenoz_rk3", "ct_plm", "ct_wenoz"])
@pytest.mark.parametrize("n", [(4, 4, 4), (5, 6, 7)])
def test_smallest_grids(mhd, scheme, n):
    """The smallest accepted grids (4 cells per active axis) and odd tiny ones, every stage
    variant: a halo wider than half the domain wraps correctly (periodic)."""
    from test_oracle_scheme import _random_ct_state
    p = I.orszag_tang_3d(8).replace(n=n, hi=(n[0] / 8, n[1] / 8, n[2] / 8))
    if scheme.startswith("ct"):
        p = p.replace(ct=1, glm=0)
    if "wenoz" in scheme:
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
    U0 = _random_ct_state(p) if p.ct else I.with_noise(I.orszag_tang_3d_ic(p), p)
    assert_parity(*run_both(mhd, p, U0, 5))


def _random_config(seed):
    """A seeded random problem: dimension and limiter cycle with the seed; extents (ragged,
    >= 4), boundary conditions per axis, Riemann solver, stepper, GLM or CT and a smooth random
    state with noise are drawn."""
    rng = np.random.default_rng(1000 + seed)
    dim = 1 + seed % 3
    limiter = (I.MINMOD, I.MC, I.WENOZ)[(seed // 3) % 3]
    n = [int(rng.integers(4, 41)) if d < dim else 1 for d in range(3)]
    ct = dim == 3 and (seed // 9) % 2 == 1
    bc = tuple(int(rng.integers(0, 2)) if (d < dim and not ct) else I.PERIODIC for d in range(3))
    glm = 1 if (dim >= 2 and not ct) else int(rng.integers(0, 2)) if not ct else 0
    p = I.Problem("rnd", tuple(n), hi=tuple(n[d] / 32 if d < dim else 1.0 for d in range(3)), bc=bc,
                  gamma=float(rng.choice([5 / 3, 1.4, 2.0])), limiter=limiter, riemann=int(rng.integers(0, 2)),
                  glm=glm, stepper=int(rng.integers(0, 2)), ct=int(ct))
    X, Y, Z = I.mesh(p)
    k = rng.uniform(1, 3, 3) * 2 * math.pi
    ph = rng.uniform(0, 2 * math.pi, 8)
    w = lambda j: np.sin(k[0] * X + ph[j]) * np.cos(k[1] * Y + ph[j]) * np.cos(k[2] * Z + 0.5 * ph[j])
    rho = 1.0 + 0.4 * w(0)
    pr = 0.6 + 0.3 * w(1)
    v = [0.5 * w(2), 0.5 * w(3), 0.5 * w(4) if dim == 3 else 0.0 * w(4)]
    B = [0.6 + 0.3 * w(5), 0.4 * w(6), 0.4 * w(7)]
    if dim == 1:
        B[0] = 0.75 + 0.0 * X  # constant normal field in 1D
    U0 = I.prim_to_cons_ic(p, rho, v[0], v[1], v[2], pr, B[0], B[1], B[2])
    if ct:
        from test_oracle_scheme import _random_ct_state
        U0 = _random_ct_state(p)
    return p, I.with_noise(U0, p, amp=1e-3, seed=int(rng.integers(1 << 30))) if not ct else U0


@pytest.mark.parametrize("seed", range(18))
def test_random_configurations(mhd, seed):
    """Seeded random problems across every option the ABI takes (dimension, ragged extents,
    per-axis periodic / outflow, minmod / MC / WENO-Z, HLL / HLLD, RK2 / RK3, GLM on / off in
    1D, CT in 3D): the GPU equals the oracle bitwise."""
    p, U0 = _random_config(seed)
    assert_parity(*run_both(mhd, p, np.ascontiguousarray(U0), 6))


@pytest.mark.parametrize("seed", [2, 5, 8, 11, 14])
def test_random_configurations_slab_group(mhd, seed):
    """The 3D random configurations split into P in-process z slabs (P the largest of 2..5 that
    divides nz with slabs at least the ghost depth): bitwise equal to one domain, equal counters."""
    p, U0 = _random_config(seed)
    gz = (3 if p.limiter == I.WENOZ else 2) + (1 if p.ct else 0)
    Ps = [P for P in (5, 4, 3, 2) if p.n[2] % P == 0 and p.n[2] // P >= gz]
    if not Ps:
        pytest.skip(f"nz = {p.n[2]} has no admissible slab count")
    s = mhd.Solver(p)
    s.set_state(np.ascontiguousarray(U0))
    log1 = s.run(4)
    U1, d1 = s.get_state(), s.diag()
    s.destroy()
    g = mhd.SolverGroup(p, Ps[0])
    g.set_state(np.ascontiguousarray(U0))
    logP = g.run(4)
    UP, dP = g.get_state(), g.diag()
    g.destroy()
    assert np.array_equal(log1, logP) and np.array_equal(U1, UP)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dP[k], (k, d1[k], dP[k])


@pytest.mark.parametrize("limiter", [I.MC, I.WENOZ])
def test_z_chunking_and_repeat_invariance(mhd, limiter):
    """The result does not depend on the z chunk length of the stage kernel's CTAs (each chunk
    re-derives its prologue: V+(kb-1), the first z face) nor on the run: kz = 1, 3, 7 and the
    model's choice, twice, all bitwise equal (the fused kernel in 2-plane-chunk corner cases)."""
    p = I.orszag_tang_3d(24, limiter=limiter).replace(n=(40, 21, 19), hi=(1.25, 0.65625, 0.59375))
    if limiter == I.WENOZ:  # the fused kernel (3D WENO-Z defaults to the split stage)
        os.environ["MHD_FUSED_WENOZ"] = "1"
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    outs = []
    try:
        for kz in ("1", "3", "7", "", ""):
            if kz:
                os.environ["MHD_KZ"] = kz
            else:
                os.environ.pop("MHD_KZ", None)
            s = mhd.Solver(p)
            s.set_state(U0)
            log = s.run(4)
            outs.append((log, s.get_state()))
            s.destroy()
    finally:
        os.environ.pop("MHD_KZ", None)
        os.environ.pop("MHD_FUSED_WENOZ", None)
    for log, U in outs[1:]:
        assert np.array_equal(log, outs[0][0]) and np.array_equal(U, outs[0][1])


def test_async_io_pipeline_equals_sync(mhd):
    """set_state_async / get_state_async / io_join (the pipelined e2e path) give the same dt
    sequence and states as the synchronous calls, step by step."""
    import torch
    p = I.orszag_tang_3d(24).replace(n=(24, 20, 16))
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    ref = mhd.Solver(p)
    s = mhd.Solver(p)
    Uh = torch.from_numpy(U0).pin_memory()
    outs = [torch.empty_like(Uh).pin_memory() for _ in range(3)]
    ins = [Uh]  # (the uploads read these until io_join: keep them alive)
    want = []
    for i in range(3):
        ref.set_state(np.ascontiguousarray(U0) if i == 0 else want[-1])
        dt_r = ref.compute_dt()
        ref.step(dt_r)
        want.append(ref.get_state())
        if i > 0:
            ins.append(torch.from_numpy(want[i - 1]).pin_memory())
        s.set_state_async(ins[-1])
        assert s.compute_dt() == dt_r
        s.step(dt_r)
        s.get_state_async(outs[i])
    s.io_join()
    torch.cuda.synchronize()
    for i in range(3):
        assert np.array_equal(outs[i].numpy(), want[i]), i
    # an unphysical state uploaded asynchronously is reported by the next synchronising call
    bad = U0.copy()
    bad[0, 3, 4, 5] = -1.0
    ins.append(torch.from_numpy(bad).pin_memory())
    s.set_state_async(ins[-1])
    with pytest.raises(mhd.MhdError):
        s.compute_dt()
    s.destroy()
    ref.destroy()


def test_unphysical_state_rejected_and_sticky(mhd):
    p = I.orszag_tang_3d(16)
    U = I.orszag_tang_3d_ic(p)
    good = U[0, 3, 2, 5]
    U[0, 3, 2, 5] = -1.0
    s = mhd.Solver(p)
    with pytest.raises(mhd.MhdError) as e:
        s.set_state(U)
    assert e.value.code == mhd.MHD_E_UNPHYSICAL
    d = s.diag()
    assert d["first_bad_cell"] == (3 * 16 + 2) * 16 + 5 and d["bad_stage"] == 0
    with pytest.raises(mhd.MhdError) as e:
        s.compute_dt()
    assert e.value.code == mhd.MHD_E_STATE
    U[0, 3, 2, 5] = good
    s.set_state(U)           # recovers
    assert s.compute_dt() > 0
    s.destroy()


def test_step_unphysical_detected(mhd):
    """an extreme rarefaction with a CFL near 1 drives rho negative inside a step; the library
    reports MHD_E_UNPHYSICAL at the next synchronising call, like the oracle."""
    p = I.Problem("vac", (64, 1, 1), bc=(I.OUTFLOW,) * 3, gamma=1.4, glm=0, riemann=I.HLL, cfl=0.95,
                  p_floor=1e-12)
    X = I.centres(p, 0)
    U = I.prim_to_cons_ic(p, 1e-6 + 0 * X, np.where(X < 0.5, -50.0, 50.0), 0, 0, 1e-8, 0, 0, 0)
    o = oracle.Oracle(p, U)
    s = mhd.Solver(p)
    s.set_state(U)
    raised_o = raised_g = None
    try:
        o.run(50)
    except oracle.OracleError as e:
        raised_o = e.counters.as_dict()
    try:
        s.run(50)
    except mhd.MhdError as e:
        raised_g = s.diag()
        assert e.code == mhd.MHD_E_UNPHYSICAL
    s.destroy()
    if raised_o is None:
        assert raised_g is None
    else:
        assert raised_g is not None
        assert raised_g["first_bad_cell"] == raised_o["first_bad_cell"]
        assert raised_g["bad_stage"] == raised_o["bad_stage"]


def test_invalid_arguments(mhd):
    with pytest.raises(mhd.MhdError) as e:
        mhd.Solver(I.orszag_tang_3d(16).replace(cfl=1.5))
    assert e.value.code == mhd.MHD_E_ARG
    with pytest.raises(mhd.MhdError):
        mhd.Solver(I.orszag_tang_2d(16, glm=0))  # GLM required in multi-D
    s = mhd.Solver(I.orszag_tang_3d(16))
    with pytest.raises(mhd.MhdError) as e:
        s.compute_dt()                              # no state yet
    assert e.value.code == mhd.MHD_E_STATE
    s.destroy()


# ---------------------------------------------------------------------------------------------
# BASELINE full size (configs[2], 256^3) in the bench's launch configuration
# ---------------------------------------------------------------------------------------------
def test_ot3d_256_full_size_parity(mhd):
    """two full steps of the 256^3 OT-3D roofline config, element by element (the oracle runs
    multi-threaded on the host; it finishes in seconds)."""
    p = I.orszag_tang_3d(256)
    U0 = I.orszag_tang_3d_ic(p)
    res = run_both(mhd, p, U0, 2)
    assert_parity(*res)


def _sampled_step_parity(mhd, workload, p, samples, halo=4, box_bc=None):
    """One step of a full-size BASELINE config on the GPU, in bench.py's launch configuration,
    checked on sampled cells: the dt equals the oracle's on the whole state (bitwise), and each
    sampled cell equals the oracle's step of its (2*halo+1)^3 neighbourhood (the PLM-RK2 update
    of a cell reads U^n within +-4 cells; outflow ghosts of the small box reach only its outer
    cells) with the whole-domain dt and c_h."""
    U0 = I.workload_ic(workload, p)
    s = mhd.Solver(p)
    s.set_state(U0)
    dt_g = s.compute_dt()
    dt_o, ch_o = oracle.compute_dt(p, U0)
    assert dt_g == dt_o, (dt_g, dt_o)
    s.step(dt_g)
    w = 2 * halo + 1
    dx = [(p.hi[d] - p.lo[d]) / p.n[d] for d in range(3)]
    bc = box_bc if box_bc is not None else I.OUTFLOW
    sub = p.replace(n=(w, w, w), lo=(0.0, 0.0, 0.0), hi=(w * dx[0], w * dx[1], w * dx[2]), bc=(bc, bc, bc))
    assert all((sub.hi[d] - sub.lo[d]) / w == dx[d] for d in range(3))  # identical dt/dx
    for (x, y, z) in samples:
        ix = [(x + o) % p.n[0] for o in range(-halo, halo + 1)]
        iy = [(y + o) % p.n[1] for o in range(-halo, halo + 1)]
        iz = [(z + o) % p.n[2] for o in range(-halo, halo + 1)]
        box = np.ascontiguousarray(U0[:, iz][:, :, iy][:, :, :, ix])
        o = oracle.Oracle(sub, box)
        o.step(dt_o, ch_o)
        want = o.U[:, halo, halo, halo]
        got = s.get_state_box((x, y, z), (1, 1, 1))[:, 0, 0, 0]
        assert np.array_equal(got, want), ((x, y, z), got - want)
    s.destroy()


def _edge_and_random_cells(n, k, rng, extra=()):
    nx, ny, nz = n
    cells = [(0, 0, 0), (nx - 1, ny - 1, nz - 1), (0, ny - 1, 1), (nx - 1, 0, nz - 2), (1, ny // 2, 0),
             (nx // 2, 1, nz - 1)]
    cells += [tuple(int(v) for v in (rng.integers(nx), rng.integers(ny), rng.integers(nz))) for _ in range(k)]
    return cells + list(extra)


def test_long_run_conservation_ot3d(mhd):
    """A long GPU run (OT-3D 128^3, 400 steps, into the turbulent phase) keeps the periodic
    invariants the scheme has at any size: total mass, momentum, energy and magnetic field
    conserved to round-off, and the GLM-controlled divergence of B stays small."""
    p = I.orszag_tang_3d(128)
    U0 = I.orszag_tang_3d_ic(p)
    s = mhd.Solver(p)
    s.set_state(np.ascontiguousarray(U0))
    log = s.run(400)
    U = s.get_state()
    d = s.diag()
    s.destroy()
    assert len(log) == 400 and np.all(np.isfinite(U)) and d["first_bad_cell"] == -1
    for f in range(8):  # (B_z starts at zero: scale by the final field as well)
        scale = max(np.abs(U0[f]).sum(), np.abs(U[f]).sum())
        assert abs(U[f].sum() - U0[f].sum()) <= 1e-11 * scale, f
    dx = 1.0 / 128
    bx, by, bz = U[5], U[6], U[7]
    div = ((np.roll(bx, -1, 2) - np.roll(bx, 1, 2)) + (np.roll(by, -1, 1) - np.roll(by, 1, 1)) +
           (np.roll(bz, -1, 0) - np.roll(bz, 1, 0))) / (2 * dx)
    assert np.sqrt((div * dx) ** 2).mean() / np.sqrt((bx * bx + by * by + bz * bz).mean()) < 0.05


@pytest.mark.slow
def test_blast_512_full_size_sampled(mhd):
    """BASELINE configs[3] per GPU (blast 512^3, one rank's slab): one step, sampled cells,
    including cells on the blast front."""
    p = I.blast_3d(512)
    rng = np.random.default_rng(11)
    front = []
    for _ in range(24):  # cells within a few cells of the r = 0.1 sphere
        v = rng.normal(size=3)
        v = 0.5 + (0.1 + rng.uniform(-3, 3) / 512) * v / np.linalg.norm(v)
        front.append(tuple(int(np.clip(c * 512, 0, 511)) for c in v))
    _sampled_step_parity(mhd, "blast3d", p, _edge_and_random_cells(p.n, 16, rng, front))


@pytest.mark.parametrize("workload,scheme", [("ot3d", "wenoz-rk3"), ("ot3d", "ct-wenoz-rk3"), ("cpa3d", "plm-rk2")])
def test_paper_schemes_256_full_size_sampled(mhd, workload, scheme):
    """The §8(f) bench lines at their full size (256^3, bench.py --workload / --scheme): one step of
    WENO-Z + HLLD + RK3 with GLM (the split stage) or with CT, and the 3D CPA workload, on sampled
    cells.  An RK3 step of a
    WENO-Z cell reads +-9 cells; the oracle box is 21^3 (outflow for GLM; periodic for CT, whose
    wrap seam reaches at most 9 cells in by the third stage, short of the centre)."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    p = bench.build_problem(workload, 1, 256, scheme)
    rng = np.random.default_rng(21)
    _sampled_step_parity(mhd, workload, p, _edge_and_random_cells(p.n, 12, rng), halo=10 if p.limiter == I.WENOZ else 4,
                         box_bc=I.PERIODIC if p.ct else I.OUTFLOW)


@pytest.mark.slow
def test_ot3d_1024_full_size_sampled(mhd):
    """BASELINE configs[4] at P = 1 (OT-3D 1024^3, 155 GB on the GPU, 77 GB host state): one
    step, sampled cells (the oracle cannot hold two copies of the whole state)."""
    import psutil
    if psutil.virtual_memory().total < 120 << 30:
        pytest.skip("needs a host with >= 120 GB of RAM for the 77 GB 1024^3 state")
    p = I.orszag_tang_3d(1024)
    _sampled_step_parity(mhd, "ot3d", p, _edge_and_random_cells(p.n, 40, np.random.default_rng(12)))


# ---------------------------------------------------------------------------------------------
# decomposition invariance: P z-slabs == 1 domain, bitwise
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("P", [2, 4, 8])
def test_slab_group_bitwise_equals_single_domain(mhd, P):
    """The group runs every slab through the NCCL ranks' stage schedule (mhd_api.cu fused_stage):
    interior planes [2, nz-2) while the halo copies run on the slab's comm stream, then the two
    2-plane boundary launches after the halo event.  P = 8: 4-plane slabs, an empty interior."""
    p = I.orszag_tang_3d(32).replace(n=(40, 21, 32))
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(6)
    U1 = s.get_state()
    d1 = s.diag()
    s.destroy()
    g = mhd.SolverGroup(p, P)
    g.set_state(U0)
    logP = g.run(6)
    UP = g.get_state()
    dP = g.diag()
    g.destroy()
    assert np.array_equal(log1, logP)
    assert np.array_equal(U1, UP)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dP[k]


def test_slab_group_outflow_z_matches_oracle(mhd):
    """the outflow shock tube along z split over 4 slabs (edge ranks copy, inner ranks exchange)"""
    n = 48
    p = I.Problem("bwz", (8, 8, n), bc=(I.OUTFLOW,) * 3, gamma=2.0, glm=1, riemann=I.HLLD)
    U1 = I.brio_wu_ic(I.brio_wu(n).replace(glm=1))[:, 0, 0, :]
    U = np.zeros(p.shape)
    for f in range(9):
        src = f
        if 1 <= f <= 3:
            src = 1 + (f - 1 - 2) % 3
        if 5 <= f <= 7:
            src = 5 + (f - 5 - 2) % 3
        U[f] = U1[src][:, None, None]
    o = oracle.Oracle(p, U)
    log_o = o.run(30)
    g = mhd.SolverGroup(p, 4)
    g.set_state(U)
    log_g = g.run(30)
    Ug = g.get_state()
    g.destroy()
    assert np.array_equal(log_o, log_g)
    assert np.all(rel_linf(Ug, o.U) <= TOL)


def test_blast_weak_layout_two_cubes(mhd):
    """configs[3] layout (one blast per unit cube along z) on 2 slabs vs the oracle"""
    p = I.blast_3d(16, cubes=2)
    U0 = I.blast_3d_ic(p)
    o = oracle.Oracle(p, U0)
    log_o = o.run(8)
    g = mhd.SolverGroup(p, 2)
    g.set_state(U0)
    log_g = g.run(8)
    Ug = g.get_state()
    g.destroy()
    assert np.array_equal(log_o, log_g)
    assert np.all(rel_linf(Ug, o.U) <= TOL)


def test_cpa3d_full_period(mhd):
    """§8(f) row 1: 3D CPA (the paper's second workload) for one full period at 24^3, bitwise."""
    p = I.cpa_3d(24)
    res = run_both(mhd, p, I.cpa_3d_ic(p), 10 ** 6, p.t_end)
    assert_parity(*res)


# ---------------------------------------------------------------------------------------------
# §8(f) row 2: SSP-RK3 (the paper's integrator), three state arrays
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("limiter,stepper", [(I.MC, I.RK2), (I.WENOZ, I.RK3)])
@pytest.mark.parametrize("bc", [(I.OUTFLOW, I.OUTFLOW, I.PERIODIC), (I.PERIODIC, I.OUTFLOW, I.OUTFLOW),
                                (I.OUTFLOW, I.PERIODIC, I.OUTFLOW)])
def test_mixed_boundaries_3d(mhd, limiter, stepper, bc):
    """Outflow x / y (index clamp in the fused and split kernels) and z (ghost copies) on a
    non-uniform ragged state (noisy OT-3D), against the oracle's materialised ghosts."""
    p = I.orszag_tang_3d(32, limiter=limiter).replace(n=(40, 21, 19), hi=(1.25, 0.65625, 0.59375), bc=bc,
                                                     stepper=stepper)
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    assert_parity(*run_both(mhd, p, U0, 8))


@pytest.mark.parametrize("case", ["ot3d", "brio_wu", "ot2d"])
def test_rk3_parity(mhd, case):
    if case == "ot3d":
        p = I.orszag_tang_3d(32).replace(n=(40, 21, 19), hi=(1.25, 0.65625, 0.59375), stepper=I.RK3)
        U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
        n = 10
    elif case == "brio_wu":
        p = I.brio_wu(512).replace(stepper=I.RK3)
        U0 = I.brio_wu_ic(p)
        n = 100000
    else:
        p = I.orszag_tang_2d(64).replace(stepper=I.RK3)
        U0 = I.orszag_tang_2d_ic(p)
        n = 60
    res = run_both(mhd, p, U0, n, p.t_end if case == "brio_wu" else 0.0)
    assert_parity(*res)


def test_rk3_slab_group_bitwise(mhd):
    p = I.orszag_tang_3d(32).replace(stepper=I.RK3)
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(5)
    U1 = s.get_state()
    s.destroy()
    g = mhd.SolverGroup(p, 4)
    g.set_state(U0)
    log4 = g.run(5)
    U4 = g.get_state()
    g.destroy()
    assert np.array_equal(log1, log4) and np.array_equal(U1, U4)


# ---------------------------------------------------------------------------------------------
# §8(f) row 3: WENO-Z reconstruction (ghost width 3), the paper's WENOZ + HLLD + RK3 + GLM
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["ot3d_rk3", "ot3d_rk2_hll", "brio_wu", "ot2d", "outflow_z"])
def test_wenoz_parity(mhd, case):
    if case.startswith("ot3d"):
        p = I.orszag_tang_3d(32, limiter=I.WENOZ).replace(n=(40, 21, 19), hi=(1.25, 0.65625, 0.59375))
        if case == "ot3d_rk3":
            p = p.replace(stepper=I.RK3)
        else:
            p = p.replace(riemann=I.HLL)
        U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
        res = run_both(mhd, p, U0, 8)
    elif case == "brio_wu":
        p = I.brio_wu(512).replace(limiter=I.WENOZ, stepper=I.RK3)
        res = run_both(mhd, p, I.brio_wu_ic(p), 100000, p.t_end)
    elif case == "ot2d":
        p = I.orszag_tang_2d(64, limiter=I.WENOZ).replace(stepper=I.RK3)
        res = run_both(mhd, p, I.orszag_tang_2d_ic(p), 60)
    else:
        n = 48
        p = I.Problem("bwz", (8, 8, n), bc=(I.OUTFLOW,) * 3, gamma=2.0, glm=1, riemann=I.HLLD, limiter=I.WENOZ,
                      stepper=I.RK3)
        U1 = I.brio_wu_ic(I.brio_wu(n).replace(glm=1))[:, 0, 0, :]
        U = np.zeros(p.shape)
        for f in range(9):
            src = f
            if 1 <= f <= 3:
                src = 1 + (f - 1 - 2) % 3
            if 5 <= f <= 7:
                src = 5 + (f - 5 - 2) % 3
            U[f] = U1[src][:, None, None]
        res = run_both(mhd, p, U, 30)
    assert_parity(*res)


def test_wenoz_slab_group_bitwise(mhd):
    p = I.orszag_tang_3d(24, limiter=I.WENOZ).replace(stepper=I.RK3)
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(4)
    U1 = s.get_state()
    s.destroy()
    g = mhd.SolverGroup(p, 4)  # slabs of 6 planes >= ghost width 3
    g.set_state(U0)
    log4 = g.run(4)
    U4 = g.get_state()
    g.destroy()
    assert np.array_equal(log1, log4) and np.array_equal(U1, U4)


# ---------------------------------------------------------------------------------------------
# §8(f) row 4: constrained transport (face-centred b, edge EMFs), 3D periodic
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("case", ["cpa_mc_rk2", "ot_hll", "random_wenoz_rk3", "ragged_minmod"])
def test_ct_parity(mhd, case):
    from test_oracle_scheme import _random_ct_state
    if case == "cpa_mc_rk2":
        p = I.ct_problem(I.cpa_3d(16))
        U0 = I.cpa_3d_ct_ic(p)
        n = 40
    elif case == "ot_hll":
        p = I.ct_problem(I.orszag_tang_3d(24, riemann=I.HLL))
        U0 = I.orszag_tang_3d_ic(p.replace(ct=0, glm=1))[:8].copy()
        n = 12
    elif case == "random_wenoz_rk3":
        p = I.orszag_tang_3d(12, limiter=I.WENOZ).replace(ct=1, glm=0, stepper=I.RK3)
        U0 = _random_ct_state(p)
        n = 10
    else:
        p = I.orszag_tang_3d(12, limiter=I.MINMOD).replace(n=(37, 14, 9), ct=1, glm=0)
        U0 = _random_ct_state(p)
        n = 10
    res = run_both(mhd, p, U0, n)
    assert_parity(*res)
    assert np.abs(oracle.ct_divb(p, res[2])).max() < 1e-10


@pytest.mark.parametrize("case,P", [("plm_rk2", 2), ("plm_rk2", 4), ("wenoz_rk3", 2), ("wenoz_rk3", 3)])
def test_ct_slab_group_bitwise(mhd, case, P):
    """CT on z slabs (ghost planes gz = G + 1, halo per stage and per dt pass): P slabs run in
    one process with the same plan, kernels and z ranges as NCCL ranks equal one domain
    bitwise, with equal counters (and so the oracle, test_ct_parity)."""
    from test_oracle_scheme import _random_ct_state
    if case == "plm_rk2":
        p = I.orszag_tang_3d(12, limiter=I.MC).replace(n=(20, 14, 24), ct=1, glm=0)
    else:
        p = I.orszag_tang_3d(12, limiter=I.WENOZ).replace(n=(16, 12, 24), ct=1, glm=0, stepper=I.RK3)
    U0 = _random_ct_state(p)
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(6)
    U1 = s.get_state()
    d1 = s.diag()
    s.destroy()
    g = mhd.SolverGroup(p, P)
    g.set_state(U0)
    logP = g.run(6)
    UP = g.get_state()
    dP = g.diag()
    g.destroy()
    assert np.array_equal(log1, logP) and np.array_equal(U1, UP)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dP[k], (k, d1[k], dP[k])


def test_slab_group_interior_split_with_z_chunks(mhd):
    """The interior/boundary split of the slab schedule combined with small z chunks (MHD_KZ=3:
    the interior range [2, 10) starts a chunk at z = 2 and the boundary launches are chunks of
    their own), on slabs of 12 planes: bitwise equal to one domain with equal counters."""
    p, U0 = _harsh_state(I.MC, 1, -13, 3.0, -2)
    p = p.replace(n=(p.n[0], p.n[1], 36))
    U0 = np.ascontiguousarray(np.concatenate([U0] * (36 // U0.shape[1] + 1), axis=1)[:, :36])
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(3)
    U1, d1 = s.get_state(), s.diag()
    s.destroy()
    os.environ["MHD_KZ"] = "3"
    try:
        g = mhd.SolverGroup(p, 3)
    finally:
        os.environ.pop("MHD_KZ", None)
    g.set_state(U0)
    logP = g.run(3)
    UP, dP = g.get_state(), g.diag()
    g.destroy()
    assert np.array_equal(log1, logP) and np.array_equal(U1, UP)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dP[k], (k, d1[k], dP[k])


@pytest.mark.parametrize("scheme", ["plm-rk2", "wenoz-rk3", "ct-rk2"])
def test_profile_units(mhd, scheme):
    """mhd_profile_*: one event pair per RK stage (whatever its launch count) and per dt pass;
    a run beyond the pool's capacity is reported, not silently truncated."""
    p = I.orszag_tang_3d(16)
    if scheme == "wenoz-rk3":
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
    if scheme == "ct-rk2":
        p = I.ct_problem(p)
    U0 = I.orszag_tang_3d_ic(p.replace(ct=0, glm=1) if p.ct else p)
    U0 = np.ascontiguousarray(U0[:8] if p.ct else U0)
    s = mhd.Solver(p)
    s.set_state(U0)
    s.run(1)
    s.profile_enable(True, capacity=64)
    s.run(5)
    prof = s.profile_read()
    ns = 3 if p.stepper == I.RK3 else 2
    assert prof["stage"][1] == 5 * ns and prof["dt"][1] == 5, prof
    assert prof["stage"][0] > 0 and prof["dt"][0] > 0
    s.profile_enable(True, capacity=4)
    s.run(2)
    with pytest.raises(mhd.MhdError):
        s.profile_read()
    s.profile_enable(False)
    s.destroy()


def test_nccl_two_ranks_bitwise(mhd, tmp_path):
    """Two NCCL ranks (torchrun, one GPU each) run the real multi-rank path — NCCL send/recv halo
    on the comm stream overlapped with the interior launch, ncclAllReduce for dt and counters —
    and must equal one domain bitwise (tools/nccl_parity.py).  Needs two GPUs (gpurun and the
    driver's GPU tier provide one: skipped there; NCCL refuses two ranks on one device)."""
    import subprocess
    import sys
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "nccl_parity.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(root, "tools", "nccl_parity.py"),
           "--out", str(out)]
    subprocess.run(cmd, check=True, timeout=600, cwd=root)
    import json
    res = json.loads(out.read_text())
    assert all(r["bitwise"] for r in res["cases"]), res


def test_profile_exposed_halo_class_on_slabs(mhd):
    """Slabs record, per stage, the compute stream's wait for the halo after the interior launch
    (mhd_profile_read_stages class 4); one slab records none."""
    p = I.orszag_tang_3d(32)
    U0 = I.orszag_tang_3d_ic(p)
    g = mhd.SolverGroup(p, 4)
    g.set_state(U0)
    g.run(1)
    for s in g.slabs:
        s.profile_enable(True, capacity=64)
    g.run(3)
    for s in g.slabs:
        pr = s.profile_read_stages()
        assert pr["halo_exposed"][1] == 6 and pr["halo_exposed"][0] >= 0.0
        assert pr["stage1"][1] == 3 and pr["stage2"][1] == 3 and pr["dt"][1] == 3
        assert pr["halo_exposed"][0] <= pr["stage1"][0] + pr["stage2"][0]
    g.destroy()
    s = mhd.Solver(p)
    s.set_state(U0)
    s.profile_enable(True)
    s.run(2)
    assert s.profile_read_stages()["halo_exposed"] == (0.0, 0)
    s.destroy()


@pytest.mark.parametrize("scheme", ["plm-rk2", "wenoz-rk3", "ct-rk2"])
def test_nccl_self_exchange_bitwise(mhd, scheme):
    """The NCCL code path of the multi-GPU run on one GPU (MHD_NCCL_SELF=1): a one-rank NCCL
    communicator exchanges the periodic z ghost planes by ncclSend/ncclRecv to itself through the
    ranks' stage schedule (interior launch while the halo runs on the comm stream, boundary
    launches after the halo event; CT and split WENO-Z wait for it) and reduces dt, counters and
    bad cells with ncclAllReduce — bitwise equal to the device-copy path with equal counters."""
    p = I.orszag_tang_3d(32).replace(n=(40, 21, 32))
    if scheme == "wenoz-rk3":
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
    if scheme == "ct-rk2":
        p = I.ct_problem(I.orszag_tang_3d(16))
    U0 = I.orszag_tang_3d_ic(p.replace(ct=0, glm=1) if p.ct else p)
    U0 = np.ascontiguousarray(U0[:8] if p.ct else I.with_noise(U0, p))
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(4)
    U1, d1 = s.get_state(), s.diag()
    s.destroy()
    os.environ["MHD_NCCL_SELF"] = "1"
    try:
        s = mhd.Solver(p)
    finally:
        os.environ.pop("MHD_NCCL_SELF", None)
    s.set_state(U0)
    s.profile_enable(True, capacity=64)
    logN = s.run(4)
    prof = s.profile_read_stages()
    UN, dN = s.get_state(), s.diag()
    s.destroy()
    assert np.array_equal(log1, logN) and np.array_equal(U1, UN)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dN[k]
    if scheme == "plm-rk2":  # the fused stage ran the split schedule (one exposed-halo pair per stage)
        assert prof["halo_exposed"][1] == 8


def _with_env(env, make):
    """construct under extra environment variables (read by mhd_create), then restore"""
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return make()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["plm-P2", "plm-P3", "plm-P4", "plm-P8", "rk3-P4", "wenoz-fused-P3", "outflow-P4"])
def test_halo_push_slab_group_bitwise(mhd, case):
    """MHD_HALO_PUSH=1 (include/mhd.h mhd_halo_push): each fused stage's epilogue also stores its
    g boundary planes into the neighbour slabs' ghost planes of the next stage's input, and every
    stage after the first runs as one launch with no exchange.  Bitwise equal to one domain with
    equal counters, also across a state change in the middle of the run (the next stage
    exchanges again); P = 8: 4-plane slabs, every plane a boundary plane."""
    scheme, P = case.rsplit("-P", 1)
    P = int(P)
    p = I.orszag_tang_3d(32).replace(n=(40, 21, 30 if P == 3 else 32))
    env = {"MHD_HALO_PUSH": "1"}
    if scheme == "rk3":
        p = p.replace(stepper=I.RK3)
    if scheme == "wenoz-fused":
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
        env["MHD_FUSED_WENOZ"] = "1"
    if scheme == "outflow":
        p = p.replace(bc=(I.PERIODIC, I.PERIODIC, I.OUTFLOW))
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    U0b = I.with_noise(I.orszag_tang_3d_ic(p), p, seed=7)
    s = _with_env({k: v for k, v in env.items() if k != "MHD_HALO_PUSH"}, lambda: mhd.Solver(p))
    s.set_state(U0)
    log1 = list(s.run(3))
    s.set_state(U0b)
    log1 += list(s.run(3))
    U1, d1 = s.get_state(), s.diag()
    s.destroy()
    g = _with_env(env, lambda: mhd.SolverGroup(p, P))
    assert all(sl.halo_push for sl in g.slabs)
    g.set_state(U0)
    logP = list(g.run(3))
    for sl in g.slabs:
        sl.profile_enable(True, capacity=64)
    g.set_state(U0b)
    logP += list(g.run(3))
    prof = [sl.profile_read_stages() for sl in g.slabs]
    UP, dP = g.get_state(), g.diag()
    g.destroy()
    assert np.array_equal(np.array(log1), np.array(logP))
    assert np.array_equal(U1, UP)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dP[k]
    # after the state change only the first stage waited for an exchange
    assert all(pr["halo_exposed"][1] == 1 for pr in prof)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme", ["plm-rk2", "plm-rk3", "wenoz-rk3", "ct-rk2"])
def test_halo_push_nccl_windows_self_bitwise(mhd, scheme):
    """The NCCL halo push on one GPU (MHD_NCCL_SELF=1 MHD_HALO_PUSH=1): the state arrays are NCCL
    symmetric windows of a one-rank communicator, the periodic z neighbour's window address comes
    from ncclGetPeerPointer, the stage epilogue stores the boundary planes through it and an LSA
    barrier kernel follows each stage — bitwise equal to one domain, with one exchange (the first
    stage) in the whole run."""
    p = I.orszag_tang_3d(32).replace(n=(40, 21, 32))
    if scheme == "plm-rk3":
        p = p.replace(stepper=I.RK3)
    if scheme == "wenoz-rk3":  # the split stage: the push from k_sp_update
        p = p.replace(limiter=I.WENOZ, stepper=I.RK3)
    if scheme == "ct-rk2":  # the push from k_ct_update (and the CT dt pass reads the pushed planes)
        p = I.ct_problem(I.orszag_tang_3d(16))
    U0 = I.orszag_tang_3d_ic(p.replace(ct=0, glm=1) if p.ct else p)
    U0 = np.ascontiguousarray(U0[:8] if p.ct else I.with_noise(U0, p))
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(5)
    U1, d1 = s.get_state(), s.diag()
    s.destroy()
    s = _with_env({"MHD_NCCL_SELF": "1", "MHD_HALO_PUSH": "1"}, lambda: mhd.Solver(p))
    assert s.halo_push
    s.set_state(U0)
    s.profile_enable(True, capacity=64)
    logN = s.run(5)
    prof = s.profile_read_stages()
    UN, dN = s.get_state(), s.diag()
    s.destroy()
    assert np.array_equal(log1, logN) and np.array_equal(U1, UN)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dN[k]
    if scheme.startswith("plm"):  # (the fused stage's split schedule ran once)
        assert prof["halo_exposed"][1] == 1


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["wenoz-split-P2", "wenoz-split-P4", "ct-plm-P4", "ct-wenoz-P3"])
def test_halo_push_split_and_ct_bitwise(mhd, case):
    """The halo push from the update kernels of the split WENO-Z stage (mhd_split.cu k_sp_update)
    and the CT stage (mhd_ct.cu k_ct_update): the next stage (and the CT dt pass, which reads
    B_z of the ghost plane) skips its exchange.  Bitwise equal to one domain with equal counters,
    across a state change; only the first stage after each state change exchanges."""
    from test_oracle_scheme import _random_ct_state
    scheme, P = case.rsplit("-P", 1)
    P = int(P)
    if scheme == "wenoz-split":
        p = I.orszag_tang_3d(32).replace(n=(40, 21, 24), limiter=I.WENOZ, stepper=I.RK3)
        U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
        U0b = I.with_noise(I.orszag_tang_3d_ic(p), p, seed=7)
    else:
        lim = I.MC if scheme == "ct-plm" else I.WENOZ
        p = I.orszag_tang_3d(12, limiter=lim).replace(n=(20, 14, 24), ct=1, glm=0,
                                                       stepper=I.RK2 if lim == I.MC else I.RK3)
        U0 = _random_ct_state(p)
        U0b = _random_ct_state(p, seed=11)
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = list(s.run(3))
    s.set_state(U0b)
    log1 += list(s.run(3))
    U1, d1 = s.get_state(), s.diag()
    s.destroy()
    g = _with_env({"MHD_HALO_PUSH": "1"}, lambda: mhd.SolverGroup(p, P))
    assert all(sl.halo_push for sl in g.slabs)
    g.set_state(U0)
    logP = list(g.run(3))
    g.set_state(U0b)
    logP += list(g.run(3))
    UP, dP = g.get_state(), g.diag()
    g.destroy()
    assert np.array_equal(np.array(log1), np.array(logP))
    assert np.array_equal(U1, UP)
    for k in ("p_floors", "plm_fallbacks", "hlld_to_hll"):
        assert d1[k] == dP[k]


@pytest.mark.gpu
def test_halo_push_one_slab_state_change(mhd):
    """A state change of ONE slab of a pushing group (its new boundary planes are its neighbours'
    ghost planes): the group falls back to the exchange for the next stage on every slab, and
    the run equals one domain given the same spliced state, bitwise."""
    p = I.orszag_tang_3d(32).replace(n=(40, 21, 32))
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    U0b = I.with_noise(I.orszag_tang_3d_ic(p), p, seed=7)
    g = _with_env({"MHD_HALO_PUSH": "1"}, lambda: mhd.SolverGroup(p, 4))
    g.set_state(U0)
    logP = list(g.run(2))
    Umid = g.get_state()
    sl = g.slabs[1]
    z0, nz = sl.offset[2], sl.extent[2]
    sl.set_state(np.ascontiguousarray(U0b[:, z0:z0 + nz]))
    logP += list(g.run(3))
    UP = g.get_state()
    g.destroy()
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = list(s.run(2))
    assert np.array_equal(s.get_state(), Umid)
    Umid[:, z0:z0 + nz] = U0b[:, z0:z0 + nz]
    s.set_state(np.ascontiguousarray(Umid))
    log1 += list(s.run(3))
    U1 = s.get_state()
    s.destroy()
    assert np.array_equal(np.array(log1), np.array(logP)) and np.array_equal(U1, UP)


@pytest.mark.gpu
@pytest.mark.parametrize("fault", [1, 2, 3, 4])
def test_halo_push_setup_failure_falls_back(mhd, fault):
    """A failed step of the NCCL halo-push set-up (injected by MHD_HALO_PUSH_FAULT: the LSA check,
    a window registration, the device communicator, the peer pointers) releases what was set up
    and leaves the context on the send/recv exchange: no push, bitwise the same run."""
    p = I.orszag_tang_3d(32).replace(n=(40, 21, 32), stepper=I.RK3)
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p)
    s = mhd.Solver(p)
    s.set_state(U0)
    log1 = s.run(3)
    U1 = s.get_state()
    s.destroy()
    s = _with_env({"MHD_NCCL_SELF": "1", "MHD_HALO_PUSH": "1", "MHD_HALO_PUSH_FAULT": str(fault)},
                  lambda: mhd.Solver(p))
    assert not s.halo_push
    s.set_state(U0)
    logN = s.run(3)
    UN = s.get_state()
    s.destroy()
    assert np.array_equal(log1, logN) and np.array_equal(U1, UN)
