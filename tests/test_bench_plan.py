"""bench.py's scaling modes on CPU (no GPU): the global problem and every rank's z slab for
N = 1, 2, 4, 8 in both modes (BASELINE.json configs[3] and configs[4]), and the
slabs' halo plans pair up (each send has the matching receive on the peer)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2510_24175_b200 import inputs as I  # noqa: E402


class A:
    def __init__(self, scaling, workload=None, n=None):
        self.scaling, self.workload, self.n = scaling, workload, n


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_weak_mode_blast_512_per_gpu(N):
    wl, n, label = bench.resolve(A("weak"))
    assert (wl, n) == ("blast3d", 512) and "configs[3]" in label
    p = bench.build_problem(wl, N, n, "plm-rk2", "weak")
    assert p.n == (512, 512, 512 * N) and p.hi[2] == float(N)  # one blast per unit cube along z
    shape, plan = bench.slab_plan(p, N)
    assert [(z0, z1) for _, z0, z1 in plan] == [(512 * r, 512 * (r + 1)) for r in range(N)]
    assert p.limiter == I.MC and p.riemann == I.HLLD and p.glm == 1 and p.stepper == I.RK2


@pytest.mark.parametrize("N", [1, 2, 4, 8])
def test_strong_mode_ot_1024_global(N):
    wl, n, label = bench.resolve(A("strong"))
    assert (wl, n) == ("ot3d", 1024) and "configs[4]" in label
    p = bench.build_problem(wl, N, n, "plm-rk2", "strong")
    assert p.n == (1024, 1024, 1024) and p.hi == (1.0, 1.0, 1.0)  # the same box at every N
    _, plan = bench.slab_plan(p, N)
    assert [(z0, z1) for _, z0, z1 in plan] == [(1024 // N * r, 1024 // N * (r + 1)) for r in range(N)]
    assert sum(z1 - z0 for _, z0, z1 in plan) == 1024


def test_overrides_and_roofline_config():
    wl, n, label = bench.resolve(A("weak", "ot3d", 256))
    assert (wl, n) == ("ot3d", 256) and "configs[2]" in label
    with pytest.raises(ValueError):
        bench.build_problem("ot3d", 3, 1024, "plm-rk2", "strong")  # 1024 planes do not split in 3


@pytest.mark.parametrize("N", [2, 4, 8])
@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_halo_plans_pair_up(N, scaling):
    """every send in a rank's halo plan meets a receive of the same size on the peer, in the
    posting order NCCL pairs them (mhd_halo_plan; pure host logic, no GPU)"""
    from paper_2510_24175_b200 import mhd
    try:
        mhd.load()
    except Exception as e:  # the library is built by __graft_entry__.build()
        pytest.skip(str(e))
    wl, n, _ = bench.resolve(A(scaling))
    p = bench.build_problem(wl, N, n, "plm-rk2", scaling)
    plans = [mhd.halo_plan(r, N, p.n[2], True, 2) for r in range(N)]
    for r in range(N):
        sends = [(peer, planes) for peer, kind, _, planes in plans[r] if kind == 0 and peer >= 0]
        for peer, planes in sends:
            recvs = [row for row in plans[peer] if row[1] == 1 and row[0] == r and row[3] == planes]
            assert recvs, (r, peer)
