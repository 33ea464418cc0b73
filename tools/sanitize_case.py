"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / initcheck / synccheck):
3D OT with ragged tiles through every stage-kernel variant in use (PLM RK2 HLLD, PLM RK3 HLL,
WENOZ RK3), the slab group, and the 2D / 1D paths.  Usage: compute-sanitizer --tool X python tools/sanitize_case.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2510_24175_b200 import inputs as I  # noqa: E402
from paper_2510_24175_b200 import mhd  # noqa: E402

cases = [
    I.orszag_tang_3d(16).replace(n=(40, 13, 12), hi=(1.25, 0.40625, 0.375)),
    I.orszag_tang_3d(16, riemann=I.HLL).replace(n=(40, 13, 12), hi=(1.25, 0.40625, 0.375), stepper=I.RK3),
    I.orszag_tang_3d(16, limiter=I.WENOZ).replace(n=(40, 13, 12), hi=(1.25, 0.40625, 0.375), stepper=I.RK3),
    I.orszag_tang_2d(24),
    I.brio_wu(64),
]
for p in cases:
    U0 = I.with_noise(I.orszag_tang_3d_ic(p), p) if p.n[2] > 1 else (
        I.orszag_tang_2d_ic(p) if p.n[1] > 1 else I.brio_wu_ic(p))
    s = mhd.Solver(p)
    s.set_state(U0)
    s.run(2)
    U = s.get_state()
    assert np.isfinite(U).all()
    s.destroy()
p = cases[2]
g = mhd.SolverGroup(p, 4)
g.set_state(I.orszag_tang_3d_ic(p))
g.run(2)
g.destroy()
print("sanitize case ok")
