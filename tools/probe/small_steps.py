"""Per-step cost on small problems (launch / host-sync bound): OT-2D 512^2 and Brio-Wu 512."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2510_24175_b200 import inputs as I, mhd

for name, p, U0 in [("ot2d_512", I.orszag_tang_2d(512), None), ("brio_wu_512", I.brio_wu(512), None)]:
    U0 = I.orszag_tang_2d_ic(p) if name.startswith("ot2d") else I.brio_wu_ic(p)
    s = mhd.Solver(p)
    s.set_state(np.ascontiguousarray(U0))
    s.run(20)
    s.profile_enable(True)
    t0 = time.perf_counter()
    log = s.run(100000, p.t_end)
    el = time.perf_counter() - t0
    pr = s.profile_read()
    (ms_stage, n_stage), (ms_dt, n_dt) = pr["stage"], pr["dt"]
    s.destroy()
    print(f"{name}: {len(log)} steps in {el:.2f} s = {1e3 * el / len(log):.3f} ms/step; kernels "
          f"{ms_stage / max(n_stage, 1):.3f} ms/stage x {n_stage / len(log):.0f}, dt {ms_dt / max(n_dt, 1):.3f} ms")
