"""Measure the reference against itself: cfg1 40 SIMP iterations at tol 1e-5 with
OPENBLAS_NUM_THREADS set by the caller, compared with tests/golden/cfg1_traj.npz
(generated with the default thread count).  Test infrastructure; needs /root/reference.

    OPENBLAS_NUM_THREADS=1 python oracle/ref_self_variation.py

Recorded (round 1): threads 1 -> max compliance diff 2.85e-7, 24/40 equal CG
counts, rho20 2.8e-6, rho40 1.9e-6."""
import sys, os, numpy as np
sys.path.insert(0, '/root/repo/oracle'); sys.path.insert(0, '/root/repo')
import make_golden as M
vt = M._vt()
from voxtop.app.presets import instantiate
problem, _ = instantiate("cantilever", (48, 24, 24))
h = problem.grid.h
opt = vt.OptConfig(volfrac=0.12, filter_radius=1.5 * h, p=3.0, max_iterations=40, ch_tol=1e-12)
recs, snaps, wall, _ = M._traj(vt, problem, opt, {20, 40}, max_levels=4)
g = np.load('/root/repo/tests/golden/cfg1_traj.npz')
w = g['recs']
d = np.abs(recs[:, 1] - w[:, 1]) / np.abs(w[:, 1])
print("threads", os.environ.get("OPENBLAS_NUM_THREADS"), "max", d.max(), "per-it", np.array2string(d, precision=1), "same", int((recs[:, 4] == w[:, 4]).sum()),
      "rho20", np.abs(snaps['rho20'] - g['rho20']).max(), "rho40", np.abs(snaps['rho40'] - g['rho40']).max())
