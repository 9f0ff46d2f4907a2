"""Measure the reference against itself: cfg1 40 SIMP iterations at tol 1e-5 with
OPENBLAS_NUM_THREADS set by the caller, compared with tests/golden/cfg1_traj.npz
(generated with the default thread count).  Test infrastructure; needs /root/reference.

    OPENBLAS_NUM_THREADS=2 python oracle/ref_self_variation.py [out.npz]
    python oracle/ref_self_variation.py --combine out1.npz out2.npz ...   # -> tests/golden/cfg1_selfvar.npz

The combined fixture holds the reference's own per-iteration compliance and CG
counts at each thread count; tests/test_gpu_solver.py bounds the GPU's
default-tolerance trajectory by this envelope.

Recorded (round 2, this container, 8 cores, default = 8 threads):
  threads 1 -> max compliance diff 2.85e-7 (24/40 equal CG counts)
  threads 2 -> max compliance diff 3.23e-5 at iterations 9-11 (20/40 equal), rho20 3.6e-5
(DESIGN.md section 4)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")

if len(sys.argv) > 1 and sys.argv[1] == "--combine":
    out = {}
    base = np.load(os.path.join(GOLD, "cfg1_traj.npz"))
    env = {"rho20": 0.0, "rho40": 0.0}
    for p in sys.argv[2:]:
        d = np.load(p)
        t = int(d["threads"])
        out[f"recs_t{t}"] = d["recs"]
        for k in env:  # the reference's own density spread, max over thread counts
            env[k] = max(env[k], float(np.abs(d[k] - base[k]).max()))
    out["threads"] = np.array(sorted(int(k[6:]) for k in out if k.startswith("recs_t")))
    out["rho20_env"] = env["rho20"]
    out["rho40_env"] = env["rho40"]
    np.savez_compressed(os.path.join(GOLD, "cfg1_selfvar.npz"), **out)
    print("wrote", sorted(out))
    sys.exit(0)

sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, ROOT)
import make_golden as M  # noqa: E402

vt = M._vt()
from voxtop.app.presets import instantiate  # noqa: E402

problem, _ = instantiate("cantilever", (48, 24, 24))
h = problem.grid.h
opt = vt.OptConfig(volfrac=0.12, filter_radius=1.5 * h, p=3.0, max_iterations=40, ch_tol=1e-12)
recs, snaps, wall, _ = M._traj(vt, problem, opt, {20, 40}, max_levels=4)
g = np.load(os.path.join(GOLD, "cfg1_traj.npz"))
w = g["recs"]
d = np.abs(recs[:, 1] - w[:, 1]) / np.abs(w[:, 1])
threads = os.environ.get("OPENBLAS_NUM_THREADS", "0")
print("threads", threads, "max", d.max(), "per-it", np.array2string(d, precision=1), "same",
      int((recs[:, 4] == w[:, 4]).sum()),
      "rho20", np.abs(snaps['rho20'] - g['rho20']).max(), "rho40", np.abs(snaps['rho40'] - g['rho40']).max())
if len(sys.argv) > 1:
    np.savez_compressed(sys.argv[1], threads=int(threads), recs=recs, rho20=snaps["rho20"], rho40=snaps["rho40"])
