"""The reference against itself on the small default-tolerance trajectories of
tests/golden (small_traj 16x8x8, bridge_traj 32x16x16, grav_traj 32x16x16
self-weight), re-run with OPENBLAS_NUM_THREADS set by the caller.  Test
infrastructure; needs /root/reference.

    OPENBLAS_NUM_THREADS=2 python oracle/ref_self_variation_small.py out_t2.npz
    python oracle/ref_self_variation_small.py --combine out_t*.npz    # -> tests/golden/selfvar_small.npz
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")
CASES = ("small", "bridge", "grav")

if len(sys.argv) > 1 and sys.argv[1] == "--combine":
    out = {}
    for p in sys.argv[2:]:
        d = np.load(p)
        t = int(d["threads"])
        for c in CASES:
            out[f"{c}_t{t}"] = d[c]
    out["threads"] = np.array(sorted({int(k.split("_t")[1]) for k in out}))
    np.savez_compressed(os.path.join(GOLD, "selfvar_small.npz"), **out)
    print("wrote", sorted(out))
    sys.exit(0)

sys.path.insert(0, os.path.join(ROOT, "oracle"))
import make_golden as M  # noqa: E402

vt = M._vt()
from voxtop.app import presets as P  # noqa: E402
from voxtop.app.presets import instantiate  # noqa: E402

res = {}
problem, _ = instantiate("cantilever", (16, 8, 8))
h = problem.grid.h
opt = vt.OptConfig(volfrac=0.12, filter_radius=2.5 * h, max_iterations=30, ch_tol=1e-12)
res["small"] = M._traj(vt, problem, opt, set(), max_levels=3)[0]
grid = vt.build_grid(32, 16, 16, 2.0)
fixed = P._fix_all(grid, P._bottom_corner_nodes(grid))
loads = P._face_pressure_loads(grid, 2, 1, 2, -100.0)
Lx, Ly, Lz = grid.domain
reg = vt.classify_regions(grid, [(vt.Box((0, 0, Lz - grid.h), (Lx, Ly, Lz)), vt.Region.PASSIVE_SOLID)])
opt = vt.OptConfig(volfrac=0.14, filter_radius=1.5 * grid.h, max_iterations=3, ch_tol=1e-12)
res["bridge"] = M._traj(vt, vt.Problem(grid, vt.make_boundary(grid, fixed, loads), reg), opt, set())[0]
problem, _ = instantiate("cantilever", (32, 16, 16))
bnd = problem.boundary
gb = vt.BoundarySpec(bnd.fixed_dofs, bnd.load_dofs, bnd.load_values, vt.GravitySpec(axis=2, g=1.0, unit_weight=1e-3))
opt = vt.OptConfig(volfrac=0.12, filter_radius=1.5 * problem.grid.h, max_iterations=4, ch_tol=1e-12)
res["grav"] = M._traj(vt, vt.Problem(problem.grid, gb, problem.regions), opt, set())[0]
threads = int(os.environ.get("OPENBLAS_NUM_THREADS", "0"))
for c in CASES:
    w = np.load(os.path.join(GOLD, f"{c}_traj.npz"))["recs"]
    d = np.abs(res[c][:, 1] - w[:, 1]) / np.abs(w[:, 1])
    print(c, "threads", threads, "max", d.max())
if len(sys.argv) > 1:
    np.savez_compressed(sys.argv[1], threads=threads, **res)
