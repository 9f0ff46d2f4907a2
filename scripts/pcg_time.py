"""Dev tool (runs ON the GPU box): ms per MGPCG iteration (60 iterations,
tolerance unreachable), both schemes, best of 4 solves.

    python scripts/pcg_time.py [homogenized|galerkin ...] [cfg=cfg2]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("cfg=")]
cfgname = next((a[4:] for a in sys.argv[1:] if a.startswith("cfg=")), "cfg2")
spec = cases.CONFIGS[cfgname]
pb = spec["builder"](*spec["dims"])
g = pb.grid
fm = pb.boundary.fixed_mask(g)
rng = np.random.default_rng(0)
st = vb.OperatorState(g, rng.uniform(0.05, 1.0, g.n_elements), pb.model, fm, pb.stiffness())
f = pb.boundary.external_force(g).copy()
f[fm] = 0.0
fd = vb.DeviceVector(st.dgrid, st.dgrid.upload(f))
for scheme in args or ["homogenized", "galerkin"]:
    H = vb.build_hierarchy(g, st, spec["levels"], scheme=scheme)
    cfg = vb.SolverConfig(tolerance=1e-30, max_iterations=60)
    best = 1e9
    for _ in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        x, rep = vb.mgcg_solve(st, H, fd, cfg=cfg)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) / rep.iterations * 1e3)
    print(f"{cfgname} {scheme}: {best:.4f} ms per CG iteration (60 iterations, best of 4 solves incl. setup)",
          flush=True)
    del H
