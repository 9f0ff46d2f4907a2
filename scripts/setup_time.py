"""Dev tool (runs ON the GPU box): where the first SIMP iteration's setup time
goes at cfg2 -- OperatorState, build_hierarchy (incl. refresh), the first
MGCG solve (PCG graph capture) -- per scheme, repeated."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402

spec = cases.CONFIGS["cfg2"]
pb = spec["builder"](*spec["dims"])
g = pb.grid
fm = pb.boundary.fixed_mask(g)
rho = np.full(g.n_elements, spec["volfrac"])
f = pb.boundary.external_force(g).copy()
f[fm] = 0.0


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


for rep in range(3):
    for scheme in ("homogenized", "galerkin"):
        t0 = t()
        st = vb.OperatorState(g, rho, pb.model, fm, pb.stiffness())
        t1 = t()
        H = vb.build_hierarchy(g, st, spec["levels"], scheme=scheme)
        t2 = t()
        vb.mgcg_solve(st, H, f, cfg=vb.SolverConfig(tolerance=1e-5))
        t3 = t()
        vb.mgcg_solve(st, H, f, cfg=vb.SolverConfig(tolerance=1e-5))
        t4 = t()
        print(f"rep {rep} {scheme:12s} state {1e3*(t1-t0):7.1f} ms  hierarchy {1e3*(t2-t1):7.1f} ms  "
              f"first solve {1e3*(t3-t2):7.1f} ms  second solve {1e3*(t4-t3):7.1f} ms", flush=True)
        del H, st
