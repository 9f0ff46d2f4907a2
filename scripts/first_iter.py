"""Dev tool (runs ON the GPU box): wall time of the first SIMP iterations of
run() at cfg2 (the first includes hierarchy build and PCG graph capture)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402

spec = cases.CONFIGS["cfg2"]
pb = spec["builder"](*spec["dims"])
opt = vb.OptConfig(volfrac=spec["volfrac"], filter_radius=1.5 * pb.grid.h, max_iterations=3, ch_tol=1e-12)
for scheme in ("homogenized", "galerkin", "homogenized"):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = vb.run(pb, opt, vb.SolverConfig(tolerance=1e-5), scheme=scheme, max_levels=spec["levels"])
    print(scheme, "total", round(time.perf_counter() - t0, 3), "wall_s", [round(r.wall_s, 4) for r in res.records],
          flush=True)
