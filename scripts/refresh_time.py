"""Dev tool: wall time of a hierarchy refresh at cfg2 (coarsening + coarsest factor)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
pb = cases.cantilever(256, 128, 128)
g = pb.grid
st = vb.OperatorState(g, np.random.default_rng(0).uniform(0, 1, g.n_elements), pb.model, pb.boundary.fixed_mask(g))
for scheme in sys.argv[1:] or ["homogenized"]:
    H = vb.build_hierarchy(g, st, 7, scheme=scheme)
    H.refresh(st); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        H.refresh(st)
    torch.cuda.synchronize()
    print(os.environ.get("VT_LIB_PATH", "default"), scheme, f"refresh {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
