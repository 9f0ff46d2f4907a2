"""Dev tool (runs ON the GPU box): the public apply() host->host at cfg2 for
several z-chunk counts (pinned and pageable input)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases, stiffness_op  # noqa: E402

spec = cases.CONFIGS["cfg2"]
pb = spec["builder"](*spec["dims"])
g = pb.grid
rng = np.random.default_rng(0)
fm = pb.boundary.fixed_mask(g)
st = vb.OperatorState(g, rng.uniform(0, 1, g.n_elements), pb.model, fm, pb.stiffness())
u = rng.standard_normal(g.n_dofs)
pinned = torch.from_numpy(u).pin_memory().numpy()
for nch in [int(x) for x in sys.argv[1:]] or [4, 6, 8, 12, 16]:
    stiffness_op.HOST_CHUNKS = nch
    for name, arr in (("pinned", pinned), ("pageable", u)):
        for _ in range(3):
            vb.apply(st, arr)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(10):
            vb.apply(st, arr)
        torch.cuda.synchronize()
        t = (time.perf_counter() - t0) / 10
        print(f"chunks {nch:2d} {name:8s}: {t*1e3:.3f} ms  {g.n_dofs/t/1e9:.2f} GDOF/s", flush=True)
