"""Dev tool: the bench's graded launch (vt_apply_projected at cfg2) a few times,
for `ncu -k regex:hex8_tile_kernel -s 3 -c 1` captures of exactly that path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402
from paper_2201_12931_b200._lib import lib  # noqa: E402
from paper_2201_12931_b200.device import ptr, stream_ptr  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
spec = cases.CONFIGS[cfg]
prob = spec["builder"](*spec["dims"])
g = prob.grid
rng = np.random.default_rng(0)
fm = prob.boundary.fixed_mask(g)
st = vb.OperatorState(g, rng.uniform(0.0, 1.0, g.n_elements), prob.model, fm, prob.stiffness())
u = rng.standard_normal(g.n_dofs)
u[fm] = 0.0
ud = st.dgrid.upload(u)
vd = st.dgrid.zeros()
for _ in range(6):
    lib.vt_apply_projected(st.dgrid.handle, ptr(st.scale_dev), ptr(ud), ptr(vd), stream_ptr())
torch.cuda.synchronize()
print("done")
