"""Dev tool: one cfg2 V-cycle (run under ncu for the per-kernel launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
from paper_2201_12931_b200._lib import lib
from paper_2201_12931_b200.device import ptr, stream_ptr
pb = cases.cantilever(256, 128, 128)
g = pb.grid
fm = pb.boundary.fixed_mask(g)
rng = np.random.default_rng(0)
st = vb.OperatorState(g, rng.uniform(0, 1, g.n_elements), pb.model, fm)
H = vb.build_hierarchy(g, st, 7, scheme="homogenized")
d = st.dgrid
r = rng.standard_normal(g.n_dofs); r[fm] = 0
f = d.upload(r); z = d.zeros()
for _ in range(3):
    lib.vt_hier_vcycle(H._h, ptr(f), ptr(z), stream_ptr())
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("vc")
lib.vt_hier_vcycle(H._h, ptr(f), ptr(z), stream_ptr())
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
