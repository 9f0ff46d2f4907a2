"""Dev tool: the z-slab apply (vt_dist_apply) with k in-process slabs on one GPU
at cfg2 -- device copies stand in for the NCCL halos -- against the
single-slab result (VT_DIST_OVERLAP=0 exchanges first, =1 overlaps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
from paper_2201_12931_b200.slabs import SlabSolver
k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
pb = cases.cantilever(256, 128, 128)
g = pb.grid
fm = pb.boundary.fixed_mask(g)
rng = np.random.default_rng(0)
rho = rng.uniform(0.0, 1.0, g.n_elements)
u = rng.standard_normal(g.n_dofs); u[fm] = 0
S = SlabSolver(g, fm, levels=7, nranks=k)
S.set_density(rho, refresh=False)
us, vs = S.upload(u), S.zeros()
for _ in range(5):
    S.apply(us, vs)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(50):
    S.apply(us, vs)
e1.record(); torch.cuda.synchronize()
t = e0.elapsed_time(e1) / 50 * 1e3
v = S.download(vs)
st = vb.OperatorState(g, rho, pb.model, fm)
ref = vb.apply(st, u)
err = float(np.abs(v - ref).max() / np.abs(ref).max())
print(f"slabs={k} overlap={os.environ.get('VT_DIST_OVERLAP', '1')} apply {t:.1f} us, rel err vs 1 slab {err:.2e}")
