"""Dev tool: repeated cfg2 MGPCG solves (wall time per solve and per CG iteration)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
pb = cases.cantilever(256, 128, 128)
g = pb.grid
fm = pb.boundary.fixed_mask(g)
rng = np.random.default_rng(0)
st = vb.OperatorState(g, rng.uniform(0, 1, g.n_elements), pb.model, fm)
scheme = sys.argv[1] if len(sys.argv) > 1 else "homogenized"
H = vb.build_hierarchy(g, st, 7, scheme=scheme)
f = pb.boundary.external_force(g); f[fm] = 0
fd = vb.DeviceVector(st.dgrid, st.dgrid.upload(f))
out = []
for k in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    x, rep = vb.mgcg_solve(st, H, fd, cfg=vb.SolverConfig(tolerance=1e-5))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    out.append(f"{rep.iterations}:{dt / rep.iterations * 1e3:.3f}")
print(scheme, "its:ms/it", " ".join(out))
