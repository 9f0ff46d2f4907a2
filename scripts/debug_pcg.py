"""Dev tool: where does the GPU MGPCG iterate drift from the oracle? (pcg.npz case)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2201_12931_b200 as vb
from oracle import cpu_path as O

g = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/pcg.npz"))
case = O.cantilever_case(16, 8, 8)
fixed = np.flatnonzero(case.fixed_mask)
k0 = O.hex8_k0(0.3, case.h)
grid = vb.build_grid(16, 8, 8, case.h)
tag = sys.argv[1] if len(sys.argv) > 1 else "r"
rho = g[f"{tag}_rho"]
scale = O.simp(rho, 3.0, 1e-9)
H = O.hier_build(case.es, case.h, case.fixed_mask, 3)
O.hier_refresh(H, rho, scale, k0, 3.0, 1e-9, 1.0)
st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
Hg = vb.build_hierarchy(grid, st, 3, scheme="homogenized")
f = g["f"]
rng = np.random.default_rng(1)
r = rng.standard_normal(grid.n_dofs); r[fixed] = 0
zg = Hg.v_cycle(r); zo = O.vcycle(H, r)
print("vcycle rel", np.abs(zg - zo).max() / np.abs(zo).max())
ag = vb.apply(st, r); ao = O.apply_k(r, case.es, fixed, k0, scale)
print("apply rel", np.abs(ag - ao).max() / np.abs(ao).max())
for k in list(range(1, 12)) + [15, 20, 25, 30, 35, 38, 39, 40]:
    xg, rg = vb.mgcg_solve(st, Hg, f, cfg=vb.SolverConfig(tolerance=1e-14, max_iterations=k))
    xo, ro = O.pcg(lambda p: O.apply_k(p, case.es, fixed, k0, scale),
                   lambda p, ff: O.resid_k(p, ff, case.es, fixed, k0, scale),
                   lambda v: O.vcycle(H, v), f, None, fixed, 1e-14, k)
    print(k, "x rel", np.abs(xg - xo).max() / np.abs(xo).max(), "res", rg.final_rel_residual, ro.final_rel_residual)
