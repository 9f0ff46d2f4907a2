"""Dev tool: iteration-1 solve of cfg1 -- run() vs mgcg_solve() vs the oracle."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2201_12931_b200 as vb
from oracle import cpu_path as O

case = O.cantilever_case(48, 24, 24)
grid = vb.build_grid(48, 24, 24, case.h)
fixed = np.flatnonzero(case.fixed_mask)
loads = [(int(d), float(case.f_ext[d])) for d in np.flatnonzero(case.f_ext)]
prob = vb.Problem(grid, vb.make_boundary(grid, fixed, loads, None), vb.classify_regions(grid, []))
seen = {}
vb.run(prob, vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, p=3.0, max_iterations=1, ch_tol=1e-12),
       vb.SolverConfig(tolerance=1e-5), scheme="homogenized", max_levels=4,
       on_iteration=lambda rec, rho, u: seen.setdefault(1, np.asarray(u).copy()))
u_run = seen[1]
k0 = O.hex8_k0(0.3, case.h)
rho0 = np.full(grid.n_elements, 0.12)
f = case.f_ext.copy(); f[fixed] = 0
H = O.hier_build(case.es, case.h, case.fixed_mask, 4)
sc0 = O.simp(rho0, 3.0, 1e-9)
O.hier_refresh(H, rho0, sc0, k0, 3.0, 1e-9, 1.0)
st = vb.OperatorState(grid, rho0, vb.MaterialModel(), case.fixed_mask)
Hg = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
r = np.random.default_rng(3).standard_normal(grid.n_dofs); r[fixed] = 0
print("vcycle rel", np.abs(Hg.v_cycle(r) - O.vcycle(H, r)).max() / np.abs(O.vcycle(H, r)).max())
for k in (8, 9, 10, 11, 12, 13):
    uo, ro = O.pcg(lambda p: O.apply_k(p, case.es, fixed, k0, sc0), lambda p, ff: O.resid_k(p, ff, case.es, fixed, k0, sc0),
                   lambda v: O.vcycle(H, v), f, None, fixed, 1e-14, k)
    ug, rg = vb.mgcg_solve(st, Hg, f, cfg=vb.SolverConfig(tolerance=1e-14, max_iterations=k))
    print(k, "mgcg vs oracle", np.abs(ug - uo).max() / np.abs(uo).max(), rg.iterations, ro.iterations,
          rg.final_rel_residual, ro.final_rel_residual)
#print("run vs oracle", np.abs(u_run - uo).max() / np.abs(uo).max(), "run vs mgcg", np.abs(u_run - ug).max() / np.abs(ug).max())
