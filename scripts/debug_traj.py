"""Dev tool: per-iteration compliance / CG-count drift of the device run() vs the cfg1 golden."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import paper_2201_12931_b200 as vb
from oracle import cpu_path as O

g = np.load(os.path.join(ROOT, "tests/golden/cfg1_traj.npz"))
want = g["recs"]
case = O.cantilever_case(48, 24, 24)
grid = vb.build_grid(48, 24, 24, case.h)
fixed = np.flatnonzero(case.fixed_mask)
loads = [(int(d), float(case.f_ext[d])) for d in np.flatnonzero(case.f_ext)]
prob = vb.Problem(grid, vb.make_boundary(grid, fixed, loads, None), vb.classify_regions(grid, []))
n_it = int(sys.argv[1]) if len(sys.argv) > 1 else 12
opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, p=3.0, max_iterations=n_it, ch_tol=1e-12)
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-5
res = vb.run(prob, opt, vb.SolverConfig(tolerance=tol, max_iterations=1000), scheme="homogenized", max_levels=4)
for r, w in zip(res.records, want):
    print(r.iteration, r.cg_iters, int(w[4]), f"{abs(r.compliance - w[1]) / abs(w[1]):.2e}", f"res {r.cg_residual:.4e} {w[5]:.4e}")

# --- iteration-2 solve in isolation: golden rho1, warm start from each side's own u1
seen = {}
def hook(rec, rho, u):
    seen[rec.iteration] = (rho.values.copy(), np.asarray(u).copy())
vb.run(prob, vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, p=3.0, max_iterations=1, ch_tol=1e-12),
       vb.SolverConfig(tolerance=tol), scheme="homogenized", max_levels=4, on_iteration=hook)
rho1_gpu, u1_gpu = seen[1]
print("rho1 max|gpu - golden|", np.abs(rho1_gpu - g["rho1"]).max())
k0 = O.hex8_k0(0.3, case.h)
rho0 = np.full(grid.n_elements, 0.12)
f = case.f_ext.copy(); f[fixed] = 0
H = O.hier_build(case.es, case.h, case.fixed_mask, 4)
sc0 = O.simp(rho0, 3.0, 1e-9)
O.hier_refresh(H, rho0, sc0, k0, 3.0, 1e-9, 1.0)
u1_o, rep = O.pcg(lambda p: O.apply_k(p, case.es, fixed, k0, sc0), lambda p, ff: O.resid_k(p, ff, case.es, fixed, k0, sc0),
                  lambda r: O.vcycle(H, r), f, None, fixed, tol, 200)
print("u1 rel diff", np.abs(u1_gpu - u1_o).max() / np.abs(u1_o).max(), rep.iterations)
rho1 = g["rho1"]
sc1 = O.simp(rho1, 3.0, 1e-9)
O.hier_refresh(H, rho1, sc1, k0, 3.0, 1e-9, 1.0)
u2_o, rep_o = O.pcg(lambda p: O.apply_k(p, case.es, fixed, k0, sc1), lambda p, ff: O.resid_k(p, ff, case.es, fixed, k0, sc1),
                    lambda r: O.vcycle(H, r), f, u1_o, fixed, tol, 200)
st = vb.OperatorState(grid, rho1, vb.MaterialModel(), case.fixed_mask)
Hg = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
u2_g, rep_g = vb.mgcg_solve(st, Hg, f, u_prev=u1_o, cfg=vb.SolverConfig(tolerance=tol))
print("it2 oracle", rep_o.iterations, rep_o.final_rel_residual, "gpu", rep_g.iterations, rep_g.final_rel_residual,
      "u2 rel", np.abs(u2_g - u2_o).max() / np.abs(u2_o).max())
for k in (1, 2, 5, 10, 15, 20, 25):
    xo, ro = O.pcg(lambda p: O.apply_k(p, case.es, fixed, k0, sc1), lambda p, ff: O.resid_k(p, ff, case.es, fixed, k0, sc1),
                   lambda r: O.vcycle(H, r), f, u1_o, fixed, 1e-14, k)
    xg, rg = vb.mgcg_solve(st, Hg, f, u_prev=u1_o, cfg=vb.SolverConfig(tolerance=1e-14, max_iterations=k))
    print(k, "x rel", np.abs(xg - xo).max() / np.abs(xo).max(), rg.final_rel_residual, ro.final_rel_residual)

# --- refreshed hierarchy (built on rho0, refreshed to rho1) vs fresh
st0 = vb.OperatorState(grid, rho0, vb.MaterialModel(), case.fixed_mask)
Hr = vb.build_hierarchy(grid, st0, 4, scheme="homogenized")
Hr.refresh(st)
u2_r, rep_r = vb.mgcg_solve(st, Hr, f, u_prev=u1_o, cfg=vb.SolverConfig(tolerance=tol))
print("refreshed hier:", rep_r.iterations, rep_r.final_rel_residual, "vs fresh", rep_g.iterations, rep_g.final_rel_residual)
rr = np.random.default_rng(5).standard_normal(grid.n_dofs); rr[fixed] = 0
print("vcycle refreshed vs fresh", np.abs(Hr.v_cycle(rr) - Hg.v_cycle(rr)).max() / np.abs(Hg.v_cycle(rr)).max())
# --- same solve twice through one hierarchy / state (graph reuse)
u2_b, rep_b = vb.mgcg_solve(st, Hg, f, u_prev=u1_o, cfg=vb.SolverConfig(tolerance=tol))
print("repeat:", rep_b.iterations, rep_b.final_rel_residual, np.abs(u2_b - u2_g).max())
