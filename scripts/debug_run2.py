"""Dev tool: DeviceRun iteration-2 solve vs a standalone mgcg_solve on the same inputs."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200.design import DeviceRun
from oracle import cpu_path as O

case = O.cantilever_case(48, 24, 24)
grid = vb.build_grid(48, 24, 24, case.h)
fixed = np.flatnonzero(case.fixed_mask)
loads = [(int(d), float(case.f_ext[d])) for d in np.flatnonzero(case.f_ext)]
prob = vb.Problem(grid, vb.make_boundary(grid, fixed, loads, None), vb.classify_regions(grid, []))
opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, p=3.0, max_iterations=3, ch_tol=1e-12)
R = DeviceRun(prob, opt, vb.SolverConfig(tolerance=1e-5), "homogenized", 4, 0.4)
m = prob.model
rep1 = R.solve(m); R.design_step(m)
rho1 = R.rho.cpu().numpy(); u1 = R.displacement(); f = R.d.download(R.f)
rep2 = R.solve(m); u2 = R.displacement()
st = vb.OperatorState(grid, rho1, vb.MaterialModel(), case.fixed_mask)
H = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
x, rep = vb.mgcg_solve(st, H, f, u_prev=u1, cfg=vb.SolverConfig(tolerance=1e-5))
print("run it2", rep2.iterations, rep2.final_rel_residual, "standalone", rep.iterations, rep.final_rel_residual,
      "u2 diff", np.abs(u2 - x).max() / np.abs(x).max())
print("f vs case f", np.abs(f - np.where(case.fixed_mask, 0, case.f_ext)).max())
# same DeviceRun buffers, fresh solve through the C ABI
R2 = DeviceRun(prob, opt, vb.SolverConfig(tolerance=1e-5), "homogenized", 4, 0.4,
               init_densities=vb.DensityField(rho1, prob.regions), init_displacement=u1)
rep3 = R2.solve(m); u3 = R2.displacement()
print("fresh DeviceRun from rho1/u1:", rep3.iterations, rep3.final_rel_residual, np.abs(u3 - x).max() / np.abs(x).max())
