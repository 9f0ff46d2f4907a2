import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
spec = cases.CONFIGS["cfg2"]
problem = spec["builder"](*spec["dims"])
grid = problem.grid; n = grid.n_dofs
rng = np.random.default_rng(0)
rho = rng.uniform(0.0, 1.0, grid.n_elements)
fm = problem.boundary.fixed_mask(grid)
u_host = rng.standard_normal(n); u_host[fm] = 0
state = vb.OperatorState(grid, rho, problem.model, fm, problem.stiffness())
pin_u = torch.from_numpy(u_host).pin_memory(); u_np = pin_u.numpy()
print("pinned?", pin_u.is_pinned(), u_np.flags['C_CONTIGUOUS'], u_np.dtype)
for i in range(8):
    t0 = time.perf_counter(); out = vb.apply(state, u_np); t1 = time.perf_counter()
    print(i, f"{(t1-t0)*1e3:.2f} ms")
u2 = torch.from_numpy(rng.standard_normal(n)).pin_memory().numpy()
for i in range(3):
    t0 = time.perf_counter(); out = vb.apply(state, u2); t1 = time.perf_counter()
    print("u2", i, f"{(t1-t0)*1e3:.2f} ms")
