"""Dev tool: cfg2 design iterations with the Galerkin vs homogenized hierarchy (solve time, CG counts)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
from paper_2201_12931_b200.design import DeviceRun
dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (256, 128, 128)
prob = cases.cantilever(*dims)
opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * prob.grid.h, ch_tol=1e-12)
for scheme in ("galerkin", "homogenized"):
    R = DeviceRun(prob, opt, vb.SolverConfig(tolerance=1e-5), scheme, None, 0.4)
    out = []
    for it in range(6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rep = R.solve(prob.model)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        c, ch, vol = R.design_step(prob.model)
        out.append((rep.iterations, round(dt * 1e3, 1), c))
    print(scheme, "(its, ms, c):", out, "mem GB", round(torch.cuda.max_memory_allocated() / 1e9, 2))
