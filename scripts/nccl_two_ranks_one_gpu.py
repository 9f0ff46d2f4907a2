"""Dev probe: can two ranks share one GPU with the library's NCCL transport?
(torchrun --nproc-per-node 2; both ranks on cuda:0, gloo for the bootstrap)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, torch.distributed as dist
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200.slabs import SlabSolver
from oracle import cpu_path as O
torch.cuda.set_device(0)
dist.init_process_group("gloo")
rank = dist.get_rank()
case = O.cantilever_case(32, 16, 16)
grid = vb.build_grid(32, 16, 16, case.h)
rng = np.random.default_rng(2)
rho = rng.uniform(0.05, 1.0, grid.n_elements)
try:
    S = SlabSolver.from_process_group(grid, case.fixed_mask, levels=4)
    S.set_density(rho)
    f = case.f_ext.copy(); f[case.fixed_mask] = 0
    x, rep = S.mgcg_solve(S.upload(f), cfg=vb.SolverConfig(tolerance=1e-8, max_iterations=300))
    xs = torch.from_numpy(np.array(S.download(x)))
    dist.all_reduce(xs)
    if rank == 0:
        st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
        H = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
        xr, rr = vb.mgcg_solve(st, H, f, cfg=vb.SolverConfig(tolerance=1e-8, max_iterations=300))
        print("2-rank NCCL slab solve:", rep.iterations, "its vs", rr.iterations,
              "rel diff", float(np.abs(xs.numpy() - xr).max() / np.abs(xr).max()))
    S.close()
except Exception as e:
    print("rank", rank, "failed:", repr(e)[:300])
dist.destroy_process_group()
