import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (4, 2, 2)
grid = vb.build_grid(*dims, 1.0)
rng = np.random.default_rng(0)
st = vb.OperatorState(grid, rng.uniform(0, 1, grid.n_elements), vb.MaterialModel(), np.zeros(grid.n_dofs, bool))
torch.cuda.synchronize(); print("scale ok", flush=True)
v = vb.apply(st, rng.standard_normal(grid.n_dofs))
print("apply ok", np.abs(v).max(), flush=True)
