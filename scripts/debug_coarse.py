"""Dev tool: coarsest solve / V-cycle accuracy at a mid-run cfg1 design (golden rho10)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, scipy.linalg
import paper_2201_12931_b200 as vb
from oracle import cpu_path as O

g = np.load(os.path.join(ROOT, "tests/golden/cfg1_traj.npz"))
case = O.cantilever_case(48, 24, 24)
grid = vb.build_grid(48, 24, 24, case.h)
k0 = O.hex8_k0(0.3, case.h)
for key in ("rho1", "rho5", "rho10", "rho20"):
    rho = g[key]
    sc = O.simp(rho, 3.0, 1e-9)
    H = O.hier_build(case.es, case.h, case.fixed_mask, 4)
    O.hier_refresh(H, rho, sc, k0, 3.0, 1e-9, 1.0)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    Hg = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
    last = H.levels[-1]
    K = O.dense_k(last.es, last.fixed, last.k0, last.scale)
    rng = np.random.default_rng(0)
    b = rng.standard_normal(K.shape[0]); b[last.fixed] = 0
    xo = scipy.linalg.cho_solve(H.chol, b)
    xg = Hg.coarse_solve(b) if hasattr(Hg, "coarse_solve") else None
    cond = np.linalg.cond(K)
    r = rng.standard_normal(grid.n_dofs); r[case.fixed_mask] = 0
    zo = O.vcycle(H, r); zg = Hg.v_cycle(r)
    print(key, f"cond {cond:.2e}", "coarse rel", None if xg is None else np.abs(xg - xo).max() / np.abs(xo).max(),
          "resid gpu", None if xg is None else np.linalg.norm(K @ xg - b) / np.linalg.norm(b),
          "resid ref", np.linalg.norm(K @ xo - b) / np.linalg.norm(b),
          "vcycle rel", np.abs(zg - zo).max() / np.abs(zo).max())
