"""Diagnose the Galerkin breakdown of the cfg5 run (runs ON the GPU box).

The 300-iteration cfg5 run with scheme="galerkin" stopped at SIMP iteration
48 with r'z < 0 at CG iteration 8 ("preconditioner is not SPD").  This script
replays iterations 1..47 through run(), rebuilds the state / hierarchy at the
47th design, and checks the two candidate causes:
  * the damped-Jacobi smoother: lambda_max(D^-1 A_l) per level by power
    iteration -- the symmetric V(1,1) cycle is SPD only if omega * lambda_max < 2;
  * the coarsest solve: its matrix M (columns = coarse_solve(e_i)) against the
    coarsest operator A (symmetry, eigenvalues, |M A - I|).
Prints one JSON line.

    python scripts/cfg5_galerkin_diag.py [iters] [cfg]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 47
cfg = sys.argv[2] if len(sys.argv) > 2 else "cfg5"
spec = cases.CONFIGS[cfg]
prob = spec["builder"](*spec["dims"])
g = prob.grid
L = spec["levels"]
opt = vb.OptConfig(volfrac=spec["volfrac"], filter_radius=1.5 * g.h, ch_tol=0.01, max_iterations=iters)
res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-5), scheme="galerkin", max_levels=L)
rho = res.densities.values
u_prev = res.displacement
fm = prob.boundary.fixed_mask(g)
out = {"cfg": cfg, "replayed_iterations": len(res.records)}
st = vb.OperatorState(g, rho, prob.model, fm, prob.stiffness())
f = prob.boundary.external_force(g).copy()
f[fm] = 0.0


def power(apply, diag, free, n_it=60, seed=0):
    rng = np.random.default_rng(seed)
    v = rng.standard_normal(free.shape[0]) * free
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(n_it):
        w = apply(v) / diag * free
        lam = float(np.linalg.norm(w))
        v = w / lam
    return lam


for scheme in ("galerkin", "homogenized"):
    H = vb.build_hierarchy(g, st, L, scheme=scheme)
    rec = {}
    try:
        x, rep = vb.mgcg_solve(st, H, f, u_prev, cfg=vb.SolverConfig(tolerance=1e-5))
        rec["solve"] = {"iterations": rep.iterations, "converged": rep.converged, "rel": rep.final_rel_residual}
    except Exception as e:  # noqa: BLE001
        rec["solve"] = {"error": str(e)}
    # V-cycle positivity on random right-hand sides
    rng = np.random.default_rng(1)
    rz = []
    for _ in range(4):
        r = rng.standard_normal(g.n_dofs)
        r[fm] = 0.0
        rz.append(float(r @ H.v_cycle(r)) / float(r @ r))
    rec["rz_over_rr_random"] = rz
    # smoother: omega * lambda_max(D^-1 A_l) < 2 on every smoothed level
    lams = []
    for l in range(0, H.n_levels - 1):
        lv = H.levels[l]
        free = (~np.asarray(lv.fixed_mask, dtype=bool)).astype(np.float64) if hasattr(lv, "fixed_mask") else None
        if free is None:
            free = np.ones(lv.n_dofs)
            free[np.asarray(lv.fixed_idx)] = 0.0
        diag = np.asarray(lv.diag)
        if l == 0:
            lam = power(lambda v: np.asarray(st.apply(v)), diag, free)
        else:
            lam = power(lambda v, l=l: np.asarray(H.coarse_apply(l, v)), diag, free)
        lams.append(lam)
    rec["lambda_max_DinvA"] = lams
    rec["omega_lambda_max"] = [0.4 * x for x in lams]
    # coarsest solve vs coarsest operator
    lc = H.n_levels - 1
    nc = H.levels[lc].n_dofs
    A = np.zeros((nc, nc))
    M = np.zeros((nc, nc))
    for i in range(nc):
        e = np.zeros(nc)
        e[i] = 1.0
        A[:, i] = H.coarse_apply(lc, e)
        M[:, i] = H.coarse_solve(e)
    ev = np.linalg.eigvalsh(0.5 * (A + A.T))
    evm = np.linalg.eigvalsh(0.5 * (M + M.T))
    rec["coarse"] = {"n": nc, "A_asym": float(np.abs(A - A.T).max() / np.abs(A).max()),
                     "A_eig_min": float(ev[0]), "A_eig_max": float(ev[-1]), "A_cond": float(ev[-1] / ev[0]),
                     "M_asym": float(np.abs(M - M.T).max() / np.abs(M).max()),
                     "M_eig_min": float(evm[0]), "M_eig_max": float(evm[-1]),
                     "MA_minus_I": float(np.abs(M @ A - np.eye(nc)).max())}
    out[scheme] = rec
    print(json.dumps({scheme: rec}), flush=True)
    del H
print(json.dumps(out))
