"""Dev experiment (CPU, oracle only): which perturbation of the reference's
numerics moves the cfg1 default-tolerance trajectory (tol 1e-5, 40 SIMP
iterations) away from the reference fixture, and by how much?

    OPENBLAS_NUM_THREADS=2 python scripts/coarse_variants.py <variant>

variants:
  ref      the oracle as is (scipy cho_factor / cho_solve)
  invref   explicit inverse + one refinement step (the round-1 GPU coarse solve)
  inv      explicit inverse alone
  rlchol   unblocked right-looking Cholesky (the GPU factor) + two triangular solves
  smooth   Jacobi update written as w*r with w = omega/d (the GPU's default epilogue)
  dots     every PCG dot product summed in a different order (pairwise by 4096 blocks)
"""
import os
import sys

import numpy as np
import scipy.linalg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import cpu_path as O  # noqa: E402

var = sys.argv[1] if len(sys.argv) > 1 else "ref"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 40

_refresh = O.hier_refresh


def rl_cholesky(A):
    L = np.array(A, dtype=np.float64)
    n = L.shape[0]
    for j in range(n):
        d = L[j, j]
        piv = np.sqrt(d)
        L[j + 1:, j] /= piv
        L[j, j] = piv
        c = L[j + 1:, j]
        L[j + 1:, j + 1:] -= np.tril(np.outer(c, c))
    return np.tril(L)


def refresh(H, *a, **k):
    _refresh(H, *a, **k)
    last = H.levels[-1]
    K = O.dense_k(last.es, last.fixed, last.k0, last.scale)
    H.K = K
    if var in ("inv", "invref"):
        L = rl_cholesky(K)
        W = scipy.linalg.solve_triangular(L, np.eye(K.shape[0]), lower=True)
        H.Kinv = W.T @ W
    if var == "rlchol":
        H.L = rl_cholesky(K)


def coarse(H, f):
    if var == "inv":
        return H.Kinv @ f
    if var == "invref":
        x0 = H.Kinv @ f
        return x0 + H.Kinv @ (f - H.K @ x0)
    if var == "rlchol":
        y = scipy.linalg.solve_triangular(H.L, f, lower=True)
        return scipy.linalg.solve_triangular(H.L.T, y, lower=False)
    return scipy.linalg.cho_solve(H.chol, f)


def smooth(H, l, sweeps):
    lv = H.levels[l]
    w = H.omega / lv.diag
    for _ in range(sweeps):
        np.subtract(lv.f, O.level_apply(H, l, lv.u), out=lv.r)
        lv.r[lv.fixed] = 0.0
        lv.u += w * lv.r


O.hier_refresh = refresh
O.coarse_solve = coarse
if var == "smooth":
    O._smooth = smooth

if var == "dots":
    _pcg = O.pcg

    class V(np.ndarray):
        def __matmul__(self, o):
            a = np.asarray(self).reshape(-1)
            b = np.asarray(o).reshape(-1)
            m = a * b
            pad = (-m.size) % 4096
            m = np.concatenate([m, np.zeros(pad)]).reshape(-1, 4096)
            return float(np.sum(m.sum(axis=1)[::-1]))

    def pcg(apply, residual, precond, f, u0, fixed_idx, tol=1e-5, maxit=200):
        wrap = lambda x: np.asarray(x).view(V)
        return _pcg(lambda p: wrap(apply(np.asarray(p))), lambda p, ff: wrap(residual(np.asarray(p), ff)),
                    lambda r: wrap(precond(np.asarray(r))), wrap(f), u0, fixed_idx, tol, maxit)

    O.pcg = pcg

g = np.load(os.path.join(ROOT, "tests", "golden", "cfg1_traj.npz"))
want = g["recs"]
case = O.cantilever_case(48, 24, 24)
out = []


def hook(rec, rho, u):
    w = want[rec.iteration - 1]
    d = abs(rec.compliance - w[1]) / abs(w[1])
    out.append((rec.iteration, d, rec.cg_iters, int(w[4])))
    print(f"{var} it {rec.iteration:2d} c_rel {d:.2e} cg {rec.cg_iters} ref {int(w[4])}", flush=True)


rho, u, recs = O.run_design(case, 0.12, 1.5 * case.h, iters, max_levels=4, ch_tol=1e-12, on_iter=hook)
print(f"{var} WORST {max(x[1] for x in out):.2e} same_counts {sum(x[2] == x[3] for x in out)}/{len(out)}",
      f"rho_final {np.abs(rho - g['rho40']).max():.2e}" if iters == 40 else "")
