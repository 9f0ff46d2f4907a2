"""CPU restatement of the voxtop MGPCG hot path (numpy / scipy).

TEST INFRASTRUCTURE ONLY -- see `oracle/__init__.py`.  The product package
never imports this module.

This is an independent restatement of the reference algorithm, written to
reproduce its floating-point operation order wherever the reference is
deterministic (gather -> dgemm -> scale -> corner-ordered scatter, axis-pass
transfers, in-place Jacobi updates, the PCG recurrences).  Each function
cites the reference location it restates (paths relative to
`/root/reference/pkg/src/voxtop/`).  It is pinned against the real reference
by `tests/test_oracle_golden.py` using fixtures made by `make_golden.py`.

Conventions (grid.py:1-10): node (i,j,k) -> i + j(nx+1) + k(nx+1)(ny+1),
dof = 3*node + comp, element arrays viewed (nz, ny, nx), node arrays viewed
(nz+1, ny+1, nx+1, 3); element corner c sits at (c&1, c>>1&1, c>>2&1).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np
import scipy.linalg
from scipy import ndimage

OFFS = np.array([[c & 1, (c >> 1) & 1, (c >> 2) & 1] for c in range(8)], np.int64)


class OracleError(Exception):
    """Base of the oracle's error kinds (mirrors errors.py:7-24 by `kind`)."""

    def __init__(self, kind: str, msg: str):
        super().__init__(msg)
        self.kind = kind


# --------------------------------------------------------------------------
# element (element.py:23-118)

_VV = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
_GG = np.array([[1.0, -1.0], [-1.0, 1.0]])
_GV = np.array([[-0.5, -0.5], [0.5, 0.5]])


def hex8_k0(nu: float, h: float) -> np.ndarray:
    """Unit-modulus hex8 stiffness, closed form (element.py:61-99).

    Block (a,b) over corner pairs is lam*G[a,b] + mu*G[b,a] (+ mu*trace on
    a == b) where G[a,b] = h * kron(T_z, kron(T_y, T_x)), T chosen per axis
    from the 1-D integral tables.
    """
    lam = nu / ((1 + nu) * (1 - 2 * nu))
    mu = 1.0 / (2 * (1 + nu))

    def table(ax, a, b):
        ga, gb = ax == a, ax == b
        if ga and gb:
            return _GG
        if ga:
            return _GV
        if gb:
            return _GV.T.copy()
        return _VV

    G = np.empty((3, 3, 8, 8))
    for a in range(3):
        for b in range(3):
            G[a, b] = np.kron(table(2, a, b), np.kron(table(1, a, b), table(0, a, b))) * h
    tr = G[0, 0] + G[1, 1] + G[2, 2]
    K = np.zeros((24, 24))
    for a in range(3):
        for b in range(3):
            blk = lam * G[a, b] + mu * G[b, a]
            if a == b:
                blk = blk + mu * tr
            K[a::3, b::3] = blk
    return K


def simp(rho, p: float, kmin: float):
    """s = kmin + rho**p (1-kmin)  (element.py:102-108)."""
    r = np.asarray(rho, dtype=np.float64)
    if np.any(r < 0) or np.any(r > 1):
        raise OracleError("value", "density outside [0, 1]")
    return kmin + r**p * (1.0 - kmin)


def simp_deriv(rho, p: float, kmin: float):
    """ds/drho (element.py:111-118)."""
    r = np.asarray(rho, dtype=np.float64)
    return p * r ** (p - 1.0) * (1.0 - kmin)


def gravity_unit(g: float, h: float, uw: float, axis: int) -> np.ndarray:
    """Self-weight of a unit-density element, lumped to its corners (element.py:121-133)."""
    f = np.zeros(24)
    f[axis::3] = -1.0 * uw * g * h**3 / 8.0
    return f


# --------------------------------------------------------------------------
# matrix-free operator (operator.py:31-105, 187-205)


def _corner(arr, c, es):
    i, j, k = OFFS[c]
    nz, ny, nx = es
    return arr[k : k + nz, j : j + ny, i : i + nx]


def gather(u, es):
    nz, ny, nx = es
    u4 = u.reshape(nz + 1, ny + 1, nx + 1, 3)
    out = np.empty((nz, ny, nx, 24))
    for c in range(8):
        out[..., 3 * c : 3 * c + 3] = _corner(u4, c, es)
    return out.reshape(-1, 24)


def scatter(ve, es):
    nz, ny, nx = es
    acc = np.zeros((nz + 1, ny + 1, nx + 1, 3))
    v4 = ve.reshape(nz, ny, nx, 24)
    for c in range(8):  # corner order fixes the summation order (operator.py:53-54)
        _corner(acc, c, es)[...] += v4[..., 3 * c : 3 * c + 3]
    return acc.reshape(-1)


def apply_k(u, es, fixed_idx, k0, scale):
    """v = K u, identity on fixed dofs (operator.py:58-81)."""
    w = u.copy()
    w[fixed_idx] = 0.0
    ve = gather(w, es) @ k0
    ve *= scale[:, None]
    v = scatter(ve, es)
    v[fixed_idx] = u[fixed_idx]
    return v


def diag_k(es, fixed_idx, k0, scale):
    """Operator diagonal, 1 on fixed (operator.py:84-105)."""
    nz, ny, nx = es
    acc = np.zeros((nz + 1, ny + 1, nx + 1, 3))
    kd = np.diag(k0)
    for c in range(8):
        blk = scale[:, None] * kd[None, 3 * c : 3 * c + 3]
        _corner(acc, c, es)[...] += blk.reshape(nz, ny, nx, 3)
    d = acc.reshape(-1)
    d[fixed_idx] = 1.0
    return d


def resid_k(u, f, es, fixed_idx, k0, scale):
    r = f - apply_k(u, es, fixed_idx, k0, scale)
    r[fixed_idx] = 0.0
    return r


def dof_table(es):
    """(nel, 24) dof ids (grid.py:128-139)."""
    nz, ny, nx = es
    k, j, i = np.indices(es)
    i, j, k = i.ravel(), j.ravel(), k.ravel()
    nodes = (i[:, None] + OFFS[None, :, 0]) + (j[:, None] + OFFS[None, :, 1]) * (nx + 1) + (
        k[:, None] + OFFS[None, :, 2]
    ) * (nx + 1) * (ny + 1)
    return (3 * nodes[:, :, None] + np.arange(3)[None, None, :]).reshape(-1, 24)


def dense_k(es, fixed_idx, k0, scale):
    """Explicit matrix with identity rows/cols on fixed dofs (operator.py:187-205)."""
    nz, ny, nx = es
    n = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    ed = dof_table(es)
    K = np.zeros((n, n))
    np.add.at(K, (ed[:, :, None], ed[:, None, :]), scale[:, None, None] * k0[None])
    K[fixed_idx, :] = 0.0
    K[:, fixed_idx] = 0.0
    K[fixed_idx, fixed_idx] = 1.0
    return K


# --------------------------------------------------------------------------
# homogenized geometric multigrid (multigrid.py:84-499)


def feasible_levels(nx, ny, nz) -> int:
    """multigrid.py:84-91."""
    L, d = 1, [nx, ny, nz]
    while all(x % 2 == 0 and x // 2 >= 2 for x in d):
        d = [x // 2 for x in d]
        L += 1
    return L


def octant_mean(rho, coarse_es):
    """Mean of the 8 children, octant index = child corner index (multigrid.py:94-104)."""
    cz, cy, cx = coarse_es
    a = rho.reshape(cz, 2, cy, 2, cx, 2)
    a = np.moveaxis(a, (1, 3, 5), (3, 4, 5)).reshape(cz * cy * cx, 8)
    return a.mean(axis=1)


def coarsen_fixed(mask, es):
    nz, ny, nx = es
    return mask.reshape(nz + 1, ny + 1, nx + 1, 3)[::2, ::2, ::2, :].reshape(-1).copy()


@dataclass
class Lvl:
    es: tuple
    h: float
    mask: np.ndarray
    fixed: np.ndarray
    k0: Optional[np.ndarray] = None
    scale: Optional[np.ndarray] = None
    mats: Optional[np.ndarray] = None  # galerkin coarse levels (nel, 24, 24)
    diag: Optional[np.ndarray] = None
    u: Optional[np.ndarray] = None
    f: Optional[np.ndarray] = None
    r: Optional[np.ndarray] = None
    tmp: Optional[np.ndarray] = None

    @property
    def n(self):
        nz, ny, nx = self.es
        return 3 * (nx + 1) * (ny + 1) * (nz + 1)


@dataclass
class Hier:
    levels: List[Lvl]
    omega: float
    sweeps: int
    chol: object = None
    scheme: str = "homogenized"
    gstack: Optional[np.ndarray] = None   # galerkin: W_c^T K0 W_c, c = 0..7
    aff: Optional[tuple] = None           # galerkin: (coarse elem, octant, correction)

    @property
    def vector_scalars(self):
        return sum(5 * lv.n for lv in self.levels)


# ---- Galerkin scheme (multigrid.py:59-81, 216-278)
def octant_weights(c: int) -> np.ndarray:
    """Trilinear weights of the 8 coarse corners at the fine corners of octant c
    (multigrid.py:59-70)."""
    off = np.array([[x & 1, (x >> 1) & 1, (x >> 2) & 1] for x in range(8)], dtype=np.float64)
    T = np.ones((8, 8))
    for a in range(8):
        pos = (off[c] + off[a]) / 2.0
        for b in range(8):
            w = 1.0
            for d in range(3):
                w *= pos[d] if off[b][d] else 1.0 - pos[d]
            T[a, b] = w
    return T


GAL_W = np.zeros((8, 24, 24))
for _c in range(8):
    _T = octant_weights(_c)
    for _ax in range(3):
        GAL_W[_c, _ax::3, _ax::3] = _T
del _c, _T, _ax


def octant_groups(arr, coarse_es, trailing=()):
    """(nel_coarse, 8, *trailing), octant = child corner index (multigrid.py:94-104)."""
    cz, cy, cx = coarse_es
    a = arr.reshape(cz, 2, cy, 2, cx, 2, *trailing)
    a = np.moveaxis(a, (1, 3, 5), (3, 4, 5))
    return a.reshape(cz * cy * cx, 8, *trailing)


def free24(mask, es):
    """(nel, 24) float mask: 1 on free local dofs (multigrid.py:144-147)."""
    return gather((~np.asarray(mask, bool)).astype(np.float64), es)


def galerkin_setup(H: "Hier", k0):
    """Static data: G_c = W_c^T K0 W_c and the fine fixed-dof corrections
    s_e W_c^T (K0 o mm^T - K0) W_c of elements touching a fixed dof
    (multigrid.py:216-223, 235-260)."""
    H.gstack = np.stack([GAL_W[c].T @ k0 @ GAL_W[c] for c in range(8)])
    fine, coarse = H.levels[0], H.levels[1]
    groups = octant_groups(free24(fine.mask, fine.es), coarse.es, (24,))
    pairs = np.argwhere(groups.min(axis=2) < 0.5)
    if pairs.size == 0:
        H.aff = None
        return
    E, C = pairs[:, 0], pairs[:, 1]
    m = groups[E, C]
    delta = k0[None, :, :] * (m[:, :, None] * m[:, None, :]) - k0[None, :, :]
    H.aff = (E, C, np.matmul(np.swapaxes(GAL_W[C], 1, 2), np.matmul(delta, GAL_W[C])))


def galerkin_level1(H: "Hier", scale0):
    """Level-1 element matrices sum_c s_c G_c (+ corrections) (multigrid.py:262-270)."""
    s_oct = octant_groups(scale0, H.levels[1].es)
    KE = (s_oct @ H.gstack.reshape(8, 576)).reshape(-1, 24, 24)
    if H.aff is not None:
        E, C, corr = H.aff
        np.add.at(KE, E, s_oct[E, C][:, None, None] * corr)
    return KE


def galerkin_coarsen(lv: Lvl, coarse_es):
    """sum_c W_c^T (K_child o mm^T) W_c (multigrid.py:272-278)."""
    m = free24(lv.mask, lv.es)
    kproj = lv.mats * (m[:, :, None] * m[:, None, :])
    groups = octant_groups(kproj, coarse_es, (24, 24))
    KE = np.zeros((groups.shape[0], 24, 24))
    for c in range(8):
        KE += np.matmul(GAL_W[c].T, np.matmul(groups[:, c], GAL_W[c]))
    return KE


def apply_mats(u, es, fixed_idx, mats):
    """operator.py:58-81 with elem_matrices."""
    uw = u.copy()
    uw[fixed_idx] = 0.0
    ve = np.matmul(mats, gather(uw, es)[:, :, None])[:, :, 0]
    out = scatter(ve, es)
    out[fixed_idx] = u[fixed_idx]
    return out


def diag_mats(es, fixed_idx, mats):
    """operator.py:84-105 with elem_matrices."""
    nz, ny, nx = es
    out = np.zeros((nz + 1, ny + 1, nx + 1, 3))
    ediag = np.einsum("eii->ei", mats).reshape(nz, ny, nx, 24)
    for c in range(8):
        _corner(out, c, es)[...] += ediag[..., 3 * c:3 * c + 3]
    d = out.reshape(-1)
    d[fixed_idx] = 1.0
    return d


def dense_mats(es, fixed_idx, mats):
    nz, ny, nx = es
    n = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    edofs = dof_table(es)
    K = np.zeros((n, n))
    np.add.at(K, (edofs[:, :, None], edofs[:, None, :]), mats)
    K[fixed_idx, :] = 0.0
    K[:, fixed_idx] = 0.0
    K[fixed_idx, fixed_idx] = 1.0
    return K


def hier_build(es, h, fixed_mask, max_levels, omega=0.4, sweeps=1, scheme="homogenized") -> Hier:
    """Level grids and masks (multigrid.py:462-499)."""
    nz, ny, nx = es
    L = min(int(max_levels), feasible_levels(nx, ny, nz))
    lv, mask, cur, hh = [], np.asarray(fixed_mask, bool), tuple(es), h
    for l in range(L):
        lv.append(Lvl(cur, hh, mask, np.flatnonzero(mask)))
        if l < L - 1:
            mask = coarsen_fixed(mask, cur)
            cur = tuple(x // 2 for x in cur)
            hh = hh * 2
    for x in lv:
        x.u, x.f, x.r, x.tmp = (np.zeros(x.n) for _ in range(4))
    return Hier(lv, float(omega), int(sweeps), scheme=scheme)


def hier_refresh(H: Hier, rho, scale0, k0, p, kmin, E):
    """Homogenized / Galerkin refresh (multigrid.py:201-233) + coarsest factor (280-316)."""
    H.levels[0].scale = scale0
    H.levels[0].k0 = k0
    if H.scheme == "homogenized":
        r = rho
        for l in range(1, len(H.levels)):
            lv = H.levels[l]
            r = octant_mean(r, lv.es)
            lv.scale = E * simp(r, p, kmin)
            lv.k0 = k0 * float(2**l)
    elif len(H.levels) > 1:
        if H.gstack is None:
            galerkin_setup(H, k0)
        H.levels[1].mats = galerkin_level1(H, scale0)
        for l in range(1, len(H.levels) - 1):
            H.levels[l + 1].mats = galerkin_coarsen(H.levels[l], H.levels[l + 1].es)
    for lv in H.levels:
        lv.diag = diag_mats(lv.es, lv.fixed, lv.mats) if lv.mats is not None else \
            diag_k(lv.es, lv.fixed, lv.k0, lv.scale)
    last = H.levels[-1]
    if last.n > 20_000:
        raise OracleError("setup", f"coarsest level has {last.n} dofs")
    if H.scheme == "homogenized" and len(H.levels) > 1 and last.fixed.size < 6:
        raise OracleError("setup", f"only {last.fixed.size} fixed dofs survive")
    K = dense_mats(last.es, last.fixed, last.mats) if last.mats is not None else \
        dense_k(last.es, last.fixed, last.k0, last.scale)
    try:
        H.chol = scipy.linalg.cho_factor(K, lower=True)
    except scipy.linalg.LinAlgError as exc:
        raise OracleError("setup", "coarsest matrix not SPD") from exc
    piv = np.abs(np.diag(H.chol[0]))
    if not np.all(np.isfinite(piv)) or piv.min() == 0.0:
        raise OracleError("setup", "zero pivot")


def _interp1(a, axis):
    src = np.moveaxis(a, axis, 0)
    shp = list(a.shape)
    shp[axis] = 2 * a.shape[axis] - 1
    out = np.zeros(shp)
    dst = np.moveaxis(out, axis, 0)
    dst[0::2] = src
    dst[1::2] = 0.5 * (src[:-1] + src[1:])
    return out


def _restrict1(a, axis):
    src = np.moveaxis(a, axis, 0)
    shp = list(a.shape)
    shp[axis] = (a.shape[axis] - 1) // 2 + 1
    out = np.zeros(shp)
    dst = np.moveaxis(out, axis, 0)
    dst[:] = src[0::2]
    odd = src[1::2]
    dst[:-1] += 0.5 * odd
    dst[1:] += 0.5 * odd
    return out


def prolong(H: Hier, l: int, ec):
    """Trilinear interpolation level l+1 -> l, axis passes z, y, x (multigrid.py:341-354)."""
    cz, cy, cx = H.levels[l + 1].es
    a = ec.reshape(cz + 1, cy + 1, cx + 1, 3)
    for ax in (0, 1, 2):
        a = _interp1(a, ax)
    out = a.reshape(-1)
    out[H.levels[l].fixed] = 0.0
    return out


def restrict(H: Hier, l: int, rf):
    """Transpose of prolong (multigrid.py:356-371)."""
    nz, ny, nx = H.levels[l].es
    a = rf.copy()
    a[H.levels[l].fixed] = 0.0
    a = a.reshape(nz + 1, ny + 1, nx + 1, 3)
    for ax in (0, 1, 2):
        a = _restrict1(a, ax)
    out = a.reshape(-1)
    out[H.levels[l + 1].fixed] = 0.0
    return out


def level_apply(H: Hier, l: int, u):
    lv = H.levels[l]
    if lv.mats is not None:
        return apply_mats(u, lv.es, lv.fixed, lv.mats)
    return apply_k(u, lv.es, lv.fixed, lv.k0, lv.scale)


def _smooth(H: Hier, l: int, sweeps: int):
    """In-place damped Jacobi (multigrid.py:387-393)."""
    lv = H.levels[l]
    for _ in range(sweeps):
        np.subtract(lv.f, level_apply(H, l, lv.u), out=lv.r)
        lv.r[lv.fixed] = 0.0
        np.divide(lv.r, lv.diag, out=lv.tmp)
        lv.u += H.omega * lv.tmp


def jacobi(H: Hier, l: int, u, f, sweeps: int):
    """Out-of-place Jacobi sweeps (multigrid.py:375-385)."""
    lv = H.levels[l]
    u = np.array(u, dtype=np.float64)
    for _ in range(sweeps):
        r = f - level_apply(H, l, u)
        r[lv.fixed] = 0.0
        u += H.omega * r / lv.diag
    return u


def coarse_solve(H: Hier, f):
    return scipy.linalg.cho_solve(H.chol, f)


def _cycle(H: Hier, l: int):
    lv = H.levels[l]
    if l == len(H.levels) - 1:
        lv.u[:] = coarse_solve(H, lv.f)
        return
    lv.u[:] = 0.0
    _smooth(H, l, H.sweeps)
    np.subtract(lv.f, level_apply(H, l, lv.u), out=lv.r)
    lv.r[lv.fixed] = 0.0
    H.levels[l + 1].f[:] = restrict(H, l, lv.r)
    _cycle(H, l + 1)
    lv.u += prolong(H, l, H.levels[l + 1].u)
    _smooth(H, l, H.sweeps)


def vcycle(H: Hier, f):
    """One V(ν,ν) cycle from zero (multigrid.py:404-430)."""
    fine = H.levels[0]
    fine.f[:] = f
    fine.f[fine.fixed] = 0.0
    _cycle(H, 0)
    return fine.u.copy()


# --------------------------------------------------------------------------
# PCG (solver.py:62-191)


@dataclass
class Report:
    iterations: int = 0
    final_rel_residual: float = 0.0
    precond_applications: int = 0
    wall_s: float = 0.0
    converged: bool = False
    aux_vector_scalars: int = 0
    residual_drift: float = 0.0


def pcg(apply, residual, precond, f, u0, fixed_idx, tol=1e-5, maxit=200):
    """Restates solver.py:62-167 step for step (same recurrences, same checks)."""
    t0 = time.perf_counter()
    n = f.shape[0]
    if not np.all(np.isfinite(f)):
        raise OracleError("breakdown", "rhs contains non-finite entries")
    rep = Report(aux_vector_scalars=4 * n)
    x = np.zeros(n) if u0 is None else np.array(u0, dtype=np.float64)
    if u0 is not None:
        x[fixed_idx] = 0.0
    fn = float(np.linalg.norm(f))
    if fn == 0.0:
        rep.converged = True
        rep.wall_s = time.perf_counter() - t0
        return x, rep
    r = residual(x, f)
    rel = float(np.linalg.norm(r)) / fn
    if rel <= tol:
        rep.converged, rep.final_rel_residual = True, rel
        rep.wall_s = time.perf_counter() - t0
        return x, rep

    def M(v):
        if precond is None:
            return v.copy()
        rep.precond_applications += 1
        return precond(v)

    z = M(r)
    p = z.copy()
    rz = float(r @ z)
    if not np.isfinite(rz) or rz <= 0.0:
        raise OracleError("breakdown", f"r'z = {rz} at iteration 0")
    k = 0
    while k < maxit:
        k += 1
        q = apply(p)
        pq = float(p @ q)
        if not np.isfinite(pq):
            raise OracleError("breakdown", f"non-finite curvature at iteration {k}")
        if pq <= 0.0:
            raise OracleError("breakdown", f"p'Kp = {pq} at iteration {k}")
        a = rz / pq
        x += a * p
        if k % 50 == 0:
            r = residual(x, f)
        else:
            r -= a * q
        rel = float(np.linalg.norm(r)) / fn
        if not np.isfinite(rel):
            raise OracleError("breakdown", f"non-finite residual at iteration {k}")
        if rel <= tol:
            tr = residual(x, f)
            trel = float(np.linalg.norm(tr)) / fn
            rep.residual_drift = abs(trel - rel) / max(trel, 1e-300)
            if trel <= tol:
                rep.converged = True
                rel = trel
                break
            r, rel = tr, trel
        z = M(r)
        rzn = float(r @ z)
        if not np.isfinite(rzn) or rzn <= 0.0:
            raise OracleError("breakdown", f"r'z = {rzn} at iteration {k}")
        p = z + (rzn / rz) * p
        rz = rzn
    if not rep.converged:
        rel = float(np.linalg.norm(residual(x, f))) / fn
    rep.iterations = k
    rep.final_rel_residual = rel
    rep.converged = rel <= tol
    rep.wall_s = time.perf_counter() - t0
    return x, rep


# --------------------------------------------------------------------------
# design-loop kernels (optimize.py:139-302)


def filter_kernel(h: float, radius: float):
    """Conic kernel r - dist over the (2R+1)^3 box, index order (dk,dj,di) (optimize.py:147-171)."""
    R = int(np.floor(radius / h + 1e-12))
    o = np.arange(-R, R + 1)
    dk, dj, di = np.meshgrid(o, o, o, indexing="ij")
    dist = h * np.sqrt(di**2 + dj**2 + dk**2)
    keep = dist <= radius + 1e-12 * radius
    return np.where(keep, radius - dist, 0.0)


def correlate0(field, kernel, es):
    return ndimage.correlate(field.reshape(es), kernel, mode="constant", cval=0.0).reshape(-1)


def filter_sens(dc, rho, kernel, wsum, gamma, es):
    """dcf = corr(rho*dc) / (max(gamma, rho) * wsum) (optimize.py:174-179)."""
    return correlate0(rho * dc, kernel, es) / (np.maximum(gamma, rho) * wsum)


def sensitivities(u, rho, es, k0, p, kmin, E, grav_unit=None):
    """-E s'(rho) u_e'K0 u_e (+ 2 u_e.g) (optimize.py:195-213)."""
    ue = gather(np.asarray(u, dtype=np.float64), es)
    quad = np.einsum("eb,eb->e", ue @ k0, ue)
    dc = -(E * simp_deriv(rho, p, kmin)) * quad
    if grav_unit is not None:
        dc += 2.0 * ue @ grav_unit
    return dc


def gravity_load(rho, es, grav_unit, f_ext=None, fixed_idx=None):
    """optimize.py:216-231."""
    f = scatter(rho[:, None] * grav_unit[None, :], es)
    if f_ext is not None:
        f = f + f_ext
    if fixed_idx is not None:
        f[fixed_idx] = 0.0
    return f


def oc_update(x_all, active, dc, dv, volfrac, move=0.2, eta=0.5, q=1.0):
    """OC with bisected multiplier (optimize.py:245-302). Returns (rho, lam, steps)."""
    x = x_all[active]
    numer = np.maximum(-dc[active], 0.0)
    dva = dv[active]
    lo = np.maximum(0.0, x - move)
    hi = np.minimum(1.0, x + move)

    def cand(lam):
        b = numer / (lam * dva)
        c = x * b**eta
        if q != 1.0:
            c = c**q
        return np.clip(c, lo, hi)

    if lo.mean() > volfrac + 1e-6 or hi.mean() < volfrac - 1e-6:
        raise OracleError("volume", "volume target unreachable within the move limits")
    l1, l2 = 0.0, 1e9
    for _ in range(200):
        if cand(l2).mean() <= volfrac:
            break
        l2 *= 16.0
    lam = 0.5 * (l1 + l2)
    steps = 0
    xn = cand(lam)
    while abs(xn.mean() - volfrac) > 1e-6:
        steps += 1
        if steps > 200:
            raise OracleError("volume", "bisection failed after 200 halvings")
        if xn.mean() > volfrac:
            l1 = lam
        else:
            l2 = lam
        lam = 0.5 * (l1 + l2)
        xn = cand(lam)
    out = x_all.copy()
    out[active] = xn
    return out, lam, steps


# --------------------------------------------------------------------------
# problem recipes (app/presets.py:48-139) and the design loop (optimize.py:344-455)


@dataclass
class Case:
    """Everything the design loop needs, as plain arrays."""

    nx: int
    ny: int
    nz: int
    h: float
    fixed_mask: np.ndarray
    f_ext: np.ndarray
    classes: np.ndarray  # int8 per element: 0 active, 1 solid, 2 void
    p: float = 3.0
    kmin: float = 1e-9
    E: float = 1.0
    nu: float = 0.3
    gravity: Optional[tuple] = None  # (axis, g, unit_weight)

    @property
    def es(self):
        return (self.nz, self.ny, self.nx)


def _node(nx, ny, i, j, k):
    return i + j * (nx + 1) + k * (nx + 1) * (ny + 1)


def _ends_half(n):
    w = np.ones(n)
    w[0] = w[-1] = 0.5
    return w


def cantilever_case(nx, ny, nz, L=64.0, gravity=None) -> Case:
    """Fixed x=0 face; -z line load -1/length along y at (i=nx, k=0) (presets.py:125-130)."""
    h = L / nx
    n = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    mask = np.zeros(n, bool)
    for k in range(nz + 1):
        for j in range(ny + 1):
            nd = _node(nx, ny, 0, j, k)
            mask[3 * nd : 3 * nd + 3] = True
    f = np.zeros(n)
    w = _ends_half(ny + 1)
    for j in range(ny + 1):
        f[3 * _node(nx, ny, nx, j, 0) + 2] += -1.0 * h * w[j]
    return Case(nx, ny, nz, h, mask, f, np.zeros(nx * ny * nz, np.int8), gravity=gravity)


def bridge_case(nx, ny, nz, L=64.0) -> Case:
    """SURVEY §8(d) cfg3 recipe: 4 bottom-corner supports, -100 top pressure,
    one passive-solid deck layer (presets.py:71-90, 133-139)."""
    h = L / nx
    n = 3 * (nx + 1) * (ny + 1) * (nz + 1)
    mask = np.zeros(n, bool)
    for i, j in ((0, 0), (nx, 0), (0, ny), (nx, ny)):
        nd = _node(nx, ny, i, j, 0)
        mask[3 * nd : 3 * nd + 3] = True
    f = np.zeros(n)
    wx, wy = _ends_half(nx + 1), _ends_half(ny + 1)
    for i in range(nx + 1):
        for j in range(ny + 1):
            f[3 * _node(nx, ny, i, j, nz) + 2] += -100.0 * h**2 * (wx[i] * wy[j])
    cls = np.zeros((nz, ny, nx), np.int8)
    cls[nz - 1] = 1
    return Case(nx, ny, nz, h, mask, f, cls.reshape(-1))


@dataclass
class Rec:
    iteration: int
    compliance: float
    volume: float
    change: float
    cg_iters: int
    cg_residual: float
    wall_s: float
    aux_scalars: int


def run_design(case: Case, volfrac, rmin, iters, tol=1e-5, maxit=200, max_levels=None,
               omega=0.4, ch_tol=0.01, move=0.2, eta=0.5, q=1.0, gamma=1e-3,
               rho0=None, u0=None, on_iter: Optional[Callable] = None, scheme="homogenized",
               p_continuation=False, obj_tol=None):
    """SIMP loop of optimize.py:344-455 with MGPCG (homogenized or galerkin);
    p_continuation ramps p = min(p, 1 + 0.5 (it // 15)) (optimize.py:78-82),
    obj_tol adds the compliance-change stop test (optimize.py:448-453)."""
    es = case.es
    k0 = hex8_k0(case.nu, case.h)
    fixed = np.flatnonzero(case.fixed_mask)
    f_ext = case.f_ext.copy()
    f_ext[fixed] = 0.0
    kern = filter_kernel(case.h, rmin)
    wsum = correlate0(np.ones(case.nx * case.ny * case.nz), kern, es)
    nel = case.nx * case.ny * case.nz
    dv = np.ones(nel)
    act = case.classes == 0
    if rho0 is None:
        rho = np.full(nel, volfrac)
        rho[case.classes == 1] = 1.0
        rho[case.classes == 2] = 0.0
    else:
        rho = np.array(rho0, dtype=np.float64)
    u = np.zeros(3 * (case.nx + 1) * (case.ny + 1) * (case.nz + 1)) if u0 is None else np.array(u0)
    if max_levels is None:
        max_levels = feasible_levels(case.nx, case.ny, case.nz)
    grav = None
    if case.gravity is not None:
        ax, g, uw = case.gravity
        grav = gravity_unit(g, case.h, uw, ax)
    H = None
    recs = []
    for it in range(iters):
        t0 = time.perf_counter()
        p_it = min(case.p, 1.0 + 0.5 * (it // 15)) if p_continuation else case.p
        scale = case.E * simp(rho, p_it, case.kmin)
        f = gravity_load(rho, es, grav, f_ext, fixed) if grav is not None else f_ext
        if H is None:
            H = hier_build(es, case.h, case.fixed_mask, max_levels, omega, scheme=scheme)
        hier_refresh(H, rho, scale, k0, p_it, case.kmin, case.E)
        n = f.shape[0]
        budget = 4 * n + H.vector_scalars
        if budget > 10.5 * n:
            raise OracleError("breakdown", "aux budget")
        ap = lambda v: apply_k(v, es, fixed, k0, scale)
        rs = lambda v, ff: resid_k(v, ff, es, fixed, k0, scale)
        u, rep = pcg(ap, rs, lambda r: vcycle(H, r), f, u, fixed, tol, maxit)
        c = float(f @ u)
        dc = sensitivities(u, rho, es, k0, p_it, case.kmin, case.E, grav)
        dcf = filter_sens(dc, rho, kern, wsum, gamma, es)
        new, lam, steps = oc_update(rho, act, dcf, dv, volfrac, move, eta, q)
        ch = float(np.abs(new - rho).max())
        rho = new
        vol = float(rho[act].mean())
        if abs(vol - volfrac) > 1e-6:
            raise OracleError("numerical", "volume constraint violated")
        rec = Rec(it + 1, c, vol, ch, rep.iterations, rep.final_rel_residual,
                  time.perf_counter() - t0, budget)
        recs.append(rec)
        if on_iter is not None:
            on_iter(rec, rho, u)
        obj_ok = obj_tol is None or len(recs) < 2 or abs(recs[-1].compliance - recs[-2].compliance) <= obj_tol
        if ch <= ch_tol and obj_ok:
            break
    return rho, u, recs


# --------------------------------------------------------------------------
# two-material SIMP (BASELINE cfg4).  NO reference counterpart: the
# reference's SPEC.md:15,178 lists multi-material design as never developed.
# This extends simp_scale / simp_scale_derivative (element.py:102-118),
# sensitivities (optimize.py:195-213) and the loop (optimize.py:344-455) with
# a second design field phi (share of the stiff phase A in the material):
#   modulus  E s(rho) m(phi),  m = eB + (1 - eB) phi^p,  eB = E_B / E_A
#   dc_rho = -E s'(rho) m(phi) q_e,   dc_phi = -E s(rho) p phi^(p-1) (1-eB) q_e
# with q_e = u_e'K0u_e; both sensitivities go through the reference filter
# (phi as the filter weight of dc_phi) and the reference OC update with their
# own volume targets (mean rho = volfrac, mean phi = phase_frac over the
# active elements).  Parity is UNPINNED against the reference except through
# the eB = 1 limit, where m = 1 exactly and the rho trajectory is the
# single-material one bit for bit (phi is then inert and not updated).


def two_material_factor(phi, p: float, eB: float):
    y = np.asarray(phi, dtype=np.float64)
    if np.any(y < 0) or np.any(y > 1):
        raise OracleError("value", "phase fraction outside [0, 1]")
    return eB + (1.0 - eB) * y**p


def two_material_scale(rho, phi, p, kmin, E, eB):
    return (E * simp(rho, p, kmin)) * two_material_factor(phi, p, eB)


def sensitivities_two_material(u, rho, phi, es, k0, p, kmin, E, eB, grav_unit=None):
    ue = gather(np.asarray(u, dtype=np.float64), es)
    quad = np.einsum("eb,eb->e", ue @ k0, ue)
    m = two_material_factor(phi, p, eB)
    dc_rho = -((E * simp_deriv(rho, p, kmin)) * m) * quad
    if grav_unit is not None:
        dc_rho += 2.0 * ue @ grav_unit
    dm = p * np.asarray(phi, dtype=np.float64) ** (p - 1.0) * (1.0 - eB)
    dc_phi = -((E * simp(rho, p, kmin)) * dm) * quad
    return dc_rho, dc_phi


def run_design_two_material(case: Case, volfrac, phase_frac, eB, rmin, iters, tol=1e-5, maxit=200,
                            max_levels=None, omega=0.4, ch_tol=0.01, move=0.2, eta=0.5, q=1.0,
                            gamma=1e-3, scheme="galerkin"):
    """Two-material SIMP loop; returns (rho, phi, u, records) with records
    (iteration, compliance, volume, phase_volume, change, cg_iters)."""
    es = case.es
    k0 = hex8_k0(case.nu, case.h)
    fixed = np.flatnonzero(case.fixed_mask)
    f_ext = case.f_ext.copy()
    f_ext[fixed] = 0.0
    kern = filter_kernel(case.h, rmin)
    wsum = correlate0(np.ones(case.nx * case.ny * case.nz), kern, es)
    nel = case.nx * case.ny * case.nz
    dv = np.ones(nel)
    act = case.classes == 0
    rho = np.full(nel, volfrac)
    rho[case.classes == 1] = 1.0
    rho[case.classes == 2] = 0.0
    phi = np.full(nel, phase_frac)
    phi[case.classes != 0] = 1.0
    u = np.zeros(3 * (case.nx + 1) * (case.ny + 1) * (case.nz + 1))
    if max_levels is None:
        max_levels = feasible_levels(case.nx, case.ny, case.nz)
    grav = None
    if case.gravity is not None:
        ax, g, uw = case.gravity
        grav = gravity_unit(g, case.h, uw, ax)
    H = None
    recs = []
    for it in range(iters):
        m = two_material_factor(phi, case.p, eB)
        scale = (case.E * simp(rho, case.p, case.kmin)) * m
        rho_mg = np.minimum(1.0, rho * m ** (1.0 / case.p))
        f = gravity_load(rho, es, grav, f_ext, fixed) if grav is not None else f_ext
        if H is None:
            H = hier_build(es, case.h, case.fixed_mask, max_levels, omega, scheme=scheme)
        hier_refresh(H, rho_mg, scale, k0, case.p, case.kmin, case.E)
        ap = lambda v: apply_k(v, es, fixed, k0, scale)
        rs = lambda v, ff: resid_k(v, ff, es, fixed, k0, scale)
        u, rep = pcg(ap, rs, lambda r: vcycle(H, r), f, u, fixed, tol, maxit)
        c = float(f @ u)
        dcr, dcp = sensitivities_two_material(u, rho, phi, es, k0, case.p, case.kmin, case.E, eB, grav)
        dcr_f = filter_sens(dcr, rho, kern, wsum, gamma, es)
        new_rho, _, _ = oc_update(rho, act, dcr_f, dv, volfrac, move, eta, q)
        ch = float(np.abs(new_rho - rho).max())
        if eB != 1.0:
            dcp_f = filter_sens(dcp, phi, kern, wsum, gamma, es)
            new_phi, _, _ = oc_update(phi, act, dcp_f, dv, phase_frac, move, eta, q)
            ch = max(ch, float(np.abs(new_phi - phi).max()))
            phi = new_phi
        rho = new_rho
        recs.append((it + 1, c, float(rho[act].mean()), float(phi[act].mean()), ch, rep.iterations))
        if ch <= ch_tol:
            break
    return rho, phi, u, recs
