"""Geometric multigrid on the device -- drop-in for multigrid.py:84-499 of
the reference, both coarse-operator schemes:

  * "galerkin" (the reference default): per-element 24x24 coarse matrices
    P^T K P with the fixed-dof projection, assembled on the device from the
    fine scales (level 1) and from the level below (csrc/galerkin.cu);
  * "homogenized": coarse operators rebuilt on the fly from averaged densities
    (E*s(mean rho) * K0(h*2^l)).

Transfers, damped Jacobi and the V-cycle run as sm_100a kernels, the
coarsest level is factored and inverted on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np
import torch

from ._lib import check, lib
from .device import DeviceGrid, DeviceVector, ptr, stream_ptr
from .errors import SetupError
from .mesh import StructuredGrid
from .stiffness_op import OperatorState, as_device, from_device

__all__ = ["MgHierarchy", "build_hierarchy", "max_feasible_levels", "SCHEMES"]

SCHEMES = ("galerkin", "homogenized")
COARSE_GUARD_DOFS = 20_000
COARSEST_MIN_ELEMS = 2


def max_feasible_levels(nelx: int, nely: int, nelz: int) -> int:
    """Halve while every dimension is even and stays >= 2 (multigrid.py:84-91)."""
    L, d = 1, (nelx, nely, nelz)
    while all(x % 2 == 0 and x // 2 >= COARSEST_MIN_ELEMS for x in d):
        d = tuple(x // 2 for x in d)
        L += 1
    return L


def _coarsen_mask(mask: np.ndarray, grid: StructuredGrid) -> np.ndarray:
    nz, ny, nx = grid.elem_shape
    return np.ascontiguousarray(mask.reshape(nz + 1, ny + 1, nx + 1, 3)[::2, ::2, ::2].reshape(-1))


@dataclass
class _Level:
    grid: StructuredGrid
    fixed_mask: np.ndarray
    fixed_idx: np.ndarray
    dgrid: DeviceGrid
    hier: "MgHierarchy"
    index: int

    @property
    def n_dofs(self):
        return self.grid.n_dofs

    @property
    def scale(self) -> np.ndarray:
        d = self.dgrid
        n = d.elem_len
        t = torch.empty(n, dtype=torch.float64, device=f"cuda:{d.device}")
        src = lib.vt_hier_level_scale(self.hier._h, self.index)
        check(lib.vt_copy(ptr(t), C.c_void_p(src), n * 8, stream_ptr()))
        return d.elem_to_plain(t).cpu().numpy()

    @property
    def mats(self) -> Optional[np.ndarray]:
        """Galerkin element matrices (n_elements, 24, 24) of this level, else None."""
        src = lib.vt_hier_level_mats(self.hier._h, self.index)
        if not src:
            return None
        n = self.grid.n_elements * 576
        t = torch.empty(n, dtype=torch.float64, device=f"cuda:{self.dgrid.device}")
        check(lib.vt_copy(ptr(t), C.c_void_p(src), n * 8, stream_ptr()))
        return t.cpu().numpy().reshape(-1, 24, 24)

    @property
    def diag(self) -> np.ndarray:
        out = self.dgrid.zeros()
        check(lib.vt_hier_level_diag(self.hier._h, self.index, ptr(out), stream_ptr()))
        return self.dgrid.download(out)


class MgHierarchy:
    """Grid hierarchy + coarse operators + coarsest factor (multigrid.py:150-430)."""

    def __init__(self, fine: DeviceGrid, levels_geom, scheme, omega, nu_pre, nu_post, model):
        self.scheme = scheme
        self.omega = float(omega)
        self.nu_pre = int(nu_pre)
        self.nu_post = int(nu_post)
        self.model = model
        self._fine = fine
        self._h = C.c_void_p()
        check(lib.vt_hier_create_ex(C.byref(self._h), fine.handle, len(levels_geom), self.omega, self.nu_pre,
                                    1 if scheme == "galerkin" else 0))
        self.levels: List[_Level] = []
        for l, (g, mask) in enumerate(levels_geom):
            if l == 0:
                dg = fine
            else:
                dg = DeviceGrid.wrap(lib.vt_hier_grid(self._h, l), g.nelx, g.nely, g.nelz, g.h,
                                     fine.nu, fine.device)
            self.levels.append(_Level(g, mask, np.flatnonzero(mask), dg, self, l))
        self._refreshed = False

    def __del__(self):
        try:
            if self._h:
                lib.vt_hier_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass

    # --------------------------------------------------------- accounting
    @property
    def n_levels(self) -> int:
        return len(self.levels)

    @property
    def vector_scalars(self) -> int:
        """u, f, r, tmp and the diagonal per level, as the reference counts them."""
        return sum(5 * lv.n_dofs for lv in self.levels)

    @property
    def operator_scalars(self) -> int:
        per = 24 * 24 if self.scheme == "galerkin" else 1
        return sum(lv.grid.n_elements * per for lv in self.levels[1:])

    @property
    def factor_scalars(self) -> int:
        n = self.levels[-1].n_dofs
        return n * n

    # --------------------------------------------------------- refresh
    def refresh(self, state: OperatorState) -> None:
        """Coarse densities/scales, diagonals and the coarsest factor (multigrid.py:201-233)."""
        if state.grid.elem_shape != self.levels[0].grid.elem_shape:
            raise ValueError("hierarchy was built for a different grid")
        self.model = state.model
        m = state.model
        check(lib.vt_hier_refresh(self._h, ptr(state.rho_dev), ptr(state.scale_dev), m.p,
                                  m.kmin_frac, m.E, stream_ptr()))
        self._refreshed = True

    def _refresh_raw(self, rho_dev, scale_dev, model):
        check(lib.vt_hier_refresh(self._h, ptr(rho_dev), ptr(scale_dev), model.p, model.kmin_frac,
                                  model.E, stream_ptr()))
        self.model = model
        self._refreshed = True

    # --------------------------------------------------------- operators
    def apply_level(self, l: int, u):
        lv = self.levels[l]
        ud = as_device(lv.dgrid, u)
        v = lv.dgrid.zeros()
        check(lib.vt_hier_level_apply(self._h, l, ptr(ud), ptr(v), stream_ptr()))
        return from_device(lv.dgrid, v, u)

    def coarse_apply(self, l: int, u):
        if not 1 <= l < self.n_levels:
            raise ValueError(f"coarse level index {l} out of range")
        if not isinstance(u, DeviceVector) and np.asarray(u).shape != (self.levels[l].n_dofs,):
            raise ValueError("dof vector has the wrong length for this level")
        return self.apply_level(l, u)

    def prolongate(self, l: int, e_coarse):
        c, f = self.levels[l + 1], self.levels[l]
        if not isinstance(e_coarse, DeviceVector) and np.asarray(e_coarse).shape != (c.n_dofs,):
            raise ValueError("coarse vector has the wrong length")
        ed = as_device(c.dgrid, e_coarse)
        out = f.dgrid.zeros()
        check(lib.vt_hier_prolong(self._h, l, ptr(ed), ptr(out), stream_ptr()))
        return from_device(f.dgrid, out, e_coarse)

    def restrict(self, l: int, r_fine):
        f, c = self.levels[l], self.levels[l + 1]
        if not isinstance(r_fine, DeviceVector) and np.asarray(r_fine).shape != (f.n_dofs,):
            raise ValueError("fine vector has the wrong length")
        rd = as_device(f.dgrid, r_fine)
        out = c.dgrid.zeros()
        check(lib.vt_hier_restrict(self._h, l, ptr(rd), ptr(out), stream_ptr()))
        return from_device(c.dgrid, out, r_fine)

    def jacobi_smooth(self, l: int, u, f, sweeps: int):
        lv = self.levels[l]
        ud = as_device(lv.dgrid, u)
        fd = as_device(lv.dgrid, f)
        out = lv.dgrid.zeros()
        check(lib.vt_hier_jacobi(self._h, l, ptr(ud), ptr(fd), int(sweeps), ptr(out), stream_ptr()))
        return from_device(lv.dgrid, out, u)

    def coarse_solve(self, f):
        if not self._refreshed:
            raise SetupError("hierarchy was not refreshed before use")
        lv = self.levels[-1]
        if not isinstance(f, DeviceVector) and np.asarray(f).shape != (lv.n_dofs,):
            raise ValueError("coarse rhs has the wrong length")
        fd = as_device(lv.dgrid, f)
        out = lv.dgrid.zeros()
        check(lib.vt_hier_coarse_solve(self._h, ptr(fd), ptr(out), stream_ptr()))
        return from_device(lv.dgrid, out, f)

    def v_cycle(self, f, out: Optional[np.ndarray] = None):
        """One V-cycle from a zero iterate: the PCG preconditioner (multigrid.py:404-416)."""
        fine = self.levels[0]
        if not isinstance(f, DeviceVector) and np.asarray(f).shape != (fine.n_dofs,):
            raise ValueError("rhs has the wrong length")
        fd = as_device(fine.dgrid, f)
        z = fine.dgrid.zeros()
        check(lib.vt_hier_vcycle(self._h, ptr(fd), ptr(z), stream_ptr()))
        res = from_device(fine.dgrid, z, f)
        if out is None:
            return res
        out[:] = res
        return out


def build_hierarchy(grid: StructuredGrid, state: OperatorState, max_levels: int,
                    scheme: str = "galerkin", omega: float = 0.4, nu_pre: int = 1,
                    nu_post: int = 1) -> MgHierarchy:
    """Validate, build levels and refresh (multigrid.py:462-499).

    Both schemes run on the device; "galerkin" (the reference default)
    stores each coarse element matrix (its packed upper triangle, 300
    doubles) on levels >= 2 (level 1 matrix-free when it is not the coarsest)."""
    if scheme not in SCHEMES:
        raise ValueError(f"unknown scheme {scheme!r}, expected one of {SCHEMES}")
    if not 0 < omega <= 1:
        raise ValueError(f"jacobi damping must lie in (0, 1], got {omega}")
    if max_levels < 1:
        raise ValueError("max_levels must be at least 1")
    if nu_pre != nu_post:
        raise ValueError("equal pre/post smoothing is required for a symmetric cycle")
    L = min(int(max_levels), max_feasible_levels(grid.nelx, grid.nely, grid.nelz))
    geoms = []
    g, mask = grid, np.asarray(state.fixed_mask, dtype=bool)
    for l in range(L):
        geoms.append((g, mask))
        if l < L - 1:
            mask = _coarsen_mask(mask, g)
            g = StructuredGrid(g.nelx // 2, g.nely // 2, g.nelz // 2, g.h * 2)
    hier = MgHierarchy(state.dgrid, geoms, scheme, omega, nu_pre, nu_post, state.model)
    hier.refresh(state)
    return hier
