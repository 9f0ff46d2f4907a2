"""SIMP design loop on the device -- drop-in for optimize.py:49-455.

Per SIMP iteration everything stays on the B200: scale refresh, self-weight
load, hierarchy refresh, MGPCG, compliance, sensitivities, the sensitivity
filter, the OC bisection (one cooperative kernel), change/volume.  The host
only sees scalars (compliance, lambda, change, volume, CG report) unless an
`on_iteration` hook asks for the fields.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, replace
from typing import Callable, List, Optional

import numpy as np
import torch

from ._lib import check, lib
from .device import DeviceGrid, DeviceVector, device_grid, ptr, require_cuda, stream_ptr
from .errors import NumericalError, SolverBreakdown
from .hierarchy import MgHierarchy, build_hierarchy, max_feasible_levels
from .krylov import AUX_BUDGET_FACTOR, SolveReport, SolverConfig, _breakdown_message
from .material import ElementStiffness, MaterialModel, gravity_coefficient, unit_stiffness
from .mesh import BoundarySpec, GravitySpec, RegionMask, StructuredGrid
from .stiffness_op import OperatorState, as_device, from_device

__all__ = ["OptConfig", "DensityField", "FilterWeights", "Problem", "RunRecord", "OptResult",
           "OcResult", "build_filter", "compliance", "sensitivities", "filter_sensitivities",
           "oc_update", "update_gravity_load", "run", "initial_densities", "VOLUME_TOL"]

VOLUME_TOL = 1e-6
_BISECTION_MAX_STEPS = 200


@dataclass(frozen=True)
class OptConfig:
    """Design-loop parameters (optimize.py:53-82)."""

    volfrac: float
    filter_radius: float
    p: float = 3.0
    move: float = 0.2
    eta: float = 0.5
    q: float = 1.0
    gamma: float = 1e-3
    ch_tol: float = 0.01
    max_iterations: int = 300
    p_continuation: bool = False
    obj_tol: Optional[float] = None

    def __post_init__(self):
        if not 0 < self.volfrac <= 1:
            raise ValueError("volfrac must lie in (0, 1]")
        if not 0 < self.move < 1:
            raise ValueError("move limit must lie in (0, 1)")
        if self.eta <= 0 or self.gamma <= 0 or self.ch_tol <= 0:
            raise ValueError("eta, gamma and ch_tol must be positive")

    def penal_at(self, iteration: int) -> float:
        if not self.p_continuation:
            return self.p
        return min(self.p, 1.0 + 0.5 * (iteration // 15))


@dataclass
class DensityField:
    values: np.ndarray
    regions: RegionMask

    def active_mean(self) -> float:
        return float(self.values[self.regions.active].mean())

    def copy(self) -> "DensityField":
        return DensityField(self.values.copy(), self.regions)


def initial_densities(regions: RegionMask, volfrac: float) -> DensityField:
    rho = np.full(regions.classes.shape, volfrac)
    rho[regions.passive_solid] = 1.0
    rho[regions.passive_void] = 0.0
    return DensityField(rho, regions)


# ---------------------------------------------------------------- filter
def filter_weights(h: float, radius: float):
    """(R, (2R+1)^3 kernel in (dk, dj, di) order): conic weights r - dist on the
    offset box, zero outside the radius (optimize.py:110-171)."""
    R = int(np.floor(radius / h + 1e-12))
    o = np.arange(-R, R + 1)
    dk, dj, di = np.meshgrid(o, o, o, indexing="ij")
    dist = h * np.sqrt(di**2 + dj**2 + dk**2)
    inside = dist <= radius + 1e-12 * radius
    return R, np.ascontiguousarray(np.where(inside, radius - dist, 0.0), dtype=np.float64)


class FilterWeights:
    """Conic weights r - dist on the (2R+1)^3 offset box (optimize.py:110-171).

    The kernel is built on the host (27 or 125 numbers); wsum and every
    filtering pass run on the device."""

    def __init__(self, grid: StructuredGrid, radius: float):
        h = grid.h
        R = int(np.floor(radius / h + 1e-12))
        o = np.arange(-R, R + 1)
        dk, dj, di = np.meshgrid(o, o, o, indexing="ij")
        dist = h * np.sqrt(di**2 + dj**2 + dk**2)
        inside = dist <= radius + 1e-12 * radius
        self.kernel = np.where(inside, radius - dist, 0.0)
        self.offsets = np.stack([di[inside], dj[inside], dk[inside]], axis=1)
        self.weights = self.kernel[inside]
        self.radius = float(radius)
        self.h = h
        self.R = R
        self.elem_shape = grid.elem_shape
        self.grid = grid
        self._dgrid = device_grid(grid, 0.3, None)
        self._h = C.c_void_p()
        k = np.ascontiguousarray(self.kernel, dtype=np.float64)
        check(lib.vt_filter_create(C.byref(self._h), self._dgrid.handle, R, k.ctypes.data_as(C.c_void_p)))
        self._wsum = None

    def __del__(self):
        try:
            if self._h:
                lib.vt_filter_destroy(self._h)
                self._h = C.c_void_p()
        except Exception:
            pass

    def _wsum_dev(self) -> torch.Tensor:
        n = self.grid.n_elements
        t = torch.empty(n, dtype=torch.float64, device=f"cuda:{self._dgrid.device}")
        check(lib.vt_copy(ptr(t), C.c_void_p(lib.vt_filter_wsum(self._h)), n * 8, stream_ptr()))
        return t

    @property
    def wsum(self) -> np.ndarray:
        if self._wsum is None:
            self._wsum = self._wsum_dev().cpu().numpy()
        return self._wsum

    def neighborhood(self, e: int):
        nz, ny, nx = self.elem_shape
        k, j, i = e // (nx * ny), (e // nx) % ny, e % nx
        ids, ws = [], []
        for (di, dj, dk), w in zip(self.offsets, self.weights):
            a, b, c = i + di, j + dj, k + dk
            if 0 <= a < nx and 0 <= b < ny and 0 <= c < nz:
                ids.append(a + b * nx + c * nx * ny)
                ws.append(w)
        return np.asarray(ids, dtype=np.int64), np.asarray(ws)

    def correlate(self, field) -> np.ndarray:
        f = self._dgrid.plain(field)
        out = torch.empty_like(f)
        check(lib.vt_filter_correlate(self._h, ptr(f), ptr(out), stream_ptr()))
        return out.cpu().numpy()


def build_filter(grid: StructuredGrid, radius: float) -> FilterWeights:
    if radius < grid.h:
        raise ValueError(f"filter radius {radius} must be at least h = {grid.h}")
    return FilterWeights(grid, radius)


def _out_like(t: torch.Tensor, like):
    return t if isinstance(like, torch.Tensor) else t.cpu().numpy()


def filter_sensitivities(dc, rho, weights: FilterWeights, gamma: float):
    """dcf = corr(rho*dc) / (max(gamma, rho) * wsum) (optimize.py:174-179)."""
    d = weights._dgrid
    dct, rt = d.plain(dc), d.plain(rho)
    out = torch.empty_like(dct)
    check(lib.vt_filter_apply(weights._h, ptr(dct), ptr(rt), float(gamma), ptr(out), stream_ptr()))
    return _out_like(out, dc)


# ---------------------------------------------------------------- objective / gradient
def compliance(f, u) -> float:
    """f'u (optimize.py:186-192)."""
    if isinstance(f, DeviceVector) and isinstance(u, DeviceVector):
        out = C.c_double()
        check(lib.vt_compliance(f.dgrid.handle, ptr(f.data), ptr(u.data), C.byref(out), stream_ptr()))
        return out.value
    fa, ua = np.asarray(f), np.asarray(u)
    if fa.shape != ua.shape:
        raise ValueError("force and displacement vectors differ in length")
    require_cuda()
    ft = torch.as_tensor(np.ascontiguousarray(fa, dtype=np.float64), device="cuda")
    ut = torch.as_tensor(np.ascontiguousarray(ua, dtype=np.float64), device="cuda")
    return float(torch.dot(ft, ut))


def sensitivities(state: OperatorState, u, gravity: Optional[GravitySpec] = None):
    """-E s'(rho) u_e'K0u_e (+ 2 u_e.g_unit) per element (optimize.py:195-213)."""
    d = state.dgrid
    ud = as_device(d, u)
    dc = torch.empty(d.n_elements, dtype=torch.float64, device=f"cuda:{d.device}")
    gax, gco = -1, 0.0
    if gravity is not None:
        gax, gco = int(gravity.axis), gravity_coefficient(gravity.g, state.grid.h, gravity.unit_weight)
    m = state.model
    check(lib.vt_sensitivities(d.handle, ptr(ud), ptr(state.rho_dev), m.p, m.kmin_frac, m.E, gax, gco,
                               ptr(dc), stream_ptr()))
    return dc if isinstance(u, DeviceVector) else dc.cpu().numpy()


def update_gravity_load(grid: StructuredGrid, rho: DensityField, gravity: GravitySpec,
                        external=None, fixed_idx=None):
    """Nodal self-weight of the current material + external loads (optimize.py:216-231)."""
    if fixed_idx is not None:
        mask = np.zeros(grid.n_dofs, dtype=bool)
        mask[np.asarray(fixed_idx, dtype=np.int64)] = True
    else:
        mask = None
    d = device_grid(grid, 0.3, mask)
    r = d.plain(rho.values if isinstance(rho, DensityField) else rho)
    fe = d.upload(external) if external is not None else None
    out = d.zeros()
    gco = gravity_coefficient(gravity.g, grid.h, gravity.unit_weight)
    check(lib.vt_gravity_load(d.handle, ptr(r), int(gravity.axis), gco, ptr(fe) if fe is not None else None,
                              1 if mask is not None else 0, ptr(out), stream_ptr()))
    return d.download(out)


# ---------------------------------------------------------------- OC
@dataclass
class OcResult:
    densities: DensityField
    lam: float
    bisection_steps: int


def _oc_device(d: DeviceGrid, rho_t, cls_t, dc_t, dv_t, cfg: OptConfig, out_t):
    lam = C.c_double()
    steps = C.c_int()
    check(lib.vt_oc_update(d.handle, ptr(rho_t), ptr(cls_t), ptr(dc_t), ptr(dv_t), float(cfg.volfrac),
                           float(cfg.move), float(cfg.eta), float(cfg.q), ptr(out_t),
                           C.byref(lam), C.byref(steps), stream_ptr()))
    return lam.value, steps.value


def oc_update(rho: DensityField, dc, dv, cfg: OptConfig) -> OcResult:
    """OC step with the bisected multiplier (optimize.py:245-302)."""
    nel = rho.values.shape[0]
    dva = np.asarray(dv, dtype=np.float64)
    if np.any(dva[rho.regions.active] <= 0):
        raise ValueError("volume gradient must be positive")
    require_cuda()
    dev = f"cuda:{torch.cuda.current_device()}"
    flat = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)
    rt = flat(rho.values)
    ct = torch.as_tensor(np.ascontiguousarray(rho.regions.classes, dtype=np.int8), device=dev)
    dct, dvt = flat(dc), flat(dva)  # keep the device copies alive across the call
    out = torch.empty_like(rt)
    lam, steps = C.c_double(), C.c_int()
    check(lib.vt_oc_update_flat(nel, ptr(rt), ptr(ct), ptr(dct), ptr(dvt), float(cfg.volfrac),
                                float(cfg.move), float(cfg.eta), float(cfg.q), ptr(out), C.byref(lam),
                                C.byref(steps), stream_ptr()))
    lam, steps = lam.value, steps.value
    return OcResult(DensityField(out.cpu().numpy(), rho.regions), lam, steps)


# ---------------------------------------------------------------- the loop
@dataclass(frozen=True)
class Problem:
    grid: StructuredGrid
    boundary: BoundarySpec
    regions: RegionMask
    model: MaterialModel = MaterialModel()
    nu: float = 0.3

    def stiffness(self) -> ElementStiffness:
        return unit_stiffness(self.nu, self.grid.h)


@dataclass
class RunRecord:
    iteration: int
    compliance: float
    volume: float
    change: float
    cg_iters: int
    cg_residual: float
    wall_s: float
    aux_scalars: int


@dataclass
class OptResult:
    densities: DensityField
    displacement: np.ndarray
    records: List[RunRecord]
    converged: bool
    iterations: int


class DeviceRun:
    """Device-resident state of one design loop; also used by bench.py."""

    def __init__(self, problem: Problem, opt: OptConfig, solver: SolverConfig, scheme: str,
                 max_levels: Optional[int], omega: float, init_densities=None, init_displacement=None):
        require_cuda()
        if scheme not in ("galerkin", "homogenized"):
            raise ValueError(f"unknown scheme {scheme!r}")
        self.scheme = scheme
        grid = problem.grid
        self.problem, self.opt, self.solver = problem, opt, solver
        self.omega = omega
        self.k0 = problem.stiffness()
        self.fixed_mask = problem.boundary.fixed_mask(grid)
        self.d = device_grid(grid, problem.nu, self.fixed_mask)
        d = self.d
        f_ext = problem.boundary.external_force(grid)
        f_ext[np.flatnonzero(self.fixed_mask)] = 0.0
        self.f_ext = d.upload(f_ext)
        self.gravity = problem.boundary.gravity
        self.filter = build_filter(grid, opt.filter_radius)
        dev = f"cuda:{d.device}"
        self.dv = torch.ones(grid.n_elements, dtype=torch.float64, device=dev)
        self.cls = torch.as_tensor(np.ascontiguousarray(problem.regions.classes, dtype=np.int8), device=dev)
        rho0 = (init_densities.values if init_densities is not None
                else initial_densities(problem.regions, opt.volfrac).values)
        self.rho = d.plain(rho0).clone()
        self.rho_new = torch.empty_like(self.rho)
        self.u = d.upload(init_displacement) if init_displacement is not None else d.zeros()
        self.f = d.zeros() if self.gravity is not None else self.f_ext
        self.scale = d.zeros_elem()
        self.dc = torch.empty_like(self.rho)
        self.dcf = torch.empty_like(self.rho)
        self.max_levels = max_levels if max_levels is not None else max_feasible_levels(
            grid.nelx, grid.nely, grid.nelz)
        self.hier: Optional[MgHierarchy] = None
        self.regions = problem.regions

    def _set_scale(self, model):
        check(lib.vt_scale_from_density(self.d.handle, ptr(self.rho), model.p, model.kmin_frac, model.E,
                                        ptr(self.scale), stream_ptr()))

    def state_view(self, model) -> OperatorState:
        st = OperatorState.__new__(OperatorState)
        st.grid, st.model, st.stiffness = self.problem.grid, model, self.k0
        st.fixed_mask, st.fixed_idx = self.fixed_mask, np.flatnonzero(self.fixed_mask)
        st.dgrid, st.rho_dev, st.scale_dev, st.densities = self.d, self.mg_rho(), self.scale, None
        return st

    def mg_rho(self) -> torch.Tensor:
        """Densities the homogenized coarse levels average (the design densities)."""
        return self.rho

    def solve(self, model):
        """refresh + MGPCG for the current densities; returns SolveReport."""
        d, sv = self.d, self.solver
        self._set_scale(model)
        if self.gravity is not None:
            gco = gravity_coefficient(self.gravity.g, self.problem.grid.h, self.gravity.unit_weight)
            check(lib.vt_gravity_load(d.handle, ptr(self.rho), int(self.gravity.axis), gco,
                                      ptr(self.f_ext), 1, ptr(self.f), stream_ptr()))
        kind, hh, aux = 0, None, 4 * d.n_dofs
        if sv.preconditioner == "multigrid":
            if self.hier is None:
                self.hier = build_hierarchy(self.problem.grid, self.state_view(model), self.max_levels,
                                            scheme=self.scheme, omega=self.omega)
            else:
                self.hier._refresh_raw(self.mg_rho(), self.scale, model)
            aux = 4 * d.n_dofs + self.hier.vector_scalars
            if aux > AUX_BUDGET_FACTOR * d.n_dofs:
                raise SolverBreakdown(f"auxiliary vector budget {aux} exceeds {AUX_BUDGET_FACTOR} * n")
            kind, hh = 2, self.hier._h
        elif sv.preconditioner == "jacobi":
            kind = 1
        from ._lib import VT_EBREAKDOWN, SolveReportC
        rep = SolveReportC()
        st = lib.vt_pcg(d.handle, ptr(self.scale), kind, hh, ptr(self.f), ptr(self.u),
                        1 if sv.warm_start else 0, float(sv.tolerance), int(sv.max_iterations),
                        C.byref(rep), stream_ptr())
        if st == VT_EBREAKDOWN:
            raise SolverBreakdown(_breakdown_message(rep))
        check(st, "vt_pcg")
        return SolveReport(iterations=rep.iterations, final_rel_residual=rep.final_rel_residual,
                           precond_applications=rep.precond_applications, converged=bool(rep.converged),
                           aux_vector_scalars=aux, residual_drift=rep.residual_drift)

    def design_step(self, model):
        """compliance, sensitivities, filter, OC; swaps rho. Returns (c, change, volume)."""
        d, opt = self.d, self.opt
        c = C.c_double()
        check(lib.vt_compliance(d.handle, ptr(self.f), ptr(self.u), C.byref(c), stream_ptr()))
        gax, gco = -1, 0.0
        if self.gravity is not None:
            gax = int(self.gravity.axis)
            gco = gravity_coefficient(self.gravity.g, self.problem.grid.h, self.gravity.unit_weight)
        check(lib.vt_sensitivities(d.handle, ptr(self.u), ptr(self.rho), model.p, model.kmin_frac, model.E,
                                   gax, gco, ptr(self.dc), stream_ptr()))
        check(lib.vt_filter_apply(self.filter._h, ptr(self.dc), ptr(self.rho), float(opt.gamma),
                                  ptr(self.dcf), stream_ptr()))
        _oc_device(d, self.rho, self.cls, self.dcf, self.dv, opt, self.rho_new)
        ch, vol = C.c_double(), C.c_double()
        check(lib.vt_change_volume(d.handle, ptr(self.rho_new), ptr(self.rho), ptr(self.cls),
                                   C.byref(ch), C.byref(vol), stream_ptr()))
        self.rho, self.rho_new = self.rho_new, self.rho
        return c.value, ch.value, vol.value

    def densities(self) -> DensityField:
        return DensityField(self.rho.cpu().numpy(), self.regions)

    def displacement(self) -> np.ndarray:
        return self.d.download(self.u)


def run(problem: Problem, opt: OptConfig, solver: SolverConfig = SolverConfig(),
        scheme: str = "galerkin", max_levels: Optional[int] = None, omega: float = 0.4,
        init_densities: Optional[DensityField] = None, init_displacement=None,
        start_iteration: int = 0,
        on_iteration: Optional[Callable[[RunRecord, DensityField, np.ndarray], None]] = None) -> OptResult:
    """The SIMP loop (optimize.py:344-455) with every kernel on the device.

    Same signature and defaults as the reference (scheme="galerkin" stores the
    Galerkin coarse element matrices on the device; "homogenized" rebuilds the
    coarse operators from averaged densities)."""
    R = DeviceRun(problem, opt, solver, scheme, max_levels, omega, init_densities, init_displacement)
    records: List[RunRecord] = []
    converged = False
    iteration = start_iteration
    while iteration < opt.max_iterations:
        t0 = time.perf_counter()
        model_k = replace(problem.model, p=opt.penal_at(iteration))
        rep = R.solve(model_k)
        c, ch, vol = R.design_step(model_k)
        iteration += 1
        if abs(vol - opt.volfrac) > VOLUME_TOL:
            raise NumericalError(f"volume constraint violated after update: {vol} vs {opt.volfrac}")
        rec = RunRecord(iteration, c, vol, ch, rep.iterations, rep.final_rel_residual,
                        time.perf_counter() - t0, rep.aux_vector_scalars)
        records.append(rec)
        if on_iteration is not None:
            on_iteration(rec, R.densities(), R.displacement())
        obj_ok = True
        if opt.obj_tol is not None and len(records) >= 2:
            obj_ok = abs(records[-1].compliance - records[-2].compliance) <= opt.obj_tol
        if ch <= opt.ch_tol and obj_ok:
            converged = True
            break
    return OptResult(R.densities(), R.displacement(), records, converged, iteration)
