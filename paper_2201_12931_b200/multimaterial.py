"""Two-material SIMP on the device (BASELINE cfg4's "two-material SIMP").

The reference has no multi-material design (its SPEC.md:15,178 lists it as
never developed), so this module extends the reference's single-material
path the standard way (two design fields per element) and keeps every other
step identical:

* ``rho`` -- material density, as in the reference; ``phi`` -- share of the
  stiff phase A in the material (phase B has modulus ``e_ratio * E``).
* modulus ``E s(rho) m(phi)``, ``s`` the reference SIMP law
  (element.py:102-108), ``m = e_ratio + (1 - e_ratio) phi^p``.
* ``dc_rho = -E s'(rho) m q_e``, ``dc_phi = -E s(rho) p phi^(p-1) (1 - e_ratio) q_e``,
  ``q_e = u_e'K0u_e`` (extends optimize.py:195-213); self-weight acts on rho.
* both go through the reference sensitivity filter (optimize.py:174-179, phi
  as the weight of dc_phi) and the reference OC update (optimize.py:245-302)
  with their own targets: mean rho = ``volfrac``, mean phi = ``phase_frac``
  over the active elements; passive elements keep phi = 1.
* the homogenized coarse levels average ``rho m^(1/p)`` (so the coarse
  modulus follows both fields); Galerkin coarsening needs nothing new.

With ``e_ratio = 1`` the modulus factor is exactly 1 and the rho trajectory is
the single-material ``run()`` bit for bit (phi is inert and not updated) --
the only anchor this extension has to the reference (tests/test_two_material.py).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, replace
from typing import Callable, List, Optional

import numpy as np
import torch

from ._lib import check, lib
from .design import VOLUME_TOL, DensityField, DeviceRun, OptConfig, Problem, RunRecord, _oc_device
from .device import ptr, stream_ptr
from .errors import NumericalError
from .krylov import SolverConfig
from .material import gravity_coefficient
from .stiffness_op import OperatorState, as_device

__all__ = ["TwoMaterialRecord", "TwoMaterialResult", "initial_phases", "sensitivities_two_material",
           "run_two_material", "run_two_material_slabs"]


@dataclass
class TwoMaterialRecord(RunRecord):
    phase_volume: float = 0.0


@dataclass
class TwoMaterialResult:
    densities: DensityField
    phases: DensityField
    displacement: np.ndarray
    records: List[TwoMaterialRecord]
    converged: bool
    iterations: int


def initial_phases(regions, phase_frac: float) -> DensityField:
    phi = np.full(regions.classes.shape, float(phase_frac))
    phi[~regions.active] = 1.0
    return DensityField(phi, regions)


def _check_ratio(e_ratio: float):
    if not 0.0 <= e_ratio <= 1.0:
        raise ValueError("e_ratio (E_B / E_A) must lie in [0, 1]")


def sensitivities_two_material(state: OperatorState, u, phi, e_ratio: float, gravity=None):
    """(dc_rho, dc_phi) for the two-material law at the state's densities."""
    _check_ratio(e_ratio)
    d = state.dgrid
    ud = as_device(d, u)
    ph = d.plain(phi.values if isinstance(phi, DensityField) else phi)
    dcr = torch.empty(d.n_elements, dtype=torch.float64, device=f"cuda:{d.device}")
    dcp = torch.empty_like(dcr)
    gax, gco = -1, 0.0
    if gravity is not None:
        gax, gco = int(gravity.axis), gravity_coefficient(gravity.g, state.grid.h, gravity.unit_weight)
    m = state.model
    check(lib.vt_sensitivities_two_material(d.handle, ptr(ud), ptr(state.rho_dev), ptr(ph), m.p,
                                            m.kmin_frac, m.E, float(e_ratio), gax, gco, ptr(dcr),
                                            ptr(dcp), stream_ptr()))
    if isinstance(u, torch.Tensor):
        return dcr, dcp
    return dcr.cpu().numpy(), dcp.cpu().numpy()


class TwoMaterialRun(DeviceRun):
    """DeviceRun with a second design field; every step stays on the device."""

    def __init__(self, problem: Problem, opt: OptConfig, phase_frac: float, e_ratio: float,
                 solver: SolverConfig, scheme: str, max_levels: Optional[int], omega: float,
                 init_densities=None, init_phases_=None):
        _check_ratio(e_ratio)
        if not 0 < phase_frac <= 1:
            raise ValueError("phase_frac must lie in (0, 1]")
        super().__init__(problem, opt, solver, scheme, max_levels, omega, init_densities, None)
        self.e_ratio, self.phase_frac = float(e_ratio), float(phase_frac)
        phi0 = (init_phases_.values if init_phases_ is not None
                else initial_phases(problem.regions, phase_frac).values)
        self.phi = self.d.plain(phi0).clone()
        self.phi_new = torch.empty_like(self.phi)
        self.rho_h = torch.empty_like(self.rho)
        self.dcp = torch.empty_like(self.rho)
        self.dcpf = torch.empty_like(self.rho)
        self.opt_phi = replace(opt, volfrac=self.phase_frac)

    def _set_scale(self, model):
        check(lib.vt_scale_two_material(self.d.handle, ptr(self.rho), ptr(self.phi), model.p,
                                        model.kmin_frac, model.E, self.e_ratio, ptr(self.scale),
                                        ptr(self.rho_h), stream_ptr()))

    def mg_rho(self) -> torch.Tensor:
        return self.rho_h

    def design_step(self, model):
        """compliance, both sensitivities, filters and OC updates; returns
        (c, change, volume, phase_volume)."""
        d, opt = self.d, self.opt
        c = C.c_double()
        check(lib.vt_compliance(d.handle, ptr(self.f), ptr(self.u), C.byref(c), stream_ptr()))
        gax, gco = -1, 0.0
        if self.gravity is not None:
            gax = int(self.gravity.axis)
            gco = gravity_coefficient(self.gravity.g, self.problem.grid.h, self.gravity.unit_weight)
        check(lib.vt_sensitivities_two_material(d.handle, ptr(self.u), ptr(self.rho), ptr(self.phi),
                                                model.p, model.kmin_frac, model.E, self.e_ratio, gax,
                                                gco, ptr(self.dc), ptr(self.dcp), stream_ptr()))
        check(lib.vt_filter_apply(self.filter._h, ptr(self.dc), ptr(self.rho), float(opt.gamma),
                                  ptr(self.dcf), stream_ptr()))
        _oc_device(d, self.rho, self.cls, self.dcf, self.dv, opt, self.rho_new)
        ch, vol = C.c_double(), C.c_double()
        check(lib.vt_change_volume(d.handle, ptr(self.rho_new), ptr(self.rho), ptr(self.cls),
                                   C.byref(ch), C.byref(vol), stream_ptr()))
        change = ch.value
        if self.e_ratio != 1.0:  # at e_ratio = 1 phi has no influence (dc_phi = 0)
            check(lib.vt_filter_apply(self.filter._h, ptr(self.dcp), ptr(self.phi), float(opt.gamma),
                                      ptr(self.dcpf), stream_ptr()))
            _oc_device(d, self.phi, self.cls, self.dcpf, self.dv, self.opt_phi, self.phi_new)
            chp = C.c_double()
            check(lib.vt_change_volume(d.handle, ptr(self.phi_new), ptr(self.phi), ptr(self.cls),
                                       C.byref(chp), None, stream_ptr()))
            change = max(change, chp.value)
            self.phi, self.phi_new = self.phi_new, self.phi
        pv = C.c_double()
        check(lib.vt_change_volume(d.handle, ptr(self.phi), ptr(self.phi), ptr(self.cls), None,
                                   C.byref(pv), stream_ptr()))
        self.rho, self.rho_new = self.rho_new, self.rho
        return c.value, change, vol.value, pv.value

    def phases(self) -> DensityField:
        return DensityField(self.phi.cpu().numpy(), self.regions)


def run_two_material(problem: Problem, opt: OptConfig, phase_frac: float, e_ratio: float = 0.5,
                     solver: SolverConfig = SolverConfig(), scheme: str = "galerkin",
                     max_levels: Optional[int] = None, omega: float = 0.4,
                     init_densities: Optional[DensityField] = None,
                     init_phases_: Optional[DensityField] = None,
                     on_iteration: Optional[Callable] = None) -> TwoMaterialResult:
    """Two-material SIMP loop: the reference's run() (optimize.py:344-455) with
    the second field updated after the density each iteration."""
    R = TwoMaterialRun(problem, opt, phase_frac, e_ratio, solver, scheme, max_levels, omega,
                       init_densities, init_phases_)
    records: List[TwoMaterialRecord] = []
    converged = False
    iteration = 0
    while iteration < opt.max_iterations:
        t0 = time.perf_counter()
        model_k = replace(problem.model, p=opt.penal_at(iteration))
        rep = R.solve(model_k)
        c, ch, vol, pvol = R.design_step(model_k)
        iteration += 1
        if abs(vol - opt.volfrac) > VOLUME_TOL:
            raise NumericalError(f"volume constraint violated after update: {vol} vs {opt.volfrac}")
        rec = TwoMaterialRecord(iteration, c, vol, ch, rep.iterations, rep.final_rel_residual,
                                time.perf_counter() - t0, rep.aux_vector_scalars, pvol)
        records.append(rec)
        if on_iteration is not None:
            on_iteration(rec, R.densities(), R.phases(), R.displacement())
        if ch <= opt.ch_tol:
            converged = True
            break
    return TwoMaterialResult(R.densities(), R.phases(), R.displacement(), records, converged, iteration)


# ---------------------------------------------------------------- on z-slabs
def _slab_run_class():
    from .slabs import SlabRun, _ptr_array

    class SlabTwoMaterialRun(SlabRun):
        """SlabRun with the second design field: per-slab two-material scale
        (+ the density the homogenized coarse levels average), the distributed
        two-material sensitivities (u halo), and the distributed filter / OC /
        change for both fields -- TwoMaterialRun's steps on slabs."""

        def __init__(self, problem, opt, phase_frac, e_ratio, solver, max_levels=None, omega=0.4, nranks=1,
                     group=None, scheme="homogenized", **kw):
            _check_ratio(e_ratio)
            if not 0 < phase_frac <= 1:
                raise ValueError("phase_frac must lie in (0, 1]")
            super().__init__(problem, opt, solver, max_levels, omega, nranks=nranks, group=group, scheme=scheme,
                             **kw)
            self.e_ratio, self.phase_frac = float(e_ratio), float(phase_frac)
            phi0 = torch.as_tensor(initial_phases(problem.regions, phase_frac).values, device=self.rho[0].device)
            nxy = problem.grid.nelx * problem.grid.nely
            self.phi = [phi0[dg.k0 * nxy:dg.k1 * nxy].clone() for dg in self.S.slab_grids]
            self.phi_new = [torch.empty_like(p) for p in self.phi]
            self.rho_h = [torch.empty_like(r) for r in self.rho]
            self.dcp = [torch.empty_like(r) for r in self.rho]
            self.dcpf = [torch.empty_like(r) for r in self.rho]

        def solve(self, model):
            S = self.S
            S.model = model
            for dg, r, ph, sc, rh in zip(S.slab_grids, self.rho, self.phi, S.scales, self.rho_h):
                check(lib.vt_scale_two_material(dg.handle, ptr(r), ptr(ph), model.p, model.kmin_frac, model.E,
                                                self.e_ratio, ptr(sc), ptr(rh), stream_ptr()))
            check(lib.vt_dist_refresh(S._h, _ptr_array(self.rho_h), _ptr_array(S.scales), model.p,
                                      model.kmin_frac, model.E, stream_ptr()), "vt_dist_refresh")
            if self.gravity is not None:
                check(lib.vt_dist_gravity_load(S._h, _ptr_array(self.rho), int(self.gravity.axis), self._gco(),
                                               _ptr_array(self.f_ext), 1, _ptr_array(self.f), stream_ptr()))
            self.u, rep = S.mgcg_solve(self.f, u_prev=self.u, cfg=self.solver)
            return rep

        def _oc(self, x, dcf, opt, out):
            lam, steps = C.c_double(), C.c_int()
            check(lib.vt_dist_oc_update(self.S._h, _ptr_array(x), _ptr_array(self.cls), _ptr_array(dcf),
                                        _ptr_array(self.dv), float(opt.volfrac), float(opt.move), float(opt.eta),
                                        float(opt.q), _ptr_array(out), C.byref(lam), C.byref(steps),
                                        stream_ptr()))

        def _change(self, a, b, want_change=True, want_mean=True):
            ch, vol = C.c_double(), C.c_double()
            check(lib.vt_dist_change_volume(self.S._h, _ptr_array(a), _ptr_array(b), _ptr_array(self.cls),
                                            C.byref(ch) if want_change else None,
                                            C.byref(vol) if want_mean else None, stream_ptr()))
            return ch.value, vol.value

        def design_step(self, model):
            """(c, change, volume, phase_volume), TwoMaterialRun.design_step on slabs."""
            S, opt = self.S, self.opt
            c = S.dot(self.f, self.u)
            gax, gco = (int(self.gravity.axis), self._gco()) if self.gravity is not None else (-1, 0.0)
            check(lib.vt_dist_sensitivities_two_material(S._h, _ptr_array(self.u), _ptr_array(self.rho),
                                                         _ptr_array(self.phi), model.p, model.kmin_frac, model.E,
                                                         self.e_ratio, gax, gco, _ptr_array(self.dc),
                                                         _ptr_array(self.dcp), stream_ptr()))
            check(lib.vt_dist_filter_apply(S._h, _ptr_array(self.dc), _ptr_array(self.rho), float(opt.gamma),
                                           _ptr_array(self.dcf), stream_ptr()))
            self._oc(self.rho, self.dcf, opt, self.rho_new)
            change, vol = self._change(self.rho_new, self.rho)
            if self.e_ratio != 1.0:  # at e_ratio = 1 phi has no influence (dc_phi = 0)
                check(lib.vt_dist_filter_apply(S._h, _ptr_array(self.dcp), _ptr_array(self.phi), float(opt.gamma),
                                               _ptr_array(self.dcpf), stream_ptr()))
                self._oc(self.phi, self.dcpf, replace(opt, volfrac=self.phase_frac), self.phi_new)
                chp, _ = self._change(self.phi_new, self.phi, want_mean=False)
                change = max(change, chp)
                self.phi, self.phi_new = self.phi_new, self.phi
            _, pv = self._change(self.phi, self.phi, want_change=False)
            self.rho, self.rho_new = self.rho_new, self.rho
            return c, change, vol, pv

        def phases(self) -> np.ndarray:
            return self._gather(self.phi).cpu().numpy()

    return SlabTwoMaterialRun


def run_two_material_slabs(problem: Problem, opt: OptConfig, phase_frac: float, e_ratio: float = 0.5,
                           solver: SolverConfig = SolverConfig(), scheme: str = "homogenized",
                           max_levels: Optional[int] = None, omega: float = 0.4, nranks: int = 1,
                           group=None, transport: str = "peer") -> TwoMaterialResult:
    """run_two_material on z-slabs: all `nranks` slabs in this process, or one
    slab per rank of `group` (peer / nccl transport), either coarse scheme."""
    Cls = _slab_run_class()
    if group is not None:
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if transport != "peer":
            raise ValueError("run_two_material_slabs with a process group uses the peer transport")
        R = Cls(problem, opt, phase_frac, e_ratio, solver, max_levels, omega, nranks=world, group=group,
                scheme=scheme, rank=rank, nlocal=1, peer=True)
    else:
        R = Cls(problem, opt, phase_frac, e_ratio, solver, max_levels, omega, nranks=nranks, scheme=scheme)
    records: List[TwoMaterialRecord] = []
    converged = False
    iteration = 0
    try:
        while iteration < opt.max_iterations:
            t0 = time.perf_counter()
            model_k = replace(problem.model, p=opt.penal_at(iteration))
            rep = R.solve(model_k)
            c, ch, vol, pvol = R.design_step(model_k)
            iteration += 1
            if abs(vol - opt.volfrac) > VOLUME_TOL:
                raise NumericalError(f"volume constraint violated after update: {vol} vs {opt.volfrac}")
            records.append(TwoMaterialRecord(iteration, c, vol, ch, rep.iterations, rep.final_rel_residual,
                                             time.perf_counter() - t0, rep.aux_vector_scalars, pvol))
            if ch <= opt.ch_tol:
                converged = True
                break
        return TwoMaterialResult(DensityField(R.densities(), problem.regions),
                                 DensityField(R.phases(), problem.regions), R.displacement(), records, converged,
                                 iteration)
    finally:
        R.S.close()
