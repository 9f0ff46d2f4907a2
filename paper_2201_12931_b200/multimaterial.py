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
           "run_two_material"]


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
