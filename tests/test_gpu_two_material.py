"""Two-material SIMP on the GPU (paper_2201_12931_b200.multimaterial) against
the oracle restatement (oracle/cpu_path.py run_design_two_material; no
reference counterpart -- see tests/test_two_material.py for how the oracle
is pinned)."""

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_2201_12931_b200")
from oracle import cpu_path as O  # noqa: E402


def _cantilever(nx, ny, nz, gravity=None):
    case = O.cantilever_case(nx, ny, nz, gravity=gravity)
    grid = vb.build_grid(nx, ny, nz, case.h)
    fixed = np.flatnonzero(case.fixed_mask)
    loads = [(int(d), float(case.f_ext[d])) for d in np.flatnonzero(case.f_ext)]
    gs = None if gravity is None else vb.GravitySpec(*gravity)
    bnd = vb.make_boundary(grid, fixed, loads, gs)
    return case, grid, vb.Problem(grid, bnd, vb.classify_regions(grid, []))


@pytest.mark.parametrize("eB", [0.4, 1.0, 0.0])
def test_two_material_sensitivities_match_oracle(eB):
    case, grid, prob = _cantilever(12, 6, 6, gravity=(2, 1.0, 1e-3))
    rng = np.random.default_rng(3)
    rho = rng.uniform(0.0, 1.0, grid.n_elements)
    phi = rng.uniform(0.0, 1.0, grid.n_elements)
    u = rng.standard_normal(grid.n_dofs)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    dcr, dcp = vb.sensitivities_two_material(st, u, phi, eB, vb.GravitySpec(2, 1.0, 1e-3))
    k0 = O.hex8_k0(0.3, case.h)
    gu = O.gravity_unit(1.0, case.h, 1e-3, 2)
    wr, wp = O.sensitivities_two_material(u, rho, phi, case.es, k0, 3.0, 1e-9, 1.0, eB, gu)
    assert rel_err(dcr, wr) <= 1e-12
    if eB == 1.0:
        assert np.all(dcp == 0.0)
        # the single-material kernel gives the same dc_rho
        assert rel_err(vb.sensitivities(st, u, vb.GravitySpec(2, 1.0, 1e-3)), dcr) <= 1e-15
    else:
        assert rel_err(dcp, wp) <= 1e-12


def test_two_material_rejects_bad_inputs():
    case, grid, prob = _cantilever(4, 2, 2)
    opt = vb.OptConfig(volfrac=0.3, filter_radius=1.5 * grid.h, max_iterations=1)
    with pytest.raises(ValueError):
        vb.run_two_material(prob, opt, 0.5, e_ratio=1.5)
    bad = vb.initial_phases(prob.regions, 0.5)
    bad.values[0] = 1.5
    with pytest.raises(ValueError):
        vb.run_two_material(prob, opt, 0.5, init_phases_=bad)


@pytest.mark.parametrize("scheme", ["galerkin", "homogenized"])
def test_two_material_trajectory_matches_oracle(scheme):
    """Every solve converged to 1e-10 on both sides (the SURVEY 8(d) protocol):
    compliance <= 1e-6 relative per iteration, rho and phi <= 1e-4."""
    case, grid, prob = _cantilever(16, 8, 8)
    its = 12
    opt = vb.OptConfig(volfrac=0.3, filter_radius=1.5 * grid.h, max_iterations=its, ch_tol=1e-12)
    res = vb.run_two_material(prob, opt, 0.4, e_ratio=0.25,
                              solver=vb.SolverConfig(tolerance=1e-10, max_iterations=1000),
                              scheme=scheme, max_levels=3)
    rho, phi, u, recs = O.run_design_two_material(case, 0.3, 0.4, 0.25, 1.5 * case.h, its, tol=1e-10,
                                                  maxit=1000, max_levels=3, ch_tol=1e-12, scheme=scheme)
    assert res.iterations == len(recs) == its
    worst = 0.0
    for r, w in zip(res.records, recs):
        worst = max(worst, abs(r.compliance - w[1]) / abs(w[1]))
        assert abs(r.volume - w[2]) <= 1e-9 and abs(r.phase_volume - w[3]) <= 1e-9
        assert abs(r.cg_iters - w[5]) <= max(2, 0.1 * w[5])
    print(f"two-material {scheme}: worst compliance rel diff {worst:.2e}, "
          f"rho {np.abs(res.densities.values - rho).max():.2e}, phi {np.abs(res.phases.values - phi).max():.2e}")
    assert worst <= 1e-6
    assert np.abs(res.densities.values - rho).max() <= 1e-4
    assert np.abs(res.phases.values - phi).max() <= 1e-4


def test_two_material_unit_ratio_is_run():
    """e_ratio = 1: the modulus factor is exactly 1, so the loop is run()."""
    case, grid, prob = _cantilever(16, 8, 8)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, max_iterations=5, ch_tol=1e-12)
    sv = vb.SolverConfig(tolerance=1e-8, max_iterations=500)
    a = vb.run(prob, opt, sv, max_levels=3)
    b = vb.run_two_material(prob, opt, 0.5, e_ratio=1.0, solver=sv, max_levels=3)
    assert [r.compliance for r in a.records] == [r.compliance for r in b.records]
    assert [r.cg_iters for r in a.records] == [r.cg_iters for r in b.records]
    assert np.array_equal(a.densities.values, b.densities.values)
    assert np.all(b.phases.values == 0.5)


def test_two_material_self_weight_matches_oracle():
    """BASELINE cfg4's combination (self-weight load + two materials) at small
    size: the gravity term acts on rho only; tight solves on both sides."""
    case, grid, prob = _cantilever(16, 8, 8, gravity=(2, 1.0, 1e-3))
    its = 6
    opt = vb.OptConfig(volfrac=0.3, filter_radius=1.5 * grid.h, max_iterations=its, ch_tol=1e-12)
    res = vb.run_two_material(prob, opt, 0.5, e_ratio=0.5,
                              solver=vb.SolverConfig(tolerance=1e-10, max_iterations=1000), max_levels=3)
    rho, phi, u, recs = O.run_design_two_material(case, 0.3, 0.5, 0.5, 1.5 * case.h, its, tol=1e-10,
                                                  maxit=1000, max_levels=3, ch_tol=1e-12)
    worst = max(abs(r.compliance - w[1]) / abs(w[1]) for r, w in zip(res.records, recs))
    assert worst <= 1e-6
    assert np.abs(res.densities.values - rho).max() <= 1e-4
    assert np.abs(res.phases.values - phi).max() <= 1e-4
