"""Two-material SIMP restatement in the oracle (oracle/cpu_path.py,
run_design_two_material).  The reference has no multi-material design
(SPEC.md:15,178), so the oracle is pinned two ways: (1) its e_ratio = 1 limit
must reproduce the reference-generated single-material fixtures exactly;
(2) both sensitivities must match central finite differences of the
compliance of a dense solve (the same check the reference's acceptance
tests apply to its own gradients, pkg/tests/test_acceptance.py:162-185)."""

import numpy as np
import pytest

from conftest import golden
from oracle import cpu_path as O


def test_unit_ratio_reproduces_reference_galerkin_trajectory():
    g = golden("galerkin_traj.npz")
    case = O.cantilever_case(16, 8, 8)
    rho, phi, u, recs = O.run_design_two_material(case, 0.12, 0.5, 1.0, 1.5 * case.h, 20,
                                                  max_levels=3, ch_tol=1e-12)
    want = g["recs"]
    assert len(recs) == want.shape[0]
    for r, w in zip(recs, want):
        assert r[0] == int(w[0]) and r[5] == int(w[4])
        assert abs(r[1] - w[1]) <= 1e-10 * abs(w[1])
    assert np.abs(rho - g["rho20"]).max() <= 1e-8
    assert np.all(phi == 0.5)


def test_unit_ratio_is_single_material_bit_for_bit():
    case = O.cantilever_case(16, 8, 8)
    rho1, u1, recs1 = O.run_design(case, 0.12, 1.5 * case.h, 4, max_levels=3, ch_tol=1e-12,
                                   scheme="homogenized")
    rho2, phi, u2, recs2 = O.run_design_two_material(case, 0.12, 0.5, 1.0, 1.5 * case.h, 4,
                                                     max_levels=3, ch_tol=1e-12, scheme="homogenized")
    assert np.array_equal(rho1, rho2) and np.array_equal(u1, u2)
    assert [r.compliance for r in recs1] == [r[1] for r in recs2]


def _compliance(case, rho, phi, eB, k0, fixed, f):
    scale = O.two_material_scale(rho, phi, case.p, case.kmin, case.E, eB)
    K = O.dense_k(case.es, fixed, k0, scale)
    u = np.linalg.solve(K, f)
    return float(f @ u), u


@pytest.mark.parametrize("eB", [0.3, 0.0])
def test_sensitivities_match_finite_differences(eB):
    case = O.cantilever_case(4, 2, 2, L=4.0)
    rng = np.random.default_rng(7)
    nel = 16
    rho = rng.uniform(0.3, 0.9, nel)
    phi = rng.uniform(0.2, 0.8, nel)
    k0 = O.hex8_k0(case.nu, case.h)
    fixed = np.flatnonzero(case.fixed_mask)
    f = case.f_ext.copy()
    f[fixed] = 0.0
    c0, u = _compliance(case, rho, phi, eB, k0, fixed, f)
    dcr, dcp = O.sensitivities_two_material(u, rho, phi, case.es, k0, case.p, case.kmin, case.E, eB)
    hstep = 1e-6
    for e in (0, 5, 11, 15):
        for field, dc in ((rho, dcr), (phi, dcp)):
            fp, fm = field.copy(), field.copy()
            fp[e] += hstep
            fm[e] -= hstep
            args_p = (fp, phi) if field is rho else (rho, fp)
            args_m = (fm, phi) if field is rho else (rho, fm)
            cp = _compliance(case, *args_p, eB, k0, fixed, f)[0]
            cm = _compliance(case, *args_m, eB, k0, fixed, f)[0]
            fd = (cp - cm) / (2 * hstep)
            assert abs(fd - dc[e]) <= 1e-5 * abs(dc[e]) + 1e-12 * abs(c0), (e, fd, dc[e])


def test_phase_bounds_rejected():
    with pytest.raises(O.OracleError):
        O.two_material_factor(np.array([0.5, 1.2]), 3.0, 0.5)


def test_two_material_loop_keeps_both_volumes():
    case = O.cantilever_case(16, 8, 8)
    rho, phi, u, recs = O.run_design_two_material(case, 0.3, 0.4, 0.25, 1.5 * case.h, 4, tol=1e-8,
                                                  maxit=500, max_levels=3)
    for r in recs:
        assert abs(r[2] - 0.3) <= 1e-6 and abs(r[3] - 0.4) <= 1e-6
    assert recs[-1][1] < recs[0][1]
