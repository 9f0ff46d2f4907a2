"""MGPCG / PCG and design-loop parity on the GPU against the reference goldens
(mirrors pkg/tests/test_solver.py, test_optimize.py, test_acceptance.py)."""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, face_fixed_mask, golden, rel_err

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


@pytest.mark.parametrize("tag", ["u", "r"])
def test_mgcg_matches_reference(tag):
    g = golden("pcg.npz")
    case, grid, _ = _cantilever(16, 8, 8)
    st = vb.OperatorState(grid, g[f"{tag}_rho"], vb.MaterialModel(), case.fixed_mask)
    H = vb.build_hierarchy(grid, st, 3, scheme="homogenized")
    f = g["f"]
    for ctag, tol, maxit in (("a", 1e-5, 200), ("b", 1e-10, 500), ("c", 1e-12, 3), ("d", 1e-8, 120)):
        u0 = g[f"{tag}{ctag}_u0"] if ctag == "d" else None
        x, rep = vb.mgcg_solve(st, H, f, u_prev=u0, cfg=vb.SolverConfig(tolerance=tol, max_iterations=maxit))
        want = g[f"{tag}{ctag}_rep"]
        # Random densities down to kmin make K ill-conditioned (cond ~1e9): the CUDA
        # kernels agree with the oracle to 1e-16 per call, yet CG amplifies the
        # rounding of the dot products (OpenBLAS ddot vs a fixed tree) exponentially
        # from ~iteration 20 (scripts/debug_pcg.py: 1e-15 -> 3e-8 by iteration 35),
        # so near the tolerance boundary the count may differ by one -- the same
        # effect the reference shows against itself across BLAS thread counts
        # (DESIGN.md §4).  The uniform-density case must match exactly.
        slack = 1 if (tag == "r" and ctag in ("a", "b")) else 0
        assert abs(rep.iterations - int(want[0])) <= slack, (ctag, rep)
        assert abs(rep.precond_applications - int(want[2])) <= slack
        assert rep.converged == bool(want[3])
        assert rep.aux_vector_scalars == int(want[4])
        if rep.iterations == int(want[0]):
            # same count: both runs stop at the same point; residuals agree to rounding x cond
            assert abs(rep.final_rel_residual - want[1]) <= 2e-2 * want[1] + 1e-15
        else:
            assert rep.converged and rep.final_rel_residual <= tol
        assert rel_err(x, g[f"{tag}{ctag}_x"]) <= max(1e-8, 0.1 * tol)


@pytest.mark.parametrize("tag", ["u", "r"])
def test_jacobi_and_plain_cg_match_reference(tag):
    g = golden("pcg.npz")
    case, grid, _ = _cantilever(16, 8, 8)
    st = vb.OperatorState(grid, g[f"{tag}_rho"], vb.MaterialModel(), case.fixed_mask)
    cfg = vb.SolverConfig(tolerance=1e-8, max_iterations=2000)
    for key, pre in (("j", vb.jacobi_preconditioner(st)), ("n", None)):
        x, rep = vb.pcg(st, pre, g["f"], cfg=cfg)
        want = g[f"{tag}{key}_rep"]
        # long unpreconditioned runs may drift by an iteration at the tolerance boundary
        assert abs(rep.iterations - int(want[0])) <= max(1, int(0.01 * want[0])), (key, rep.iterations, want)
        assert rep.converged == bool(want[3])
        assert rel_err(x, g[f"{tag}{key}_x"]) <= 1e-6


def test_pcg_breakdown_and_zero_rhs(rng):
    case, grid, _ = _cantilever(8, 4, 4)
    st = vb.OperatorState(grid, np.full(grid.n_elements, 0.5), vb.MaterialModel(), case.fixed_mask)
    x, rep = vb.pcg(st, None, np.zeros(grid.n_dofs), u0=rng.standard_normal(grid.n_dofs))
    assert rep.converged and rep.iterations == 0
    assert np.all(x[st.fixed_idx] == 0.0)
    with pytest.raises(vb.SolverBreakdown, match="SPD"):
        vb.pcg(st, lambda r: -r, case.f_ext * (~case.fixed_mask))
    bad = np.zeros(grid.n_dofs)
    bad[5] = np.nan
    with pytest.raises(vb.SolverBreakdown):
        vb.pcg(st, None, bad)
    f = case.f_ext * (~case.fixed_mask)
    x, rep = vb.pcg(st, None, f, cfg=vb.SolverConfig(tolerance=1e-12, max_iterations=3))
    assert not rep.converged and rep.iterations == 3


def test_design_kernels_match_reference():
    g = golden("design.npz")
    grid = vb.build_grid(12, 6, 5, 0.75)
    st = vb.OperatorState(grid, g["rho"], vb.MaterialModel(), face_fixed_mask(12, 6, 5),
                          vb.unit_stiffness(0.3, 0.75))
    assert rel_err(vb.sensitivities(st, g["u"]), g["dc"]) <= 1e-12
    grav = vb.GravitySpec(axis=2, g=9.81, unit_weight=0.7)
    assert rel_err(vb.sensitivities(st, g["u"], grav), g["dcg"]) <= 1e-12
    regions = vb.classify_regions(grid, [])
    fld = vb.DensityField(g["rho"], regions)
    assert np.array_equal(vb.update_gravity_load(grid, fld, grav, g["f_ext"], st.fixed_idx), g["fgrav"])
    assert np.array_equal(vb.update_gravity_load(grid, fld, grav), g["fgrav_plain"])
    for tag, r in (("r15", 1.5 * 0.75), ("r25", 2.5 * 0.75), ("r18", 1.8 * 0.75)):
        w = vb.build_filter(grid, r)
        assert np.array_equal(w.kernel, g[f"{tag}_kernel"])
        assert np.array_equal(w.wsum, g[f"{tag}_wsum"])
        out = vb.filter_sensitivities(g["dcin"], g["rho"], w, 1e-3)
        assert np.array_equal(out, g[f"{tag}_dcf"])
    reg = vb.RegionMask(g["oc_classes"])
    for tag, kw in (("a", dict(volfrac=0.3)), ("b", dict(volfrac=0.3, move=0.1, q=2.0)), ("c", dict(volfrac=0.25, eta=0.3))):
        res = vb.oc_update(vb.DensityField(g["oc_x0"], reg), g["dcin"], np.ones(grid.n_elements),
                           vb.OptConfig(filter_radius=1.0, **kw))
        assert res.bisection_steps == int(g[f"oc{tag}_steps"])
        assert abs(res.lam - float(g[f"oc{tag}_lam"])) <= 1e-12 * abs(float(g[f"oc{tag}_lam"]))
        assert np.abs(res.densities.values - g[f"oc{tag}_rho"]).max() <= 1e-12


def test_oc_infeasible_raises():
    grid = vb.build_grid(2, 2, 2, 1.0)
    rho = vb.DensityField(np.full(8, 0.1), vb.classify_regions(grid, []))
    with pytest.raises(vb.VolumeInfeasible):
        vb.oc_update(rho, -np.ones(8), np.ones(8), vb.OptConfig(volfrac=0.9, filter_radius=1.0, move=0.1))


def _ref_envelope(fixture, key, want):
    """The reference's own compliance spread on a default-tolerance trajectory:
    max over the re-runs at 1/2/3/4/8 OpenBLAS threads (oracle/ref_self_variation*.py)
    of the relative distance to the fixture it was made from (8 threads)."""
    sv = golden(fixture)
    return max(float(np.max(np.abs(sv[f"{key}_t{t}"][:, 1] - want[:, 1]) / np.abs(want[:, 1])))
               for t in sv["threads"])


def _default_tol_bar(env):
    """North-star 1e-6, widened to twice the reference's own measured spread
    where the reference cannot meet 1e-6 against itself (the spread is sampled
    from five thread counts, so it is a lower bound)."""
    return max(1e-6, 2.0 * env)


def _traj_check(res, want, rho_ref, c_tol=1e-6, rho_tol=1e-4, res_tol=1e-5, cg_rel=0.05):
    """Trajectory bars: compliance <= c_tol relative on every iteration (the
    north-star 1e-6 by default), rho <= rho_tol max-abs, same volume, residual
    below the solve tolerance, CG counts within a few percent.  Under the tight
    protocol (both sides' solves converged to 1e-10, the *_tight tests) the
    trajectories no longer depend on rounding order (measured ~1e-10).  At the
    reference default tolerance the bar is _default_tol_bar of the reference's
    own measured spread (tests/golden/selfvar_*.npz)."""
    recs = res.records
    assert len(recs) == want.shape[0]
    for r, w in zip(recs, want):
        assert r.iteration == int(w[0])
        assert abs(r.cg_iters - int(w[4])) <= max(2, int(cg_rel * w[4])), (r.iteration, r.cg_iters, w[4])
        assert abs(r.compliance - w[1]) <= c_tol * abs(w[1]), (r.iteration, r.compliance, w[1], r.cg_iters, w[4])
        assert abs(r.volume - w[2]) <= 2e-6
        assert r.aux_scalars == int(w[6])
        assert r.cg_residual <= res_tol
    assert np.abs(res.densities.values - rho_ref).max() <= rho_tol


def test_small_trajectory_matches_reference():
    g = golden("small_traj.npz")
    case, grid, prob = _cantilever(16, 8, 8)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=2.5 * grid.h, max_iterations=30, ch_tol=1e-12)
    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-5), scheme="homogenized", max_levels=3)
    _traj_check(res, g["recs"], g["rho30"],
                c_tol=_default_tol_bar(_ref_envelope("selfvar_small.npz", "small", g["recs"])))


def test_small_tight_trajectory_matches_reference():
    """North-star bars under the SURVEY 8(d) protocol: both sides converge every
    solve to 1e-10, so the trajectory no longer depends on rounding order and
    compliance must agree to <= 1e-6 (measured ~1e-10), rho to <= 1e-4."""
    g = golden("small_tight.npz")
    case, grid, prob = _cantilever(16, 8, 8)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=2.5 * grid.h, max_iterations=30, ch_tol=1e-12)
    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-10, max_iterations=1000), scheme="homogenized",
                 max_levels=3)
    want = g["recs"]
    worst = max(abs(r.compliance - w[1]) / abs(w[1]) for r, w in zip(res.records, want))
    print(f"small tight: worst compliance rel diff {worst:.2e}")
    _traj_check(res, want, g["rho30"], c_tol=1e-6, rho_tol=1e-4, res_tol=1e-10)


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "cfg1_tight.npz")), reason="cfg1 tight fixture missing")
def test_cfg1_tight_trajectory_parity():
    """BASELINE config 1 (48x24x24, p=3, rmin=1.5h, 4-level homogenized MG, 40 SIMP
    iterations) against the reference run with every solve converged to 1e-10:
    compliance <= 1e-6 relative per iteration, rho <= 1e-4 after 20 and 40."""
    g = golden("cfg1_tight.npz")
    case, grid, prob = _cantilever(48, 24, 24)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, p=3.0, max_iterations=40, ch_tol=1e-12)
    seen = {}

    def hook(rec, rho, u):
        if rec.iteration in (20, 40):
            seen[rec.iteration] = rho.values.copy()

    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-10, max_iterations=1000), scheme="homogenized",
                 max_levels=4, on_iteration=hook)
    want = g["recs"]
    worst = max(abs(r.compliance - w[1]) / abs(w[1]) for r, w in zip(res.records, want))
    print(f"cfg1 tight: worst compliance rel diff {worst:.2e}, "
          f"rho20 {np.abs(seen[20] - g['rho20']).max():.2e}, rho40 {np.abs(seen[40] - g['rho40']).max():.2e}")
    # 300+ CG iterations at 1e-10: finite-precision CG loses orthogonality and the
    # count itself becomes rounding-dependent (the design does not: c ~1e-10)
    _traj_check(res, want, g["rho40"], c_tol=1e-6, rho_tol=1e-4, res_tol=1e-10, cg_rel=0.10)
    assert np.abs(seen[20] - g["rho20"]).max() <= 1e-4


def test_tight_tolerance_trajectory_matches_oracle():
    """SURVEY 8(d) fallback protocol: both sides at tol 1e-10 make the design
    trajectory preconditioner- and rounding-independent (CPU oracle on the box)."""
    case, grid, prob = _cantilever(16, 8, 8)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, max_iterations=8, ch_tol=1e-12)
    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-10, max_iterations=1000), scheme="homogenized",
                 max_levels=3)
    rho, u, recs = O.run_design(case, 0.12, 1.5 * case.h, 8, tol=1e-10, maxit=1000, max_levels=3,
                                ch_tol=1e-12)
    for r, w in zip(res.records, recs):
        assert abs(r.compliance - w.compliance) <= 1e-9 * abs(w.compliance)
        assert abs(r.cg_iters - w.cg_iters) <= 2
    assert np.abs(res.densities.values - rho).max() <= 1e-7


def test_bridge_trajectory_matches_reference():
    g = golden("bridge_traj.npz")
    case = O.bridge_case(32, 16, 16)
    grid = vb.build_grid(32, 16, 16, case.h)
    loads = [(int(d), float(case.f_ext[d])) for d in np.flatnonzero(case.f_ext)]
    bnd = vb.make_boundary(grid, np.flatnonzero(case.fixed_mask), loads)
    Lx, Ly, Lz = grid.domain
    reg = vb.classify_regions(grid, [(vb.Box((0, 0, Lz - grid.h), (Lx, Ly, Lz)), vb.Region.PASSIVE_SOLID)])
    assert np.array_equal(reg.classes, case.classes)
    opt = vb.OptConfig(volfrac=0.14, filter_radius=1.5 * grid.h, max_iterations=3, ch_tol=1e-12)
    res = vb.run(vb.Problem(grid, bnd, reg), opt, vb.SolverConfig(tolerance=1e-5), scheme="homogenized")
    _traj_check(res, g["recs"], g["rho3"],
                c_tol=_default_tol_bar(_ref_envelope("selfvar_small.npz", "bridge", g["recs"])))


def test_gravity_trajectory_and_failure():
    g = golden("grav_traj.npz")
    case, grid, prob = _cantilever(32, 16, 16, gravity=(2, 1.0, 1e-3))
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, max_iterations=4, ch_tol=1e-12)
    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-5), scheme="homogenized")
    _traj_check(res, g["recs"], g["rho4"],
                c_tol=_default_tol_bar(_ref_envelope("selfvar_small.npz", "grav", g["recs"])))
    info = json.load(open(os.path.join(GOLDEN, "grav_fail.json")))
    case, grid, prob = _cantilever(32, 16, 16, gravity=(2, 1.0, 1.0))
    seen = []
    with pytest.raises(vb.VolumeInfeasible):
        vb.run(prob, opt, vb.SolverConfig(tolerance=1e-5), scheme="homogenized",
               on_iteration=lambda r, a, b: seen.append(r.compliance))
    assert info["raised"] == "VolumeInfeasible"
    assert len(seen) == len(info["compliance"])
    assert abs(seen[0] - info["compliance"][0]) <= 1e-9 * abs(seen[0])


@pytest.mark.skipif(not os.path.exists(os.path.join(GOLDEN, "cfg1_traj.npz")), reason="cfg1 fixture missing")
def test_cfg1_trajectory_parity():
    """BASELINE config 1: 48x24x24 cantilever, p=3, rmin=1.5h, 4-level homogenized MG,
    40 SIMP iterations at the reference's default tolerance (1e-5).

    Bar: the north-star 1e-6 compliance / 1e-4 density wherever the reference
    itself is reproducible to that level, and otherwise the reference's OWN
    spread: tests/golden/cfg1_selfvar.npz holds the real reference re-run with
    1, 2, 3, 4 and 8 OpenBLAS threads (8 = the fixture's, bit-identical).  With
    2 threads the reference moves by 3.2e-5 in compliance at iterations 9-11
    and 3.6e-5 in density at iteration 20: a solve stopped at a relative
    residual of 1e-5 does not pin the compliance of those iterations closer
    than that.  The GPU must stay inside twice that
    envelope on every iteration (_default_tol_bar)."""
    g = golden("cfg1_traj.npz")
    sv = golden("cfg1_selfvar.npz")
    want = g["recs"]
    env_c = max(float(np.max(np.abs(sv[f"recs_t{t}"][:, 1] - want[:, 1]) / np.abs(want[:, 1])))
                for t in sv["threads"])
    c_bar = _default_tol_bar(env_c)
    rho_bar = max(1e-4, 2.0 * float(sv["rho20_env"]))
    case, grid, prob = _cantilever(48, 24, 24)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, p=3.0, max_iterations=40, ch_tol=1e-12)
    seen = {}

    def hook(rec, rho, u):
        if rec.iteration in (20, 40):
            seen[rec.iteration] = rho.values.copy()

    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-5), scheme="homogenized", max_levels=4,
                 on_iteration=hook)
    worst_c = max(abs(r.compliance - w[1]) / abs(w[1]) for r, w in zip(res.records, want))
    same_its = sum(int(r.cg_iters == int(w[4])) for r, w in zip(res.records, want))
    print(f"cfg1: worst compliance rel diff {worst_c:.2e} (reference self-variation envelope {env_c:.2e}), "
          f"equal CG counts {same_its}/40, rho20 {np.abs(seen[20] - g['rho20']).max():.2e}, "
          f"rho40 {np.abs(seen[40] - g['rho40']).max():.2e}")
    _traj_check(res, want, g["rho40"], c_tol=c_bar, rho_tol=rho_bar)
    assert np.abs(seen[20] - g["rho20"]).max() <= rho_bar


def test_pcg_graph_not_reused_across_hierarchies():
    """The per-grid PCG iteration graph is keyed by the hierarchy's identity, not
    its address: a hierarchy destroyed and rebuilt (often at the same address,
    with different device buffers and level count) must trigger a recapture."""
    import gc

    case, grid, prob = _cantilever(16, 8, 8)
    rng = np.random.default_rng(11)
    rho = rng.uniform(0.05, 1.0, grid.n_elements)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    f = case.f_ext.copy()
    f[case.fixed_mask] = 0.0
    cfg = vb.SolverConfig(tolerance=1e-8, max_iterations=300)
    k0 = O.hex8_k0(0.3, case.h)
    scale = O.simp(rho, 3.0, 1e-9)
    fixed = np.flatnonzero(case.fixed_mask)
    for levels in (2, 3, 2, 3):
        H = vb.build_hierarchy(grid, st, levels, scheme="homogenized")
        x, rep = vb.mgcg_solve(st, H, f, cfg=cfg)
        OH = O.hier_build(case.es, case.h, case.fixed_mask, levels)
        O.hier_refresh(OH, rho, scale, k0, 3.0, 1e-9, 1.0)
        xo, ro = O.pcg(lambda p: O.apply_k(p, case.es, fixed, k0, scale),
                       lambda p, ff: O.resid_k(p, ff, case.es, fixed, k0, scale),
                       lambda r: O.vcycle(OH, r), f, None, fixed, 1e-8, 300)
        assert rep.iterations == ro.iterations, (levels, rep.iterations, ro.iterations)
        assert rel_err(x, xo) <= 1e-7
        del H
        gc.collect()
