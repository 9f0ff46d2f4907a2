"""Z-slab decomposition on one GPU: all slabs in one process,
halos by device copies -- the same planes, order and arithmetic the NCCL
transport uses across GPUs.  The distributed operator / V-cycle / MGPCG must
reproduce the single-slab path (which is pinned to the reference goldens)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_2201_12931_b200")
from paper_2201_12931_b200.slabs import SlabSolver, plan_slabs  # noqa: E402
from oracle import cpu_path as O  # noqa: E402


def _setup(nx, ny, nz, seed=0):
    case = O.cantilever_case(nx, ny, nz)
    grid = vb.build_grid(nx, ny, nz, case.h)
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.05, 1.0, grid.n_elements)
    return case, grid, rho, rng


@pytest.mark.parametrize("nranks", [2, 4])
def test_slab_apply_matches_single(nranks):
    case, grid, rho, rng = _setup(32, 16, 16)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    S = SlabSolver(grid, case.fixed_mask, levels=4, nranks=nranks)
    S.set_density(rho, refresh=False)
    u = rng.standard_normal(grid.n_dofs)
    u[case.fixed_mask] = 0.0
    ref = vb.apply(st, u)
    ref[case.fixed_mask] = 0.0  # solver-internal apply: zero on fixed
    got = S.download(S.apply(S.upload(u)))
    assert np.abs(got - ref).max() <= 1e-15 * np.abs(ref).max()


@pytest.mark.parametrize("nranks", [2, 4])
def test_slab_vcycle_matches_single(nranks):
    case, grid, rho, rng = _setup(32, 16, 16, seed=1)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    H = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
    S = SlabSolver(grid, case.fixed_mask, levels=4, nranks=nranks)
    S.set_density(rho)
    r = rng.standard_normal(grid.n_dofs)
    r[case.fixed_mask] = 0.0
    ref = H.v_cycle(r)
    got = S.download(S.v_cycle(S.upload(r)))
    assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_slab_mgcg_matches_single(nranks):
    """1-GPU vs k-slab MGPCG: same iteration count, iterates within 1e-10 (the
    rank-ordered dot products round differently from the single-slab tree)."""
    case, grid, rho, rng = _setup(32, 16, 32, seed=2)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    H = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
    f = case.f_ext.copy()
    f[case.fixed_mask] = 0.0
    cfg = vb.SolverConfig(tolerance=1e-8, max_iterations=300)
    x_ref, rep_ref = vb.mgcg_solve(st, H, f, cfg=cfg)
    S = SlabSolver(grid, case.fixed_mask, levels=4, nranks=nranks)
    S.set_density(rho)
    x, rep = S.mgcg_solve(S.upload(f), cfg=cfg)
    got = S.download(x)
    assert rep.converged and rep.iterations == rep_ref.iterations, (rep, rep_ref)
    assert abs(rep.final_rel_residual - rep_ref.final_rel_residual) <= 1e-6 * rep_ref.final_rel_residual
    assert np.abs(got - x_ref).max() <= 1e-10 * np.abs(x_ref).max()
    # warm start from the solution converges immediately, like the reference
    x2, rep2 = S.mgcg_solve(S.upload(f), u_prev=x, cfg=cfg)
    assert rep2.converged and rep2.iterations == 0


def test_slab_plan_of_baseline_configs():
    # cfg2 / cfg3 / cfg5 on 8 GPUs: balanced slabs, deep distributed hierarchy
    p = plan_slabs(128, 7, 8)
    assert p.dist_level == 4 and p.bounds[1] == 16
    p = plan_slabs(256, 8, 8)
    assert p.dist_level == 5 and p.bounds[1] == 32
    p = plan_slabs(384, 8, 8)
    assert p.dist_level == 4 and p.bounds[1] == 48


def test_nccl_transport_single_rank_matches_single():
    """The NCCL code path (library-owned communicator bootstrapped over a
    torch.distributed group, all-gathers / broadcasts captured in the iteration
    graph) at world size 1 -- the only size one GPU allows -- solves like the
    single-slab path."""
    import os
    import socket

    import torch.distributed as dist

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        case, grid, rho, rng = _setup(32, 16, 16, seed=3)
        st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
        H = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
        f = case.f_ext.copy()
        f[case.fixed_mask] = 0.0
        cfg = vb.SolverConfig(tolerance=1e-8, max_iterations=300)
        x_ref, rep_ref = vb.mgcg_solve(st, H, f, cfg=cfg)
        S = SlabSolver.from_process_group(grid, case.fixed_mask, levels=4)
        S.set_density(rho)
        x, rep = S.mgcg_solve(S.upload(f), cfg=cfg)
        assert rep.converged and rep.iterations == rep_ref.iterations
        assert np.abs(S.download(x) - x_ref).max() <= 1e-10 * np.abs(x_ref).max()
        S.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nranks", [2, 4])
def test_slab_design_loop_matches_single(nranks):
    """The whole SIMP loop on slabs (solve, sensitivities with the u halo, filter
    with R-layer halos, OC with rank-ordered sums) against run() on one slab,
    both with tight solves: same trajectory to rounding."""
    from paper_2201_12931_b200 import cases
    from paper_2201_12931_b200.slabs import run_slabs

    prob = cases.cantilever(32, 16, 16)
    for radius in (1.5, 2.5):
        opt = vb.OptConfig(volfrac=0.12, filter_radius=radius * prob.grid.h, max_iterations=6, ch_tol=1e-12)
        cfg = vb.SolverConfig(tolerance=1e-10, max_iterations=1000)
        ref = vb.run(prob, opt, cfg, scheme="homogenized", max_levels=4)
        got = run_slabs(prob, opt, cfg, max_levels=4, nranks=nranks)
        for a, b in zip(got.records, ref.records):
            assert abs(a.compliance - b.compliance) <= 1e-9 * abs(b.compliance), (a, b)
            assert abs(a.volume - b.volume) <= 1e-9
            assert a.aux_scalars == b.aux_scalars
        assert np.abs(got.densities.values - ref.densities.values).max() <= 1e-8
        assert np.abs(got.displacement - ref.displacement).max() <= 1e-8 * np.abs(ref.displacement).max()


def test_slab_filter_bit_identical():
    """R-layer halo filter on 4 slabs == the single-GPU filter, bit for bit."""
    import ctypes as C

    import torch

    from paper_2201_12931_b200.design import filter_weights
    from paper_2201_12931_b200.slabs import _ptr_array

    case, grid, rho, rng = _setup(16, 8, 16, seed=5)
    S = SlabSolver(grid, case.fixed_mask, levels=3, nranks=4)
    dc = -rng.uniform(0.0, 1.0, grid.n_elements)
    for radius in (1.5, 2.5):
        w = vb.build_filter(grid, radius * grid.h)
        ref = vb.filter_sensitivities(dc, rho, w, 1e-3)
        R, kern = filter_weights(grid.h, radius * grid.h)
        from paper_2201_12931_b200._lib import lib
        from paper_2201_12931_b200.device import stream_ptr

        assert lib.vt_dist_filter_create(S._h, R, kern.ctypes.data_as(C.c_void_p)) == 0
        rs, ds = S._slab_rho(rho), S._slab_rho(dc)
        out = [torch.empty_like(r) for r in rs]
        assert lib.vt_dist_filter_apply(S._h, _ptr_array(ds), _ptr_array(rs), 1e-3, _ptr_array(out),
                                        stream_ptr()) == 0
        got = torch.cat(out).cpu().numpy()
        assert np.array_equal(got, ref), radius


def test_slab_design_loop_with_self_weight():
    """Design-dependent (self-weight) load on slabs: the load lumping reads the
    element layer below each slab (exchanged), sensitivities carry 2 u.g."""
    from paper_2201_12931_b200 import cases
    from paper_2201_12931_b200.slabs import run_slabs

    prob = cases.selfweight(32, 16, 16, 1e-3)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * prob.grid.h, max_iterations=4, ch_tol=1e-12)
    cfg = vb.SolverConfig(tolerance=1e-10, max_iterations=1000)
    ref = vb.run(prob, opt, cfg, scheme="homogenized", max_levels=4)
    got = run_slabs(prob, opt, cfg, max_levels=4, nranks=4)
    for a, b in zip(got.records, ref.records):
        assert abs(a.compliance - b.compliance) <= 1e-9 * abs(b.compliance), (a, b)
    assert np.abs(got.densities.values - ref.densities.values).max() <= 1e-8


# ---------------------------------------------------------------- Galerkin (the reference default) on slabs
@pytest.mark.parametrize("nranks", [2, 4])
def test_galerkin_slab_vcycle_matches_single(nranks):
    """Galerkin V-cycle on slabs (levels 0/1 distributed, level 1 matrix-free,
    stored-matrix tail replicated) against the single-GPU Galerkin V-cycle."""
    case, grid, rho, rng = _setup(32, 16, 16, seed=4)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    H = vb.build_hierarchy(grid, st, 4, scheme="galerkin")
    S = SlabSolver(grid, case.fixed_mask, levels=4, nranks=nranks, scheme="galerkin")
    assert S.plan.dist_level == 1
    S.set_density(rho)
    r = rng.standard_normal(grid.n_dofs)
    r[case.fixed_mask] = 0.0
    ref = H.v_cycle(r)
    got = S.download(S.v_cycle(S.upload(r)))
    assert np.abs(got - ref).max() <= 1e-14 * np.abs(ref).max()


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_galerkin_slab_mgcg_matches_single(nranks):
    case, grid, rho, rng = _setup(32, 16, 32, seed=5)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    H = vb.build_hierarchy(grid, st, 4, scheme="galerkin")
    f = case.f_ext.copy()
    f[case.fixed_mask] = 0.0
    cfg = vb.SolverConfig(tolerance=1e-8, max_iterations=300)
    x_ref, rep_ref = vb.mgcg_solve(st, H, f, cfg=cfg)
    S = SlabSolver(grid, case.fixed_mask, levels=4, nranks=nranks, scheme="galerkin")
    S.set_density(rho)
    x, rep = S.mgcg_solve(S.upload(f), cfg=cfg)
    assert rep.converged and rep.iterations == rep_ref.iterations, (rep, rep_ref)
    assert np.abs(S.download(x) - x_ref).max() <= 1e-10 * np.abs(x_ref).max()


def test_galerkin_slab_design_loop_matches_single():
    """run_slabs(scheme="galerkin") against run() with the reference's default
    scheme, tight solves: same trajectory to rounding."""
    from paper_2201_12931_b200 import cases
    from paper_2201_12931_b200.slabs import run_slabs

    prob = cases.cantilever(32, 16, 16)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * prob.grid.h, max_iterations=5, ch_tol=1e-12)
    cfg = vb.SolverConfig(tolerance=1e-10, max_iterations=1000)
    ref = vb.run(prob, opt, cfg, scheme="galerkin", max_levels=4)
    got = run_slabs(prob, opt, cfg, max_levels=4, nranks=2, scheme="galerkin")
    for a, b in zip(got.records, ref.records):
        assert abs(a.compliance - b.compliance) <= 1e-9 * abs(b.compliance), (a, b)
        assert a.aux_scalars == b.aux_scalars
    assert np.abs(got.densities.values - ref.densities.values).max() <= 1e-8


def test_galerkin_slab_plan_needs_even_layers():
    case, grid, rho, rng = _setup(16, 8, 8)
    with pytest.raises(ValueError, match="even number"):
        SlabSolver(grid, case.fixed_mask, levels=3, nranks=8, scheme="galerkin")


@pytest.mark.parametrize("scheme", ["homogenized", "galerkin"])
def test_two_material_slabs_match_single(scheme):
    """Two-material SIMP (BASELINE cfg4's extension) on 2 slabs against the
    single-GPU run_two_material, tight solves."""
    from paper_2201_12931_b200 import cases
    from paper_2201_12931_b200.multimaterial import run_two_material, run_two_material_slabs

    prob = cases.cantilever(32, 16, 16)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * prob.grid.h, max_iterations=4, ch_tol=1e-12)
    cfg = vb.SolverConfig(tolerance=1e-10, max_iterations=1000)
    ref = run_two_material(prob, opt, phase_frac=0.5, e_ratio=0.5, solver=cfg, scheme=scheme, max_levels=4)
    got = run_two_material_slabs(prob, opt, phase_frac=0.5, e_ratio=0.5, solver=cfg, scheme=scheme,
                                 max_levels=4, nranks=2)
    for a, b in zip(got.records, ref.records):
        assert abs(a.compliance - b.compliance) <= 1e-9 * abs(b.compliance), (a, b)
        assert abs(a.phase_volume - b.phase_volume) <= 1e-9
    assert np.abs(got.densities.values - ref.densities.values).max() <= 1e-8
    assert np.abs(got.phases.values - ref.phases.values).max() <= 1e-8
