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
