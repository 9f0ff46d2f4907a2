"""Fused coarse tail (csrc/tail.cu): the V-cycle levels from the first one
with at most vt_tail_config() nodes down to the coarsest solve and back run as
one thread-block-cluster kernel (an option, off by default: measured slower
than the PDL kernel chain).  Checked against the multi-kernel V-cycle of
the same hierarchy (tail disabled): bit-identical for the Galerkin scheme (same
element products, corner-order node sums, transfers and coarse mat-vecs),
within 1e-12 for the homogenized one (the tile kernel sums the element
products in another order), and with the tail on against the reference's
own V-cycle fixtures (tests/golden/multigrid.npz, galerkin.npz)
[ref: multigrid.py:404-430]."""

import contextlib

import numpy as np
import pytest

from conftest import face_fixed_mask, golden, rel_err

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_2201_12931_b200")
from paper_2201_12931_b200._lib import lib  # noqa: E402


@contextlib.contextmanager
def tail_nodes(n):
    prev = lib.vt_tail_config(n)
    try:
        yield
    finally:
        lib.vt_tail_config(prev)


def _setup(dims, levels, scheme, nu, seed=7):
    rng = np.random.default_rng(seed)
    grid = vb.build_grid(*dims, 1.0)
    fm = face_fixed_mask(*dims)
    st = vb.OperatorState(grid, rng.uniform(0.05, 1.0, grid.n_elements), vb.MaterialModel(), fm,
                          vb.unit_stiffness(0.3, 1.0))
    f = rng.standard_normal(grid.n_dofs)
    f[fm] = 0.0
    return grid, st, f, dict(max_levels=levels, scheme=scheme, nu_pre=nu, nu_post=nu)


CASES = [((64, 32, 32), 5, "homogenized", 1), ((64, 32, 32), 5, "galerkin", 1),
         ((32, 16, 16), 4, "homogenized", 2), ((32, 16, 16), 4, "galerkin", 2),
         ((48, 24, 24), 4, "homogenized", 1)]


@pytest.mark.parametrize("dims,levels,scheme,nu", CASES)
def test_tail_matches_multikernel_vcycle(dims, levels, scheme, nu):
    grid, st, f, kw = _setup(dims, levels, scheme, nu)
    with tail_nodes(0):
        H0 = vb.build_hierarchy(grid, st, **kw)
        assert lib.vt_hier_tail_level(H0._h) == -1
        z0 = H0.v_cycle(f)
    with tail_nodes(12000):
        H1 = vb.build_hierarchy(grid, st, **kw)
        t = lib.vt_hier_tail_level(H1._h)
        assert 1 <= t < H1.n_levels
        l0 = vb.launch_count()
        z1 = H1.v_cycle(f)
        fused_launches = vb.launch_count() - l0
    l0 = vb.launch_count()
    H0.v_cycle(f)
    assert fused_launches < vb.launch_count() - l0
    if scheme == "galerkin":
        assert np.array_equal(z1, z0)
    else:
        assert rel_err(z1, z0) <= 1e-12
    assert np.array_equal(H1.v_cycle(f), z1)  # deterministic


@pytest.mark.parametrize("scheme", ["homogenized", "galerkin"])
def test_tail_whole_cycle_and_solve(scheme):
    """A budget that covers every level below the fine one (tail from level 1
    homogenized / 2 galerkin), then MGCG with and without the tail."""
    grid, st, f, kw = _setup((32, 16, 16), 4, scheme, 1, seed=3)
    with tail_nodes(1 << 30):
        H1 = vb.build_hierarchy(grid, st, **kw)
        assert lib.vt_hier_tail_level(H1._h) == (1 if scheme == "homogenized" else 2)
        x1, r1 = vb.mgcg_solve(st, H1, f, cfg=vb.SolverConfig(tolerance=1e-8, max_iterations=300))
    with tail_nodes(0):
        H0 = vb.build_hierarchy(grid, st, **kw)
        x0, r0 = vb.mgcg_solve(st, H0, f, cfg=vb.SolverConfig(tolerance=1e-8, max_iterations=300))
    assert r1.converged and r0.converged
    assert abs(r1.iterations - r0.iterations) <= (0 if scheme == "galerkin" else 1)
    assert rel_err(x1, x0) <= 1e-7
    if scheme == "galerkin":
        assert np.array_equal(x1, x0)


def test_tail_coarsest_only():
    """A budget only the coarsest level meets: the tail is the direct solve alone."""
    grid, st, f, kw = _setup((32, 16, 16), 3, "homogenized", 1, seed=5)
    coarsest = (32 // 4 + 1) * (16 // 4 + 1) * (16 // 4 + 1)
    with tail_nodes(coarsest):
        H1 = vb.build_hierarchy(grid, st, **kw)
        assert lib.vt_hier_tail_level(H1._h) == 2
        z1 = H1.v_cycle(f)
    with tail_nodes(0):
        z0 = vb.build_hierarchy(grid, st, **kw).v_cycle(f)
    assert np.array_equal(z1, z0)


@pytest.mark.parametrize("fixture,scheme,tags,bar", [("multigrid.npz", "homogenized", ["t", "v", "w"], 1e-10),
                                                     ("galerkin.npz", "galerkin", ["t", "v", "x"], 1e-11)])
def test_tail_vcycle_matches_reference_fixtures(fixture, scheme, tags, bar):
    g = golden(fixture)
    for tag in tags:
        dims = tuple(int(x) for x in g[f"{tag}_dims"])
        grid = vb.build_grid(*dims, 1.0)
        kw = {} if scheme == "homogenized" else {"stiffness": vb.unit_stiffness(0.3, 1.0)}
        st = vb.OperatorState(grid, g[f"{tag}_rho"], vb.MaterialModel(), face_fixed_mask(*dims), **kw)
        with tail_nodes(1 << 30):
            H = vb.build_hierarchy(grid, st, int(g[f"{tag}_levels"]), scheme=scheme)
            used = lib.vt_hier_tail_level(H._h) >= 1
        assert used or H.n_levels <= (1 if scheme == "homogenized" else 2), tag
        assert rel_err(H.v_cycle(g[f"{tag}_f"]), g[f"{tag}_z"]) <= bar, tag
