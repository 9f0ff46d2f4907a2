"""Galerkin coarse operators (the reference's default multigrid scheme) on the
GPU against the reference fixtures tests/golden/galerkin*.npz
(mirrors pkg/tests/test_multigrid.py's galerkin cases)."""

import numpy as np
import pytest

from conftest import face_fixed_mask, golden, rel_err

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_2201_12931_b200")
from oracle import cpu_path as O  # noqa: E402


def _hier(g, tag):
    dims = tuple(int(x) for x in g[f"{tag}_dims"])
    grid = vb.build_grid(*dims, 1.0)
    st = vb.OperatorState(grid, g[f"{tag}_rho"], vb.MaterialModel(), face_fixed_mask(*dims),
                          vb.unit_stiffness(0.3, 1.0))
    H = vb.build_hierarchy(grid, st, int(g[f"{tag}_levels"]), scheme="galerkin")
    return grid, st, H


@pytest.mark.parametrize("tag", ["t", "v", "x"])
def test_galerkin_levels_match_reference(tag):
    g = golden("galerkin.npz")
    grid, st, H = _hier(g, tag)
    assert H.n_levels == int(g[f"{tag}_levels"])
    assert H.vector_scalars == int(g[f"{tag}_vector_scalars"])
    assert H.operator_scalars == int(g[f"{tag}_operator_scalars"])
    assert H.factor_scalars == int(g[f"{tag}_factor_scalars"])
    for l, lv in enumerate(H.levels):
        if l >= 1:
            want = g[f"{tag}_mats{l}"]
            got = lv.mats
            assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max(), l
            # stored as packed upper triangles: the expanded copy is exactly symmetric
            assert np.array_equal(got, got.transpose(0, 2, 1)), l
        assert rel_err(lv.diag, g[f"{tag}_diag{l}"]) <= 1e-13
    for l in range(1, H.n_levels):
        assert rel_err(H.coarse_apply(l, g[f"{tag}_cu{l}"]), g[f"{tag}_cv{l}"]) <= 1e-13
    assert rel_err(H.coarse_solve(g[f"{tag}_fL"]), g[f"{tag}_uL"]) <= 1e-11
    assert rel_err(H.v_cycle(g[f"{tag}_f"]), g[f"{tag}_z"]) <= 1e-11


@pytest.mark.parametrize("tag", ["t", "v", "x"])
def test_galerkin_mgcg_matches_reference(tag):
    g = golden("galerkin.npz")
    grid, st, H = _hier(g, tag)
    for ctag, tol, maxit in (("a", 1e-5, 200), ("b", 1e-10, 500)):
        x, rep = vb.mgcg_solve(st, H, g[f"{tag}_f"], cfg=vb.SolverConfig(tolerance=tol, max_iterations=maxit))
        want = g[f"{tag}{ctag}_rep"]
        assert abs(rep.iterations - int(want[0])) <= (1 if ctag == "b" else 0), (ctag, rep, want)
        assert rep.converged == bool(want[3])
        assert rep.aux_vector_scalars == int(want[4])
        assert rel_err(x, g[f"{tag}{ctag}_x"]) <= max(1e-8, 0.1 * tol)


def test_galerkin_trajectory_matches_reference():
    """run() with the reference's defaults (scheme="galerkin"), 16x8x8, 20 SIMP
    iterations: tight protocol (1e-10) at the north-star bars, default tolerance
    at the chaos-aware bars of test_gpu_solver._traj_check."""
    from test_gpu_solver import _cantilever, _traj_check

    g = golden("galerkin_traj.npz")
    case, grid, prob = _cantilever(16, 8, 8)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * grid.h, max_iterations=20, ch_tol=1e-12)
    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-10, max_iterations=1000), max_levels=3)
    worst = max(abs(r.compliance - w[1]) / abs(w[1]) for r, w in zip(res.records, g["recs_tight"]))
    print(f"galerkin tight: worst compliance rel diff {worst:.2e}")
    _traj_check(res, g["recs_tight"], g["rho20_tight"], c_tol=1e-6, res_tol=1e-10, cg_rel=0.10)
    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-5), max_levels=3)
    _traj_check(res, g["recs"], g["rho20"])
