"""The one-launch coarse tail of the homogenized V-cycle (csrc/tail.cu) against
the kernel-per-pass V-cycle it replaces: same arithmetic operation for
operation, so the V-cycle output -- and a whole MGCG solve -- must be
bit-identical (VT_TAIL=0 switches the tail off; the variable is read at every
V-cycle build).  Parity with the reference goes through the default (tail on)
path in test_gpu_operator / test_gpu_solver."""

import os

import numpy as np
import pytest

from conftest import rel_err

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_2201_12931_b200")
from oracle import cpu_path as O  # noqa: E402


def _setup(nx, ny, nz, levels, seed=3):
    case = O.cantilever_case(nx, ny, nz)
    grid = vb.build_grid(nx, ny, nz, case.h)
    rng = np.random.default_rng(seed)
    rho = rng.uniform(0.01, 1.0, grid.n_elements)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
    f = rng.standard_normal(grid.n_dofs)
    f[case.fixed_mask] = 0.0
    return case, grid, st, f


def _vcycle(st, grid, levels, f, tail):
    os.environ["VT_TAIL"] = "1" if tail else "0"
    try:
        H = vb.build_hierarchy(grid, st, levels, scheme="homogenized")
        l0 = vb.launch_count()
        z = H.v_cycle(f)
        return z, vb.launch_count() - l0, H
    finally:
        os.environ.pop("VT_TAIL", None)


@pytest.mark.parametrize("dims,levels", [((16, 8, 8), 3), ((48, 24, 24), 4), ((64, 32, 32), 5),
                                         ((256, 128, 128), 7)])
def test_tail_vcycle_bit_identical(dims, levels):
    case, grid, st, f = _setup(*dims, levels)
    z1, n1, _ = _vcycle(st, grid, levels, f, True)
    z0, n0, _ = _vcycle(st, grid, levels, f, False)
    assert n1 < n0, (n1, n0)  # the tail replaced launches
    assert np.array_equal(z1, z0), rel_err(z1, z0)


def test_tail_mgcg_bit_identical():
    case, grid, st, f = _setup(48, 24, 24, 4)
    out = {}
    for tail in (True, False):
        os.environ["VT_TAIL"] = "1" if tail else "0"
        try:
            H = vb.build_hierarchy(grid, st, 4, scheme="homogenized")
            x, rep = vb.mgcg_solve(st, H, f, cfg=vb.SolverConfig(tolerance=1e-8, max_iterations=300))
            out[tail] = (x, rep.iterations, rep.final_rel_residual)
        finally:
            os.environ.pop("VT_TAIL", None)
    assert out[True][1] == out[False][1]
    assert out[True][2] == out[False][2]
    assert np.array_equal(out[True][0], out[False][0])
