"""CUDA operator / multigrid parity against the reference golden fixtures and
the oracle (mirrors pkg/tests/test_operator.py and test_multigrid.py)."""

import numpy as np
import pytest

from conftest import face_fixed_mask, golden, rel_err

pytestmark = pytest.mark.gpu

vb = pytest.importorskip("paper_2201_12931_b200")
from oracle import cpu_path as O  # noqa: E402


def _op_state(g, ci):
    dims = tuple(int(x) for x in g[f"c{ci}_dims"])
    h = float(g[f"c{ci}_h"])
    grid = vb.build_grid(*dims, h)
    st = vb.OperatorState(grid, g[f"c{ci}_rho"], vb.MaterialModel(), g[f"c{ci}_fixed"],
                          vb.unit_stiffness(0.3, h))
    return grid, st


def test_scale_matches_reference():
    g = golden("operator.npz")
    for ci in range(int(g["ncases"])):
        _, st = _op_state(g, ci)
        ref = g[f"c{ci}_scale"]
        # correctly-rounded rho^3 vs glibc pow: at most 1 ulp apart
        assert np.abs(st.scale - ref).max() <= 2.3e-16 * np.abs(ref).max()


def test_apply_diag_residual_match_reference():
    g = golden("operator.npz")
    for ci in range(int(g["ncases"])):
        grid, st = _op_state(g, ci)
        v = vb.apply(st, g[f"c{ci}_u"])
        assert rel_err(v, g[f"c{ci}_v"]) <= 1e-12, ci
        fx = g[f"c{ci}_fixed"]
        assert np.array_equal(v[fx], g[f"c{ci}_u"][fx])
        d = vb.diagonal(st)
        assert rel_err(d, g[f"c{ci}_d"]) <= 1e-15, ci
        r = vb.residual(st, g[f"c{ci}_u"], g[f"c{ci}_f"])
        assert rel_err(r, g[f"c{ci}_r"]) <= 1e-12, ci
        assert np.all(r[fx] == 0.0)


@pytest.mark.parametrize("dims", [(2, 1, 1), (3, 2, 2), (31, 15, 4), (32, 16, 3), (33, 17, 5),
                                  (62, 30, 7), (64, 5, 9), (7, 47, 3), (40, 33, 20)])
def test_apply_matches_oracle_tile_edges(dims, rng):
    """Sizes straddling the 31x15 tile and the z-chunking of the kernel."""
    grid = vb.build_grid(*dims, 0.7)
    rho = rng.uniform(0.0, 1.0, grid.n_elements)
    fixed = rng.choice(grid.n_dofs, size=grid.n_dofs // 10 + 3, replace=False)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), fixed, vb.unit_stiffness(0.3, 0.7))
    u = rng.standard_normal(grid.n_dofs)
    es = (dims[2], dims[1], dims[0])
    ref = O.apply_k(u, es, np.sort(fixed), O.hex8_k0(0.3, 0.7), O.simp(rho, 3.0, 1e-9))
    v = vb.apply(st, u)
    assert rel_err(v, ref) <= 1e-12


def test_apply_properties(rng):
    grid = vb.build_grid(12, 9, 7, 1.0)
    rho = rng.uniform(0.1, 1.0, grid.n_elements)
    st0 = vb.OperatorState(grid, rho, vb.MaterialModel(), np.zeros(grid.n_dofs, bool))
    t = np.zeros(grid.n_dofs)
    t[0::3] = 1.0
    assert np.abs(vb.apply(st0, t)).max() <= 1e-13  # translation nullspace
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), face_fixed_mask(12, 9, 7))
    a = rng.standard_normal(grid.n_dofs)
    b = rng.standard_normal(grid.n_dofs)
    a[st.fixed_idx] = 0
    b[st.fixed_idx] = 0
    x, y = vb.apply(st, a) @ b, a @ vb.apply(st, b)
    assert abs(x - y) <= 1e-12 * abs(x)  # symmetry
    assert vb.apply(st, a) @ a > 0
    v1, v2 = vb.apply(st, a), vb.apply(st, a)
    assert np.array_equal(v1, v2)  # bitwise determinism
    assert np.array_equal(vb.apply(st, np.zeros(grid.n_dofs)), np.zeros(grid.n_dofs))
    with pytest.raises(ValueError):
        vb.apply(st, np.zeros(5))


def _hier(g, tag):
    dims = tuple(int(x) for x in g[f"{tag}_dims"])
    grid = vb.build_grid(*dims, 1.0)
    st = vb.OperatorState(grid, g[f"{tag}_rho"], vb.MaterialModel(), face_fixed_mask(*dims))
    return st, vb.build_hierarchy(grid, st, int(g[f"{tag}_levels"]), scheme="homogenized")


@pytest.mark.parametrize("dims", [(264, 36, 12), (128, 16, 8), (4, 4, 4), (136, 72, 64)])
def test_transfers_bit_identical_across_blocks(dims):
    """Restriction / prolongation stay bit-identical to the axis passes when the
    coarse level spans several (row block, node block) units of the staged
    kernels (multigrid.py:341-371)."""
    nx, ny, nz = dims
    rng = np.random.default_rng(7)
    fm = face_fixed_mask(nx, ny, nz)
    grid = vb.build_grid(nx, ny, nz, 1.0)
    st = vb.OperatorState(grid, rng.uniform(0.1, 1.0, grid.n_elements), vb.MaterialModel(), fm)
    H = vb.build_hierarchy(grid, st, 4 if nz >= 64 else 3, scheme="homogenized")
    OH = O.hier_build((nz, ny, nx), 1.0, fm, H.n_levels)
    for l in range(H.n_levels - 1):
        rf = rng.standard_normal(H.levels[l].n_dofs)
        assert np.array_equal(H.restrict(l, rf), O.restrict(OH, l, rf)), l
        ec = rng.standard_normal(H.levels[l + 1].n_dofs)
        assert np.array_equal(H.prolongate(l, ec), O.prolong(OH, l, ec)), l


@pytest.mark.parametrize("tag", ["t", "v", "w"])
def test_multigrid_matches_reference(tag):
    g = golden("multigrid.npz")
    st, H = _hier(g, tag)
    assert H.n_levels == int(g[f"{tag}_levels"])
    assert H.vector_scalars == int(g[f"{tag}_vector_scalars"])
    assert H.operator_scalars == int(g[f"{tag}_operator_scalars"])
    assert H.factor_scalars == int(g[f"{tag}_factor_scalars"])
    for l, lv in enumerate(H.levels):
        assert np.array_equal(lv.fixed_idx, g[f"{tag}_fixed{l}"])
        ref = g[f"{tag}_scale{l}"]
        assert np.abs(lv.scale - ref).max() <= 2.3e-16 * np.abs(ref).max()
        assert rel_err(lv.diag, g[f"{tag}_diag{l}"]) <= 1e-15
    for l in range(H.n_levels - 1):
        # transfers: bit-identical to the reference's axis passes
        assert np.array_equal(H.restrict(l, g[f"{tag}_rf{l}"]), g[f"{tag}_rc{l}"])
        assert np.array_equal(H.prolongate(l, g[f"{tag}_ec{l}"]), g[f"{tag}_ef{l}"])
    for l in range(1, H.n_levels):
        assert rel_err(H.coarse_apply(l, g[f"{tag}_cu{l}"]), g[f"{tag}_cv{l}"]) <= 1e-12
    assert rel_err(H.coarse_solve(g[f"{tag}_fL"]), g[f"{tag}_uL"]) <= 1e-9
    assert rel_err(H.jacobi_smooth(0, g[f"{tag}_ju"], g[f"{tag}_f"], 2), g[f"{tag}_js"]) <= 1e-12
    assert rel_err(H.v_cycle(g[f"{tag}_f"]), g[f"{tag}_z"]) <= 1e-10


def test_vcycle_linear_symmetric_spd(rng):
    grid = vb.build_grid(16, 8, 8, 1.0)
    rho = rng.uniform(0.05, 1.0, grid.n_elements)
    st = vb.OperatorState(grid, rho, vb.MaterialModel(), face_fixed_mask(16, 8, 8))
    H = vb.build_hierarchy(grid, st, 3, scheme="homogenized")
    f1 = rng.standard_normal(grid.n_dofs)
    f2 = rng.standard_normal(grid.n_dofs)
    f1[st.fixed_idx] = 0
    f2[st.fixed_idx] = 0
    v1, v2 = H.v_cycle(f1), H.v_cycle(f2)
    lin = H.v_cycle(1.3 * f1 - 0.6 * f2) - 1.3 * v1 + 0.6 * v2
    assert np.abs(lin).max() <= 1e-12 * np.abs(v1).max()
    assert abs(v1 @ f2 - f1 @ v2) <= 1e-12 * abs(v1 @ f2)
    assert v1 @ f1 > 0
    assert np.array_equal(H.v_cycle(np.zeros(grid.n_dofs)), np.zeros(grid.n_dofs))


def test_setup_errors():
    grid = vb.build_grid(4, 4, 4, 1.0)
    mask = np.zeros(grid.n_dofs, bool)
    for node in (grid.node_id(1, 1, 1), grid.node_id(3, 1, 3), grid.node_id(1, 3, 3)):
        mask[3 * node: 3 * node + 3] = True
    st = vb.OperatorState(grid, np.ones(grid.n_elements), vb.MaterialModel(), mask)
    with pytest.raises(vb.SetupError):
        vb.build_hierarchy(grid, st, 2, scheme="homogenized")
    g32 = vb.build_grid(32, 32, 32, 1.0)
    st32 = vb.OperatorState(g32, np.ones(g32.n_elements), vb.MaterialModel(), face_fixed_mask(32, 32, 32))
    with pytest.raises(vb.SetupError):
        vb.build_hierarchy(g32, st32, 1, scheme="homogenized")
    with pytest.raises(ValueError):
        vb.OperatorState(grid, np.full(grid.n_elements, 1.5), vb.MaterialModel(), mask)


@pytest.mark.parametrize("dims", [(16, 8, 8), (33, 17, 9), (6, 5, 2)])
def test_streamed_host_apply_matches_device_apply(dims, rng):
    """vt_apply_host (H2D / operator / D2H overlapped in z-chunks) is bit-identical
    to the device-resident vt_apply for every chunk count, identity on fixed."""
    import ctypes as C

    import torch

    from paper_2201_12931_b200._lib import lib
    from paper_2201_12931_b200.device import DeviceVector, ptr, stream_ptr

    grid = vb.build_grid(*dims, 0.5)
    fm = face_fixed_mask(*dims)
    st = vb.OperatorState(grid, rng.uniform(0.01, 1.0, grid.n_elements), vb.MaterialModel(), fm,
                          vb.unit_stiffness(0.3, 0.5))
    u = rng.standard_normal(grid.n_dofs)
    ref = vb.apply(st, DeviceVector(st.dgrid, st.dgrid.upload(u))).numpy()
    assert np.array_equal(ref[fm], u[fm])
    for nch in (1, 2, 3, 8, 16):
        out = np.zeros(grid.n_dofs)
        assert lib.vt_apply_host(st.dgrid.handle, ptr(st.scale_dev), u.ctypes.data_as(C.c_void_p),
                                 out.ctypes.data_as(C.c_void_p), nch, stream_ptr()) == 0
        assert np.array_equal(out, ref), nch
    pinned = vb.apply(st, u)  # pageable in (threaded page-locked staging), page-locked out
    assert np.array_equal(pinned, ref)
    u_pin = torch.from_numpy(u.copy()).pin_memory().numpy()  # page-locked both ways: direct copies
    assert np.array_equal(vb.apply(st, u_pin), ref)
