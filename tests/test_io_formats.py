"""TPF1 checkpoints and VTI exports byte-for-byte against
files the reference wrote (tests/golden/io_*, oracle/make_golden.py gen_io);
mirrors pkg/tests/test_io.py.  CPU part: host arrays; GPU part: device
tensors, DeviceVector and the slab-parallel checkpoint."""

import os

import numpy as np
import pytest

from conftest import GOLDEN, golden

vb = pytest.importorskip("paper_2201_12931_b200")
from paper_2201_12931_b200 import io as vio  # noqa: E402


def _case():
    g = golden("io.npz")
    dims = tuple(int(x) for x in g["dims"])
    return g, vb.build_grid(*dims, float(g["h"]))


def _bytes(name):
    with open(os.path.join(GOLDEN, name), "rb") as fh:
        return fh.read()


def test_checkpoint_bytes_and_roundtrip(tmp_path):
    g, grid = _case()
    p = tmp_path / "c.bin"
    vio.checkpoint_save(p, grid, int(g["it"]), g["rho"], g["u"])
    assert p.read_bytes() == _bytes("io_ckpt.bin")
    ck = vio.checkpoint_load(os.path.join(GOLDEN, "io_ckpt.bin"), expect_grid=grid)
    assert (ck.nelx, ck.nely, ck.nelz, ck.iteration) == (4, 3, 2, 7)
    assert np.array_equal(ck.densities, g["rho"]) and np.array_equal(ck.displacement, g["u"])


def test_checkpoint_rejects_bad_files(tmp_path):
    _, grid = _case()
    data = _bytes("io_ckpt.bin")
    cases = {"short": data[:10], "magic": b"XXXX" + data[4:], "trunc": data[:-8],
             "version": data[:4] + (2).to_bytes(4, "little") + data[8:]}
    for name, blob in cases.items():
        p = tmp_path / f"{name}.bin"
        p.write_bytes(blob)
        with pytest.raises(vb.ConfigError):
            vio.checkpoint_load(p)
    with pytest.raises(vb.ConfigError, match="written for 4x3x2"):
        vio.checkpoint_load(os.path.join(GOLDEN, "io_ckpt.bin"), expect_grid=vb.build_grid(4, 3, 4, 1.0))
    with pytest.raises(ValueError):
        vio.checkpoint_save(tmp_path / "x.bin", grid, 0, np.zeros(3), np.zeros(grid.n_dofs))


@pytest.mark.parametrize("binary,name", [(True, "io_bin.vti"), (False, "io_ascii.vti")])
def test_vti_bytes_and_read(tmp_path, binary, name):
    g, grid = _case()
    p = tmp_path / "d.vti"
    vio.export_vti(g["rho"], grid, p, binary=binary)
    assert p.read_bytes() == _bytes(name)
    vals, dims, sp = vio.read_vti(os.path.join(GOLDEN, name))
    assert dims == (4, 3, 2) and sp == 0.75
    assert np.array_equal(vals, g["rho"].astype(np.float32))


@pytest.mark.gpu
def test_checkpoint_from_device_and_slabs(tmp_path):
    import torch

    from paper_2201_12931_b200 import cases
    from paper_2201_12931_b200.device import DeviceVector
    from paper_2201_12931_b200.slabs import SlabRun

    g, grid = _case()
    st = vb.OperatorState(grid, g["rho"], vb.MaterialModel(), np.zeros(grid.n_dofs, bool),
                          vb.unit_stiffness(0.3, grid.h))
    rho_d = torch.as_tensor(g["rho"], device="cuda")
    u_d = DeviceVector(st.dgrid, st.dgrid.upload(g["u"]))
    p = tmp_path / "dev.bin"
    vio.checkpoint_save(p, grid, int(g["it"]), rho_d, u_d)
    assert p.read_bytes() == _bytes("io_ckpt.bin")
    q = tmp_path / "dev.vti"
    vio.export_vti(rho_d, grid, q)
    assert q.read_bytes() == _bytes("io_bin.vti")
    # parallel checkpoint of a 4-slab run == checkpoint of its gathered state
    prob = cases.cantilever(16, 8, 16)
    opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * prob.grid.h, max_iterations=2, ch_tol=1e-12)
    R = SlabRun(prob, opt, vb.SolverConfig(tolerance=1e-6), 3, nranks=4)
    R.solve(prob.model)
    R.design_step(prob.model)
    a, b = tmp_path / "slabs.bin", tmp_path / "gathered.bin"
    vio.checkpoint_save_slabs(a, R, 1)
    vio.checkpoint_save(b, prob.grid, 1, R.densities(), R.displacement())
    assert a.read_bytes() == b.read_bytes()
    ck = vio.checkpoint_load(a, expect_grid=prob.grid)
    assert ck.iteration == 1
    # streamed load straight to the device == the host load
    ckd = vio.checkpoint_load(a, expect_grid=prob.grid, device="cuda")
    assert ckd.densities.is_cuda and ckd.displacement.is_cuda
    assert np.array_equal(ckd.densities.cpu().numpy(), ck.densities)
    assert np.array_equal(ckd.displacement.cpu().numpy(), ck.displacement)


def test_vti_chunked_payload_matches_single_shot(tmp_path, monkeypatch):
    """The chunked base64 writer (chunks aligned to 3 bytes) produces exactly the
    single-shot encoding of the reference, whatever the chunk size."""
    import base64
    import struct

    g, grid = _case()
    ref = (tmp_path / "a.vti")
    vio.export_vti(g["rho"], grid, ref)
    for chunk in (1, 2, 3, 5, 7):
        monkeypatch.setattr(vio, "_VTI_CHUNK", chunk)
        p = tmp_path / f"c{chunk}.vti"
        vio.export_vti(g["rho"], grid, p)
        assert p.read_bytes() == ref.read_bytes()
    raw = g["rho"].astype("<f4").tobytes()
    assert base64.b64encode(struct.pack("<I", len(raw)) + raw).decode() in ref.read_text()


def test_checkpoint_load_rejects_size_mismatch_without_reading(tmp_path):
    g, grid = _case()
    p = tmp_path / "t.bin"
    vio.checkpoint_save(p, grid, 3, g["rho"], g["u"])
    with open(p, "ab") as fh:
        fh.write(b"x")
    with pytest.raises(vb.ConfigError, match="bytes, expected"):
        vio.checkpoint_load(p)
