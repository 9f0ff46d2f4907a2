"""On-disk formats of the reference at 100M+-element scale:
the TPF1 binary checkpoint and the VTI voxel export of app/io.py:33-149,
byte-for-byte identical to the reference's files, written from device-resident
state without materialising host copies of whole fields.

  * checkpoint_save / checkpoint_load / Checkpoint  (app/io.py:97-149)
  * export_vti / read_vti                             (app/io.py:36-94)
  * checkpoint_save_slabs: every rank of a z-slab run writes its own byte
    ranges of one checkpoint file (element layers and node planes are
    contiguous in the reference order), so a 100M-element state is written in
    parallel from all GPUs.

Device inputs (torch CUDA tensors in the reference order, or DeviceVector in
the vt layout) are streamed through two page-locked staging buffers: the
device->host copy of chunk k+1 overlaps the file write of chunk k.
"""

from __future__ import annotations

import base64
import ctypes as C
import os
import struct
import xml.etree.ElementTree as ET
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Tuple

import numpy as np
import torch

from ._lib import check, lib
from .device import DeviceVector, ptr, stream_ptr
from .errors import ConfigError
from .mesh import StructuredGrid

__all__ = ["Checkpoint", "checkpoint_save", "checkpoint_load", "checkpoint_save_slabs", "export_vti",
           "read_vti"]

_CKPT_MAGIC = b"TPF1"
_CKPT_VERSION = 1
_CHUNK = 1 << 24  # doubles per staging chunk (128 MB)


@dataclass
class Checkpoint:
    nelx: int
    nely: int
    nelz: int
    iteration: int
    densities: np.ndarray
    displacement: np.ndarray


def _header(grid: StructuredGrid, iteration: int) -> bytes:
    return _CKPT_MAGIC + struct.pack("<IIIII", _CKPT_VERSION, grid.nelx, grid.nely, grid.nelz, int(iteration))


def _as_flat(x, n: int, what: str):
    """numpy / CUDA tensor (reference order) or DeviceVector (vt layout) -> numpy or
    a contiguous float64 CUDA tensor of length n."""
    if isinstance(x, DeviceVector):
        return x.numpy()
    if isinstance(x, torch.Tensor):
        t = x.detach().reshape(-1).to(torch.float64).contiguous()
        if t.numel() != n:
            raise ValueError("checkpoint arrays do not match the grid")
        return t if t.is_cuda else t.numpy()
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).reshape(-1)
    if a.shape != (n,):
        raise ValueError("checkpoint arrays do not match the grid")
    return a


def _write_array(fd: int, offset: int, arr) -> int:
    """pwrite a float64 array (numpy or CUDA tensor) at offset; returns the end."""
    if isinstance(arr, np.ndarray):
        os.pwrite(fd, arr.astype("<f8", copy=False).tobytes(), offset)
        return offset + 8 * arr.size
    n = arr.numel()
    bufs = [torch.empty(min(_CHUNK, n), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    stream = torch.cuda.current_stream()
    starts = list(range(0, n, _CHUNK))
    for k, s in enumerate(starts[:2]):  # prime both buffers
        e = min(s + _CHUNK, n)
        bufs[k][: e - s].copy_(arr[s:e], non_blocking=True)
        evs[k].record(stream)
    for k, s in enumerate(starts):
        e = min(s + _CHUNK, n)
        b = k & 1
        evs[b].synchronize()
        os.pwrite(fd, bufs[b][: e - s].numpy().tobytes(), offset + 8 * s)
        if k + 2 < len(starts):  # refill this buffer with chunk k+2 while the next write runs
            s2 = starts[k + 2]
            e2 = min(s2 + _CHUNK, n)
            bufs[b][: e2 - s2].copy_(arr[s2:e2], non_blocking=True)
            evs[b].record(stream)
    return offset + 8 * n


def checkpoint_save(path, grid: StructuredGrid, iteration: int, rho, u) -> None:
    """Binary state dump: magic, version, dims, iteration, rho, displacement
    (app/io.py:97-110); device arrays are streamed from the GPU."""
    r = _as_flat(rho, grid.n_elements, "rho")
    d = _as_flat(u, grid.n_dofs, "u")
    fd = os.open(os.fspath(path), os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
    try:
        os.pwrite(fd, _header(grid, iteration), 0)
        off = _write_array(fd, 24, r)
        _write_array(fd, off, d)
    finally:
        os.close(fd)


def _read_header(path):
    size = os.stat(os.fspath(path)).st_size
    with open(path, "rb") as fh:
        head = fh.read(24)
    if len(head) < 24:
        raise ConfigError(f"checkpoint {path} is truncated (no header)")
    if head[:4] != _CKPT_MAGIC:
        raise ConfigError(f"checkpoint {path} has wrong magic {head[:4]!r}")
    version, nelx, nely, nelz, iteration = struct.unpack("<IIIII", head[4:24])
    if version != _CKPT_VERSION:
        raise ConfigError(f"checkpoint {path} has unsupported version {version}")
    nel = nelx * nely * nelz
    n = 3 * (nelx + 1) * (nely + 1) * (nelz + 1)
    expected = 24 + 8 * (nel + n)
    if size != expected:
        raise ConfigError(f"checkpoint {path} has {size} bytes, expected {expected}")
    return nelx, nely, nelz, iteration, nel, n


def _read_to_device(fd: int, offset: int, n: int, device) -> torch.Tensor:
    """n float64 values at `offset` -> a CUDA tensor, through two page-locked
    buffers: the file read of chunk k+1 overlaps the host->device copy of chunk k."""
    out = torch.empty(n, dtype=torch.float64, device=device)
    if n == 0:
        return out
    bufs = [torch.empty(min(_CHUNK, n), dtype=torch.float64, pin_memory=True) for _ in range(2)]
    evs = [torch.cuda.Event(), torch.cuda.Event()]
    stream = torch.cuda.current_stream(device)
    for k, s in enumerate(range(0, n, _CHUNK)):
        e = min(s + _CHUNK, n)
        b = k & 1
        if k >= 2:
            evs[b].synchronize()  # the copy that last used this buffer is done
        view = memoryview(bufs[b].numpy()[: e - s]).cast("B")
        got = os.preadv(fd, [view], offset + 8 * s)
        if got != 8 * (e - s):
            raise ConfigError("checkpoint file shrank while being read")
        with torch.cuda.stream(stream):
            out[s:e].copy_(bufs[b][: e - s], non_blocking=True)
        evs[b].record(stream)
    stream.synchronize()
    return out


def checkpoint_load(path, expect_grid: Optional[StructuredGrid] = None, device=None) -> Checkpoint:
    """Read and validate a checkpoint; refuses partial or mismatched files
    (app/io.py:113-149).  The size is checked against the header before any
    payload is read (no whole-file read).  device=None returns numpy arrays
    like the reference; device="cuda[:i]" streams both fields straight into
    CUDA tensors (reference order) through pinned double buffers."""
    nelx, nely, nelz, iteration, nel, n = _read_header(path)
    if expect_grid is not None and (nelx, nely, nelz) != (expect_grid.nelx, expect_grid.nely, expect_grid.nelz):
        raise ConfigError(
            f"checkpoint {path} was written for {nelx}x{nely}x{nelz}, the active "
            f"configuration is {expect_grid.nelx}x{expect_grid.nely}x{expect_grid.nelz}"
        )
    if device is None:
        rho = np.fromfile(path, dtype="<f8", count=nel, offset=24)
        u = np.fromfile(path, dtype="<f8", count=n, offset=24 + 8 * nel)
        return Checkpoint(nelx, nely, nelz, iteration, rho, u)
    fd = os.open(os.fspath(path), os.O_RDONLY)
    try:
        rho = _read_to_device(fd, 24, nel, device)
        u = _read_to_device(fd, 24 + 8 * nel, n, device)
    finally:
        os.close(fd)
    return Checkpoint(nelx, nely, nelz, iteration, rho, u)


def checkpoint_save_slabs(path, run, iteration: int, group=None) -> None:
    """Parallel checkpoint of a z-slab run (slabs.SlabRun): every rank writes the
    byte ranges of its element layers (rho) and owned node planes (u) into one
    file; rank 0 writes the header and sizes the file.  Same bytes as
    checkpoint_save of the gathered state."""
    S = run.S
    grid = S.grid
    nxy = grid.nelx * grid.nely
    node_plane = 3 * (grid.nelx + 1) * (grid.nely + 1)
    total = 24 + 8 * (grid.n_elements + grid.n_dofs)
    remote = S.nlocal != S.nranks
    if remote:
        import torch.distributed as dist
    if not remote or S.rank == 0:
        fd = os.open(os.fspath(path), os.O_WRONLY | os.O_CREAT | os.O_TRUNC, 0o644)
        os.pwrite(fd, _header(grid, iteration), 0)
        os.ftruncate(fd, total)
        os.close(fd)
    if remote:
        dist.barrier(group=group)
    fd = os.open(os.fspath(path), os.O_WRONLY)
    try:
        for dg, rho, u in zip(S.slab_grids, run.rho, run.u):
            _write_array(fd, 24 + 8 * dg.k0 * nxy, rho)
            # owned node planes [k0, k1) (+ plane nz on the last slab): contiguous in reference order
            k_end = dg.k1 + (1 if dg.k1 == grid.nelz else 0)
            host = np.empty(grid.n_dofs)  # vt layout -> reference order (owned planes only touched)
            check(lib.vt_vec_download(dg.handle, ptr(u), host.ctypes.data_as(C.c_void_p), stream_ptr()))
            torch.cuda.current_stream().synchronize()
            a, b = dg.k0 * node_plane, k_end * node_plane
            _write_array(fd, 24 + 8 * grid.n_elements + 8 * a, host[a:b])
    finally:
        os.close(fd)
    if remote:
        dist.barrier(group=group)


_VTI_HEAD = """<?xml version="1.0"?>
<VTKFile type="ImageData" version="1.0" byte_order="LittleEndian" header_type="UInt32">
  <ImageData WholeExtent="{extent}" Origin="0 0 0" Spacing="{h!r} {h!r} {h!r}">
    <Piece Extent="{extent}">
      <CellData Scalars="density">
        <DataArray type="Float32" Name="density" NumberOfComponents="1" format="{fmt}">
          """
_VTI_TAIL = """
        </DataArray>
      </CellData>
    </Piece>
  </ImageData>
</VTKFile>
"""
_VTI_CHUNK = 3 * (1 << 22)  # float32 values per base64 chunk (a multiple of 3 bytes keeps chunks aligned)


def export_vti(rho, grid: StructuredGrid, path, binary: bool = True) -> None:
    """Cell-centred float32 density field as XML ImageData (app/io.py:36-71),
    byte-identical to the reference's file.  The binary payload is
    base64(UInt32 byte count + float32 values); it is encoded and written in
    chunks aligned to 3 bytes, so a 100M-cell field never exists as one host
    string.  A CUDA tensor is converted to float32 on the device and copied
    down chunk by chunk."""
    path = Path(path)
    if isinstance(rho, torch.Tensor):
        t = rho.detach().reshape(-1)
        if t.numel() != grid.n_elements:
            raise ValueError(f"expected {grid.n_elements} cell values")
        values = t.to(torch.float32)
    else:
        values = np.asarray(rho, dtype=np.float32).reshape(-1) if np.ndim(rho) else np.asarray(rho)
        if values.shape != (grid.n_elements,):
            raise ValueError(f"expected {grid.n_elements} cell values")
    nx, ny, nz = grid.nelx, grid.nely, grid.nelz
    extent = f"0 {nx} 0 {ny} 0 {nz}"
    head = _VTI_HEAD.format(extent=extent, h=grid.h, fmt="binary" if binary else "ascii")
    try:
        with open(path, "w", encoding="ascii", newline="") as fh:
            fh.write(head)
            if binary:
                n = grid.n_elements
                carry = struct.pack("<I", 4 * n)  # the UInt32 header, then the values
                for s in range(0, n, _VTI_CHUNK):
                    e = min(s + _VTI_CHUNK, n)
                    blk = values[s:e]
                    raw = (blk.cpu().numpy() if isinstance(blk, torch.Tensor) else blk).astype("<f4").tobytes()
                    buf = carry + raw
                    cut = len(buf) - len(buf) % 3 if e < n else len(buf)
                    fh.write(base64.b64encode(buf[:cut]).decode("ascii"))
                    carry = buf[cut:]
            else:
                vals = values.cpu().numpy() if isinstance(values, torch.Tensor) else values
                fh.write(" ".join(repr(float(v)) for v in vals))
            fh.write(_VTI_TAIL)
    except OSError as exc:
        raise OSError(f"failed writing VTI file {path}: {exc}") from exc


def read_vti(path) -> Tuple[np.ndarray, Tuple[int, int, int], float]:
    """Parse a file written by export_vti: (values, (nelx, nely, nelz), spacing) (app/io.py:74-94)."""
    root = ET.parse(path).getroot()
    image = root.find("ImageData")
    ext = [int(t) for t in image.attrib["WholeExtent"].split()]
    dims = (ext[1] - ext[0], ext[3] - ext[2], ext[5] - ext[4])
    spacing = float(image.attrib["Spacing"].split()[0])
    arr = image.find("Piece").find("CellData").find("DataArray")
    text = arr.text.strip()
    if arr.attrib["format"] == "binary":
        raw = base64.b64decode(text)
        (nbytes,) = struct.unpack("<I", raw[:4])
        values = np.frombuffer(raw[4:4 + nbytes], dtype="<f4")
    else:
        values = np.array([float(t) for t in text.split()], dtype=np.float32)
    return values, dims, spacing
