"""Matrix-free stiffness operator on the device: OperatorState, apply,
diagonal, residual -- the drop-in for operator.py:108-184 of the reference.

The element scale field E*s(rho) lives on the device in the vt element
layout; v = K(rho) u runs as the TMA-pipelined factorized hex8 kernel
(csrc/hex8_apply.cu).  numpy in -> numpy out, like the reference; pass a
DeviceVector to stay on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from ._lib import check, lib
from .device import DeviceGrid, DeviceVector, device_grid, ptr, require_cuda, stream_ptr
from .material import ElementStiffness, MaterialModel, unit_stiffness
from .mesh import StructuredGrid

__all__ = ["OperatorState", "apply", "diagonal", "residual", "assemble_dense", "as_device", "from_device",
           "DENSE_GUARD_DOFS"]

DENSE_GUARD_DOFS = 20_000  # [ref: operator.py:28]


def _check_stiffness(st: ElementStiffness, grid: StructuredGrid):
    ref = unit_stiffness(st.nu, st.h).matrix
    if st.matrix.shape != (24, 24) or not np.allclose(st.matrix, ref, rtol=1e-14, atol=1e-14 * np.abs(ref).max()):
        raise ValueError(
            "the device operator supports the closed-form hex8 stiffness unit_stiffness(nu, h) only"
        )


@dataclass
class OperatorState:
    """Device-resident K(rho): grid, densities, material, constraints (operator.py:108-151)."""

    grid: StructuredGrid
    densities: np.ndarray
    model: MaterialModel
    fixed_mask: np.ndarray
    stiffness: ElementStiffness = None
    scale_dev: torch.Tensor = field(init=False, repr=False)
    fixed_idx: np.ndarray = field(init=False)
    dgrid: DeviceGrid = field(init=False, repr=False)
    rho_dev: torch.Tensor = field(init=False, repr=False)

    def __post_init__(self):
        require_cuda()
        if isinstance(self.densities, torch.Tensor):
            rho_t = self.densities
            if rho_t.shape != (self.grid.n_elements,):
                raise ValueError(f"densities must have length {self.grid.n_elements}, got {tuple(rho_t.shape)}")
            self.densities = None
        else:
            rho = np.asarray(self.densities, dtype=np.float64)
            if rho.shape != (self.grid.n_elements,):
                raise ValueError(f"densities must have length {self.grid.n_elements}, got {rho.shape}")
            self.densities = rho
            rho_t = None
        if self.stiffness is None:
            self.stiffness = unit_stiffness(0.3, self.grid.h)
        _check_stiffness(self.stiffness, self.grid)
        if abs(self.stiffness.h - self.grid.h) > 1e-12 * self.grid.h:
            raise ValueError("stiffness was integrated for a different element size")
        mask = np.asarray(self.fixed_mask)
        if mask.dtype != bool:
            idx = np.unique(np.asarray(mask, dtype=np.int64))
            mask = np.zeros(self.grid.n_dofs, dtype=bool)
            mask[idx] = True
        if mask.shape != (self.grid.n_dofs,):
            raise ValueError("fixed mask has wrong length")
        self.fixed_mask = mask
        self.fixed_idx = np.flatnonzero(mask)
        self.dgrid = device_grid(self.grid, self.stiffness.nu, mask)
        self.rho_dev = self.dgrid.plain(rho_t if rho_t is not None else self.densities)
        if self.densities is None:
            self.densities = self.rho_dev.cpu().numpy()
        self.scale_dev = self.dgrid.zeros_elem()
        m = self.model
        check(lib.vt_scale_from_density(self.dgrid.handle, ptr(self.rho_dev), m.p, m.kmin_frac, m.E,
                                        ptr(self.scale_dev), stream_ptr()))

    @property
    def scale(self) -> np.ndarray:
        """E * s(rho) per element (downloaded from the device)."""
        return self.dgrid.elem_to_plain(self.scale_dev).cpu().numpy()

    def apply(self, u):
        return apply(self, u)

    def diagonal(self):
        return diagonal(self)

    def residual(self, u, f):
        return residual(self, u, f)


def as_device(dgrid: DeviceGrid, v) -> torch.Tensor:
    if isinstance(v, DeviceVector):
        if v.dgrid.vec_len != dgrid.vec_len:
            raise ValueError("device vector belongs to a different grid")
        return v.data
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (dgrid.n_dofs,):
        raise ValueError(f"expected dof vector of length {dgrid.n_dofs}")
    return dgrid.upload(a)


def from_device(dgrid: DeviceGrid, t: torch.Tensor, like) -> object:
    if isinstance(like, DeviceVector):
        return DeviceVector(dgrid, t)
    return dgrid.download(t)


HOST_CHUNKS = 8  # z-chunks of the streamed host apply (H2D / kernel / D2H overlap)


def _pinned_empty(n: int) -> np.ndarray:
    """A fresh numpy array in page-locked memory (torch's caching host allocator)."""
    return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()


def apply(state: OperatorState, u):
    """v = K(rho) u (operator.py:154-165).

    numpy in -> a new numpy array out, streamed through the GPU in z-chunks
    (vt_apply_host: the host->device copy of the next chunk, the operator on
    this one and the device->host copy of the previous one overlap); the
    result lives in page-locked memory.  A DeviceVector stays on the device."""
    d = state.dgrid
    if isinstance(u, DeviceVector):
        ud = as_device(d, u)
        v = d.zeros()
        check(lib.vt_apply(d.handle, ptr(state.scale_dev), ptr(ud), ptr(v), stream_ptr()))
        return from_device(d, v, u)
    a = np.ascontiguousarray(np.asarray(u, dtype=np.float64))
    if a.shape != (d.n_dofs,):
        raise ValueError(f"expected dof vector of length {d.n_dofs}")
    out = _pinned_empty(d.n_dofs)
    check(lib.vt_apply_host(d.handle, ptr(state.scale_dev), a.ctypes.data_as(C.c_void_p),
                            out.ctypes.data_as(C.c_void_p), HOST_CHUNKS, stream_ptr()))
    return out


def diagonal(state: OperatorState):
    d = state.dgrid
    out = d.zeros()
    check(lib.vt_diagonal(d.handle, ptr(state.scale_dev), ptr(out), stream_ptr()))
    return d.download(out)


def residual(state: OperatorState, u, f):
    """r = f - K u, zero on fixed (operator.py:177-184)."""
    d = state.dgrid
    fd = as_device(d, f)
    ud = as_device(d, u)
    r = d.zeros()
    check(lib.vt_residual(d.handle, ptr(state.scale_dev), ptr(ud), ptr(fd), ptr(r), stream_ptr()))
    return from_device(d, r, u)


def assemble_dense(state: OperatorState, guard: int = DENSE_GUARD_DOFS) -> np.ndarray:
    """Explicit global stiffness with identity rows/columns on fixed dofs
    (operator.py:187-205).  Assembled on the device in the reference's
    element order from the reference's scale E*s(rho) (numpy's pow, as
    operator.py:142 evaluates it), so the result is bit-identical to its
    np.add.at sum; refuses grids above the guard limit like the reference."""
    from .material import simp_scale

    n = state.grid.n_dofs
    if n > guard:
        raise ValueError(f"dense assembly of {n} dofs exceeds the guard limit {guard}")
    d = state.dgrid
    sc = torch.as_tensor(state.model.E * simp_scale(state.densities, state.model), device=f"cuda:{d.device}")
    k0 = torch.as_tensor(np.ascontiguousarray(state.stiffness.matrix, dtype=np.float64).reshape(-1),
                         device=f"cuda:{d.device}")
    K = torch.empty((n, n), dtype=torch.float64, device=f"cuda:{d.device}")
    check(lib.vt_assemble_dense(d.handle, ptr(sc), ptr(k0), ptr(K), stream_ptr()),
          "vt_assemble_dense")
    return K.cpu().numpy()
