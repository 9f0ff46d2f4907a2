"""Device residency: vt_grid handles and vectors in the vt layouts.

PyTorch is plumbing here: it allocates device memory (caching allocator)
and supplies the current CUDA stream.  All arithmetic runs in libvoxb200.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import threading
import weakref

import numpy as np
import torch

from . import _lib
from ._lib import check, lib
from .mesh import StructuredGrid, node_mask_bytes

__all__ = ["DeviceGrid", "device_grid", "stream_ptr", "require_cuda", "DeviceVector"]


def require_cuda():
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2201_12931_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback"
        )


def stream_ptr():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t: torch.Tensor):
    return C.c_void_p(t.data_ptr())


class DeviceGrid:
    """One vt_grid: geometry + fixed mask of a level on the current device."""

    def __init__(self, nelx, nely, nelz, h, nu=0.3, fixed_mask=None, k0=0, k1=None, device=None):
        require_cuda()
        self.nelx, self.nely, self.nelz, self.h, self.nu = int(nelx), int(nely), int(nelz), float(h), float(nu)
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.k0 = int(k0)
        self.k1 = self.nelz if k1 is None else int(k1)
        self.handle = C.c_void_p()
        owned = None
        if fixed_mask is not None:
            owned = node_mask_bytes(fixed_mask)
        mp = owned.ctypes.data_as(C.c_void_p) if owned is not None else None
        check(lib.vt_grid_create(C.byref(self.handle), self.nelx, self.nely, self.nelz, self.h,
                                 self.nu, mp, self.k0, self.k1, self.device), "vt_grid_create")
        self._owns = True
        self._init_sizes()

    @classmethod
    def wrap(cls, handle, nelx, nely, nelz, h, nu, device):
        g = cls.__new__(cls)
        g.nelx, g.nely, g.nelz, g.h, g.nu = nelx, nely, nelz, h, nu
        g.device, g.k0, g.k1 = device, 0, nelz
        g.handle = C.c_void_p(handle)
        g._owns = False
        g._init_sizes()
        return g

    def _init_sizes(self):
        self.vec_len = int(lib.vt_vec_len(self.handle))
        self.elem_len = int(lib.vt_elem_len(self.handle))
        self.n_fixed = int(lib.vt_n_fixed(self.handle))
        self.n_dofs = 3 * (self.nelx + 1) * (self.nely + 1) * (self.nelz + 1)
        self.n_elements = self.nelx * self.nely * self.nelz
        self.rp = self.nelx + 1 if (self.nelx + 1) % 2 == 0 else self.nelx + 2
        self.ep = self.nelx if self.nelx % 2 == 0 else self.nelx + 1

    def __del__(self):
        try:
            if getattr(self, "_owns", False) and self.handle:
                lib.vt_grid_destroy(self.handle)
                self.handle = C.c_void_p()
        except Exception:
            pass

    @property
    def grid(self) -> StructuredGrid:
        return StructuredGrid(self.nelx, self.nely, self.nelz, self.h)

    # ---------------------------------------------------------------- vectors
    def zeros(self) -> torch.Tensor:
        return torch.zeros(self.vec_len, dtype=torch.float64, device=f"cuda:{self.device}")

    def zeros_elem(self) -> torch.Tensor:
        return torch.zeros(self.elem_len, dtype=torch.float64, device=f"cuda:{self.device}")

    def upload(self, host) -> torch.Tensor:
        h = np.ascontiguousarray(np.asarray(host, dtype=np.float64))
        if h.shape != (self.n_dofs,):
            raise ValueError(f"expected dof vector of length {self.n_dofs}")
        d = self.zeros()
        check(lib.vt_vec_upload(self.handle, h.ctypes.data_as(C.c_void_p), ptr(d), stream_ptr()))
        torch.cuda.current_stream().synchronize()  # h may be a temporary
        return d

    def download(self, dev: torch.Tensor) -> np.ndarray:
        out = np.empty(self.n_dofs)
        check(lib.vt_vec_download(self.handle, ptr(dev), out.ctypes.data_as(C.c_void_p), stream_ptr()))
        torch.cuda.current_stream().synchronize()
        return out

    def elem_to_plain(self, field: torch.Tensor) -> torch.Tensor:
        """vt element layout (ghost layer + row pitch) -> plain (n_elements,)"""
        q = self.k1 - self.k0
        v = field.view(q + 1, self.nely, self.ep)[1:, :, : self.nelx]
        return v.reshape(-1).contiguous()

    def plain(self, host_or_dev, n=None) -> torch.Tensor:
        n = self.n_elements if n is None else n
        if isinstance(host_or_dev, torch.Tensor):
            t = host_or_dev.to(dtype=torch.float64, device=f"cuda:{self.device}")
        else:
            t = torch.as_tensor(np.ascontiguousarray(np.asarray(host_or_dev, dtype=np.float64)),
                                device=f"cuda:{self.device}")
        if t.shape != (n,):
            raise ValueError(f"expected an element field of length {n}, got {tuple(t.shape)}")
        return t.contiguous()


class DeviceVector:
    """A node vector that stays on the device (vt layout) with its grid."""

    __slots__ = ("dgrid", "data")

    def __init__(self, dgrid: DeviceGrid, data: torch.Tensor):
        self.dgrid = dgrid
        self.data = data

    def numpy(self) -> np.ndarray:
        return self.dgrid.download(self.data)

    @property
    def shape(self):
        return (self.dgrid.n_dofs,)


_cache_lock = threading.Lock()
_grid_cache: "weakref.WeakValueDictionary" = weakref.WeakValueDictionary()


def device_grid(grid: StructuredGrid, nu: float, fixed_mask) -> DeviceGrid:
    """Shared DeviceGrid per (grid, nu, fixed set); lives while referenced."""
    fm = None if fixed_mask is None else np.asarray(fixed_mask, dtype=bool)
    digest = "none" if fm is None else hashlib.blake2b(np.packbits(fm).tobytes(), digest_size=16).hexdigest()
    key = (grid.nelx, grid.nely, grid.nelz, float(grid.h), float(nu), digest, torch.cuda.current_device())
    with _cache_lock:
        g = _grid_cache.get(key)
        if g is None:
            g = DeviceGrid(grid.nelx, grid.nely, grid.nelz, grid.h, nu, fm)
            _grid_cache[key] = g
        return g
