"""Z-slab decomposition of the MGPCG solve: one slab per rank.

The reference is single-process; this module distributes its state-equation
solve -- the matrix-free K(rho)u, the homogenized V-cycle and PCG -- over
z-slabs (csrc/dist.cu).  Levels 0..D are slab-distributed with one ghost node
plane per side (NCCL send/recv halos); the coarse tail D+1..L-1, including the
dense coarsest solve, is replicated on every rank; dot products are reduced
per rank, all-gathered and summed in rank order so every rank takes the same
scalar decisions.

Three transports, same arithmetic:
  * ``SlabSolver(..., nranks=N)`` without a process group keeps all N slabs in
    this process on one GPU (halos are device copies) -- used by the parity
    tests, which compare it with the single-slab solve;
  * ``SlabSolver.from_process_group(..., transport="peer")`` (the default)
    runs one slab per rank of an initialised ``torch.distributed`` group
    (torchrun, one process per GPU); each exchange is one kernel that loads
    the neighbours' staged planes from their device memory (CUDA IPC over
    NVLink / NVSwitch; csrc/peer.cu).  The IPC handles travel over the group.
    Ranks may also share one GPU, which is how the multi-process path is
    tested on a single B200;
  * ``transport="nccl"``: the same with NCCL send/recv/broadcast/all-gather
    on a library-owned communicator (id broadcast over the group).

``plan_slabs`` (pure host logic, gloo-tested on CPU) chooses the partition.
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from ._lib import SolveReportC, check, lib
from .device import DeviceGrid, ptr, require_cuda, stream_ptr
from .hierarchy import max_feasible_levels
from .krylov import AUX_BUDGET_FACTOR, SolveReport, SolverConfig
from .material import MaterialModel
from .mesh import StructuredGrid, node_mask_bytes

__all__ = ["SlabPlan", "plan_slabs", "SlabSolver"]


@dataclass(frozen=True)
class SlabPlan:
    """Partition of the element layers: rank g owns [bounds[g], bounds[g+1])."""

    nranks: int
    levels: int
    dist_level: int          # levels 0..dist_level are slab-distributed
    bounds: Tuple[int, ...]  # nranks + 1 layer boundaries, multiples of 2**dist_level

    def slab(self, rank: int) -> Tuple[int, int]:
        return self.bounds[rank], self.bounds[rank + 1]

    def tail_planes(self, rank: int, nz: int) -> Tuple[int, int]:
        """Coarse node planes of level dist_level+1 restricted by `rank` (those
        whose centre fine plane 2K the rank owns at level dist_level)."""
        d = self.dist_level
        a = self.bounds[rank] >> d
        b = (self.bounds[rank + 1] >> d) + (1 if self.bounds[rank + 1] == nz else 0)
        return (a + 1) // 2, (b + 1) // 2

    def halo_pattern(self, rank: int) -> List[Tuple[str, int, int]]:
        """Per-apply node-plane exchange of `rank` as (op, peer, local plane p):
        send the first owned plane down / the last owned plane up, receive the
        ghost planes p = 0 and p = n + 1 (mirrors csrc/dist.cu halo_nodes)."""
        k0, k1 = self.slab(rank)
        n = k1 - k0
        ops = []
        if rank > 0:
            ops += [("send", rank - 1, 1), ("recv", rank - 1, 0)]
        if rank < self.nranks - 1:
            ops += [("send", rank + 1, n), ("recv", rank + 1, n + 1)]
        return ops


def plan_slabs(nz: int, levels: int, nranks: int, max_dist_level: Optional[int] = None) -> SlabPlan:
    """Even z-slabs whose boundaries survive the deepest possible coarsening.

    D = the largest level d <= levels-2 (and <= max_dist_level) at which
    nz / 2**d layers split evenly into nranks slabs (so every distributed level
    is balanced and every slab boundary falls on an even coarse layer); levels
    d+1.. are replicated.  The Galerkin scheme distributes exactly levels 0 and
    1 (max_dist_level=1, and D must reach 1)."""
    if nranks < 1:
        raise ValueError("nranks must be positive")
    if levels < 2:
        raise ValueError("the slab solver needs at least 2 multigrid levels")
    if nz % (1 << (levels - 1)):
        raise ValueError(f"nz={nz} does not support {levels} levels")
    top = levels - 2 if max_dist_level is None else min(levels - 2, int(max_dist_level))
    for d in range(top, -1, -1):
        t = nz >> d
        if t % nranks == 0:
            per = (t // nranks) << d
            return SlabPlan(nranks, levels, d, tuple(per * g for g in range(nranks + 1)))
    raise ValueError(f"cannot split nz={nz} element layers evenly into {nranks} slabs")


def _ptr_array(tensors: Sequence[torch.Tensor]):
    arr = (C.c_void_p * len(tensors))()
    for i, t in enumerate(tensors):
        arr[i] = t.data_ptr()
    return arr


class SlabSolver:
    """Slab-decomposed operator + MGPCG (homogenized or Galerkin V-cycle) for one problem.

    grid / fixed_mask are the global problem (every rank passes the same).
    Vectors are lists of per-local-slab device tensors in the vt node layout
    of the slab grid (``upload`` / ``download`` convert global numpy arrays)."""

    def __init__(self, grid: StructuredGrid, fixed_mask, levels: Optional[int] = None, omega: float = 0.4,
                 nranks: int = 1, rank: int = 0, nlocal: Optional[int] = None, nccl_id: Optional[bytes] = None,
                 nu: float = 0.3, device: Optional[int] = None, peer: bool = False, scheme: str = "homogenized"):
        require_cuda()
        if scheme not in ("homogenized", "galerkin"):
            raise ValueError(f"unknown scheme {scheme!r}")
        self.grid = grid
        self.scheme = scheme
        self.levels = int(levels) if levels is not None else max_feasible_levels(grid.nelx, grid.nely, grid.nelz)
        if scheme == "galerkin":
            if self.levels < 3:
                raise ValueError("the Galerkin slab scheme needs at least 3 multigrid levels")
            self.plan = plan_slabs(grid.nelz, self.levels, nranks, max_dist_level=1)
            if self.plan.dist_level != 1:
                raise ValueError(f"the Galerkin slab scheme needs an even number of element layers per slab "
                                 f"(nz={grid.nelz}, {nranks} slabs)")
        else:
            self.plan = plan_slabs(grid.nelz, self.levels, nranks)
        self.nranks, self.rank = nranks, rank
        self.nlocal = nranks if nlocal is None else int(nlocal)
        self.device = torch.cuda.current_device() if device is None else int(device)
        mask = np.asarray(fixed_mask, dtype=bool)
        if mask.shape != (grid.n_dofs,):
            raise ValueError("fixed mask has wrong length")
        self.fixed_mask = mask
        nm = node_mask_bytes(mask)
        kb = (C.c_int * (nranks + 1))(*self.plan.bounds)
        idbuf = None
        if nccl_id is not None:
            idbuf = (C.c_uint8 * len(nccl_id)).from_buffer_copy(nccl_id)
        self._h = C.c_void_p()
        self.transport = "peer" if peer else ("nccl" if nccl_id is not None else "local")
        if peer:
            if self.nlocal != 1:
                raise ValueError("the peer transport runs one slab per process")
            check(lib.vt_dist_create_peer(C.byref(self._h), grid.nelx, grid.nely, grid.nelz, grid.h, nu,
                                          nm.ctypes.data_as(C.c_void_p), self.levels, omega, nranks, rank, kb,
                                          self.plan.dist_level, self.device), "vt_dist_create_peer")
        else:
            check(lib.vt_dist_create(C.byref(self._h), grid.nelx, grid.nely, grid.nelz, grid.h, nu,
                                     nm.ctypes.data_as(C.c_void_p), self.levels, omega, nranks, rank,
                                     self.nlocal, kb, self.plan.dist_level, idbuf, self.device),
                  "vt_dist_create")
        if scheme == "galerkin":
            check(lib.vt_dist_set_scheme(self._h, 1), "vt_dist_set_scheme")
        self.slab_grids = []
        for i in range(self.nlocal):
            g = lib.vt_dist_grid(self._h, i, 0)
            k0, k1 = self.plan.slab(rank + i)
            dg = DeviceGrid.wrap(g, grid.nelx, grid.nely, grid.nelz, grid.h, nu, self.device)
            dg.k0, dg.k1 = k0, k1
            dg.vec_len = int(lib.vt_vec_len(C.c_void_p(g)))
            dg.elem_len = int(lib.vt_elem_len(C.c_void_p(g)))
            self.slab_grids.append(dg)
        self.scales = [dg.zeros_elem() for dg in self.slab_grids]
        self.model: Optional[MaterialModel] = None

    @classmethod
    def from_process_group(cls, grid: StructuredGrid, fixed_mask, levels=None, omega=0.4, group=None,
                           transport: str = "peer", nu: float = 0.3, scheme: str = "homogenized"):
        """One slab per rank of the initialised torch.distributed group.
        transport="peer": IPC handles of every rank's staging block are
        all-gathered over the group; "nccl": the library's NCCL communicator is
        bootstrapped from an id broadcast over it."""
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if transport == "peer":
            S = cls(grid, fixed_mask, levels, omega, nranks=world, rank=rank, nlocal=1, nu=nu, peer=True,
                    scheme=scheme)
            S.connect_peers(group)
            return S
        if transport != "nccl":
            raise ValueError(f"unknown transport {transport!r}")
        nbytes = int(lib.vt_nccl_id_bytes())
        obj = [None]
        if rank == 0:
            buf = (C.c_uint8 * nbytes)()
            check(lib.vt_nccl_unique_id(buf, nbytes), "vt_nccl_unique_id")
            obj[0] = bytes(buf)
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(grid, fixed_mask, levels, omega, nranks=world, rank=rank, nlocal=1, nccl_id=obj[0], nu=nu,
                   scheme=scheme)

    def connect_peers(self, group=None):
        """All-gather the ranks' IPC handles over `group` and map the peers'
        staging blocks (peer transport)."""
        import torch.distributed as dist

        hb = int(lib.vt_peer_handle_bytes())
        buf = (C.c_uint8 * hb)()
        check(lib.vt_dist_peer_handle(self._h, buf, hb), "vt_dist_peer_handle")
        allh = [None] * self.nranks
        dist.all_gather_object(allh, bytes(buf), group=group)
        cat = b"".join(allh)
        arr = (C.c_uint8 * len(cat)).from_buffer_copy(cat)
        check(lib.vt_dist_peer_open(self._h, arr, len(cat)), "vt_dist_peer_open")

    def close(self):
        if getattr(self, "_h", None):
            lib.vt_dist_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ data movement
    def upload(self, host) -> List[torch.Tensor]:
        return [dg.upload(host) for dg in self.slab_grids]

    def download(self, vecs: Sequence[torch.Tensor], out: Optional[np.ndarray] = None) -> np.ndarray:
        """Owned planes of the local slabs into a global (n_dofs,) array."""
        if out is None:  # page-locked, zero outside this process's planes
            out = torch.zeros(self.grid.n_dofs, dtype=torch.float64, pin_memory=True).numpy()
        for dg, v in zip(self.slab_grids, vecs):
            check(lib.vt_vec_download(dg.handle, ptr(v), out.ctypes.data_as(C.c_void_p), stream_ptr()))
        torch.cuda.current_stream().synchronize()
        return out

    def zeros(self) -> List[torch.Tensor]:
        return [dg.zeros() for dg in self.slab_grids]

    def _slab_rho(self, rho) -> List[torch.Tensor]:
        nxy = self.grid.nelx * self.grid.nely
        rho_t = rho if isinstance(rho, torch.Tensor) else torch.as_tensor(np.asarray(rho, dtype=np.float64))
        rho_t = rho_t.to(device=f"cuda:{self.device}", dtype=torch.float64)
        if rho_t.shape != (self.grid.n_elements,):
            raise ValueError(f"densities must have length {self.grid.n_elements}")
        return [rho_t[dg.k0 * nxy:dg.k1 * nxy].contiguous() for dg in self.slab_grids]

    # ------------------------------------------------------------ operator / MG
    def set_density(self, rho, model: MaterialModel = MaterialModel(), refresh: bool = True):
        """scale = E s(rho) per slab (+ ghost layer); refresh = coarse levels + coarsest factor."""
        self.model = model
        self._rho = self._slab_rho(rho)
        for dg, r, sc in zip(self.slab_grids, self._rho, self.scales):
            check(lib.vt_scale_from_density(dg.handle, ptr(r), model.p, model.kmin_frac, model.E, ptr(sc),
                                            stream_ptr()))
        if refresh:
            check(lib.vt_dist_refresh(self._h, _ptr_array(self._rho), _ptr_array(self.scales), model.p,
                                      model.kmin_frac, model.E, stream_ptr()), "vt_dist_refresh")
        else:
            check(lib.vt_dist_set_scale(self._h, _ptr_array(self.scales), stream_ptr()))

    def apply(self, u: List[torch.Tensor], v: Optional[List[torch.Tensor]] = None) -> List[torch.Tensor]:
        """v = K u on every local slab (u zero on fixed dofs; its ghost planes are refreshed)."""
        v = self.zeros() if v is None else v
        check(lib.vt_dist_apply(self._h, _ptr_array(u), _ptr_array(v), stream_ptr()))
        return v

    def dot(self, x: List[torch.Tensor], y: List[torch.Tensor]) -> float:
        out = C.c_double()
        check(lib.vt_dist_dot(self._h, _ptr_array(x), _ptr_array(y), C.byref(out), stream_ptr()))
        return out.value

    def v_cycle(self, f: List[torch.Tensor]) -> List[torch.Tensor]:
        z = self.zeros()
        check(lib.vt_dist_vcycle(self._h, _ptr_array(f), _ptr_array(z), stream_ptr()), "vt_dist_vcycle")
        return z

    def mgcg_solve(self, f: List[torch.Tensor], u_prev: Optional[List[torch.Tensor]] = None,
                   cfg: SolverConfig = SolverConfig()) -> Tuple[List[torch.Tensor], SolveReport]:
        """MGPCG over all ranks (solver.py:170-191 with the pcg of 62-167)."""
        if cfg.preconditioner != "multigrid":
            raise ValueError("the slab solver implements the multigrid preconditioner")
        n = self.grid.n_dofs
        aux = 4 * n + sum(5 * 3 * ((self.grid.nelx >> l) + 1) * ((self.grid.nely >> l) + 1) * ((self.grid.nelz >> l) + 1)
                          for l in range(self.levels))
        if aux > AUX_BUDGET_FACTOR * n:  # [ref: solver.py:183-187]
            from .errors import SolverBreakdown

            raise SolverBreakdown(f"auxiliary vector budget {aux} exceeds {AUX_BUDGET_FACTOR} * n")
        x = [t.clone() for t in u_prev] if (u_prev is not None and cfg.warm_start) else self.zeros()
        rep = SolveReportC()
        t0 = time.perf_counter()
        check(lib.vt_dist_pcg(self._h, _ptr_array(f), _ptr_array(x), 1 if u_prev is not None and cfg.warm_start else 0,
                              float(cfg.tolerance), int(cfg.max_iterations), C.byref(rep), stream_ptr()),
              "vt_dist_pcg")
        return x, SolveReport(iterations=rep.iterations, final_rel_residual=rep.final_rel_residual,
                              precond_applications=rep.precond_applications, wall_s=time.perf_counter() - t0,
                              converged=bool(rep.converged), aux_vector_scalars=aux,
                              residual_drift=rep.residual_drift)


# ---------------------------------------------------------------------------
# the design loop on slabs
class SlabRun:
    """Device-resident SIMP loop over z-slabs (optimize.py:344-455): refresh +
    slab MGPCG, compliance, sensitivities (u halo), filter (R-layer halos of
    rho*dc), OC (rank-ordered sums per lambda step), change / volume.  Element
    fields live as per-slab plain ranges of the reference element order."""

    def __init__(self, problem, opt, solver: SolverConfig, max_levels=None, omega: float = 0.4,
                 nranks: int = 1, rank: int = 0, nlocal: Optional[int] = None, nccl_id: Optional[bytes] = None,
                 init_densities=None, group=None, init_displacement=None, peer: bool = False,
                 scheme: str = "homogenized"):
        from .design import filter_weights, initial_densities

        if solver.preconditioner != "multigrid":
            raise ValueError("the slab solver implements the multigrid preconditioner")
        grid = problem.grid
        self.problem, self.opt, self.solver, self.group = problem, opt, solver, group
        fm = problem.boundary.fixed_mask(grid)
        self.S = S = SlabSolver(grid, fm, max_levels, omega, nranks=nranks, rank=rank, nlocal=nlocal,
                                nccl_id=nccl_id, nu=problem.nu, peer=peer, scheme=scheme)
        if peer:
            S.connect_peers(group)
        f_ext = problem.boundary.external_force(grid)
        f_ext[fm] = 0.0
        self.f_ext = S.upload(f_ext)
        self.gravity = problem.boundary.gravity
        self.f = S.zeros() if self.gravity is not None else self.f_ext
        rho0 = (init_densities.values if init_densities is not None
                else initial_densities(problem.regions, opt.volfrac).values)
        self.rho = S._slab_rho(rho0)
        self.rho = [r.clone() for r in self.rho]
        self.rho_new = [torch.empty_like(r) for r in self.rho]
        nxy = grid.nelx * grid.nely
        cls = torch.as_tensor(np.ascontiguousarray(problem.regions.classes, dtype=np.int8),
                              device=f"cuda:{S.device}")
        self.cls = [cls[dg.k0 * nxy:dg.k1 * nxy].contiguous() for dg in S.slab_grids]
        self.dv = [torch.ones_like(r) for r in self.rho]
        self.dc = [torch.empty_like(r) for r in self.rho]
        self.dcf = [torch.empty_like(r) for r in self.rho]
        # a resumed run warm-starts its first solve from the stored displacement,
        # as the reference's run() does (optimize.py:344-360)
        if init_displacement is not None:
            u0 = np.array(init_displacement, dtype=np.float64)
            if u0.shape != (grid.n_dofs,):
                raise ValueError(f"initial displacement must have length {grid.n_dofs}")
            u0[fm] = 0.0
            self.u = S.upload(u0)
        else:
            self.u = S.zeros()
        R, kern = filter_weights(grid.h, opt.filter_radius)
        check(lib.vt_dist_filter_create(S._h, R, kern.ctypes.data_as(C.c_void_p)), "vt_dist_filter_create")

    @classmethod
    def from_process_group(cls, problem, opt, solver, max_levels=None, omega=0.4, init_densities=None,
                           group=None, init_displacement=None, transport: str = "peer",
                           scheme: str = "homogenized"):
        import torch.distributed as dist

        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if transport == "peer":
            return cls(problem, opt, solver, max_levels, omega, nranks=world, rank=rank, nlocal=1,
                       init_densities=init_densities, group=group, init_displacement=init_displacement, peer=True,
                       scheme=scheme)
        if transport != "nccl":
            raise ValueError(f"unknown transport {transport!r}")
        obj = [None]
        if rank == 0:
            n = int(lib.vt_nccl_id_bytes())
            buf = (C.c_uint8 * n)()
            check(lib.vt_nccl_unique_id(buf, n), "vt_nccl_unique_id")
            obj[0] = bytes(buf)
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(problem, opt, solver, max_levels, omega, nranks=world, rank=rank, nlocal=1,
                   nccl_id=obj[0], init_densities=init_densities, group=group,
                   init_displacement=init_displacement, scheme=scheme)

    def solve(self, model) -> SolveReport:
        S = self.S
        S.model = model
        for dg, r, sc in zip(S.slab_grids, self.rho, S.scales):
            check(lib.vt_scale_from_density(dg.handle, ptr(r), model.p, model.kmin_frac, model.E, ptr(sc),
                                            stream_ptr()))
        check(lib.vt_dist_refresh(S._h, _ptr_array(self.rho), _ptr_array(S.scales), model.p,
                                  model.kmin_frac, model.E, stream_ptr()), "vt_dist_refresh")
        if self.gravity is not None:  # design-dependent load (optimize.py:216-231, 397-400)
            check(lib.vt_dist_gravity_load(S._h, _ptr_array(self.rho), int(self.gravity.axis), self._gco(),
                                           _ptr_array(self.f_ext), 1, _ptr_array(self.f), stream_ptr()))
        self.u, rep = S.mgcg_solve(self.f, u_prev=self.u, cfg=self.solver)
        return rep

    def _gco(self) -> float:
        from .material import gravity_coefficient

        g = self.gravity
        return gravity_coefficient(g.g, self.problem.grid.h, g.unit_weight)

    def design_step(self, model):
        """compliance, sensitivities, filter, OC; swaps rho. Returns (c, change, volume)."""
        S, opt = self.S, self.opt
        c = S.dot(self.f, self.u)
        gax, gco = (int(self.gravity.axis), self._gco()) if self.gravity is not None else (-1, 0.0)
        check(lib.vt_dist_sensitivities(S._h, _ptr_array(self.u), _ptr_array(self.rho), model.p,
                                        model.kmin_frac, model.E, gax, gco, _ptr_array(self.dc), stream_ptr()))
        check(lib.vt_dist_filter_apply(S._h, _ptr_array(self.dc), _ptr_array(self.rho), float(opt.gamma),
                                       _ptr_array(self.dcf), stream_ptr()))
        lam, steps = C.c_double(), C.c_int()
        check(lib.vt_dist_oc_update(S._h, _ptr_array(self.rho), _ptr_array(self.cls), _ptr_array(self.dcf),
                                    _ptr_array(self.dv), float(opt.volfrac), float(opt.move), float(opt.eta),
                                    float(opt.q), _ptr_array(self.rho_new), C.byref(lam), C.byref(steps),
                                    stream_ptr()))
        ch, vol = C.c_double(), C.c_double()
        check(lib.vt_dist_change_volume(S._h, _ptr_array(self.rho_new), _ptr_array(self.rho),
                                        _ptr_array(self.cls), C.byref(ch), C.byref(vol), stream_ptr()))
        self.rho, self.rho_new = self.rho_new, self.rho
        return c, ch.value, vol.value

    def _gather(self, parts: List[torch.Tensor]) -> torch.Tensor:
        if self.S.nlocal == self.S.nranks:
            return torch.cat(parts)
        import torch.distributed as dist

        x = parts[0].contiguous()
        if dist.get_backend(self.group) != "nccl":  # gloo gathers host tensors
            x = x.cpu()
        out = [torch.empty_like(x) for _ in range(self.S.nranks)]
        dist.all_gather(out, x, group=self.group)
        return torch.cat(out)

    def densities(self) -> np.ndarray:
        return self._gather(self.rho).cpu().numpy()

    def displacement(self) -> np.ndarray:
        out = self.S.download(self.u)
        if self.S.nlocal != self.S.nranks:
            import torch.distributed as dist

            # disjoint owned planes: the sum assembles the field.  NCCL groups
            # reduce device tensors only; gloo takes host tensors
            dev = "cuda" if dist.get_backend(self.group) == "nccl" else "cpu"
            t = torch.from_numpy(np.array(out)).to(dev)
            dist.all_reduce(t, group=self.group)
            out = t.cpu().numpy()
        return out


def run_slabs(problem, opt, solver: SolverConfig = SolverConfig(), max_levels=None, omega: float = 0.4,
              nranks: int = 1, group=None, init_densities=None, start_iteration: int = 0, on_iteration=None,
              init_displacement=None, transport: str = "peer", scheme: str = "homogenized"):
    """run() (optimize.py:323-455) on z-slabs: all `nranks` slabs in this
    process, or -- with `group` -- one slab per rank of the group over the
    `transport` ("peer" or "nccl"); scheme "homogenized" or "galerkin" (the
    reference default, optimize.py:348)."""
    from dataclasses import replace

    from .design import DensityField, OptResult, RunRecord, VOLUME_TOL
    from .errors import NumericalError

    if group is not None:
        R = SlabRun.from_process_group(problem, opt, solver, max_levels, omega, init_densities, group,
                                       init_displacement=init_displacement, transport=transport, scheme=scheme)
    else:
        R = SlabRun(problem, opt, solver, max_levels, omega, nranks=nranks, init_densities=init_densities,
                    init_displacement=init_displacement, scheme=scheme)
    records: List = []
    converged = False
    iteration = start_iteration
    while iteration < opt.max_iterations:
        t0 = time.perf_counter()
        model_k = replace(problem.model, p=opt.penal_at(iteration))
        rep = R.solve(model_k)
        c, ch, vol = R.design_step(model_k)
        iteration += 1
        if abs(vol - opt.volfrac) > VOLUME_TOL:
            raise NumericalError(f"volume constraint violated after update: {vol} vs {opt.volfrac}")
        rec = RunRecord(iteration, c, vol, ch, rep.iterations, rep.final_rel_residual,
                        time.perf_counter() - t0, rep.aux_vector_scalars)
        records.append(rec)
        if on_iteration is not None:
            on_iteration(rec, DensityField(R.densities(), problem.regions), R.displacement())
        obj_ok = True
        if opt.obj_tol is not None and len(records) >= 2:
            obj_ok = abs(records[-1].compliance - records[-2].compliance) <= opt.obj_tol
        if ch <= opt.ch_tol and obj_ok:
            converged = True
            break
    res = OptResult(DensityField(R.densities(), problem.regions), R.displacement(), records, converged, iteration)
    R.S.close()
    return res
