"""Multi-rank host logic of the z-slab decomposition on CPU (gloo, world 2):
every rank derives the same plan, the NCCL bootstrap id travels over the
process group, and the halo pattern of csrc/dist.cu (send first/last owned
node plane, receive ghost planes 0 / n+1) reproduces the neighbours' planes
of the global vector."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

slabs = pytest.importorskip("paper_2201_12931_b200.slabs")  # needs the built libvoxb200.so
plan_slabs = slabs.plan_slabs


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, nx, ny, nz, levels, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        plan = plan_slabs(nz, levels, world)
        plans = [None] * world
        dist.all_gather_object(plans, plan)
        assert all(p == plan for p in plans)
        # NCCL bootstrap id over the group (what SlabSolver.from_process_group does)
        import ctypes as C
        from paper_2201_12931_b200._lib import lib

        obj = [None]
        if rank == 0:  # NCCL may be absent on a CPU-only host: then an empty id travels
            n = lib.vt_nccl_id_bytes()
            buf = (C.c_uint8 * n)()
            obj[0] = bytes(buf) if lib.vt_nccl_unique_id(buf, n) == 0 else b""
        dist.broadcast_object_list(obj, src=0)
        assert isinstance(obj[0], bytes) and len(obj[0]) in (0, lib.vt_nccl_id_bytes())
        # the peer transport's IPC handles have a fixed size that travels the same way
        assert lib.vt_peer_handle_bytes() == 64
        # halo exchange of a global node vector, vt slab layout (ghost planes 0, n+1)
        rng = np.random.default_rng(7)
        glob = torch.from_numpy(rng.standard_normal((nz + 1, ny + 1, nx + 1, 3)))
        k0, k1 = plan.slab(rank)
        n = k1 - k0
        last = rank == world - 1
        loc = torch.zeros((n + 2, ny + 1, nx + 1, 3), dtype=torch.float64)
        loc[1:n + 1 + (1 if last else 0)] = glob[k0:k1 + (1 if last else 0)]
        reqs = []
        for op, peer, p in plan.halo_pattern(rank):
            buf = loc[p]
            if op == "send":
                reqs.append(dist.isend(buf.clone(), peer))
            else:
                tmp = torch.empty_like(buf)
                dist.recv(tmp, peer)
                loc[p] = tmp
        for r in reqs:
            r.wait()
        ok = True
        if rank > 0:
            ok &= torch.equal(loc[0], glob[k0 - 1])
        if not last:
            ok &= torch.equal(loc[n + 1], glob[k1])
        # tail planes: the ranks' coarse restriction ranges tile the coarse grid
        tb = plan.tail_planes(rank, nz)
        ranges = [None] * world
        dist.all_gather_object(ranges, tb)
        q.put((rank, bool(ok), ranges))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims,levels", [((8, 4, 16), 3), ((16, 8, 32), 4)])
def test_two_rank_plan_halo_and_tail(dims, levels):
    nx, ny, nz = dims
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, nx, ny, nz, levels, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok, ranges in out:
        assert ok, f"rank {rank} ghost planes differ from the global vector"
        plan = plan_slabs(nz, levels, world)
        nzc = nz >> (plan.dist_level + 1)
        assert ranges[0][0] == 0 and ranges[-1][1] == nzc + 1
        assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))


def test_plan_rejects_unsplittable():
    with pytest.raises(ValueError):
        plan_slabs(6, 2, 4)
    p = plan_slabs(12, 3, 3)
    assert p.bounds == (0, 4, 8, 12) and p.dist_level == 1
