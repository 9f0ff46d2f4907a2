"""Load cases of BASELINE.json built through the public setup API
(recipes of SURVEY.md section 8(d), using the reference preset geometry,
app/presets.py:48-139).

  cantilever(nx, ny, nz)      cfg1 / cfg2 / cfg5: fixed x=0 face, -z line load
                              along y at (i=nx, k=0), 64 x 32 x 32 domain
  bridge(nx, ny, nz)          cfg3: 4 bottom-corner supports, -100 top pressure,
                              one passive-solid deck layer, volfrac 0.14
  selfweight(nx, ny, nz, uw)  cfg4: cantilever + GravitySpec(axis=2, g=1, uw)
"""

from __future__ import annotations

import numpy as np

from .design import Problem
from .mesh import Box, GravitySpec, Region, build_grid, classify_regions, make_boundary

__all__ = ["cantilever", "bridge", "selfweight", "CONFIGS"]


def _half_ends(n):
    w = np.ones(n)
    w[0] = w[-1] = 0.5
    return w


def _all_dofs(nodes):
    nodes = np.asarray(nodes, dtype=np.int64).ravel()
    return (3 * nodes[:, None] + np.arange(3)[None, :]).ravel()


def cantilever(nx, ny, nz, L=64.0, gravity=None) -> Problem:
    g = build_grid(nx, ny, nz, L / nx)
    j, k = np.meshgrid(np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    fixed = _all_dofs(g.node_id(0, j.ravel(), k.ravel()))
    w = _half_ends(ny + 1)
    loads = [(3 * int(g.node_id(nx, jj, 0)) + 2, float(-1.0 * g.h * w[jj])) for jj in range(ny + 1)]
    return Problem(g, make_boundary(g, fixed, loads, gravity), classify_regions(g, []))


def selfweight(nx, ny, nz, unit_weight=1e-3, L=64.0) -> Problem:
    return cantilever(nx, ny, nz, L, GravitySpec(axis=2, g=1.0, unit_weight=unit_weight))


def bridge(nx, ny, nz, L=64.0) -> Problem:
    g = build_grid(nx, ny, nz, L / nx)
    corners = [g.node_id(0, 0, 0), g.node_id(nx, 0, 0), g.node_id(0, ny, 0), g.node_id(nx, ny, 0)]
    fixed = _all_dofs(corners)
    wx, wy = _half_ends(nx + 1), _half_ends(ny + 1)
    loads = []
    for i in range(nx + 1):
        for j in range(ny + 1):
            loads.append((3 * int(g.node_id(i, j, nz)) + 2, float(-100.0 * g.h**2 * (wx[i] * wy[j]))))
    Lx, Ly, Lz = g.domain
    regions = classify_regions(g, [(Box((0.0, 0.0, Lz - g.h), (Lx, Ly, Lz)), Region.PASSIVE_SOLID)])
    return Problem(g, make_boundary(g, fixed, loads), regions)


CONFIGS = {
    "cfg1": dict(builder=cantilever, dims=(48, 24, 24), volfrac=0.12, levels=4),
    "cfg2": dict(builder=cantilever, dims=(256, 128, 128), volfrac=0.12, levels=7),
    "cfg3": dict(builder=bridge, dims=(512, 256, 256), volfrac=0.14, levels=8),
    "cfg4": dict(builder=selfweight, dims=(384, 192, 192), volfrac=0.12, levels=7),
    "cfg5": dict(builder=cantilever, dims=(768, 384, 384), volfrac=0.12, levels=8),
}
