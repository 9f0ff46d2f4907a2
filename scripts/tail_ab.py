"""A/B of the fused coarse tail at cfg2 (runs ON the GPU box): ms per PCG
iteration (50 iterations, tolerance unreachable) and per V-cycle, with the
tail on (default budget) and off, for both schemes.

    python scripts/tail_ab.py [nodes ...]
"""

import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402
from paper_2201_12931_b200._lib import lib  # noqa: E402
from paper_2201_12931_b200.device import ptr, stream_ptr  # noqa: E402


def main():
    budgets = [int(x) for x in sys.argv[1:]] or [0, 12000]
    spec = cases.CONFIGS["cfg2"]
    problem = spec["builder"](*spec["dims"])
    grid = problem.grid
    rng = np.random.default_rng(0)
    rho = rng.uniform(0.05, 1.0, grid.n_elements)
    fm = problem.boundary.fixed_mask(grid)
    st = vb.OperatorState(grid, rho, problem.model, fm, problem.stiffness())
    f = problem.boundary.external_force(grid) if hasattr(problem.boundary, "external_force") else None
    if f is None or not np.any(f):
        f = rng.standard_normal(grid.n_dofs)
        f[fm] = 0.0
    out = []
    for scheme in ("homogenized", "galerkin"):
        for b in budgets:
            lib.vt_tail_config(b)
            H = vb.build_hierarchy(grid, st, spec["levels"], scheme=scheme)
            t = lib.vt_hier_tail_level(H._h)
            cfg = vb.SolverConfig(tolerance=1e-30, max_iterations=60)
            vb.mgcg_solve(st, H, f, cfg=cfg)  # capture + warm
            torch.cuda.synchronize()
            res = []
            for _ in range(3):
                t0 = time.perf_counter()
                x, rep = vb.mgcg_solve(st, H, f, cfg=cfg)
                torch.cuda.synchronize()
                res.append((time.perf_counter() - t0) / rep.iterations * 1e3)
            fd = st.dgrid.upload(f)
            zd = st.dgrid.zeros()
            for _ in range(3):
                lib.vt_hier_vcycle(H._h, ptr(fd), ptr(zd), stream_ptr())
            torch.cuda.synchronize()
            l0 = vb.launch_count()
            t0 = time.perf_counter()
            for _ in range(20):
                lib.vt_hier_vcycle(H._h, ptr(fd), ptr(zd), stream_ptr())
            torch.cuda.synchronize()
            vc = (time.perf_counter() - t0) / 20 * 1e3
            if b > 0:
                import ctypes as C
                lib.vt_tail_trace(1, None, 0)
                buf = (C.c_uint64 * 64)()
                for _ in range(3):
                    lib.vt_hier_vcycle(H._h, ptr(fd), ptr(zd), stream_ptr())
                lib.vt_tail_trace(1, buf, 64)
                lib.vt_tail_trace(0, None, 0)
                ts = [buf[63]] + [buf[i] for i in range(63) if buf[i]]
                print("phases_us", [round((ts[i + 1] - ts[i]) / 1e3, 2) for i in range(len(ts) - 1)],
                      "total_us", round((ts[-1] - ts[0]) / 1e3, 1), flush=True)
            rec = {"scheme": scheme, "tail_nodes": b, "tail_level": t, "ms_per_pcg_iter": min(res),
                   "ms_per_vcycle_call": vc, "launches_per_vcycle": (vb.launch_count() - l0) / 20,
                   "final_rel": rep.final_rel_residual}
            print(json.dumps(rec), flush=True)
            out.append(rec)
            del H
    return out


if __name__ == "__main__":
    main()
