"""Dev tool: BASELINE configs 3 and 4 (and 2 for reference) on ONE B200.

For each config: K(rho)u at the config's size (CUDA events, device-resident
inputs larger than L2) and two timed SIMP iterations (iterations 2-3: refresh
+ homogenized MGPCG + design step; iteration 1 untimed: hierarchy build and
graph capture).  Prints one JSON object; the committed copy lives in
profiles/r1_configs_1gpu.json.

    python scripts/configs_1gpu.py [cfg3 cfg4 ...]
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
from paper_2201_12931_b200.design import DeviceRun  # noqa: E402
from paper_2201_12931_b200.device import ptr, stream_ptr  # noqa: E402

try:  # driver-measured copy bandwidth of this pool's B200s, else the B200_PROFILING.md fallback
    with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                           "MEASURED_PEAKS.json")) as _fh:
        HBM = float(json.load(_fh)["hbm_gbs"])
except (OSError, KeyError, ValueError):
    HBM = 6650.0


def measure(name):
    c = cases.CONFIGS[name]
    prob = c["builder"](*c["dims"])
    g = prob.grid
    opt = vb.OptConfig(volfrac=c["volfrac"], filter_radius=1.5 * g.h, ch_tol=1e-12)
    R = DeviceRun(prob, opt, vb.SolverConfig(tolerance=1e-5), "homogenized", c["levels"], 0.4)
    R._set_scale(prob.model)
    d = R.d
    rng = np.random.default_rng(0)
    u = d.upload(rng.standard_normal(g.n_dofs) * (~R.fixed_mask))
    v = d.zeros()
    sp = stream_ptr()
    for _ in range(3):
        lib.vt_apply_projected(d.handle, ptr(R.scale), ptr(u), ptr(v), sp)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(10):
        lib.vt_apply_projected(d.handle, ptr(R.scale), ptr(u), ptr(v), sp)
    e1.record(s)
    e1.synchronize()
    t = e0.elapsed_time(e1) * 1e-4
    del u, v
    alg = 16.0 * g.n_dofs + 8.0 * g.n_elements
    R.solve(prob.model)
    R.design_step(prob.model)
    its, secs = [], []
    for _ in range(2):
        torch.cuda.synchronize()
        ts = time.perf_counter()
        rep = R.solve(prob.model)
        R.design_step(prob.model)
        torch.cuda.synchronize()
        secs.append(time.perf_counter() - ts)
        its.append(rep.iterations)
    return {"dims": list(c["dims"]), "levels": c["levels"], "dofs": g.n_dofs, "elements": g.n_elements,
            "builder": c["builder"].__name__, "apply_ms": t * 1e3, "apply_gdofs": g.n_dofs / t / 1e9,
            "roofline_frac": alg / t / 1e9 / HBM, "simp_iter_s": sum(secs) / len(secs), "cg_iters": its,
            "ms_per_cg_iter": 1e3 * sum(secs) / max(1, sum(its))}


def measure_two_material(name, phase_frac=0.5, e_ratio=0.5, scheme="galerkin"):
    """BASELINE cfg4's two-material SIMP (paper_2201_12931_b200.multimaterial):
    two timed SIMP iterations (iterations 2-3) with both design fields updated."""
    from paper_2201_12931_b200.multimaterial import TwoMaterialRun
    c = cases.CONFIGS[name]
    prob = c["builder"](*c["dims"])
    g = prob.grid
    opt = vb.OptConfig(volfrac=c["volfrac"], filter_radius=1.5 * g.h, ch_tol=1e-12)
    R = TwoMaterialRun(prob, opt, phase_frac, e_ratio, vb.SolverConfig(tolerance=1e-5), scheme,
                       c["levels"], 0.4)
    R.solve(prob.model)
    R.design_step(prob.model)
    its, secs, comp = [], [], []
    for _ in range(2):
        torch.cuda.synchronize()
        ts = time.perf_counter()
        rep = R.solve(prob.model)
        cc, ch, vol, pvol = R.design_step(prob.model)
        torch.cuda.synchronize()
        secs.append(time.perf_counter() - ts)
        its.append(rep.iterations)
        comp.append(cc)
    return {"dims": list(c["dims"]), "levels": c["levels"], "dofs": g.n_dofs, "elements": g.n_elements,
            "builder": c["builder"].__name__, "scheme": scheme, "phase_frac": phase_frac,
            "e_ratio": e_ratio, "simp_iter_s": sum(secs) / len(secs), "cg_iters": its,
            "compliance": comp, "ms_per_cg_iter": 1e3 * sum(secs) / max(1, sum(its))}


if __name__ == "__main__":
    names = sys.argv[1:] or ["cfg2", "cfg3", "cfg4"]
    out = {"gpu": torch.cuda.get_device_name(0), "peak_gbs": HBM,
           "note": "1 GPU; SIMP iterations 2-3 (refresh + homogenized MGPCG tol 1e-5 + design step), "
                   "device resident; apply = vt_apply_projected, 10 launches"}
    for n in names:
        if n.endswith("_two_material"):
            out[n] = measure_two_material(n[: -len("_two_material")])
        else:
            out[n] = measure(n)
        torch.cuda.empty_cache()
    print(json.dumps(out))
