"""BASELINE cfg5 on ONE B200: 768x384x384 cantilever (113M elements, 342M dofs).
Times K(rho)u (CUDA events) and the first SIMP iterations end to end
(refresh + homogenized MGPCG + design step, all device-resident)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
from paper_2201_12931_b200._lib import lib
from paper_2201_12931_b200.design import DeviceRun
from paper_2201_12931_b200.device import ptr, stream_ptr

dims = tuple(int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (768, 384, 384)
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 3
t0 = time.perf_counter()
prob = cases.cantilever(*dims)
g = prob.grid
opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * g.h, ch_tol=1e-12)
R = DeviceRun(prob, opt, vb.SolverConfig(tolerance=1e-5), "homogenized", None, 0.4)
R._set_scale(prob.model)
torch.cuda.synchronize()
setup = time.perf_counter() - t0
# K(rho)u on a random vector (device resident)
d = R.d
u = d.upload(np.random.default_rng(0).standard_normal(g.n_dofs) * (~R.fixed_mask))
v = d.zeros()
s = torch.cuda.current_stream()
for _ in range(3):
    lib.vt_apply_projected(d.handle, ptr(R.scale), ptr(u), ptr(v), stream_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(10):
    lib.vt_apply_projected(d.handle, ptr(R.scale), ptr(u), ptr(v), stream_ptr())
e1.record(s); e1.synchronize()
t_apply = e0.elapsed_time(e1) / 10 * 1e-3
del u, v
alg = 16.0 * g.n_dofs + 8.0 * g.n_elements
recs = []
for it in range(iters):
    torch.cuda.synchronize(); ts = time.perf_counter()
    rep = R.solve(prob.model)
    torch.cuda.synchronize(); tsol = time.perf_counter() - ts
    c, ch, vol = R.design_step(prob.model)
    torch.cuda.synchronize(); tit = time.perf_counter() - ts
    recs.append({"iteration": it + 1, "cg_iters": rep.iterations, "solve_s": round(tsol, 3),
                 "simp_iter_s": round(tit, 3), "compliance": c, "rel_res": rep.final_rel_residual})
    print(recs[-1], flush=True)
out = {"dims": dims, "elements": g.n_elements, "dofs": g.n_dofs, "levels": R.hier.n_levels,
       "setup_s": round(setup, 1), "apply_ms": t_apply * 1e3, "apply_gdofs": g.n_dofs / t_apply / 1e9,
       "apply_tbs_alg": alg / t_apply / 1e12, "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
       "simp": recs}
print(json.dumps(out))
