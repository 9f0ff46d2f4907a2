"""BASELINE cfg5 (768x384x384: 113M elements, 342M dofs) solved end to end on
ONE B200 through the public run(): the reference defaults (tol 1e-5, cap 200,
ch_tol 0.01, max 300 iterations, p = 3, rmin = 1.5h, volfrac 0.12), the
north-star homogenized scheme with 8 levels.  Prints one JSON line; every
iteration is appended to gpurun_out/cfg5_run_progress.jsonl as it completes.

    python scripts/cfg5_full_run.py [scheme] [max_minutes] [omega]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402

scheme = sys.argv[1] if len(sys.argv) > 1 else "homogenized"
budget = float(sys.argv[2]) * 60 if len(sys.argv) > 2 else 40 * 60
omega = float(sys.argv[3]) if len(sys.argv) > 3 else 0.4
tag = scheme if omega == 0.4 else f"{scheme}_omega{omega:g}"
spec = cases.CONFIGS["cfg5"]
prob = spec["builder"](*spec["dims"])
g = prob.grid
opt = vb.OptConfig(volfrac=0.12, filter_radius=1.5 * g.h, ch_tol=0.01, max_iterations=300)
os.makedirs("gpurun_out", exist_ok=True)
log = open(f"gpurun_out/cfg5_run_progress_{tag}.jsonl", "w")
t_start = time.perf_counter()


class Stop(Exception):
    pass


def hook(rec, rho, u):
    log.write(json.dumps({"it": rec.iteration, "c": rec.compliance, "change": rec.change, "cg": rec.cg_iters,
                          "res": rec.cg_residual, "wall_s": rec.wall_s,
                          "elapsed_s": time.perf_counter() - t_start}) + "\n")
    log.flush()
    if time.perf_counter() - t_start > budget:
        raise Stop()


torch.cuda.synchronize()
stopped = False
try:
    res = vb.run(prob, opt, vb.SolverConfig(tolerance=1e-5), scheme=scheme, max_levels=spec["levels"],
                 omega=omega, on_iteration=hook)
    recs, converged, iters = res.records, res.converged, res.iterations
except Stop:
    stopped = True
    recs = None
total = time.perf_counter() - t_start
lines = [json.loads(x) for x in open(f"gpurun_out/cfg5_run_progress_{tag}.jsonl")]
out = {"workload": "cfg5 cantilever 768x384x384, 113246208 elements, 341955075 dofs, 1 B200",
       "scheme": scheme, "omega": omega, "levels": spec["levels"], "iterations": len(lines),
       "converged": (not stopped) and bool(converged), "stopped_by_time_budget": stopped,
       "total_s": total, "s_per_simp_iter": sum(x["wall_s"] for x in lines) / len(lines),
       "cg_iters_total": sum(x["cg"] for x in lines),
       "compliance_first_last": [lines[0]["c"], lines[-1]["c"]], "change_last": lines[-1]["change"],
       "device_memory_used_gb": (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 1e9,
       "note": "public run() at the reference defaults (tol 1e-5, CG cap 200, ch_tol 0.01, max 300 iterations)"}
print(json.dumps(out))
