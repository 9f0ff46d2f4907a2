"""Dev tool: one cfg2 MGPCG solve; run under ncu, then `python scripts/pcg_profile.py table X.csv`
prints the kernels of one CG iteration (between two pcg_s1 launches)."""
import csv, os, sys
if len(sys.argv) > 2 and sys.argv[1] == "table":
    rows = list(csv.reader(open(sys.argv[2])))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[hi]; ix = {h: i for i, h in enumerate(hdr)}
    recs = {}
    for r in rows[hi + 1:]:
        if len(r) < len(hdr): continue
        d = recs.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]][:48]})
        d[r[ix["Metric Name"]]] = (r[ix["Metric Value"]], r[ix["Metric Unit"]])
    ids = sorted(recs)
    s1 = [i for i in ids if "pcg_s1" in recs[i]["name"]]
    a, b = s1[-3], s1[-2]
    tot = 0.0
    for i in ids[ids.index(a) + 1: ids.index(b) + 1]:
        v, u = recs[i]["gpu__time_duration.sum"]
        t = float(v.replace(",", "")) / (1000.0 if u == "ns" else 1.0)
        tot += t
        print(f"{recs[i]['name']:50s} {t:8.1f} us")
    print(f"iteration total {tot:.1f} us")
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
pb = cases.cantilever(256, 128, 128)
g = pb.grid
fm = pb.boundary.fixed_mask(g)
rng = np.random.default_rng(0)
st = vb.OperatorState(g, rng.uniform(0, 1, g.n_elements), pb.model, fm)
H = vb.build_hierarchy(g, st, 7, scheme=sys.argv[1] if len(sys.argv) > 1 else "homogenized")
f = pb.boundary.external_force(g); f[fm] = 0
fd = vb.DeviceVector(st.dgrid, st.dgrid.upload(f))
x, rep = vb.mgcg_solve(st, H, fd, cfg=vb.SolverConfig(tolerance=1e-5, max_iterations=6))
torch.cuda.synchronize()
