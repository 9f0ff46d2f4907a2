"""Dev tool: device time of the cfg2 V-cycle (CUDA events, 50 cycles after warm-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
from paper_2201_12931_b200._lib import lib
from paper_2201_12931_b200.device import ptr, stream_ptr
pb = cases.cantilever(256, 128, 128)
g = pb.grid
fm = pb.boundary.fixed_mask(g)
rng = np.random.default_rng(0)
st = vb.OperatorState(g, rng.uniform(0, 1, g.n_elements), pb.model, fm)
H = vb.build_hierarchy(g, st, 7, scheme=sys.argv[1] if len(sys.argv) > 1 else "homogenized")
d = st.dgrid
r = rng.standard_normal(g.n_dofs); r[fm] = 0
f = d.upload(r); z = d.zeros()
for _ in range(5):
    lib.vt_hier_vcycle(H._h, ptr(f), ptr(z), stream_ptr())
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
for _ in range(50):
    lib.vt_hier_vcycle(H._h, ptr(f), ptr(z), stream_ptr())
e1.record()
torch.cuda.synchronize()
import hashlib
zh = hashlib.sha1(d.download(z).tobytes()).hexdigest()[:12]
print(os.environ.get("VT_LIB_PATH", "default"), f"vcycle {e0.elapsed_time(e1) / 50 * 1e3:.1f} us z-hash {zh}")
