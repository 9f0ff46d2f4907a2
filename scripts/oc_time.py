"""Dev tool: device time of the OC bisection (vt_oc_update) at cfg2 size."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
from paper_2201_12931_b200._lib import lib
from paper_2201_12931_b200.device import ptr, stream_ptr
pb = cases.cantilever(256, 128, 128)
g = pb.grid
st = vb.OperatorState(g, np.full(g.n_elements, 0.12), pb.model, pb.boundary.fixed_mask(g))
rng = np.random.default_rng(0)
n = g.n_elements
rho = torch.tensor(rng.uniform(0.05, 0.3, n), device="cuda")
dc = torch.tensor(-rng.uniform(0.0, 1.0, n) ** 3, device="cuda")
dv = torch.ones(n, dtype=torch.float64, device="cuda")
cls = torch.zeros(n, dtype=torch.int8, device="cuda")
out = torch.empty_like(rho)
lam = C.c_double(); steps = C.c_int()
def run():
    r = lib.vt_oc_update(st.dgrid.handle, ptr(rho), ptr(cls), ptr(dc), ptr(dv), C.c_double(0.12), C.c_double(0.2),
                         C.c_double(0.5), C.c_double(1.0), ptr(out), C.byref(lam), C.byref(steps), stream_ptr())
    assert r == 0, r
run(); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10): run()
torch.cuda.synchronize()
print(os.environ.get("VT_LIB_PATH", "default"), f"oc_update {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms, steps {steps.value}, lam {lam.value:.6e}, sum {float(out.sum()):.12e}")
