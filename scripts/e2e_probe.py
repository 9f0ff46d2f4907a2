"""Dev tool: where does the host->host apply time go (PCIe vs kernel vs allocation)?"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200 import cases
from paper_2201_12931_b200._lib import lib
from paper_2201_12931_b200.device import ptr, stream_ptr

pb = cases.cantilever(256, 128, 128)
g = pb.grid
n = g.n_dofs
rng = np.random.default_rng(0)
fm = pb.boundary.fixed_mask(g)
st = vb.OperatorState(g, rng.uniform(0, 1, g.n_elements), pb.model, fm)
hu = torch.from_numpy(rng.standard_normal(n)).pin_memory()
hv = torch.empty(n, dtype=torch.float64).pin_memory()
dv = torch.empty(n, dtype=torch.float64, device="cuda")
def t(fn, k=10):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / k * 1e3
print("H2D pinned 103MB ms", t(lambda: dv.copy_(hu, non_blocking=True)))
print("D2H pinned 103MB ms", t(lambda: hv.copy_(dv, non_blocking=True)))
def both():
    dv.copy_(hu, non_blocking=True); hv.copy_(dv, non_blocking=True)
print("H2D+D2H serial ms", t(both))
for nch in (1, 2, 4, 8, 16):
    f = lambda: lib.vt_apply_host(st.dgrid.handle, ptr(st.scale_dev), C.c_void_p(hu.data_ptr()), C.c_void_p(hv.data_ptr()), nch, stream_ptr())
    print("vt_apply_host nch", nch, "ms", t(f))
un = hu.numpy()
print("vb.apply (pinned in, new pinned out) ms", t(lambda: vb.apply(st, un)))
print("pinned alloc ms", t(lambda: torch.empty(n, dtype=torch.float64, pin_memory=True)))
pageable = np.array(un)
print("vb.apply (pageable in) ms", t(lambda: vb.apply(st, pageable), k=3))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
dv2 = torch.empty_like(dv)
hv2 = torch.empty(n, dtype=torch.float64).pin_memory()
def bidir():
    with torch.cuda.stream(s1):
        dv.copy_(hu, non_blocking=True)
    with torch.cuda.stream(s2):
        hv2.copy_(dv2, non_blocking=True)
    torch.cuda.synchronize()
print("concurrent H2D || D2H 103MB each ms", t(bidir))
