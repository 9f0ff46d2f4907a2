"""Dev tool: per-CTA timing of one hex8 apply launch (vt_debug_trace)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import cases  # noqa: E402
from paper_2201_12931_b200._lib import lib  # noqa: E402
from paper_2201_12931_b200.device import ptr, stream_ptr  # noqa: E402

nx, ny, nz = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 128, 128)))
pb = cases.cantilever(nx, ny, nz)
g = pb.grid
rng = np.random.default_rng(0)
fm = pb.boundary.fixed_mask(g)
st = vb.OperatorState(g, rng.uniform(0, 1, g.n_elements), pb.model, fm)
d = st.dgrid
u = d.upload(rng.standard_normal(g.n_dofs) * (~fm))
v = d.zeros()
lib.vt_debug_trace(d.handle, 1, None, 0)
for _ in range(5):
    lib.vt_apply_projected(d.handle, ptr(st.scale_dev), ptr(u), ptr(v), stream_ptr())
buf = np.zeros(4 * 4096, dtype=np.uint64)
lib.vt_debug_trace(d.handle, 1, buf.ctypes.data_as(C.c_void_p), 4096)
rec = buf.reshape(-1, 4).astype(np.int64)
rec = rec[rec[:, 0] > 0]
ncta = rec.shape[0]
print("grid", ncta, "SMs used", len(np.unique(rec[:, 2])))
t0 = rec[:, 0].min()
start, end = (rec[:, 0] - t0) / 1e3, (rec[:, 1] - t0) / 1e3
dur = end - start
print(f"launch span {end.max():.1f} us; CTA duration min {dur.min():.1f} mean {dur.mean():.1f} "
      f"max {dur.max():.1f}; start spread {start.max():.1f} us")
items = rec[:, 3] >> 32
ex0 = (rec[:, 3] >> 16) & 0xffff
ey0 = rec[:, 3] & 0xffff
ey0 = np.where(ey0 > 32767, ey0 - 65536, ey0)
ex0 = np.where(ex0 > 32767, ex0 - 65536, ex0)
smid = rec[:, 2]
order = np.argsort(dur)
print("fastest (smid,us,items,ex0,ey0):", [(int(smid[i]), round(float(dur[i]), 1), int(items[i]), int(ex0[i]), int(ey0[i])) for i in order[:8]])
print("slowest:", [(int(smid[i]), round(float(dur[i]), 1), int(items[i]), int(ex0[i]), int(ey0[i])) for i in order[-8:]])
for key, arr in (("items", items), ("smid%2", smid % 2), ("smid<74", smid < 74), ("cta<74", np.arange(ncta) < 74)):
    for val in np.unique(arr):
        m = arr == val
        print(f"  {key}={val}: n={m.sum()} mean dur {dur[m].mean():.1f}")
edge = (ex0 >= 247) | (ey0 >= 119)
print(f"  edge tiles: n={edge.sum()} mean {dur[edge].mean():.1f}; interior mean {dur[~edge].mean():.1f}")
print("dur by cta index (first 40):", np.round(dur[:40], 0).tolist())
