"""TPF1 checkpoint / VTI export at BASELINE cfg5 scale (768x384x384: 113M
elements, 342M dofs) on one GPU: device-resident state -> file -> device.

    python scripts/io_scale.py [outdir]      (prints one JSON line)

Times checkpoint_save (device tensors streamed through pinned double
buffers), checkpoint_load to numpy and straight to the device, export_vti
(float32 on the device, chunked base64) and checks the round trip bit for bit."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from paper_2201_12931_b200 import io as vio  # noqa: E402

out_dir = sys.argv[1] if len(sys.argv) > 1 else "/tmp/vt_io"
os.makedirs(out_dir, exist_ok=True)
nx, ny, nz = (int(x) for x in os.environ.get("VT_IO_DIMS", "768,384,384").split(","))
grid = vb.build_grid(nx, ny, nz, 64.0 / nx)
g = torch.Generator(device="cuda").manual_seed(0)
rho = torch.rand(grid.n_elements, dtype=torch.float64, device="cuda", generator=g)
u = torch.randn(grid.n_dofs, dtype=torch.float64, device="cuda", generator=g)
torch.cuda.synchronize()
res = {"grid": [nx, ny, nz], "elements": grid.n_elements, "dofs": grid.n_dofs}
ck = os.path.join(out_dir, "state.bin")


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, time.perf_counter() - t0


_, t = timed(lambda: vio.checkpoint_save(ck, grid, 7, rho, u))
size = os.path.getsize(ck)
res["checkpoint_bytes"] = size
res["save_s"], res["save_gbs"] = t, size / t / 1e9
ckd, t = timed(lambda: vio.checkpoint_load(ck, expect_grid=grid, device="cuda"))
res["load_device_s"], res["load_device_gbs"] = t, size / t / 1e9
res["round_trip_bit_identical"] = bool(torch.equal(ckd.densities, rho) and torch.equal(ckd.displacement, u))
del ckd
ckh, t = timed(lambda: vio.checkpoint_load(ck, expect_grid=grid))
res["load_host_s"], res["load_host_gbs"] = t, size / t / 1e9
del ckh
vti = os.path.join(out_dir, "rho.vti")
_, t = timed(lambda: vio.export_vti(rho, grid, vti))
res["vti_bytes"] = os.path.getsize(vti)
res["vti_s"] = t
os.remove(ck)
os.remove(vti)
res["note"] = ("one B200 box, files under %s; save/load stream through two 128 MB pinned buffers "
               "(D2H of chunk k+1 overlaps the write of chunk k; read of k+1 overlaps H2D of k)" % out_dir)
print(json.dumps(res))
