"""Dev tool: time one homogenized V-cycle at cfg2 with the one-launch tail on
and off (CUDA events), for A/B and for ncu captures of tail_vcycle_kernel."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_12931_b200 as vb  # noqa: E402
from oracle import cpu_path as O  # noqa: E402

nx, ny, nz = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 128, 128)))
case = O.cantilever_case(nx, ny, nz)
grid = vb.build_grid(nx, ny, nz, case.h)
rng = np.random.default_rng(0)
st = vb.OperatorState(grid, rng.uniform(0.01, 1.0, grid.n_elements), vb.MaterialModel(), case.fixed_mask)
f = st.dgrid.upload(rng.standard_normal(grid.n_dofs) * (~case.fixed_mask))
fv = vb.DeviceVector(st.dgrid, f)
levels = vb.max_feasible_levels(nx, ny, nz)
for tail in ("1", "0"):
    os.environ["VT_TAIL"] = tail
    H = vb.build_hierarchy(grid, st, levels, scheme="homogenized")
    for _ in range(3):
        H.v_cycle(fv)
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(20):
        H.v_cycle(fv)
    e1.record(s)
    e1.synchronize()
    print(f"tail={tail} vcycle {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
