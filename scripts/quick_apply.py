"""Dev tool: time the hex8 apply / residual / smoother kernels and one MGPCG solve
at a given size (CUDA events on the launching stream)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
import paper_2201_12931_b200 as vb
from paper_2201_12931_b200._lib import lib
from paper_2201_12931_b200.device import ptr, stream_ptr
from oracle import cpu_path as O

nx, ny, nz = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (256, 128, 128)))
case = O.cantilever_case(nx, ny, nz)
grid = vb.build_grid(nx, ny, nz, case.h)
rng = np.random.default_rng(0)
rho = rng.uniform(0.0, 1.0, grid.n_elements)
st = vb.OperatorState(grid, rho, vb.MaterialModel(), case.fixed_mask)
d = st.dgrid
u = d.upload(rng.standard_normal(grid.n_dofs) * (~case.fixed_mask))
v = d.zeros()
n = grid.n_dofs
B = 16 * n + 8 * grid.n_elements
s = torch.cuda.current_stream()
def timeit(fn, reps=20):
    for _ in range(3): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps): fn()
    e1.record(s); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3
t = timeit(lambda: lib.vt_apply(d.handle, ptr(st.scale_dev), ptr(u), ptr(v), stream_ptr()))
print(f"apply(+project) {nx}x{ny}x{nz}: {t*1e6:.1f} us  {n/t/1e9:.2f} GDOF/s  {B/t/1e9:.0f} GB/s alg")
f = d.upload(case.f_ext * (~case.fixed_mask))
t = timeit(lambda: lib.vt_residual(d.handle, ptr(st.scale_dev), ptr(u), ptr(f), ptr(v), stream_ptr()))
print(f"residual(+project): {t*1e6:.1f} us")
H = vb.build_hierarchy(grid, st, vb.max_feasible_levels(nx, ny, nz), scheme="homogenized")
z = d.zeros()
t = timeit(lambda: lib.vt_hier_vcycle(H._h, ptr(f), ptr(z), stream_ptr()), reps=10)
print(f"vcycle: {t*1e3:.3f} ms")
for it in range(2):
    t0 = time.perf_counter()
    x, rep = vb.mgcg_solve(st, H, vb.DeviceVector(d, f), cfg=vb.SolverConfig(tolerance=1e-5))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"mgcg: {rep.iterations} its, {dt*1e3:.1f} ms, {dt/max(rep.iterations,1)*1e3:.3f} ms/it, rel {rep.final_rel_residual:.2e}")
print("launches", vb.launch_count())
