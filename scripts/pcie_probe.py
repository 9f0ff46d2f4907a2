"""Dev tool: PCIe duplex throughput of chunked H2D || D2H pipelines (no kernels)."""
import sys, time
import torch
n = 12830211
hu = torch.randn(n, dtype=torch.float64).pin_memory()
hv = torch.empty(n, dtype=torch.float64).pin_memory()
du = torch.empty(n, dtype=torch.float64, device="cuda")
dv = torch.empty(n, dtype=torch.float64, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def run(nch, dep):
    b = [n * c // nch for c in range(nch + 1)]
    ev = [torch.cuda.Event() for _ in range(nch)]
    for c in range(nch):
        with torch.cuda.stream(sa):
            du[b[c]:b[c + 1]].copy_(hu[b[c]:b[c + 1]], non_blocking=True)
            ev[c].record(sa)
    for c in range(nch):
        with torch.cuda.stream(sb):
            if dep:
                sb.wait_event(ev[c])
            hv[b[c]:b[c + 1]].copy_(dv[b[c]:b[c + 1]], non_blocking=True)
    torch.cuda.synchronize()
for nch in (1, 2, 4, 8, 16):
    for dep in (False, True):
        run(nch, dep)
        t0 = time.perf_counter()
        for _ in range(10):
            run(nch, dep)
        print(f"nch {nch:2d} dep {dep}: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms")
