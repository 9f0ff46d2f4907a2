#include <algorithm>
#include <cstring>
#include <thread>
#include <atomic>
// libvoxb200 runtime: grids, TMA descriptors, layout conversion, the C ABI
// of the operator, and the PCG driver [ref: solver.py:62-191].
//
// PCG runs as a CUDA graph per iteration whose scalar decisions (alpha,
// beta, convergence candidate, true-residual swap, breakdown) are made by
// one-warp kernels on device-resident state; every vector kernel reads a
// skip word, so the host only enqueues graph launches and polls a pinned
// copy of the control block one iteration behind the device.
#include <cudaTypedefs.h>
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>

#include <mutex>
#include <string>
#include <vector>

#include "vt_internal.h"
#include "vt_pcg.cuh"

namespace vt {

static thread_local std::string g_err;
unsigned long long g_launches = 0;
bool g_pdl = [] {
  const char* e = getenv("VT_PDL");
  return !(e && e[0] == '0');
}();

void set_error(const std::string& msg) { g_err = msg; }
vt_status fail(vt_status code, const std::string& msg) {
  g_err = msg;
  return code;
}
vt_status cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
          ") at " + what;
  return e == cudaErrorMemoryAllocation ? VT_ENOMEM : VT_ECUDA;
}

// ------------------------------------------------------------ element constants
// Closed-form unit-modulus hex8 stiffness, same operation order as the
// reference [ref: element.py:23-28, 61-99].
void hex8_k0_host(double nu, double h, double* K) {
  const double VV[2][2] = {{1.0 / 3.0, 1.0 / 6.0}, {1.0 / 6.0, 1.0 / 3.0}};
  const double GG[2][2] = {{1.0, -1.0}, {-1.0, 1.0}};
  const double GV[2][2] = {{-0.5, -0.5}, {0.5, 0.5}};
  const double lam = nu / ((1 + nu) * (1 - 2 * nu));
  const double mu = 1.0 / (2 * (1 + nu));
  static double G[3][3][8][8];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      for (int p = 0; p < 8; ++p)
        for (int q = 0; q < 8; ++q) {
          double f[3];
          for (int ax = 0; ax < 3; ++ax) {
            const int pa = (p >> ax) & 1, qa = (q >> ax) & 1;
            const bool ga = ax == a, gb = ax == b;
            f[ax] = (ga && gb) ? GG[pa][qa] : ga ? GV[pa][qa] : gb ? GV[qa][pa] : VV[pa][qa];
          }
          // np.kron(f2, np.kron(f1, f0)) * h
          G[a][b][p][q] = (f[2] * (f[1] * f[0])) * h;
        }
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b)
      for (int p = 0; p < 8; ++p)
        for (int q = 0; q < 8; ++q) {
          double v = lam * G[a][b][p][q] + mu * G[b][a][p][q];
          if (a == b) v = v + mu * ((G[0][0][p][q] + G[1][1][p][q]) + G[2][2][p][q]);
          K[(3 * p + a) * 24 + 3 * q + b] = v;
        }
}

Hex8Coef hex8_coef(double nu, double h) {
  const double lam = nu / ((1 + nu) * (1 - 2 * nu));
  const double mu = 1.0 / (2 * (1 + nu));
  Hex8Coef c;
  c.kc[0] = h * lam / 16.0;
  c.kc[1] = h * mu / 8.0;
  c.kc[2] = h * mu / 16.0;
  c.kc[3] = h * lam / 48.0;
  c.kc[4] = h * mu / 48.0;
  c.kc[5] = h * (lam / 144.0 + mu / 36.0);
  double K[576];
  hex8_k0_host(nu, h, K);
  c.kd = K[0];
  return c;
}

// ------------------------------------------------------------ TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static bool encode3d(CUtensorMap* m, const void* ptr, unsigned long long d0, unsigned long long d1,
                     unsigned long long d2, unsigned long long s1, unsigned long long s2,
                     unsigned b0, unsigned b1) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {s1, s2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(ptr), dims, strides, box,
                  es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

const CUtensorMap* vec_map(vt_grid* G, const void* ptr) {
  auto it = G->vec_maps.find(ptr);
  if (it != G->vec_maps.end()) return &it->second;
  CUtensorMap m;
  const Geom& g = G->g;
  if (!encode3d(&m, ptr, 3ull * (g.nx + 1), g.ny + 1, g.P, 24ull * g.rp,
                24ull * g.rp * (g.ny + 1), 100, H8_TY + 1))
    return nullptr;
  if (G->vec_maps.size() > 256) G->vec_maps.clear();
  return &(G->vec_maps[ptr] = m);
}

// rhs vector of the residual / smoother: the same layout, box of the owned
// node rows only (TY - 1 rows)
const CUtensorMap* fvec_map(vt_grid* G, const void* ptr) {
  auto it = G->fvec_maps.find(ptr);
  if (it != G->fvec_maps.end()) return &it->second;
  CUtensorMap m;
  const Geom& g = G->g;
  if (!encode3d(&m, ptr, 3ull * (g.nx + 1), g.ny + 1, g.P, 24ull * g.rp,
                24ull * g.rp * (g.ny + 1), 100, H8_TY - 1))
    return nullptr;
  if (G->fvec_maps.size() > 256) G->fvec_maps.clear();
  return &(G->fvec_maps[ptr] = m);
}

// fine-level node vector seen as (dofs of a row, rows, planes) with a
// (box_x dofs, box_y rows, 1 plane) box: the staged blocks of the restriction
const CUtensorMap* xfer_map(vt_grid* G, const void* ptr, unsigned box_x, unsigned box_y) {
  auto it = G->xfer_maps.find(ptr);
  if (it != G->xfer_maps.end()) return &it->second;
  CUtensorMap m;
  const Geom& g = G->g;
  if (!encode3d(&m, ptr, 3ull * (g.nx + 1), g.ny + 1, g.P, 24ull * g.rp, 24ull * g.rp * (g.ny + 1), box_x, box_y))
    return nullptr;
  if (G->xfer_maps.size() > 256) G->xfer_maps.clear();
  return &(G->xfer_maps[ptr] = m);
}

const CUtensorMap* elem_map(vt_grid* G, const void* ptr) {
  auto it = G->elem_maps.find(ptr);
  if (it != G->elem_maps.end()) return &it->second;
  CUtensorMap m;
  const Geom& g = G->g;
  if (!encode3d(&m, ptr, g.nx, g.ny, g.Q, 8ull * g.ep, 8ull * g.ep * g.ny, 34, H8_TY)) return nullptr;  // 32 + even-alignment slack
  if (G->elem_maps.size() > 256) G->elem_maps.clear();
  return &(G->elem_maps[ptr] = m);
}

vt_status launch_scale(vt_grid* G, const double* rho, double p, double kmin, double E,
                       double* scale, int* bad, cudaStream_t s);


static vt_status alloc_vec(vt_grid* G, double** p) {
  if (*p) return VT_OK;
  VT_CUDA(cudaMalloc(p, G->vec_len() * sizeof(double)));
  VT_CUDA(cudaMemset(*p, 0, G->vec_len() * sizeof(double)));
  return VT_OK;
}

static double host_sum_partials(vt_grid* G, const double* dev, int n, cudaStream_t s) {
  // deterministic: same one-warp device reduction the PCG graph uses
  launch_sum_partials(dev, n, G->scalars, s);
  cudaMemcpyAsync(G->host_scalars, G->scalars, sizeof(double), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  return G->host_scalars[0];
}

}  // namespace vt

using namespace vt;

extern "C" {

const char* vt_last_error(void) { return g_err.c_str(); }
int vt_version(void) { return 1; }
uint64_t vt_launch_count(void) { return g_launches; }

vt_status vt_debug_trace(vt_grid* G, int enable, uint64_t* host_out, int max_ctas) {
  if (enable && !G->trace) {
    VT_CUDA(cudaMalloc(&G->trace, 4 * 8192 * sizeof(unsigned long long)));
    VT_CUDA(cudaMemset(G->trace, 0, 4 * 8192 * sizeof(unsigned long long)));
  }
  if (host_out && G->trace) {
    VT_CUDA(cudaDeviceSynchronize());
    const int n = max_ctas < 8192 ? max_ctas : 8192;
    VT_CUDA(cudaMemcpy(host_out, G->trace, 4 * (size_t)n * sizeof(unsigned long long),
                       cudaMemcpyDeviceToHost));
  }
  if (!enable && G->trace) {
    cudaFree(G->trace);
    G->trace = nullptr;
  }
  return VT_OK;
}

vt_status vt_copy(void* dst, const void* src, int64_t bytes, void* stream) {
  VT_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return VT_OK;
}

vt_status vt_grid_create(vt_grid** out, int nx, int ny, int nz, double h, double nu,
                         const uint8_t* node_mask, int k0, int k1, int device) {
  if (!out) return fail(VT_EINVAL, "null output handle");
  if (nx < 1 || ny < 1 || nz < 1) return fail(VT_EINVAL, "grid dimensions must be positive");
  if (!(h > 0)) return fail(VT_EINVAL, "element edge length must be positive");
  if (!(nu >= 0 && nu < 0.5)) return fail(VT_EINVAL, "Poisson ratio must lie in [0, 0.5)");
  if (k0 < 0 || k1 > nz || k0 >= k1) return fail(VT_EINVAL, "bad slab range");
  VT_CUDA(cudaSetDevice(device));
  vt_grid* G = new vt_grid();
  G->device = device;
  G->h = h;
  G->nu = nu;
  Geom& g = G->g;
  g.nx = nx; g.ny = ny; g.nz = nz; g.k0 = k0; g.k1 = k1;
  g.last = (k1 == nz) ? 1 : 0;
  g.rp = ((nx + 1) % 2 == 0) ? nx + 1 : nx + 2;
  g.ep = (nx % 2 == 0) ? nx : nx + 1;
  g.P = k1 - k0 + 2;
  g.Q = k1 - k0 + 1;
  g.pA = 1;
  g.pB = k1 - k0 + 1 + g.last;
  g.nplane = (long long)(ny + 1) * g.rp * 3;
  g.mp = ((nx + 1 + 15) / 16) * 16;
  g.mplane = (long long)(ny + 1) * g.mp;
  g.eplane = (long long)ny * g.ep;
  G->coef = hex8_coef(nu, h);
  VT_CUDA(cudaDeviceGetAttribute(&G->nsm, cudaDevAttrMultiProcessorCount, device));
  G->h8 = hex8_plan(g, G->nsm);
  VT_TRY(hex8_configure());
  VT_CUDA(cudaMalloc(&G->mask, (size_t)g.P * g.mplane));
  VT_CUDA(cudaMemset(G->mask, 0, (size_t)g.P * g.mplane));
  if (node_mask) {
    const int nown = g.pB - g.pA;
    const size_t row = (size_t)nx + 1;
    VT_CUDA(cudaMemcpy2D(G->mask + (size_t)g.pA * g.mplane, g.mp,
                         node_mask + (size_t)k0 * (ny + 1) * row, row, row,
                         (size_t)nown * (ny + 1), cudaMemcpyHostToDevice));
    long long nf = 0;
    const size_t nb = (size_t)nown * (ny + 1) * row;
    const uint8_t* src = node_mask + (size_t)k0 * (ny + 1) * row;
    for (size_t i = 0; i < nb; ++i) nf += __builtin_popcount(src[i] & 7u);
    G->n_fixed = nf;
  }
  VT_CUDA(cudaMalloc(&G->partial, 8 * 4096 * sizeof(double)));
  VT_CUDA(cudaMalloc(&G->scalars, 64 * sizeof(double)));
  VT_CUDA(cudaMemset(G->scalars, 0, 64 * sizeof(double)));
  VT_CUDA(cudaMallocHost(&G->host_scalars, 64 * sizeof(double)));
  VT_TRY(alloc_vec(G, &G->scratch));
  VT_TRY(alloc_vec(G, &G->scratch2));
  // fixed-dof mask tiles travel with the TMA pipeline of the hex8 kernel
  {
    auto fn = encode_fn();
    if (!fn) return fail(VT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {(cuuint64_t)nx + 1, (cuuint64_t)ny + 1, (cuuint64_t)g.P};
    cuuint64_t strides[2] = {(cuuint64_t)g.mp, (cuuint64_t)g.mplane};
    cuuint32_t box[3] = {48, (cuuint32_t)H8_TY, 1}, es[3] = {1, 1, 1};
    if (fn(&G->mask_map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, G->mask, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return fail(VT_ECUDA, "mask tensor map encoding failed");
  }
  *out = G;
  return VT_OK;
}

vt_status vt_grid_destroy(vt_grid* G) {
  if (!G) return VT_OK;
  cudaSetDevice(G->device);
  if (G->pcg_graph) cudaGraphExecDestroy(G->pcg_graph);
  if (G->stream) cudaStreamDestroy(G->stream);
  cudaFree(G->mask); cudaFree(G->partial); cudaFree(G->scalars); cudaFreeHost(G->host_scalars);
  cudaFree(G->scratch); cudaFree(G->scratch2);
  cudaFree(G->io_stage); cudaFree(G->io_stage_out); cudaFree(G->io_raw); cudaFree(G->io_proj); cudaFree(G->io_v);
  if (G->io_pin_in) cudaFreeHost(G->io_pin_in);
  if (G->io_pin_out) cudaFreeHost(G->io_pin_out);
  if (G->io_in) cudaStreamDestroy(G->io_in);
  if (G->io_out) cudaStreamDestroy(G->io_out);
  for (cudaEvent_t e : G->io_ev)
    if (e) cudaEventDestroy(e);
  double* ws[] = {G->w_x, G->w_f, G->w_r, G->w_p, G->w_q, G->w_z, G->w_t, G->w_d};
  for (double* w : ws) cudaFree(w);
  cudaFree(G->pcg_ctl);
  cudaFreeHost(G->pcg_ctl_host);
  delete G;
  return VT_OK;
}

int64_t vt_vec_len(const vt_grid* G) { return G->vec_len(); }
int64_t vt_elem_len(const vt_grid* G) { return G->elem_len(); }
int64_t vt_n_fixed(const vt_grid* G) { return G->n_fixed; }

vt_status vt_vec_upload(const vt_grid* G, const double* host, double* dev, void* stream) {
  const Geom& g = G->g;
  const size_t row = (size_t)(g.nx + 1) * 3 * sizeof(double);
  const size_t rows = (size_t)(g.pB - g.pA) * (g.ny + 1);
  const double* src = host + (size_t)g.k0 * (g.ny + 1) * (g.nx + 1) * 3;
  VT_CUDA(cudaMemcpy2DAsync(dev + (size_t)g.pA * g.nplane, (size_t)g.rp * 24, src, row, row, rows,
                            cudaMemcpyHostToDevice, (cudaStream_t)stream));
  return VT_OK;
}

vt_status vt_vec_download(const vt_grid* G, const double* dev, double* host, void* stream) {
  const Geom& g = G->g;
  const size_t row = (size_t)(g.nx + 1) * 3 * sizeof(double);
  const size_t rows = (size_t)(g.pB - g.pA) * (g.ny + 1);
  double* dst = host + (size_t)g.k0 * (g.ny + 1) * (g.nx + 1) * 3;
  VT_CUDA(cudaMemcpy2DAsync(dst, row, dev + (size_t)g.pA * g.nplane, (size_t)g.rp * 24, row, rows,
                            cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  return VT_OK;
}

vt_status vt_scale_from_density(vt_grid* G, const double* rho, double p, double kmin, double E,
                                double* scale, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int* bad = reinterpret_cast<int*>(G->scalars + 1);
  VT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  VT_TRY(launch_scale(G, rho, p, kmin, E, scale, bad, s));
  int hb = 0;
  VT_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  if (hb) return fail(VT_EDENSITY, "density outside [0, 1]");
  return VT_OK;
}

vt_status vt_apply(vt_grid* G, const double* scale, const double* u, double* v, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  VT_TRY(launch_project(G, u, G->scratch, s));
  return launch_hex8(G, H8_APPLY, false, scale, G->scratch, u, nullptr, v, 0.0, nullptr, nullptr,
                     s);
}

vt_status vt_apply_projected(vt_grid* G, const double* scale, const double* u, double* v,
                             void* stream) {
  return launch_hex8(G, H8_APPLY, false, scale, u, nullptr, nullptr, v, 0.0, nullptr, nullptr,
                     (cudaStream_t)stream);
}

// v = K(rho) u from host memory to host memory, streamed in z-chunks: the
// H2D copy of chunk c+1 (copy engine 1), the operator on chunk c (SMs) and the
// D2H copy of chunk c-1 (copy engine 2) overlap, so the call costs about one
// PCIe transfer instead of two plus the kernel [ref: operator.py:154-165].
// Host arrays are the reference's flat (n_dofs,) order.  Page-locked arrays
// are copied directly; pageable ones (a stock numpy array) go through the
// grid's page-locked staging buffers, filled / drained chunk by chunk by a few
// host threads so the host copies overlap the PCIe transfers (the driver's own
// pageable path serialises a bounce-buffer copy per transfer).  Blocking.
static bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

static int io_threads() {
  const unsigned hc = std::thread::hardware_concurrency();
  return (int)std::max(1u, std::min(8u, hc ? hc : 1u));
}

vt_status vt_apply_host(vt_grid* G, const double* scale, const double* hu, double* hv,
                        int nchunks, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const Geom& g = G->g;
  const int nown = g.pB - g.pA;
  const size_t row = (size_t)(g.nx + 1) * 3;              // doubles per dense node row
  const size_t dplane = row * (g.ny + 1);                 // doubles per dense node plane
  if (!G->io_stage) {
    VT_CUDA(cudaMalloc(&G->io_stage, (size_t)nown * dplane * sizeof(double)));
    VT_CUDA(cudaMalloc(&G->io_stage_out, (size_t)nown * dplane * sizeof(double)));
    VT_TRY(alloc_vec(G, &G->io_raw));
    VT_TRY(alloc_vec(G, &G->io_proj));
    VT_TRY(alloc_vec(G, &G->io_v));
    VT_CUDA(cudaStreamCreateWithFlags(&G->io_in, cudaStreamNonBlocking));
    VT_CUDA(cudaStreamCreateWithFlags(&G->io_out, cudaStreamNonBlocking));
    for (cudaEvent_t& e : G->io_ev) VT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  int nch = nchunks < 1 ? 1 : nchunks;
  if (nch > 16) nch = 16;  // (io_ev holds 2 x 16 + 1 events)
  if (nch > nown) nch = nown;
  std::vector<int> pb(nch + 1);
  for (int c = 0; c <= nch; ++c) pb[c] = g.pA + (int)((long long)nown * c / nch);
  cudaEvent_t* ev_in = G->io_ev;
  cudaEvent_t* ev_k = G->io_ev + 16;
  cudaEvent_t ev_done = G->io_ev[32];
  const double* hsrc = hu + (size_t)g.k0 * dplane;
  double* hdst = hv + (size_t)g.k0 * dplane;
  const bool stage_in = !host_pinned(hu), stage_out = !host_pinned(hv);
  if ((stage_in && !G->io_pin_in) || (stage_out && !G->io_pin_out)) {
    double** bufs[2] = {&G->io_pin_in, &G->io_pin_out};
    for (double** b : bufs)
      if (!*b) VT_CUDA(cudaMallocHost(b, (size_t)nown * dplane * sizeof(double)));
  }
  const double* src = stage_in ? G->io_pin_in : hsrc;
  double* dst = stage_out ? G->io_pin_out : hdst;
  auto chunk = [&](int c, size_t* off, size_t* cnt) {
    *off = (size_t)(pb[c] - g.pA) * dplane;
    *cnt = (size_t)(pb[c + 1] - pb[c]) * dplane;
  };
  // host staging of the input: the threads copy chunk after chunk, each a
  // slice of it; the H2D of chunk c is issued once all slices of c are in
  const int T = (stage_in || stage_out) ? io_threads() : 0;
  std::vector<std::atomic<int>> in_done(nch);
  for (auto& a : in_done) a.store(0);
  std::vector<std::thread> workers;
  if (stage_in) {
    for (int t = 0; t < T; ++t)
      workers.emplace_back([&, t]() {
        for (int c = 0; c < nch; ++c) {
          size_t off, cnt;
          chunk(c, &off, &cnt);
          const size_t a = off + cnt * t / T, b = off + cnt * (t + 1) / T;
          memcpy(G->io_pin_in + a, hsrc + a, (b - a) * sizeof(double));
          in_done[c].fetch_add(1, std::memory_order_release);
        }
      });
  }
  // the copy streams must not run ahead of work already queued on s
  VT_CUDA(cudaEventRecord(ev_done, s));
  VT_CUDA(cudaStreamWaitEvent(G->io_in, ev_done, 0));
  VT_CUDA(cudaStreamWaitEvent(G->io_out, ev_done, 0));
  vt_status st = VT_OK;
  // the input copy stream carries copies only, so the H2D engine never waits
  // for a kernel between chunks
  for (int c = 0; c < nch && st == VT_OK; ++c) {
    size_t off, cnt;
    chunk(c, &off, &cnt);
    if (stage_in)
      while (in_done[c].load(std::memory_order_acquire) < T) std::this_thread::yield();
    cudaError_t e = cudaMemcpyAsync(G->io_stage + off, src + off, cnt * sizeof(double), cudaMemcpyHostToDevice,
                                    G->io_in);
    if (e == cudaSuccess) e = cudaEventRecord(ev_in[c], G->io_in);
    if (e != cudaSuccess) st = cuda_fail(e, "vt_apply_host H2D");
  }
  for (auto& w : workers) w.join();
  workers.clear();
  if (st != VT_OK) return st;
  std::vector<int> has_out(nch, 0);
  for (int c = 0; c < nch; ++c) {
    // output planes [pb[c]-1, pb[c+1]-1): they read input planes up to pb[c+1]-1,
    // all inside chunks <= c, so the operator on chunk c starts as soon as its
    // own copy has landed (the last range runs to the end)
    const int ob = c == 0 ? pb[0] : pb[c] - 1;
    const int oe = c == nch - 1 ? pb[nch] : pb[c + 1] - 1;
    VT_CUDA(cudaStreamWaitEvent(s, ev_in[c], 0));
    const size_t ioff = (size_t)(pb[c] - g.pA) * dplane;
    VT_TRY(launch_unpack_project(G, G->io_stage + ioff, pb[c], pb[c + 1], G->io_raw, G->io_proj, s));
    if (oe > ob) {
      VT_TRY(launch_hex8(G, H8_APPLY, false, scale, G->io_proj, G->io_raw, nullptr, G->io_v, 0.0,
                         nullptr, nullptr, s, ob, oe));
      const size_t off = (size_t)(ob - g.pA) * dplane;
      const size_t cnt = (size_t)(oe - ob) * dplane;
      VT_TRY(launch_pack(G, G->io_v, ob, oe, G->io_stage_out + off, s));
      VT_CUDA(cudaEventRecord(ev_k[c], s));
      VT_CUDA(cudaStreamWaitEvent(G->io_out, ev_k[c], 0));
      VT_CUDA(cudaMemcpyAsync(dst + off, G->io_stage_out + off, cnt * sizeof(double),
                              cudaMemcpyDeviceToHost, G->io_out));
      if (stage_out) VT_CUDA(cudaEventRecord(ev_in[c], G->io_out));  // (ev_in reused: D2H of c landed)
      has_out[c] = 1;
    }
  }
  if (stage_out) {  // drain the page-locked output chunk by chunk as the D2H copies land
    std::atomic<int> bad{0};
    for (int t = 0; t < T; ++t)
      workers.emplace_back([&, t]() {
        for (int c = 0; c < nch; ++c) {
          if (!has_out[c]) continue;
          const int ob = c == 0 ? pb[0] : pb[c] - 1;
          const int oe = c == nch - 1 ? pb[nch] : pb[c + 1] - 1;
          const size_t off = (size_t)(ob - g.pA) * dplane, cnt = (size_t)(oe - ob) * dplane;
          if (cudaEventSynchronize(ev_in[c]) != cudaSuccess) {
            bad.store(1);
            return;
          }
          const size_t a = off + cnt * t / T, b = off + cnt * (t + 1) / T;
          memcpy(hdst + a, G->io_pin_out + a, (b - a) * sizeof(double));
        }
      });
    for (auto& w : workers) w.join();
    if (bad.load()) return fail(VT_ECUDA, "vt_apply_host: D2H copy failed");
  }
  VT_CUDA(cudaEventRecord(ev_done, G->io_out));
  VT_CUDA(cudaStreamWaitEvent(s, ev_done, 0));
  VT_CUDA(cudaStreamSynchronize(s));
  return VT_OK;
}


vt_status vt_diagonal(vt_grid* G, const double* scale, double* d, void* stream) {
  return launch_diag(G, scale, d, (cudaStream_t)stream);
}

vt_status vt_residual(vt_grid* G, const double* scale, const double* u, const double* f,
                      double* r, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  VT_TRY(launch_project(G, u, G->scratch, s));
  return launch_hex8(G, H8_RESID, false, scale, G->scratch, G->scratch, f, r, 0.0, nullptr,
                     nullptr, s);
}

vt_status vt_dot(vt_grid* G, const double* x, const double* y, double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int n = 0;
  VT_TRY(launch_dot(G, x, y, G->partial, &n, s));
  *out = host_sum_partials(G, G->partial, n, s);
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status vt_axpy(vt_grid* G, int mode, double a, const double* x, double* y, void* stream) {
  if (mode < 0 || mode > 2) return fail(VT_EINVAL, "axpy mode must be 0, 1 or 2");
  return launch_axpy(G, mode, a, x, y, (cudaStream_t)stream);
}

vt_status vt_project(vt_grid* G, const double* src, double* dst, void* stream) {
  return launch_project(G, src, dst, (cudaStream_t)stream);
}

vt_status vt_assemble_dense(vt_grid* G, const double* scale, const double* k0, double* K,
                            void* stream) {
  if (G->g.k0 != 0 || G->g.k1 != G->g.nz) return fail(VT_EINVAL, "dense assembly needs the whole grid");
  return launch_assemble_dense(G, scale, k0, K, (cudaStream_t)stream);
}

vt_status vt_compliance(vt_grid* G, const double* f, const double* u, double* c, void* stream) {
  return vt_dot(G, f, u, c, stream);
}

// ------------------------------------------------------------------ PCG
static vt_status pcg_capture(vt_grid* G, const double* scale, int precond, vt_hier* H,
                             cudaStream_t s, unsigned long long* nodes) {
  PcgCtl* ctl = reinterpret_cast<PcgCtl*>(G->pcg_ctl);
  double* P0 = G->partial;
  double* P1 = G->partial + 4096;
  double* P2 = G->partial + 2 * 4096;
  double* P3 = G->partial + 3 * 4096;
  const int h8g = G->h8.grid, dg = dot_grid(G);
  const unsigned long long before = g_launches;
  VT_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  vt_status st = VT_OK;
  do {
    // q = K p, p.q                                    [ref: solver.py:123-124]
    if ((st = launch_hex8(G, H8_APPLY, true, scale, G->w_p, nullptr, nullptr, G->w_q, 0.0, P0,
                          &ctl->stop, s)) != VT_OK) break;
    if ((st = launch_pcg_s1(ctl, P0, h8g, s)) != VT_OK) break;
    // r -= alpha q | x += alpha p, r = f - K x         [ref: solver.py:131-136]
    // (MG preconditioner: the same pass writes the V-cycle's first Jacobi sweep).
    // x += alpha p is deferred to the p update at the end of the iteration (it
    // reads p there anyway: one 8 B/dof stream fewer), except when the true
    // residual needs x earlier -- every 50th iteration (mode 0 here) and on a
    // convergence candidate (mode 2 after S2).
    static const bool fuse_env = !getenv("VT_FUSE_J0") || atoi(getenv("VT_FUSE_J0")) != 0;
    const bool fuse_j0 = fuse_env && precond == 2 && H->lv.size() >= 2 && H->sweeps >= 1 && H->wd[0];
    if ((st = launch_pcg_update(G, ctl, nullptr, G->w_p, G->w_r, G->w_q, P1, 1, s,
                                fuse_j0 ? H->wd[0] : nullptr, fuse_j0 ? H->u[0] : nullptr)) != VT_OK)
      break;
    if ((st = launch_pcg_update(G, ctl, G->w_x, G->w_p, G->w_r, G->w_q, P1, 0, s)) != VT_OK) break;
    if ((st = launch_hex8(G, H8_RESID, true, scale, G->w_x, G->w_x, G->w_f, G->w_r, 0.0, P1,
                          &ctl->skip_true50, s)) != VT_OK) break;
    if ((st = launch_pcg_s2(ctl, P1, dg, h8g, s)) != VT_OK) break;
    if ((st = launch_pcg_update(G, ctl, G->w_x, G->w_p, G->w_r, G->w_q, P1, 2, s)) != VT_OK) break;
    // convergence candidate: true residual          [ref: solver.py:140-149]
    if ((st = launch_hex8(G, H8_RESID, true, scale, G->w_x, G->w_x, G->w_f, G->w_t, 0.0, P2,
                          &ctl->skip_cand, s)) != VT_OK) break;
    if ((st = launch_pcg_s3(ctl, P2, h8g, s)) != VT_OK) break;
    if ((st = launch_copy(G, &ctl->skip_swap, G->w_t, G->w_r, s, G->nsm * 2)) != VT_OK) break;
    // z = M r ; r.z                                   [ref: solver.py:150-151]
    const double* z = G->w_z;
    int nrz = dg;
    if (precond == 2) {
      if ((st = hier_vcycle_launch(H, G->w_r, &ctl->stop, P3, true, s, &z, 0,
                                   fuse_j0 ? ctl : nullptr)) != VT_OK)
        break;
      nrz = hier_rz_parts(H);
      if (nrz == 0) {
        if ((st = launch_dot(G, G->w_r, z, P3, &nrz, s, &ctl->stop)) != VT_OK) break;
      }
    } else if (precond == 1) {
      if ((st = launch_jacobi_precond(G, &ctl->stop, G->w_r, G->w_d, G->w_z, P3, s)) != VT_OK) break;
    } else {
      if ((st = launch_copy(G, &ctl->stop, G->w_r, G->w_z, s)) != VT_OK) break;
      if ((st = launch_dot(G, G->w_r, G->w_z, P3, &nrz, s, &ctl->stop)) != VT_OK) break;
    }
    if ((st = launch_pcg_s4(ctl, P3, nrz, precond != 0, s)) != VT_OK) break;
    // p = z + beta p                                  [ref: solver.py:158]
    if ((st = launch_pcg_xpby(G, ctl, z, G->w_p, s, G->w_x)) != VT_OK) break;
    // measurement hook: VT_PCG_NOOPS extra skipped kernels per iteration (the
    // in-graph cost of a conditional no-op node; not for production)
    static const int noops = getenv("VT_PCG_NOOPS") ? atoi(getenv("VT_PCG_NOOPS")) : 0;
    static const int noop_grid = getenv("VT_PCG_NOOP_GRID") ? atoi(getenv("VT_PCG_NOOP_GRID")) : 0;
    for (int i = 0; i < noops && st == VT_OK; ++i)
      st = launch_copy(G, &ctl->skip_swap, G->w_t, G->w_t, s, noop_grid);
    if (st != VT_OK) break;
  } while (0);
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(s, &graph);
  if (st != VT_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture");
  *nodes = g_launches - before;
  g_launches = before;
  if (G->pcg_graph) cudaGraphExecDestroy(G->pcg_graph);
  G->pcg_graph = nullptr;
  ce = cudaGraphInstantiate(&G->pcg_graph, graph, 0);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate");
  return VT_OK;
}

vt_status vt_pcg(vt_grid* G, const double* scale, int precond, vt_hier* H, const double* f,
                 double* x, int warm, double tol, int maxit, vt_solve_report* rep, void* stream) {
  // The solve is blocking; it runs on a private non-blocking stream so that the
  // iteration graph can be captured whatever stream (even legacy 0) the caller uses.
  VT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  if (!G->stream) VT_CUDA(cudaStreamCreateWithFlags(&G->stream, cudaStreamNonBlocking));
  cudaStream_t s = G->stream;
  if (!rep) return fail(VT_EINVAL, "null report");
  memset(rep, 0, sizeof(*rep));
  if (precond == 2 && !H) return fail(VT_EINVAL, "multigrid preconditioner needs a hierarchy");
  if (precond == 2) {
    const Geom& hg = vt_hier_grid(H, 0)->g;
    if (hg.nx != G->g.nx || hg.ny != G->g.ny || hg.nz != G->g.nz)
      return fail(VT_EINVAL, "hierarchy was built for a different grid");
  }
  double** ws[] = {&G->w_x, &G->w_f, &G->w_r, &G->w_p, &G->w_q, &G->w_z, &G->w_t, &G->w_d};
  for (double** w : ws) VT_TRY(alloc_vec(G, w));
  if (!G->pcg_ctl) {
    VT_CUDA(cudaMalloc(&G->pcg_ctl, sizeof(PcgCtl)));
    VT_CUDA(cudaMallocHost(&G->pcg_ctl_host, 2 * sizeof(PcgCtl)));
  }
  const size_t vb = G->vec_len() * sizeof(double);
  int n = 0;
  // ||f||, non-finite rhs                         [ref: solver.py:81-95]
  VT_TRY(launch_dot(G, f, f, G->partial, &n, s));
  const double ff = host_sum_partials(G, G->partial, n, s);
  const double fnorm = sqrt(ff);
  if (!isfinite(fnorm)) {
    rep->breakdown = 5;
    return fail(VT_EBREAKDOWN, "rhs contains non-finite entries");
  }
  // x0 = u0 with fixed dofs zeroed
  if (warm) {
    VT_TRY(launch_project(G, x, G->w_x, s));
  } else {
    VT_CUDA(cudaMemsetAsync(G->w_x, 0, vb, s));
  }
  if (fnorm == 0.0) {
    VT_CUDA(cudaMemcpyAsync(x, G->w_x, vb, cudaMemcpyDeviceToDevice, s));
    VT_CUDA(cudaStreamSynchronize(s));
    rep->converged = 1;
    return VT_OK;
  }
  VT_CUDA(cudaMemcpyAsync(G->w_f, f, vb, cudaMemcpyDeviceToDevice, s));
  double* P1 = G->partial + 4096;
  double* P3 = G->partial + 3 * 4096;
  VT_TRY(launch_hex8(G, H8_RESID, true, scale, G->w_x, G->w_x, G->w_f, G->w_r, 0.0, P1, nullptr, s));
  double rel = sqrt(host_sum_partials(G, P1, G->h8.grid, s)) / fnorm;
  if (rel <= tol) {
    VT_CUDA(cudaMemcpyAsync(x, G->w_x, vb, cudaMemcpyDeviceToDevice, s));
    VT_CUDA(cudaStreamSynchronize(s));
    rep->converged = 1;
    rep->final_rel_residual = rel;
    return VT_OK;
  }
  // z = M r, p = z, rz = r.z                      [ref: solver.py:105-118]
  const double* z = G->w_z;
  int nrz = 0;
  int apps = 0;
  if (precond == 2) {
    VT_TRY(hier_vcycle_launch(H, G->w_r, nullptr, P3, true, s, &z));
    nrz = hier_rz_parts(H);
    if (nrz == 0) VT_TRY(launch_dot(G, G->w_r, z, P3, &nrz, s));
    apps = 1;
  } else if (precond == 1) {
    VT_TRY(vt_diagonal(G, scale, G->w_d, s));
    VT_TRY(launch_jacobi_precond(G, nullptr, G->w_r, G->w_d, G->w_z, P3, s));
    nrz = dot_grid(G);
    apps = 1;
  } else {
    VT_CUDA(cudaMemcpyAsync(G->w_z, G->w_r, vb, cudaMemcpyDeviceToDevice, s));
    VT_TRY(launch_dot(G, G->w_r, G->w_z, P3, &nrz, s));
  }
  VT_CUDA(cudaMemcpyAsync(G->w_p, z, vb, cudaMemcpyDeviceToDevice, s));
  const double rz = host_sum_partials(G, P3, nrz, s);
  rep->precond_applications = apps;
  if (!isfinite(rz) || rz <= 0.0) {
    rep->breakdown = 1;
    rep->breakdown_iter = 0;
    rep->breakdown_value = rz;
    return fail(VT_EBREAKDOWN, "preconditioned product r'z is not positive at iteration 0; "
                               "preconditioner is not SPD");
  }
  // device control block
  PcgCtl c0;
  memset(&c0, 0, sizeof(c0));
  c0.rz = rz;
  c0.fnorm = fnorm;
  c0.tol = tol;
  c0.rel = rel;
  c0.precond_apps = apps;
  c0.skip_cand = 1;
  c0.skip_swap = 1;
  VT_CUDA(cudaMemcpyAsync(G->pcg_ctl, &c0, sizeof(c0), cudaMemcpyHostToDevice, s));
  // (re)capture the iteration graph when the operator / preconditioner changed.
  // The hierarchy is keyed by its unique id, not its address: a destroyed
  // hierarchy's address (and its scale buffer's) can come back for a new one
  // whose device buffers differ -- a stale graph would read freed memory.
  const void* key[4] = {scale, (const void*)(uintptr_t)(H ? H->uid : 0),
                        (const void*)(intptr_t)(precond + 1), G};
  if (!G->pcg_graph || memcmp(key, G->pcg_key, sizeof(key)) != 0) {
    VT_CUDA(cudaStreamSynchronize(s));
    VT_TRY(pcg_capture(G, scale, precond, H, s, &G->pcg_nodes));
    memcpy(G->pcg_key, key, sizeof(key));
  }
  PcgCtl* ring = reinterpret_cast<PcgCtl*>(G->pcg_ctl_host);
  cudaEvent_t ev[2];
  VT_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  VT_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  auto launch_iter = [&](int i) -> vt_status {
    VT_CUDA(cudaGraphLaunch(G->pcg_graph, s));
    g_launches += G->pcg_nodes;
    VT_CUDA(cudaMemcpyAsync(&ring[i & 1], G->pcg_ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
    VT_CUDA(cudaEventRecord(ev[i & 1], s));
    return VT_OK;
  };
  vt_status st = VT_OK;
  if (maxit >= 1) st = launch_iter(1);
  for (int i = 1; st == VT_OK && i <= maxit; ++i) {
    if (i + 1 <= maxit) {
      st = launch_iter(i + 1);
      if (st != VT_OK) break;
    }
    cudaError_t e = cudaEventSynchronize(ev[i & 1]);
    if (e != cudaSuccess) { st = cuda_fail(e, "pcg iteration"); break; }
    if (ring[i & 1].stop) break;
  }
  cudaStreamSynchronize(s);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (st != VT_OK) return st;
  PcgCtl c;
  VT_CUDA(cudaMemcpy(&c, G->pcg_ctl, sizeof(c), cudaMemcpyDeviceToHost));
  rep->iterations = c.k;
  rep->precond_applications = c.precond_apps;
  rep->residual_drift = c.drift;
  if (c.err) {
    rep->breakdown = c.err;
    rep->breakdown_iter = c.err_iter;
    rep->breakdown_value = c.err == 3 || c.err == 2 ? c.pq : c.err_val;
    return fail(VT_EBREAKDOWN, "pcg breakdown");
  }
  double final_rel = c.rel;
  if (!c.converged) {
    // report the true residual [ref: solver.py:161-167]
    VT_TRY(launch_hex8(G, H8_RESID, true, scale, G->w_x, G->w_x, G->w_f, G->w_t, 0.0, P1, nullptr, s));
    final_rel = sqrt(host_sum_partials(G, P1, G->h8.grid, s)) / fnorm;
  }
  rep->final_rel_residual = final_rel;
  rep->converged = final_rel <= tol;
  VT_CUDA(cudaMemcpyAsync(x, G->w_x, vb, cudaMemcpyDeviceToDevice, s));
  VT_CUDA(cudaStreamSynchronize(s));
  return VT_OK;
}

}  // extern "C"
