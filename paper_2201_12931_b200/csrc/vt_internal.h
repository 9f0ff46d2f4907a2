// Host-side runtime structures of libvoxb200 (not part of the C ABI).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <map>
#include <utility>
#include <string>
#include <vector>

#include "../../include/voxb200.h"
#include "vt_device.cuh"

namespace vt {

// ----------------------------------------------------------------- errors
void set_error(const std::string& msg);
vt_status fail(vt_status code, const std::string& msg);
vt_status cuda_fail(cudaError_t e, const char* what);
#define VT_CUDA(call)                                     \
  do {                                                    \
    cudaError_t e_ = (call);                              \
    if (e_ != cudaSuccess) return ::vt::cuda_fail(e_, #call); \
  } while (0)
#define VT_TRY(call)                  \
  do {                                \
    vt_status s_ = (call);            \
    if (s_ != VT_OK) return s_;       \
  } while (0)

extern unsigned long long g_launches;  // kernels launched by this library
extern bool g_pdl;                     // launch with programmatic stream serialization (VT_PDL=0 off)

// grid for `work` independent items of `per_cta` each, capped (small coarse
// levels would otherwise launch a full-GPU grid of mostly idle CTAs)
inline int fit_grid(long long work, long long per_cta, int cap) {
  long long g = (work + per_cta - 1) / per_cta;
  if (g < 1) g = 1;
  return (int)(g < cap ? g : cap);
}

template <typename... ExpTypes, typename... ActTypes>
inline cudaError_t launch_pdl(void (*kernel)(ExpTypes...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, ActTypes&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<ActTypes>(args)...);
}
inline void count_launch(int n = 1) { g_launches += (unsigned long long)n; }

// Element-operator constants of one level (factorized hex8):
// kc = h*{lam/16, mu/8, mu/16, lam/48, mu/48, lam/144+mu/36}, kd = K0 diagonal.
struct Hex8Coef {
  double kc[6];
  double kd;
};
Hex8Coef hex8_coef(double nu, double h);

// hex8 tile height (element rows per CTA); the TMA boxes of runtime.cu follow it.
#ifndef VT_H8_TY
#define VT_H8_TY 8
#endif
constexpr int H8_TY = VT_H8_TY;

// Apply-family kernel modes.
enum Hex8Mode { H8_APPLY = 0, H8_RESID = 1, H8_SMOOTH = 2 };

struct Hex8Launch {
  int grid;        // persistent CTAs
  int tiles_x, tiles_y;
  long long work;  // tiles_x * tiles_y * owned planes
};

}  // namespace vt

// ------------------------------------------------------------------- grid
struct vt_grid {
  int device = 0;
  vt::Geom g{};
  double h = 1.0, nu = 0.3;
  vt::Hex8Coef coef{};
  uint8_t* mask = nullptr;          // P planes x (ny+1) rows x mp bytes, 1 byte per node
  CUtensorMap mask_map{};           // TMA descriptor of the mask (48x16 byte boxes)
  unsigned long long* trace = nullptr;  // per-CTA timing of hex8 launches (vt_debug_trace)
  long long n_fixed = 0;
  double* partial = nullptr;        // reduction partials (>= 4096 doubles)
  double* scalars = nullptr;        // small device scalar scratch (64 doubles)
  double* host_scalars = nullptr;   // pinned mirror
  double* scratch = nullptr;        // one node vector (projected inputs)
  double* scratch2 = nullptr;       // a second node vector
  vt::Hex8Launch h8{};
  int nsm = 148;
  std::map<const void*, CUtensorMap> vec_maps;   // node-vector TMA descriptors
  std::map<const void*, CUtensorMap> elem_maps;  // element-field TMA descriptors
  std::map<const void*, CUtensorMap> xfer_maps;  // node-vector descriptors of the TMA restriction
  std::map<const void*, CUtensorMap> fvec_maps;  // rhs tiles of the residual / smoother (owned rows)
  // PCG workspace (lazily allocated)
  double *w_x = nullptr, *w_f = nullptr, *w_r = nullptr, *w_p = nullptr, *w_q = nullptr,
         *w_z = nullptr, *w_t = nullptr, *w_d = nullptr;
  void* pcg_ctl = nullptr;          // device control block
  void* pcg_ctl_host = nullptr;     // pinned mirror (ring of 2)
  cudaGraphExec_t pcg_graph = nullptr;
  const void* pcg_key[4] = {nullptr, nullptr, nullptr, nullptr};
  unsigned long long pcg_nodes = 0;   // kernel nodes per PCG iteration graph
  cudaStream_t stream = nullptr;      // private stream of the blocking solver
  // streamed host-to-host apply (vt_apply_host): staging + copy streams
  double *io_stage = nullptr, *io_raw = nullptr, *io_proj = nullptr, *io_v = nullptr;
  double* io_stage_out = nullptr;
  double *io_pin_in = nullptr, *io_pin_out = nullptr;  // page-locked staging for pageable host arrays
  cudaStream_t io_in = nullptr, io_out = nullptr;
  cudaEvent_t io_ev[33] = {};

  long long vec_len() const { return (long long)g.P * g.nplane; }
  long long elem_len() const { return (long long)g.Q * g.eplane; }
  long long nel_local() const { return (long long)g.nx * g.ny * (g.k1 - g.k0); }
};

// ------------------------------------------------------------------- hierarchy
struct vt_hier {
  unsigned long long uid = 0;      // unique per hierarchy (graph cache key: addresses get reused)
  std::vector<vt_grid*> lv;        // lv[0] = caller's fine grid (not owned)
  std::vector<double*> u, u2, r, f, scale, rho;
  double omega = 0.4;
  int sweeps = 1;
  int nL = 0;                      // coarsest dofs
  double *A = nullptr, *W = nullptr, *Kinv = nullptr, *k0l = nullptr;
  double* A0 = nullptr;             // assembled coarsest matrix (refinement residual)
  double* cvec = nullptr;           // 3 dense coarsest vectors: fc, x0, r
  std::vector<double*> wd;          // omega / diag per dof (0 on fixed), smoothed levels
  int* status = nullptr;
  bool factored = false;
  const double* last_z = nullptr;  // buffer that holds the V-cycle output
  // Galerkin scheme (galerkin.cu): scheme 1 stores per-element matrices on levels >= 1
  int scheme = 0;                   // 0 homogenized, 1 galerkin
  double *gG = nullptr, *gcorr = nullptr, *gve = nullptr;
  int* gcorr_of = nullptr;
  std::vector<double*> mats, gdiag;  // per level (index >= 1)
  bool gal_mf = false;              // level 1 applied matrix-free (P^T K0 P)
  bool mats1_fresh = false;         // mats[1] materialized for the current refresh
  double* mats_full = nullptr;      // full 24x24 copy of one level (vt_hier_level_mats)
  long long mats_full_n = 0;
  double *gfa = nullptr, *gfb = nullptr, *gc1 = nullptr;  // fine x2 / level-1 scratch
  // fused coarse tail (tail.cu): element-product scratch, first eligible level
  double* tail_ve = nullptr;
  void* tail_bar = nullptr;        // grid-barrier words (VT_TAIL_MODE=grid)
  int tail_first = -1;
};

namespace vt {
vt_status hier_refresh_levels(vt_hier* H, double p, double kmin, double E, cudaStream_t s);
// TMA descriptors (cached per device pointer)
const CUtensorMap* vec_map(vt_grid* G, const void* ptr);
const CUtensorMap* elem_map(vt_grid* G, const void* ptr);
const CUtensorMap* xfer_map(vt_grid* G, const void* ptr, unsigned box_x, unsigned box_y);
const CUtensorMap* fvec_map(vt_grid* G, const void* ptr);

// kernel launchers (hex8_apply.cu)
Hex8Launch hex8_plan(const Geom& g, int nsm);
Hex8Launch hex8_plan_range(const Geom& g, int nsm, int nout);
vt_status hex8_configure();
vt_status launch_hex8(vt_grid* G, int mode, bool dot, const double* scale, const double* u,
                      const double* ufix, const double* f, double* out, double omega,
                      double* partial, const int* stop, cudaStream_t s, int pbeg = -1,
                      int pend = -1);
// (vectors.cu)
vt_status launch_project(vt_grid* G, const double* src, double* dst, cudaStream_t s);
vt_status launch_axpy(vt_grid* G, int mode, double a, const double* x, double* y, cudaStream_t s);
vt_status launch_assemble_dense(vt_grid* G, const double* scale, const double* k0, double* K,
                                cudaStream_t s);
vt_status launch_unpack_project(vt_grid* G, const double* dense, int pa, int pb, double* raw,
                                double* proj, cudaStream_t s);
vt_status launch_pack(vt_grid* G, const double* src, int pa, int pb, double* dense, cudaStream_t s);
vt_status launch_dot(vt_grid* G, const double* x, const double* y, double* partial, int* nparts,
                     cudaStream_t s, const int* stop = nullptr);
vt_status launch_sum_partials(const double* partial, int n, double* out, cudaStream_t s);
vt_status launch_diag(vt_grid* G, const double* scale, double* d, cudaStream_t s);
vt_status launch_zero_owned(vt_grid* G, double* v, cudaStream_t s);
int dot_grid(vt_grid* G);
// (multigrid.cu)
struct PcgCtl;
vt_status hier_vcycle_launch(vt_hier* H, const double* f0, const int* stop, double* rz_partial,
                             bool want_rz, cudaStream_t s, const double** z_out, int top = 0,
                             const PcgCtl* fused_j0 = nullptr);
int hier_rz_parts(vt_hier* H);
vt_status launch_prolong_add(vt_grid* C, vt_grid* F, const double* uc, double* uf,
                             const int* stop, cudaStream_t s);
vt_status launch_coarsen_mask(vt_grid* F, vt_grid* C, cudaStream_t s);
vt_status launch_coarsen_rho(vt_grid* F, vt_grid* C, const double* rf, double* rc, cudaStream_t s);
vt_status launch_scale(vt_grid* G, const double* rho, double p, double kmin, double E,
                       double* scale, int* bad, cudaStream_t s);
vt_status launch_restrict(vt_grid* F, vt_grid* C, const double* rf, double* fc, const int* stop,
                          int kb, int ke, cudaStream_t s);
void hex8_k0_host(double nu, double h, double* K);
// (galerkin.cu)
vt_status gal_setup(vt_hier* H);
void gal_free(vt_hier* H);
vt_status gal_refresh(vt_hier* H, cudaStream_t s);
vt_status gal_level_op(vt_hier* H, int l, int mode, const double* u, const double* f, double* out,
                       const int* stop, cudaStream_t s);
vt_status gal_jacobi0(vt_hier* H, int l, const double* f, double* u, const int* stop, cudaStream_t s);
vt_status gal_materialize_level1(vt_hier* H, cudaStream_t s);
vt_status gal_expand(vt_hier* H, int l, cudaStream_t s);
vt_status launch_gal_jacobi0(vt_grid* G, const double* f, const double* d, double omega, double* u,
                             const int* stop, cudaStream_t s);
vt_status launch_gal_vec_epilogue(vt_grid* G, int mode, const double* v, const double* u, const double* f,
                                  const double* d, double omega, double* out, const int* stop,
                                  cudaStream_t s);
vt_status launch_prolong_set(vt_grid* C, vt_grid* F, const double* uc, double* uf, const int* stop,
                             cudaStream_t s);
// (tail.cu)
vt_status tail_setup(vt_hier* H);
int hier_tail_start(vt_hier* H, int top);
vt_status launch_tail(vt_hier* H, int t, const double* ft, const int* stop, cudaStream_t s,
                      const double** z_out);
}  // namespace vt
