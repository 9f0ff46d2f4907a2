// Vector passes, deterministic reductions and the device-resident PCG scalar
// logic [ref: solver.py:62-167].  All element-wise updates reproduce the
// reference's numpy rounding (separate multiply and add, no contraction).
#include <math.h>

#include "vt_internal.h"
#include "vt_pcg.cuh"

namespace vt {

constexpr int VT_THREADS = 256;
#ifndef VT_EW_B
#define VT_EW_B 2
#endif
constexpr int EW_B = VT_EW_B;  // elements in flight per thread in the streaming kernels

int dot_grid(vt_grid* G) { return G->nsm * 4; }

// owned region of a node vector: planes [pA, pB) are contiguous
__device__ __forceinline__ void owned_range(const Geom& g, long long& b, long long& e) {
  b = (long long)g.pA * g.nplane;
  e = (long long)g.pB * g.nplane;
}

// ---------------------------------------------------------------- projection
__global__ void project_kernel(Geom g, const uint8_t* mask, const double* src, double* dst) {
  griddep_wait();
  long long b, e;
  owned_range(g, b, e);
  const long long nn = (e - b) / 3;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const long long node = b / 3 + t;
    const int i = (int)(node % g.rp);
    const long long r = node / g.rp;
    const unsigned m = i <= g.nx ? mask[(r / (g.ny + 1)) * g.mplane + (r % (g.ny + 1)) * g.mp + i] : 0u;
#pragma unroll
    for (int c = 0; c < 3; ++c) dst[node * 3 + c] = ((m >> c) & 1u) ? 0.0 : src[node * 3 + c];
  }
}

vt_status launch_project(vt_grid* G, const double* src, double* dst, cudaStream_t s) {
  launch_pdl(project_kernel, fit_grid((long long)(G->g.pB - G->g.pA) * G->g.nplane / 3, VT_THREADS, G->nsm * 8), VT_THREADS, 0, s, G->g, G->mask, src, dst);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// dense reference-order planes [pa, pb) (host order, first plane at `dense`)
// -> vt layout: raw copy (identity values on fixed dofs) and the projected copy
// the operator multiplies (fixed dofs zero) [ref: operator.py:71-81]
__global__ void unpack_project_kernel(Geom g, const uint8_t* mask, const double* __restrict__ dense,
                                      int pa, int pb, double* __restrict__ raw,
                                      double* __restrict__ proj) {
  griddep_wait();
  const long long row = (long long)(g.nx + 1);
  const long long nn = (long long)(pb - pa) * (g.ny + 1) * row;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % row);
    const long long r = t / row;
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + pa;
    const long long node = ((long long)p * (g.ny + 1) + j) * g.rp + i;
    const unsigned m = mask[(long long)p * g.mplane + (long long)j * g.mp + i];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const double v = dense[t * 3 + c];
      raw[node * 3 + c] = v;
      proj[node * 3 + c] = ((m >> c) & 1u) ? 0.0 : v;
    }
  }
}
// vt layout planes [pa, pb) -> dense reference-order rows (contiguous D2H)
__global__ void pack_kernel(Geom g, const double* __restrict__ src, int pa, int pb,
                            double* __restrict__ dense) {
  griddep_wait();
  const long long w = (long long)(g.nx + 1) * 3;
  const long long nn = (long long)(pb - pa) * (g.ny + 1) * w;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / w;
    const long long d = t - r * w;
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + pa;
    dense[t] = src[((long long)p * (g.ny + 1) + j) * g.rp * 3 + d];
  }
}
vt_status launch_pack(vt_grid* G, const double* src, int pa, int pb, double* dense, cudaStream_t s) {
  launch_pdl(pack_kernel, G->nsm * 4, VT_THREADS, 0, s, G->g, src, pa, pb, dense);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status launch_unpack_project(vt_grid* G, const double* dense, int pa, int pb, double* raw,
                                double* proj, cudaStream_t s) {
  launch_pdl(unpack_project_kernel, G->nsm * 4, VT_THREADS, 0, s, G->g, G->mask, dense, pa, pb, raw, proj);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

__global__ void zero_owned_kernel(Geom g, double* v) {
  griddep_wait();
  long long b, e;
  owned_range(g, b, e);
  for (long long i = b + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e;
       i += (long long)gridDim.x * blockDim.x)
    v[i] = 0.0;
}
vt_status launch_zero_owned(vt_grid* G, double* v, cudaStream_t s) {
  launch_pdl(zero_owned_kernel, fit_grid((long long)(G->g.pB - G->g.pA) * G->g.nplane, VT_THREADS, G->nsm * 8), VT_THREADS, 0, s, G->g, v);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// ---------------------------------------------------------------- axpy
// numpy-rounded vector updates over the whole vt vector (ghosts / pads stay 0):
//   mode 0: y = y + a*x   (`y += a * x`)     mode 1: y = y - a*x   (`y -= a * x`)
//   mode 2: y = x + a*y   (`y = x + a * y`)
__global__ void axpy_kernel(long long n, int mode, double a, const double* __restrict__ x,
                            double* __restrict__ y) {
  griddep_wait();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double yi = y[i], xi = x[i];
    if (mode == 0) y[i] = __dadd_rn(yi, __dmul_rn(a, xi));
    else if (mode == 1) y[i] = __dsub_rn(yi, __dmul_rn(a, xi));
    else y[i] = __dadd_rn(xi, __dmul_rn(a, yi));
  }
}
vt_status launch_axpy(vt_grid* G, int mode, double a, const double* x, double* y, cudaStream_t s) {
  const long long n = (long long)G->vec_len();
  launch_pdl(axpy_kernel, fit_grid(n, VT_THREADS, G->nsm * 8), VT_THREADS, 0, s, n, mode, a, x, y);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// Dense global stiffness with identity rows / columns on fixed dofs
// [ref: operator.py:187-205].  One CTA of 576 threads walks the elements in the
// reference's order; thread (a, b) adds s_e K0[a][b] into K[dof_a][dof_b].
// `scale` is plain (n_elements,) in the reference element order.
// An element's 24 dofs are distinct, so its 576 targets are too, and the
// barrier per element makes every entry accumulate in ascending element order
// -- the order of np.add.at -- so K is bit-identical to the reference's.
__global__ void __launch_bounds__(576, 1)
    assemble_dense_kernel(Geom g, const double* scale, const double* k0, const uint8_t* mask, int n,
                          double* K) {
  griddep_wait();
  const int nx1 = g.nx + 1, ny1 = g.ny + 1;
  const long long nn = (long long)n * n;
  for (long long t = threadIdx.x; t < nn; t += blockDim.x) K[t] = 0.0;
  __syncthreads();
  const int t = threadIdx.x, a = t / 24, b = t % 24, ca = a / 3, cb = b / 3;
  const double kab = k0[t];
  const int nel = g.nx * g.ny * (g.k1 - g.k0);
  for (int e = 0; e < nel; ++e) {
    const int i = e % g.nx, j = (e / g.nx) % g.ny, k = e / (g.nx * g.ny);
    const double s = scale[e];
    const long long na = (i + (ca & 1)) + (long long)(j + ((ca >> 1) & 1)) * nx1 + (long long)(k + (ca >> 2)) * nx1 * ny1;
    const long long nb = (i + (cb & 1)) + (long long)(j + ((cb >> 1) & 1)) * nx1 + (long long)(k + (cb >> 2)) * nx1 * ny1;
    double* dst = K + (3 * na + a % 3) * n + 3 * nb + b % 3;
    *dst = __dadd_rn(*dst, __dmul_rn(s, kab));
    __syncthreads();
  }
  // fixed rows / columns -> identity
  for (long long q = threadIdx.x; q < nn; q += blockDim.x) {
    const int r = (int)(q / n), c = (int)(q % n);
    const int nr = r / 3, nc = c / 3;
    const unsigned mr = mask[mask_off(g, nr / (nx1 * ny1) + 1, (nr / nx1) % ny1, nr % nx1)];
    const unsigned mc = mask[mask_off(g, nc / (nx1 * ny1) + 1, (nc / nx1) % ny1, nc % nx1)];
    if (((mr >> (r % 3)) & 1u) || ((mc >> (c % 3)) & 1u)) K[q] = (r == c) ? 1.0 : 0.0;
  }
}
vt_status launch_assemble_dense(vt_grid* G, const double* scale, const double* k0, double* K,
                                cudaStream_t s) {
  const int n = (int)(3LL * (G->g.nx + 1) * (G->g.ny + 1) * (G->g.k1 - G->g.k0 + 1));
  launch_pdl(assemble_dense_kernel, 1, 576, 0, s, G->g, scale, k0, G->mask, n, K);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// ---------------------------------------------------------------- dots
__global__ void dot_kernel(Geom g, const double* __restrict__ x, const double* __restrict__ y,
                           double* partial, const int* stop) {
  griddep_wait();
  __shared__ double red[VT_THREADS / 32];
  if (stop && *(volatile const int*)stop) return;
  long long b, e;
  owned_range(g, b, e);
  double acc = 0.0;
  const double2* x2 = reinterpret_cast<const double2*>(x + b);
  const double2* y2 = reinterpret_cast<const double2*>(y + b);
  const long long n2 = (e - b) / 2;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n2;
       i += (long long)gridDim.x * blockDim.x) {
    const double2 a = x2[i], c = y2[i];
    acc = fma(a.x, c.x, acc);
    acc = fma(a.y, c.y, acc);
  }
  const double s = block_sum<VT_THREADS>(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

vt_status launch_dot(vt_grid* G, const double* x, const double* y, double* partial, int* nparts,
                     cudaStream_t s, const int* stop) {
  const int grid = dot_grid(G);
  launch_pdl(dot_kernel, grid, VT_THREADS, 0, s, G->g, x, y, partial, stop);
  count_launch();
  if (nparts) *nparts = grid;
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

__global__ void sum_partials_kernel(const double* p, int n, double* out) {
  griddep_wait();
  const double s = warp_sum_partials(p, n);
  if (threadIdx.x == 0) *out = s;
}
vt_status launch_sum_partials(const double* partial, int n, double* out, cudaStream_t s) {
  launch_pdl(sum_partials_kernel, 1, 32, 0, s, partial, n, out);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// ---------------------------------------------------------------- diagonal
// d = K0_ii * sum over incident elements (corner order c = 0..7), 1 on fixed
// [ref: operator.py:84-105].  Node plane p gets corners ck=0 from element
// layer q=p and ck=1 from q=p-1 (local coords, see voxb200.h).
__device__ __forceinline__ double node_diag(const Geom& g, const double* scale, int p, int j,
                                            int i, double kd) {
  double d = 0.0;
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int ei = i - (c & 1), ej = j - ((c >> 1) & 1), q = p - ((c >> 2) & 1);
    const int k = q + g.k0 - 1;  // global element layer
    if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || q < 0 || q >= g.Q || k < 0 || k >= g.nz)
      continue;
    d = __dadd_rn(d, __dmul_rn(scale[elem_off(g, q, ej, ei)], kd));
  }
  return d;
}

__global__ void diag_kernel(Geom g, const uint8_t* mask, const double* scale, double kd,
                            double* out) {
  griddep_wait();
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (g.nx + 1));
    const long long r = t / (g.nx + 1);
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const long long node = node_off(g, p, j, i);
    const double d = node_diag(g, scale, p, j, i, kd);
    const unsigned m = mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int c = 0; c < 3; ++c) out[node * 3 + c] = ((m >> c) & 1u) ? 1.0 : d;
  }
}

vt_status launch_diag(vt_grid* G, const double* scale, double* d, cudaStream_t s) {
  launch_pdl(diag_kernel, G->nsm * 8, VT_THREADS, 0, s, G->g, G->mask, scale, G->coef.kd, d);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// u = omega * (f / d) on free dofs, 0 on fixed: the first pre-smoothing sweep
// from a zero iterate, bit-identical to the reference's
// u += omega * ((f - K 0) / d) [ref: multigrid.py:387-393, 423-424].
// One thread per node pair (i, i+1), i even: the row pitch is even, so the
// pair's 6 doubles are 16-byte aligned and move as 3 vector loads / stores
// (scalar per-node access was L2-request bound at 3 doubles per node).
__global__ void jacobi0_kernel(Geom g, const uint8_t* __restrict__ mask,
                               const double* __restrict__ scale, double kd, double omega,
                               const double* __restrict__ f, double* __restrict__ u,
                               const int* stop) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  const int hp = (g.nx + 2) / 2;  // node pairs per row (last may hold the pad node)
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * hp;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = 2 * (int)(t % hp);
    const long long r = t / hp;
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const long long node = node_off(g, p, j, i);
    const unsigned m2 = *reinterpret_cast<const uint16_t*>(mask + mask_off(g, p, j, i));
    const double d0 = node_diag(g, scale, p, j, i, kd);
    const bool two = i + 1 <= g.nx;
    const double d1 = two ? node_diag(g, scale, p, j, i + 1, kd) : 1.0;
    const double2* fv = reinterpret_cast<const double2*>(f + node * 3);
    const double2 a = fv[0], b = fv[1], c = fv[2];
    const double fin[6] = {a.x, a.y, b.x, b.y, c.x, c.y};
    double o[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      const int nd = q / 3, comp = q % 3;
      const unsigned m = (m2 >> (8 * nd)) & 0xffu;
      const double d = nd ? d1 : d0;
      o[q] = ((m >> comp) & 1u) || (nd && !two) ? 0.0 : __dmul_rn(omega, __ddiv_rn(fin[q], d));
    }
    double2* uv = reinterpret_cast<double2*>(u + node * 3);
    uv[0] = make_double2(o[0], o[1]);
    uv[1] = make_double2(o[2], o[3]);
    uv[2] = make_double2(o[4], o[5]);
  }
}

vt_status launch_jacobi0(vt_grid* G, const double* scale, double omega, const double* f,
                         double* u, const int* stop, cudaStream_t s) {
  launch_pdl(jacobi0_kernel, fit_grid((long long)(G->g.pB - G->g.pA) * (G->g.ny + 1) * ((G->g.nx + 2) / 2), VT_THREADS, G->nsm * 8), VT_THREADS, 0, s, G->g, G->mask, scale, G->coef.kd, omega, f, u,
                                                   stop);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// Damped inverse diagonal per dof, w = omega / d (0 on fixed dofs and row
// pads), computed once per refresh so the first Jacobi sweep of every V-cycle
// is a pure stream u = w f (diag assembly in the reference corner order,
// operator.py:116-124; one rounding of omega/d shared with the smoother
// epilogue, see hex8_apply.cu).
__global__ void wdiag_kernel(Geom g, const uint8_t* __restrict__ mask,
                             const double* __restrict__ scale, double kd, double omega,
                             double* __restrict__ w) {
  griddep_wait();
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (g.nx + 1));
    const long long r = t / (g.nx + 1);
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const long long node = node_off(g, p, j, i);
    const double wv = __ddiv_rn(omega, node_diag(g, scale, p, j, i, kd));
    const unsigned m = mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int c = 0; c < 3; ++c) w[node * 3 + c] = ((m >> c) & 1u) ? 0.0 : wv;
  }
}

vt_status launch_wdiag(vt_grid* G, const double* scale, double omega, double* w, cudaStream_t s) {
  VT_CUDA(cudaMemsetAsync(w, 0, G->vec_len() * sizeof(double), s));
  launch_pdl(wdiag_kernel, G->nsm * 8, VT_THREADS, 0, s, G->g, (const uint8_t*)G->mask, scale,
             G->coef.kd, omega, w);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// u = w f over the owned node planes (first damped Jacobi sweep from zero,
// multigrid.py:387-393); 16-byte accesses, fully coalesced.
__global__ void jacobi0w_kernel(long long n2, const double2* __restrict__ w,
                                const double2* __restrict__ f, double2* __restrict__ u,
                                const int* stop, const PcgCtl* fused) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  // already produced by this iteration's pcg_update, unless r was replaced
  // by a true residual (skip_rec: periodic one; !skip_swap: candidate copy)
  if (fused && !fused->skip_rec && fused->skip_swap) return;
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; t0 < n2; t0 += EW_B * st) {
    double2 a[EW_B], b[EW_B];
#pragma unroll
    for (int k = 0; k < EW_B; ++k) {
      const long long t = t0 + k * st;
      if (t < n2) {
        a[k] = w[t];
        b[k] = f[t];
      }
    }
#pragma unroll
    for (int k = 0; k < EW_B; ++k) {
      const long long t = t0 + k * st;
      if (t < n2)
        u[t] = make_double2(a[k].x == 0.0 ? 0.0 : __dmul_rn(a[k].x, b[k].x),
                            a[k].y == 0.0 ? 0.0 : __dmul_rn(a[k].y, b[k].y));
    }
  }
}

vt_status launch_jacobi0w(vt_grid* G, const double* w, const double* f, double* u, const int* stop,
                          cudaStream_t s, const PcgCtl* fused) {
  const long long a = (long long)G->g.pA * G->g.nplane, b = (long long)G->g.pB * G->g.nplane;
  const long long n2 = (b - a) / 2;  // nplane is even (rp even)
  // fused: a no-op in most PCG iterations, where a launch's cost grows with its
  // CTA count (measured in-graph: ~0.8 us at 1 CTA, 2.2 us at 592, 3.7 us at 1184)
  launch_pdl(jacobi0w_kernel, fit_grid(n2, VT_THREADS * EW_B, G->nsm * (fused ? 2 : 8)), VT_THREADS, 0, s, n2,
             reinterpret_cast<const double2*>(w + a), reinterpret_cast<const double2*>(f + a),
             reinterpret_cast<double2*>(u + a), stop, fused);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// ---------------------------------------------------------------- PCG passes
// x += alpha p ; r -= alpha q ; partial ||r||^2   [ref: solver.py:131-136]
// (16-byte vector accesses: owned ranges start and end on even indices)
// mode 1: the recursive update (skipped on k % 50 == 0), plus x += alpha p when
//         x != nullptr (the slab solver; the single-GPU graph defers x to xpby);
// mode 0: x += alpha p only, on the k % 50 == 0 iterations (before the true
//         residual needs it);
// mode 2: x += alpha p only, for a convergence candidate whose x was deferred.
// With w != nullptr (MG-preconditioned solves) mode 1 also writes the
// V-cycle's first damped Jacobi sweep u0 = w r of the updated residual
// (multigrid.py:387-393), which the V-cycle then skips unless r was replaced
// by a true residual this iteration (jacobi0w_kernel's ctl test).
__global__ void pcg_update_kernel(Geom g, const PcgCtl* ctl, double* __restrict__ x,
                                  const double* __restrict__ p, double* __restrict__ r,
                                  const double* __restrict__ q, double* partial, int mode,
                                  const double* __restrict__ w, double* __restrict__ u0) {
  griddep_wait();
  __shared__ double red[VT_THREADS / 32];
  // The host enqueues iteration k+1 before it sees that iteration k stopped, so
  // every pass of an iteration checks `stop` itself: S1 of a stopped solve
  // returns early and leaves the skip flags of the last live iteration behind.
  const int skip = mode == 1 ? ctl->skip_rec : (mode == 0 ? ctl->skip_true50 : ctl->skip_xc);
  if (skip || ctl->stop) return;
  const bool with_r = mode == 1, with_x = x != nullptr;
  const double alpha = ctl->alpha;
  long long b, e;
  owned_range(g, b, e);
  double2* x2 = reinterpret_cast<double2*>(x + b);
  const double2* p2 = reinterpret_cast<const double2*>(p + b);
  double2* r2 = reinterpret_cast<double2*>(r + b);
  const double2* q2 = reinterpret_cast<const double2*>(q + b);
  const double2* w2 = reinterpret_cast<const double2*>(w + b);
  double2* u2 = reinterpret_cast<double2*>(u0 + b);
  const bool fuse = with_r && w != nullptr;
  const long long n2 = (e - b) / 2;
  double acc = 0.0;
  // EW_B independent elements per thread in flight (same per-thread element
  // order as a plain grid-stride loop, so the partial sums are unchanged)
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n2; i0 += EW_B * st) {
    double2 pv[EW_B], xv[EW_B], qv[EW_B], rv[EW_B], wv[EW_B];
#pragma unroll
    for (int k = 0; k < EW_B; ++k) {
      const long long i = i0 + k * st;
      if (i < n2) {
        if (with_x) {
          pv[k] = p2[i];
          xv[k] = x2[i];
        }
        if (with_r) {
          qv[k] = q2[i];
          rv[k] = r2[i];
        }
        if (fuse) wv[k] = w2[i];
      }
    }
#pragma unroll
    for (int k = 0; k < EW_B; ++k) {
      const long long i = i0 + k * st;
      if (i >= n2) break;
      if (with_x) {
        xv[k].x = __dadd_rn(xv[k].x, __dmul_rn(alpha, pv[k].x));
        xv[k].y = __dadd_rn(xv[k].y, __dmul_rn(alpha, pv[k].y));
        x2[i] = xv[k];
      }
      if (with_r) {
        rv[k].x = __dsub_rn(rv[k].x, __dmul_rn(alpha, qv[k].x));
        rv[k].y = __dsub_rn(rv[k].y, __dmul_rn(alpha, qv[k].y));
        r2[i] = rv[k];
        acc = fma(rv[k].x, rv[k].x, acc);
        acc = fma(rv[k].y, rv[k].y, acc);
        if (fuse)
          u2[i] = make_double2(wv[k].x == 0.0 ? 0.0 : __dmul_rn(wv[k].x, rv[k].x),
                               wv[k].y == 0.0 ? 0.0 : __dmul_rn(wv[k].y, rv[k].y));
      }
    }
  }
  if (with_r) {
    const double s = block_sum<VT_THREADS>(acc, red);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
  }
}

// p = z + beta p   [ref: solver.py:158]; with x: first x += alpha p (old p),
// the update pcg_update deferred, unless x is already current this iteration
__global__ void pcg_xpby_kernel(Geom g, const PcgCtl* ctl, const double* __restrict__ z,
                                double* __restrict__ p, double* __restrict__ x) {
  griddep_wait();
  if (ctl->stop) return;
  const double beta = ctl->beta, alpha = ctl->alpha;
  const bool with_x = x != nullptr && !ctl->x_done;
  long long b, e;
  owned_range(g, b, e);
  const double2* z2 = reinterpret_cast<const double2*>(z + b);
  double2* p2 = reinterpret_cast<double2*>(p + b);
  double2* x2 = reinterpret_cast<double2*>(x + b);
  const long long n2 = (e - b) / 2;
  const long long st = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n2; i0 += EW_B * st) {
    double2 zv[EW_B], pv[EW_B], xv[EW_B];
#pragma unroll
    for (int k = 0; k < EW_B; ++k) {
      const long long i = i0 + k * st;
      if (i < n2) {
        zv[k] = z2[i];
        pv[k] = p2[i];
        if (with_x) xv[k] = x2[i];
      }
    }
#pragma unroll
    for (int k = 0; k < EW_B; ++k) {
      const long long i = i0 + k * st;
      if (i >= n2) break;
      if (with_x) {
        xv[k].x = __dadd_rn(xv[k].x, __dmul_rn(alpha, pv[k].x));
        xv[k].y = __dadd_rn(xv[k].y, __dmul_rn(alpha, pv[k].y));
        x2[i] = xv[k];
      }
      pv[k].x = __dadd_rn(zv[k].x, __dmul_rn(beta, pv[k].x));
      pv[k].y = __dadd_rn(zv[k].y, __dmul_rn(beta, pv[k].y));
      p2[i] = pv[k];
    }
  }
}

// conditional copy dst = src (skip flag)
__global__ void copy_kernel(Geom g, const int* skip, const double* __restrict__ src,
                            double* __restrict__ dst) {
  griddep_wait();
  if (skip && *(volatile const int*)skip) return;  // (skip_swap is 1 once stopped)
  long long b, e;
  owned_range(g, b, e);
  for (long long i = b + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// z = r / d (+ partial r.z) -- Jacobi preconditioner [ref: solver.py:57-59]
__global__ void jacobi_precond_kernel(Geom g, const int* stop, const double* __restrict__ r,
                                      const double* __restrict__ d, double* __restrict__ z,
                                      double* partial) {
  griddep_wait();
  __shared__ double red[VT_THREADS / 32];
  if (stop && *(volatile const int*)stop) return;
  long long b, e;
  owned_range(g, b, e);
  double acc = 0.0;
  for (long long i = b + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < e;
       i += (long long)gridDim.x * blockDim.x) {
    const double rv = r[i];
    // pad entries carry d = 0 -> treat as 0/1
    const double dv = d[i];
    const double zv = dv != 0.0 ? __ddiv_rn(rv, dv) : 0.0;
    z[i] = zv;
    acc = fma(rv, zv, acc);
  }
  const double s = block_sum<VT_THREADS>(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// ---------------------------------------------------------------- scalar steps
// S1: pq -> alpha, iteration counter, curvature checks [ref: solver.py:121-132]
__global__ void pcg_s1_kernel(PcgCtl* c, const double* partial, int n) {
  griddep_wait();
  if (c->stop) return;
  const double pq = warp_sum_partials(partial, n);
  if (threadIdx.x != 0) return;
  c->k += 1;
  c->pq = pq;
  if (!isfinite(pq)) {
    c->err = 2; c->err_iter = c->k; c->err_val = pq; c->stop = 1;
  } else if (pq <= 0.0) {
    c->err = 3; c->err_iter = c->k; c->err_val = pq; c->stop = 1;
  }
  const int stop = c->stop;
  c->alpha = c->rz / pq;
  const int is50 = (c->k % 50) == 0;
  c->skip_rec = stop || is50;
  c->skip_true50 = stop || !is50;
  c->skip_cand = 1;
  c->skip_swap = 1;
  c->skip_xc = 1;
  c->x_done = is50;  // the mode-0 pass brings x up to date before the true residual
}

// S2: rel = ||r|| / ||f|| ; candidate convergence [ref: solver.py:137-140]
__global__ void pcg_s2_kernel(PcgCtl* c, const double* partial, int n_rec, int n_true) {
  griddep_wait();
  if (c->stop) return;
  const int is50 = (c->k % 50) == 0;
  const double rr = warp_sum_partials(partial, is50 ? n_true : n_rec);
  if (threadIdx.x != 0) return;
  const double rel = sqrt(rr) / c->fnorm;
  c->rel = rel;
  if (!isfinite(rel)) {
    c->err = 4; c->err_iter = c->k; c->err_val = rel; c->stop = 1;
    return;
  }
  c->skip_cand = !(rel <= c->tol);
  // a candidate's true residual needs the current x: update it now if deferred
  c->skip_xc = c->skip_cand || c->x_done;
  if (!c->skip_cand) c->x_done = 1;
}

// S3: true residual check on a convergence candidate [ref: solver.py:140-149]
__global__ void pcg_s3_kernel(PcgCtl* c, const double* partial, int n) {
  griddep_wait();
  if (c->skip_cand || c->stop) return;
  const double tr = warp_sum_partials(partial, n);
  if (threadIdx.x != 0) return;
  const double trel = sqrt(tr) / c->fnorm;
  c->drift = fabs(trel - c->rel) / fmax(trel, 1e-300);
  c->rel = trel;
  if (trel <= c->tol) {
    c->converged = 1;
    c->stop = 1;
    c->skip_rec = c->skip_true50 = c->skip_cand = c->skip_swap = 1;
  } else {
    c->skip_swap = 0;
  }
}

// S4: r.z -> beta [ref: solver.py:150-159]
__global__ void pcg_s4_kernel(PcgCtl* c, const double* partial, int n, int counts) {
  griddep_wait();
  if (c->stop) return;
  const double rz = warp_sum_partials(partial, n);
  if (threadIdx.x != 0) return;
  if (counts) c->precond_apps += 1;
  if (!isfinite(rz) || rz <= 0.0) {
    c->err = 1; c->err_iter = c->k; c->err_val = rz; c->stop = 1;
    return;
  }
  c->beta = rz / c->rz;
  c->rz = rz;
}

vt_status launch_pcg_update(vt_grid* G, PcgCtl* ctl, double* x, const double* p, double* r,
                            const double* q, double* partial, int with_r, cudaStream_t s,
                            const double* w, double* u0) {
  // modes 0 / 2 (x only) are no-ops in most iterations: a smaller grid costs
  // less per skipped launch and still streams at full rate when they run
  launch_pdl(pcg_update_kernel, with_r == 1 ? dot_grid(G) : G->nsm * 2, VT_THREADS, 0, s, G->g, ctl, x, p, r,
             q, partial, with_r, w, u0);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}
vt_status launch_pcg_xpby(vt_grid* G, PcgCtl* ctl, const double* z, double* p, cudaStream_t s,
                          double* x) {
  launch_pdl(pcg_xpby_kernel, G->nsm * 8, VT_THREADS, 0, s, G->g, ctl, z, p, x);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}
vt_status launch_copy(vt_grid* G, const int* skip, const double* src, double* dst,
                      cudaStream_t s, int grid) {
  if (grid <= 0) grid = fit_grid((long long)(G->g.pB - G->g.pA) * G->g.nplane, VT_THREADS, G->nsm * 8);
  launch_pdl(copy_kernel, grid, VT_THREADS, 0, s, G->g, skip, src, dst);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}
vt_status launch_jacobi_precond(vt_grid* G, const int* stop, const double* r, const double* d,
                                double* z, double* partial, cudaStream_t s) {
  launch_pdl(jacobi_precond_kernel, dot_grid(G), VT_THREADS, 0, s, G->g, stop, r, d, z, partial);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}
vt_status launch_pcg_s1(PcgCtl* c, const double* partial, int n, cudaStream_t s) {
  launch_pdl(pcg_s1_kernel, 1, 32, 0, s, c, partial, n);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}
vt_status launch_pcg_s2(PcgCtl* c, const double* partial, int n_rec, int n_true,
                        cudaStream_t s) {
  launch_pdl(pcg_s2_kernel, 1, 32, 0, s, c, partial, n_rec, n_true);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}
vt_status launch_pcg_s3(PcgCtl* c, const double* partial, int n, cudaStream_t s) {
  launch_pdl(pcg_s3_kernel, 1, 32, 0, s, c, partial, n);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}
vt_status launch_pcg_s4(PcgCtl* c, const double* partial, int n, int counts, cudaStream_t s) {
  launch_pdl(pcg_s4_kernel, 1, 32, 0, s, c, partial, n, counts);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

}  // namespace vt
