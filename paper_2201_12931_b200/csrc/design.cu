// Per-SIMP-iteration kernels [ref: optimize.py:139-302]:
//  compliance (dot), adjoint sensitivities (factorized u_e'K0u_e), the
//  self-weight load, the sensitivity filter (bit-identical to
//  scipy.ndimage.correlate with zero padding) and the OC update, whose
//  whole lambda bisection runs inside one cooperative kernel.
#include <cooperative_groups.h>
#include <float.h>
#include <math.h>

#include "vt_internal.h"

namespace cg = cooperative_groups;

namespace vt {

constexpr int DS_THREADS = 256;
#ifndef VT_OC_B
#define VT_OC_B 1
#endif
constexpr int OC_B = VT_OC_B;  // OC bisection: elements in flight per thread

__device__ __forceinline__ double corner_u(const Geom& g, const double* u, int i, int j, int k,
                                           int c, int comp) {
  const int p = k + ((c >> 2) & 1) - g.k0 + 1;
  return u[node_off(g, p, j + ((c >> 1) & 1), i + (c & 1)) * 3 + comp];
}

// dc_e = -(E p rho^(p-1) (1-kmin)) * u_e'K0u_e  (+ 2 u_e.g_unit)
// u_e'K0u_e = sum over the 21 coefficient pairs C.O of the factorized form.
// TWO: two-material SIMP (no reference counterpart): the
// element modulus is E s(rho) m(phi), m = eB + (1 - eB) phi^p, and the kernel
// also writes dc_phi = -E s(rho) p phi^(p-1) (1 - eB) u_e'K0u_e.
template <bool TWO>
__global__ void sens_kernel(Geom g, const double* __restrict__ u, const double* __restrict__ rho,
                            double p, double kmin, double E, int gax, double gcoef,
                            const double kc0, const double kc1, const double kc2, const double kc3,
                            const double kc4, const double kc5, double* __restrict__ dc,
                            const double* __restrict__ phi, double eB,
                            double* __restrict__ dcphi) {
  const long long nel = (long long)g.nx * g.ny * (g.k1 - g.k0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % g.nx);
    const long long r = e / g.nx;
    const int j = (int)(r % g.ny);
    const int k = (int)(r / g.ny) + g.k0;
    double C[3][8];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      double v[8];
#pragma unroll
      for (int c = 0; c < 8; ++c) v[c] = corner_u(g, u, i, j, k, c, a);
      // x pass
      double s1[8];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        s1[2 * q] = v[2 * q + 1] + v[2 * q];
        s1[2 * q + 1] = v[2 * q + 1] - v[2 * q];
      }
      // y pass (pairs differ in bit 1)
      double s2[8];
#pragma unroll
      for (int z = 0; z < 2; ++z)
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          const double lo = s1[z * 4 + x], hi = s1[z * 4 + 2 + x];
          s2[z * 4 + x] = hi + lo;
          s2[z * 4 + 2 + x] = hi - lo;
        }
      // z pass (bit 2)
#pragma unroll
      for (int xy = 0; xy < 4; ++xy) {
        C[a][xy] = s2[4 + xy] + s2[xy];
        C[a][4 + xy] = s2[4 + xy] - s2[xy];
      }
    }
    const double d0 = C[0][1] + C[1][2] + C[2][4];
    double O[3][8];
    O[0][1] = kc0 * d0 + kc1 * C[0][1];
    O[1][2] = kc0 * d0 + kc1 * C[1][2];
    O[2][4] = kc0 * d0 + kc1 * C[2][4];
    const double t01 = kc2 * (C[0][2] + C[1][1]);
    const double t02 = kc2 * (C[0][4] + C[2][1]);
    const double t12 = kc2 * (C[1][4] + C[2][2]);
    O[0][2] = t01; O[1][1] = t01; O[0][4] = t02; O[2][1] = t02; O[1][4] = t12; O[2][2] = t12;
    double w = kc3 * (C[0][3] + C[2][6]);
    O[0][3] = w + kc2 * C[0][3]; O[2][6] = w + kc2 * C[2][6];
    w = kc3 * (C[0][5] + C[1][6]);
    O[0][5] = w + kc2 * C[0][5]; O[1][6] = w + kc2 * C[1][6];
    w = kc3 * (C[1][3] + C[2][5]);
    O[1][3] = w + kc2 * C[1][3]; O[2][5] = w + kc2 * C[2][5];
    const double tt = C[0][6] + C[1][5] + C[2][3];
    O[0][6] = kc4 * (tt + C[0][6]); O[1][5] = kc4 * (tt + C[1][5]); O[2][3] = kc4 * (tt + C[2][3]);
#pragma unroll
    for (int a = 0; a < 3; ++a) O[a][7] = kc5 * C[a][7];
    double quad = 0.0;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int pt = 1; pt < 8; ++pt) quad = fma(C[a][pt], O[a][pt], quad);
    const double x = rho[e];
    // p * r**(p-1) * (1-kmin)   [ref: element.py:117]; r**2.0 is r*r in numpy
    const double pm1 = p - 1.0;
    double rp;
    if (pm1 == 2.0) rp = x * x;
    else if (pm1 == 1.0) rp = x;
    else if (pm1 == 0.0) rp = 1.0;
    else if (pm1 == 0.5) rp = sqrt(x);
    else rp = pow(x, pm1);
    double ds = __dmul_rn(E, __dmul_rn(__dmul_rn(p, rp), 1.0 - kmin));
    if (TWO) {
      const double y = phi[e];
      const double m = __dadd_rn(eB, __dmul_rn(1.0 - eB, simp_pow(y, p)));
      ds = __dmul_rn(ds, m);
      // E * s(rho) * (p * phi^(p-1) * (1 - eB))
      const double s = __dmul_rn(E, __dadd_rn(kmin, __dmul_rn(simp_pow(x, p), 1.0 - kmin)));
      const double dm = __dmul_rn(__dmul_rn(p, simp_pow(y, pm1)), 1.0 - eB);
      dcphi[e] = __dmul_rn(-__dmul_rn(s, dm), quad);
    }
    double out = __dmul_rn(-ds, quad);
    if (gax >= 0) out += 2.0 * (gcoef * C[gax][0]);
    dc[e] = out;
  }
}

// Two-material element scale (vt element layout) and the density the
// homogenized coarse levels average: rho_mg = rho m(phi)^(1/p), so that
// s(rho_mg) ~ s(rho) m(phi) up to kmin (preconditioner only; the fine operator
// uses the exact scale).
__global__ void two_scale_kernel(Geom g, const double* __restrict__ rho,
                                 const double* __restrict__ phi, double p, double kmin, double E,
                                 double eB, double* __restrict__ scale, double* __restrict__ rho_mg,
                                 int* bad) {
  const long long nel = (long long)g.nx * g.ny * (g.k1 - g.k0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % g.nx);
    const long long r = e / g.nx;
    const int j = (int)(r % g.ny);
    const int q = (int)(r / g.ny) + 1;
    const double x = rho[e], y = phi[e];
    if (!(x >= 0.0 && x <= 1.0 && y >= 0.0 && y <= 1.0)) *bad = 1;
    const double m = __dadd_rn(eB, __dmul_rn(1.0 - eB, simp_pow(y, p)));
    const double s = __dmul_rn(E, __dadd_rn(kmin, __dmul_rn(simp_pow(x, p), 1.0 - kmin)));
    scale[elem_off(g, q, j, i)] = __dmul_rn(s, m);
    if (rho_mg) rho_mg[e] = fmin(1.0, x * pow(m, 1.0 / p));
  }
}

// f = sum over incident elements (corner order) of rho_e g_unit, + f_ext, fixed -> 0
// [ref: optimize.py:216-231]
__global__ void gravity_kernel(Geom g, const uint8_t* mask, const double* __restrict__ rho,
                               int gax, double gcoef, const double* __restrict__ fext,
                               int zero_fixed, double* __restrict__ f) {
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (g.nx + 1));
    const long long r = t / (g.nx + 1);
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const int k = p - 1 + g.k0;
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int ei = i - (c & 1), ej = j - ((c >> 1) & 1), ek = k - ((c >> 2) & 1);
      if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < g.k0 || ek >= g.k1) continue;
      const long long e = ((long long)(ek - g.k0) * g.ny + ej) * g.nx + ei;
      acc = __dadd_rn(acc, __dmul_rn(rho[e], gcoef));
    }
    const long long node = node_off(g, p, j, i);
    const unsigned m = mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double v = (c == gax) ? acc : 0.0;
      if (fext) v = __dadd_rn(v, fext[node * 3 + c]);
      if (zero_fixed && ((m >> c) & 1u)) v = 0.0;
      f[node * 3 + c] = v;
    }
  }
}

// sensitivity filter: num = sum_{kernel order, |w|>eps} (rho*dc)[nb] * w  (zero outside),
// dcf = num / (max(gamma, rho) * wsum)   [ref: optimize.py:139-144, 174-179]
__global__ void filter_kernel(int nx, int ny, int nz, int R, const double* __restrict__ w,
                              const double* __restrict__ dc, const double* __restrict__ rho,
                              const double* __restrict__ wsum, double gamma, int mode,
                              double* __restrict__ out) {
  const long long nel = (long long)nx * ny * nz;
  const int D = 2 * R + 1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx);
    const long long r = e / nx;
    const int j = (int)(r % ny);
    const int k = (int)(r / ny);
    double acc = 0.0;
    for (int t = 0; t < D * D * D; ++t) {
      const double wt = w[t];
      if (!(fabs(wt) > DBL_EPSILON)) continue;
      const int dk = t / (D * D) - R, dj = (t / D) % D - R, di = t % D - R;
      const int kk = k + dk, jj = j + dj, ii = i + di;
      if (kk < 0 || kk >= nz || jj < 0 || jj >= ny || ii < 0 || ii >= nx) continue;
      const long long nb = ((long long)kk * ny + jj) * nx + ii;
      const double v = mode == 1 ? 1.0 : mode == 2 ? dc[nb] : __dmul_rn(rho[nb], dc[nb]);
      acc = __dadd_rn(acc, __dmul_rn(v, wt));
    }
    if (mode != 0) {
      out[e] = acc;
    } else {
      const double den = __dmul_rn(fmax(gamma, rho[e]), wsum[e]);
      out[e] = __ddiv_rn(acc, den);
    }
  }
}

// ------------------------------------------------------------------ OC
struct OcArgs {
  long long nel;
  const double* x;
  const int8_t* cls;
  const double* dc;
  const double* dv;
  double volfrac, move, eta, q;
  double* out;
  double* part;   // 2 * gridDim doubles (double-buffered partial sums)
  double* res;    // [0] lam, [1] steps, [2] status (0 ok, 1 infeasible, 2 bisection fail), [3] n_active
};

__device__ __forceinline__ double oc_cand(double x, double numer, double dva, double lam,
                                          double eta, double q, double lo, double hi) {
  const double b = __ddiv_rn(numer, __dmul_rn(lam, dva));
  const double pe = (eta == 0.5) ? sqrt(b) : pow(b, eta);
  double c = __dmul_rn(x, pe);
  if (q != 1.0) c = (q == 2.0) ? c * c : pow(c, q);
  return fmin(fmax(c, lo), hi);
}

// grid-wide deterministic sum: each block writes its partial, grid sync, every
// block re-sums the partials in index order.
__device__ double grid_sum(cg::grid_group& grid, double v, double* part, int parity,
                           double* red) {
  const double s = block_sum<DS_THREADS>(v, red);
  double* buf = part + parity * gridDim.x;
  if (threadIdx.x == 0) buf[blockIdx.x] = s;
  grid.sync();
  __shared__ double tot;
  if (threadIdx.x < 32) {
    const double t = warp_sum_partials(buf, gridDim.x);
    if (threadIdx.x == 0) tot = t;
  }
  __syncthreads();
  return tot;
}

__global__ void oc_kernel(OcArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double red[DS_THREADS / 32];
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int parity = 0;
  // active count, lo / hi means
  double cnt = 0.0, slo = 0.0, shi = 0.0;
  for (long long e = t0; e < a.nel; e += stride) {
    if (a.cls[e] != 0) continue;
    const double x = a.x[e];
    cnt += 1.0;
    slo += fmax(0.0, x - a.move);
    shi += fmin(1.0, x + a.move);
  }
  const double n = grid_sum(grid, cnt, a.part, parity, red); parity ^= 1;
  const double mlo = grid_sum(grid, slo, a.part, parity, red) / n; parity ^= 1;
  const double mhi = grid_sum(grid, shi, a.part, parity, red) / n; parity ^= 1;
  if (mlo > a.volfrac + 1e-6 || mhi < a.volfrac - 1e-6) {
    if (t0 == 0) { a.res[2] = 1.0; a.res[4] = mlo; a.res[5] = mhi; }
    return;
  }
  auto mean_at = [&](double lam) {
    double s = 0.0;
    // OC_B elements in flight per thread (same per-thread order as a plain
    // grid-stride loop: the partial sums are unchanged)
    for (long long e0 = t0; e0 < a.nel; e0 += OC_B * stride) {
      double xv[OC_B], dcv[OC_B], dvv[OC_B];
      bool act[OC_B];
#pragma unroll
      for (int k = 0; k < OC_B; ++k) {
        const long long e = e0 + k * stride;
        act[k] = e < a.nel && a.cls[e] == 0;
        if (act[k]) {
          xv[k] = a.x[e];
          dcv[k] = a.dc[e];
          dvv[k] = a.dv[e];
        }
      }
#pragma unroll
      for (int k = 0; k < OC_B; ++k)
        if (act[k])
          s += oc_cand(xv[k], fmax(-dcv[k], 0.0), dvv[k], lam, a.eta, a.q, fmax(0.0, xv[k] - a.move),
                       fmin(1.0, xv[k] + a.move));
    }
    const double tot = grid_sum(grid, s, a.part, parity, red);
    parity ^= 1;
    return tot / n;
  };
  double l1 = 0.0, l2 = 1e9;
  for (int it = 0; it < 200; ++it) {  // [ref: optimize.py:279-282]
    if (mean_at(l2) <= a.volfrac) break;
    l2 *= 16.0;
  }
  double lam = 0.5 * (l1 + l2);
  int steps = 0;
  double m = mean_at(lam);
  int status = 0;
  while (fabs(m - a.volfrac) > 1e-6) {  // [ref: optimize.py:283-298]
    ++steps;
    if (steps > 200) { status = 2; break; }
    if (m > a.volfrac) l1 = lam; else l2 = lam;
    lam = 0.5 * (l1 + l2);
    m = mean_at(lam);
  }
  if (status == 0) {
    for (long long e = t0; e < a.nel; e += stride) {
      const double x = a.x[e];
      if (a.cls[e] != 0) { a.out[e] = x; continue; }
      a.out[e] = oc_cand(x, fmax(-a.dc[e], 0.0), a.dv[e], lam, a.eta, a.q, fmax(0.0, x - a.move),
                         fmin(1.0, x + a.move));
    }
  }
  if (t0 == 0) { a.res[0] = lam; a.res[1] = steps; a.res[2] = status; a.res[3] = n; }
}

// max |a - b| over all elements and mean of a over active elements
__global__ void change_kernel(long long nel, const double* a, const double* b, const int8_t* cls,
                              double* part) {
  __shared__ double red[DS_THREADS / 32];
  double mx = 0.0, s = 0.0, c = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    mx = fmax(mx, fabs(a[e] - b[e]));
    if (cls[e] == 0) { s += a[e]; c += 1.0; }
  }
  const double m = block_max<DS_THREADS>(mx, red);
  const double ss = block_sum<DS_THREADS>(s, red);
  const double cc = block_sum<DS_THREADS>(c, red);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 3 + 0] = m;
    part[blockIdx.x * 3 + 1] = ss;
    part[blockIdx.x * 3 + 2] = cc;
  }
}

}  // namespace vt

struct vt_filter {
  vt_grid* G = nullptr;
  int R = 0;
  double* w = nullptr;
  double* wsum = nullptr;
};

using namespace vt;

namespace vt {
// whole OC bisection in one cooperative launch [ref: optimize.py:245-302];
// part: 2 x (resident blocks, <= 2048) doubles, res: 6 doubles
static vt_status oc_run(long long nel, int nsm, double* part, double* res_dev, const double* rho,
                        const int8_t* classes, const double* dc, const double* dv, double volfrac,
                        double move, double eta, double q, double* rho_out, double* lam, int* steps,
                        cudaStream_t s) {
  static int per_sm = 0;
  if (!per_sm) VT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, oc_kernel, DS_THREADS, 0));
  // every resident block (one grid barrier per bisection step, so latency
  // hiding matters more than the partial count)
  int grid = per_sm * nsm;
  if (grid > 2048) grid = 2048;
  OcArgs a;
  a.nel = nel;
  a.x = rho;
  a.cls = classes;
  a.dc = dc;
  a.dv = dv;
  a.volfrac = volfrac;
  a.move = move;
  a.eta = eta;
  a.q = q;
  a.out = rho_out;
  a.part = part;
  a.res = res_dev;
  void* args[] = {&a};
  VT_CUDA(cudaLaunchCooperativeKernel((void*)oc_kernel, grid, DS_THREADS, args, 0, s));
  count_launch();
  double res[6];
  VT_CUDA(cudaMemcpyAsync(res, a.res, sizeof(res), cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  if (res[2] == 1.0) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "volume target unreachable within the move limits (reachable [%.6f, %.6f], target %g)",
             res[4], res[5], volfrac);
    return fail(VT_EVOLUME, buf);
  }
  if (res[2] == 2.0)
    return fail(VT_EVOLUME, "bisection failed to reach the volume target after 200 halvings");
  if (lam) *lam = res[0];
  if (steps) *steps = (int)res[1];
  return VT_OK;
}
}  // namespace vt

extern "C" {

vt_status vt_sensitivities(vt_grid* G, const double* u, const double* rho, double p, double kmin,
                           double E, int grav_axis, double grav_coef, double* dc, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const double* k = G->coef.kc;
  sens_kernel<false><<<G->nsm * 8, DS_THREADS, 0, s>>>(G->g, u, rho, p, kmin, E, grav_axis, grav_coef,
                                                       k[0], k[1], k[2], k[3], k[4], k[5], dc,
                                                       nullptr, 1.0, nullptr);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status vt_sensitivities_two_material(vt_grid* G, const double* u, const double* rho,
                                        const double* phi, double p, double kmin, double E,
                                        double eB, int grav_axis, double grav_coef, double* dc_rho,
                                        double* dc_phi, void* stream) {
  if (!(eB >= 0.0 && eB <= 1.0)) return fail(VT_EINVAL, "modulus ratio must lie in [0, 1]");
  cudaStream_t s = (cudaStream_t)stream;
  const double* k = G->coef.kc;
  sens_kernel<true><<<G->nsm * 8, DS_THREADS, 0, s>>>(G->g, u, rho, p, kmin, E, grav_axis, grav_coef,
                                                      k[0], k[1], k[2], k[3], k[4], k[5], dc_rho,
                                                      phi, eB, dc_phi);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status vt_scale_two_material(vt_grid* G, const double* rho, const double* phi, double p,
                                double kmin, double E, double eB, double* scale, double* rho_mg,
                                void* stream) {
  if (!(eB >= 0.0 && eB <= 1.0)) return fail(VT_EINVAL, "modulus ratio must lie in [0, 1]");
  cudaStream_t s = (cudaStream_t)stream;
  int* bad = reinterpret_cast<int*>(G->scalars + 1);
  VT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  two_scale_kernel<<<G->nsm * 8, DS_THREADS, 0, s>>>(G->g, rho, phi, p, kmin, E, eB, scale, rho_mg,
                                                     bad);
  count_launch();
  VT_CUDA(cudaGetLastError());
  int hb = 0;
  VT_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  if (hb) return fail(VT_EDENSITY, "density or phase fraction outside [0, 1]");
  return VT_OK;
}

vt_status vt_gravity_load(vt_grid* G, const double* rho, int grav_axis, double grav_coef,
                          const double* f_ext, int zero_fixed, double* f, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  gravity_kernel<<<G->nsm * 8, DS_THREADS, 0, s>>>(G->g, G->mask, rho, grav_axis, grav_coef, f_ext,
                                                   zero_fixed, f);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status vt_filter_create(vt_filter** out, vt_grid* G, int R, const double* kernel_host) {
  if (R < 0) return fail(VT_EINVAL, "filter half-width must be non-negative");
  if (G->g.k0 != 0 || G->g.k1 != G->g.nz)
    return fail(VT_EINVAL, "filter on a slab needs the distributed runtime");
  vt_filter* F = new vt_filter();
  F->G = G;
  F->R = R;
  const int D = 2 * R + 1;
  VT_CUDA(cudaMalloc(&F->w, (size_t)D * D * D * sizeof(double)));
  VT_CUDA(cudaMemcpy(F->w, kernel_host, (size_t)D * D * D * sizeof(double), cudaMemcpyHostToDevice));
  VT_CUDA(cudaMalloc(&F->wsum, (size_t)G->nel_local() * sizeof(double)));
  filter_kernel<<<G->nsm * 8, DS_THREADS>>>(G->g.nx, G->g.ny, G->g.nz, R, F->w, nullptr, nullptr,
                                            nullptr, 0.0, 1, F->wsum);
  count_launch();
  VT_CUDA(cudaGetLastError());
  VT_CUDA(cudaDeviceSynchronize());
  *out = F;
  return VT_OK;
}

vt_status vt_filter_destroy(vt_filter* F) {
  if (!F) return VT_OK;
  cudaFree(F->w);
  cudaFree(F->wsum);
  delete F;
  return VT_OK;
}

const double* vt_filter_wsum(vt_filter* F) { return F->wsum; }

vt_status vt_filter_apply(vt_filter* F, const double* dc, const double* rho, double gamma,
                          double* dcf, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  vt_grid* G = F->G;
  filter_kernel<<<G->nsm * 8, DS_THREADS, 0, s>>>(G->g.nx, G->g.ny, G->g.nz, F->R, F->w, dc, rho,
                                                  F->wsum, gamma, 0, dcf);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status vt_filter_correlate(vt_filter* F, const double* field, double* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  vt_grid* G = F->G;
  filter_kernel<<<G->nsm * 8, DS_THREADS, 0, s>>>(G->g.nx, G->g.ny, G->g.nz, F->R, F->w, field,
                                                  nullptr, nullptr, 0.0, 2, out);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status vt_oc_update(vt_grid* G, const double* rho, const int8_t* classes, const double* dc,
                       const double* dv, double volfrac, double move, double eta, double q,
                       double* rho_out, double* lam, int* steps, void* stream) {
  return vt::oc_run(G->nel_local(), G->nsm, G->partial, G->scalars + 8, rho, classes, dc, dv, volfrac,
                    move, eta, q, rho_out, lam, steps, (cudaStream_t)stream);
}

vt_status vt_oc_update_flat(long long nel, const double* rho, const int8_t* classes, const double* dc,
                            const double* dv, double volfrac, double move, double eta, double q,
                            double* rho_out, double* lam, int* steps, void* stream) {
  if (nel <= 0) return fail(VT_EINVAL, "element count must be positive");
  // per-device scratch: 2 x 2048 block partials + the result words
  static double* scratch[64] = {};
  int dev = 0, nsm = 0;
  VT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(VT_EINVAL, "device ordinal out of range");
  VT_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  if (!scratch[dev]) VT_CUDA(cudaMalloc(&scratch[dev], (2 * 2048 + 16) * sizeof(double)));
  return vt::oc_run(nel, nsm, scratch[dev], scratch[dev] + 2 * 2048, rho, classes, dc, dv, volfrac,
                    move, eta, q, rho_out, lam, steps, (cudaStream_t)stream);
}

vt_status vt_change_volume(vt_grid* G, const double* a, const double* b, const int8_t* classes,
                           double* max_abs_diff, double* active_mean, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int grid = G->nsm * 2;
  change_kernel<<<grid, DS_THREADS, 0, s>>>(G->nel_local(), a, b, classes, G->partial);
  count_launch();
  VT_CUDA(cudaGetLastError());
  std::vector<double> h(3 * grid);
  VT_CUDA(cudaMemcpyAsync(h.data(), G->partial, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  double mx = 0.0, sm = 0.0, cn = 0.0;
  for (int i = 0; i < grid; ++i) {
    mx = fmax(mx, h[3 * i]);
    sm += h[3 * i + 1];
    cn += h[3 * i + 2];
  }
  if (max_abs_diff) *max_abs_diff = mx;
  if (active_mean) *active_mean = cn > 0 ? sm / cn : 0.0;
  return VT_OK;
}

}  // extern "C"
