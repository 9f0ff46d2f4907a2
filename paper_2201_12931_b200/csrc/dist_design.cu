// Per-SIMP-iteration design kernels on the z-slab decomposition
// [ref: optimize.py:139-302; "filter halo R planes of rho*dc;
// allreduce c, ch (max), and the sum for each OC lambda step"].
//
//  * sensitivities: one node-plane halo of u, then the single-GPU kernel on
//    each slab (global plane index arithmetic);
//  * filter: rho*dc is formed into a slab buffer with R ghost element layers
//    on both sides, the ghost layers come from the neighbours, and the
//    correlation runs in global coordinates with the global zero padding --
//    same neighbour order and arithmetic as scipy.ndimage.correlate /
//    filter_kernel, so the result is bit-identical to the single-GPU filter;
//  * OC: the lambda bisection of optimize.py:245-302 driven from the host;
//    every global sum is a per-slab fixed-order sum, all-gathered and added in
//    rank order, so every rank takes the same bisection decisions;
//  * change / volume: per-rank max and sums, gathered.
#include <float.h>
#include <math.h>
#include <stdio.h>

#include "dist_internal.h"

namespace vt {

constexpr int DD_THREADS = 256;

// prod[(k - k0 + R) layer] = rho * dc for the slab's own layers
__global__ void dfilter_prod_kernel(long long nel, long long layer, int R,
                                    const double* __restrict__ rho, const double* __restrict__ dc,
                                    double* __restrict__ prod) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x)
    prod[e + R * layer] = __dmul_rn(rho[e], dc[e]);
}

// mode 1: wsum = correlate(1); mode 0: dcf = correlate(prod) / (max(gamma, rho) wsum)
__global__ void dfilter_kernel(int nx, int ny, int nzg, int k0, int nloc, int R,
                               const double* __restrict__ w, const double* __restrict__ prod,
                               const double* __restrict__ rho, const double* __restrict__ wsum,
                               double gamma, int mode, double* __restrict__ out) {
  const long long nel = (long long)nx * ny * nloc;
  const int D = 2 * R + 1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % nx);
    const long long r = e / nx;
    const int j = (int)(r % ny);
    const int kl = (int)(r / ny);
    const int k = kl + k0;
    double acc = 0.0;
    for (int t = 0; t < D * D * D; ++t) {
      const double wt = w[t];
      if (!(fabs(wt) > DBL_EPSILON)) continue;
      const int dk = t / (D * D) - R, dj = (t / D) % D - R, di = t % D - R;
      const int kk = k + dk, jj = j + dj, ii = i + di;
      if (kk < 0 || kk >= nzg || jj < 0 || jj >= ny || ii < 0 || ii >= nx) continue;
      const double v =
          mode == 1 ? 1.0 : prod[((long long)(kk - k0 + R) * ny + jj) * nx + ii];
      acc = __dadd_rn(acc, __dmul_rn(v, wt));
    }
    if (mode == 1) {
      out[e] = acc;
    } else {
      const double den = __dmul_rn(fmax(gamma, rho[e]), wsum[e]);
      out[e] = __ddiv_rn(acc, den);
    }
  }
}

__device__ __forceinline__ double doc_cand(double x, double numer, double dva, double lam,
                                           double eta, double q, double lo, double hi) {
  const double b = __ddiv_rn(numer, __dmul_rn(lam, dva));
  const double pe = (eta == 0.5) ? sqrt(b) : pow(b, eta);
  double c = __dmul_rn(x, pe);
  if (q != 1.0) c = (q == 2.0) ? c * c : pow(c, q);
  return fmin(fmax(c, lo), hi);
}

// per-CTA partial sums of the OC quantities over one slab:
//   mode 0: [count, sum lo, sum hi] of active elements
//   mode 1: sum of the candidates at lam
//   mode 2: write the candidates at lam (passives copied)
//   mode 3: [max |a - b|, sum a (active), count active] (change / volume)
__global__ void doc_kernel(int mode, long long nel, const double* __restrict__ x,
                           const int8_t* __restrict__ cls, const double* __restrict__ dc,
                           const double* __restrict__ dv, double lam, double move, double eta,
                           double q, double* __restrict__ out, double* part) {
  __shared__ double red[DD_THREADS / 32];
  double s0 = 0.0, s1 = 0.0, s2 = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    const double xe = x[e];
    if (mode == 3) {
      s0 = fmax(s0, fabs(xe - dc[e]));
      if (cls[e] == 0) { s1 += xe; s2 += 1.0; }
      continue;
    }
    if (cls[e] != 0) {
      if (mode == 2) out[e] = xe;
      continue;
    }
    const double lo = fmax(0.0, xe - move), hi = fmin(1.0, xe + move);
    if (mode == 0) {
      s0 += 1.0; s1 += lo; s2 += hi;
    } else {
      const double c = doc_cand(xe, fmax(-dc[e], 0.0), dv[e], lam, eta, q, lo, hi);
      if (mode == 1) s0 += c; else out[e] = c;
    }
  }
  if (mode == 2) return;
  const int nq = (mode == 1) ? 1 : 3;
  double v[3] = {s0, s1, s2};
  for (int c = 0; c < nq; ++c) {
    const double t = (mode == 3 && c == 0) ? block_max<DD_THREADS>(v[c], red)
                                           : block_sum<DD_THREADS>(v[c], red);
    if (threadIdx.x == 0) part[c * 4096 + blockIdx.x] = t;
  }
}

__global__ void part_max_kernel(const double* part, int n, double* out) {
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += 32) m = fmax(m, part[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (threadIdx.x == 0) *out = m;
}

static int doc_grid(vt_grid* G) { return G->nsm * 2; }

// self-weight load on a slab: f = sum over incident elements (corner order) of
// rho_e g_unit (+ f_ext), fixed -> 0 [ref: optimize.py:216-231]; rho_pad holds
// element layers k0-1 .. k1-1 (the first one from the rank below)
__global__ void dgrav_kernel(Geom g, const uint8_t* __restrict__ mask, const double* __restrict__ rho_pad,
                             int gax, double gcoef, const double* __restrict__ fext, int zero_fixed,
                             double* __restrict__ f) {
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
      if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek < g.k0 - 1 || ek >= g.k1) continue;
      const long long e = ((long long)(ek - g.k0 + 1) * g.ny + ej) * g.nx + ei;
      acc = __dadd_rn(acc, __dmul_rn(rho_pad[e], gcoef));
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

// R ghost element layers of prod on both sides (plain layout, layer = nx*ny)
static vt_status halo_prod(vt_dist* D, cudaStream_t s) {
  if (D->N == 1 || D->fR == 0) return VT_OK;
  const int R = D->fR;
  const long long layer = (long long)D->nx * D->ny;
  const size_t blk = (size_t)R * layer;
  auto nl = [&](int i) { const Geom& g = D->sl[i].lv[0]->g; return g.k1 - g.k0; };
  if (!D->remote()) {
    for (int i = 0; i < D->N; ++i) {
      double* p = D->fprod[i];
      if (i > 0)  // below: the neighbour's top R own layers
        VT_CUDA(cudaMemcpyAsync(p, D->fprod[i - 1] + (size_t)nl(i - 1) * layer, blk * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
      if (i < D->N - 1)  // above: the neighbour's bottom R own layers
        VT_CUDA(cudaMemcpyAsync(p + (size_t)(R + nl(i)) * layer, D->fprod[i + 1] + blk,
                                blk * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    return VT_OK;
  }
  const int r = D->sl[0].rank, n = nl(0);
  double* p = D->fprod[0];
  if (D->px)
    return peer_halo(D, p + blk, p + (size_t)n * layer, p, p + (size_t)(R + n) * layer, (long long)blk, s);
  auto& A = nccl();
  VT_NCCL(A.GroupStart());
  if (r > 0) {
    VT_NCCL(A.Send(p + blk, blk, ncclDouble, r - 1, D->comm, s));
    VT_NCCL(A.Recv(p, blk, ncclDouble, r - 1, D->comm, s));
  }
  if (r < D->N - 1) {
    VT_NCCL(A.Send(p + (size_t)n * layer, blk, ncclDouble, r + 1, D->comm, s));
    VT_NCCL(A.Recv(p + (size_t)(R + n) * layer, blk, ncclDouble, r + 1, D->comm, s));
  }
  VT_NCCL(A.GroupEnd());
  return VT_OK;
}

// OC sums: per slab partials -> slot per rank -> rank-ordered host sums
static vt_status oc_sums(vt_dist* D, int mode, const double* const* x, const int8_t* const* cls,
                         const double* const* dc, const double* const* dv, double lam,
                         double move, double eta, double q, cudaStream_t s, double* out3) {
  const int nq = (mode == 1) ? 1 : 3;
  const int slot0 = 8;
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    const int grid = doc_grid(G);
    double* part = D->opart + (size_t)i * 4 * 4096;
    doc_kernel<<<grid, DD_THREADS, 0, s>>>(mode, G->nel_local(), x[i], cls[i], dc ? dc[i] : nullptr,
                                           dv ? dv[i] : nullptr, lam, move, eta, q, nullptr, part);
    count_launch();
    for (int c = 0; c < nq; ++c) {
      if (mode == 3 && c == 0) {
        part_max_kernel<<<1, 32, 0, s>>>(part, grid, D->scal + (size_t)(slot0 + c) * D->N + D->sl[i].rank);
        count_launch();
      } else {
        VT_TRY(slab_sum(D, i, part + c * 4096, grid, 0, slot0 + c, nullptr, s));
      }
    }
  }
  VT_CUDA(cudaGetLastError());
  std::vector<double> h(D->N);
  for (int c = 0; c < nq; ++c) {
    VT_TRY(host_slot_values(D, slot0 + c, s, h.data()));
    double acc = 0.0;
    for (int g = 0; g < D->N; ++g) acc = (mode == 3 && c == 0) ? fmax(acc, h[g]) : acc + h[g];
    out3[c] = acc;
  }
  return VT_OK;
}

}  // namespace vt

using namespace vt;

extern "C" {

// dc_e on every local slab [ref: optimize.py:195-213]; u's ghost planes are refreshed
vt_status vt_dist_sensitivities(vt_dist* D, double* const* u, const double* const* rho, double p,
                                double kmin, double E, int grav_axis, double grav_coef,
                                double* const* dc, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double*> uu(u, u + D->nlocal);
  VT_TRY(halo_nodes(D, 0, uu, s));
  for (int i = 0; i < D->nlocal; ++i)
    VT_TRY(vt_sensitivities(D->sl[i].lv[0], u[i], rho[i], p, kmin, E, grav_axis, grav_coef, dc[i],
                            stream));
  return VT_OK;
}

// (dc_rho, dc_phi) of the two-material law on every local slab (u's ghost
// planes refreshed first) [extends optimize.py:195-213; DESIGN.md 3.5]
vt_status vt_dist_sensitivities_two_material(vt_dist* D, double* const* u, const double* const* rho,
                                             const double* const* phi, double p, double kmin, double E,
                                             double e_ratio, int grav_axis, double grav_coef,
                                             double* const* dc_rho, double* const* dc_phi, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double*> uu(u, u + D->nlocal);
  VT_TRY(halo_nodes(D, 0, uu, s));
  for (int i = 0; i < D->nlocal; ++i)
    VT_TRY(vt_sensitivities_two_material(D->sl[i].lv[0], u[i], rho[i], phi[i], p, kmin, E, e_ratio,
                                         grav_axis, grav_coef, dc_rho[i], dc_phi[i], stream));
  return VT_OK;
}

// f = gravity load of rho (+ f_ext), zero on fixed dofs when zero_fixed
vt_status vt_dist_gravity_load(vt_dist* D, const double* const* rho, int grav_axis, double grav_coef,
                               const double* const* f_ext, int zero_fixed, double* const* f,
                               void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const long long layer = (long long)D->nx * D->ny;
  if (D->gpad.empty()) {
    D->gpad.assign(D->nlocal, nullptr);
    for (int i = 0; i < D->nlocal; ++i) {
      vt_grid* G = D->sl[i].lv[0];
      const size_t n = (size_t)(G->g.k1 - G->g.k0 + 1) * layer;
      VT_CUDA(cudaMalloc(&D->gpad[i], n * sizeof(double)));
      VT_CUDA(cudaMemset(D->gpad[i], 0, n * sizeof(double)));
    }
  }
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    VT_CUDA(cudaMemcpyAsync(D->gpad[i] + layer, rho[i], G->nel_local() * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
  }
  if (D->N > 1) {  // layer k0-1 from the rank below
    auto nl = [&](int i) { const Geom& g = D->sl[i].lv[0]->g; return g.k1 - g.k0; };
    if (!D->remote()) {
      for (int i = 1; i < D->N; ++i)
        VT_CUDA(cudaMemcpyAsync(D->gpad[i], D->gpad[i - 1] + (size_t)nl(i - 1) * layer,
                                layer * sizeof(double), cudaMemcpyDeviceToDevice, s));
    } else if (D->px) {  // rank+1 pulls my top layer, I pull rank-1's
      const int r = D->sl[0].rank;
      PeerOps o;
      if (r < D->N - 1) {
        o.pack(D->gpad[0] + (size_t)nl(0) * layer, (long long)D->px->half, layer);
        o.wait(r + 1);
      }
      if (r > 0) {
        o.pull(r - 1, (long long)D->px->half, D->gpad[0], layer);
        o.wait(r - 1);
      }
      VT_TRY(peer_exchange(D, o, s));
    } else {
      const int r = D->sl[0].rank;
      auto& A = nccl();
      VT_NCCL(A.GroupStart());
      if (r < D->N - 1)
        VT_NCCL(A.Send(D->gpad[0] + (size_t)nl(0) * layer, layer, ncclDouble, r + 1, D->comm, s));
      if (r > 0) VT_NCCL(A.Recv(D->gpad[0], layer, ncclDouble, r - 1, D->comm, s));
      VT_NCCL(A.GroupEnd());
    }
  }
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    dgrav_kernel<<<G->nsm * 8, DD_THREADS, 0, s>>>(G->g, G->mask, D->gpad[i], grav_axis, grav_coef,
                                                   f_ext ? f_ext[i] : nullptr, zero_fixed, f[i]);
    count_launch();
  }
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// sensitivity filter of half-width R (kernel in (dk, dj, di) order) [ref: optimize.py:110-171]
vt_status vt_dist_filter_create(vt_dist* D, int R, const double* kernel_host) {
  if (R < 0) return fail(VT_EINVAL, "filter half-width must be non-negative");
  if (D->px && R > PEER_MAX_R)
    return fail(VT_EINVAL, "filter half-width exceeds the peer transport's staging area (8 layers)");
  for (int i = 0; i < D->nlocal; ++i) {
    const Geom& g = D->sl[i].lv[0]->g;
    if (D->N > 1 && g.k1 - g.k0 < R)
      return fail(VT_EINVAL, "every slab needs at least R element layers for the filter halo");
  }
  const int K = 2 * R + 1;
  cudaFree(D->fw);
  for (double* p : D->fwsum) cudaFree(p);
  for (double* p : D->fprod) cudaFree(p);
  D->fwsum.assign(D->nlocal, nullptr);
  D->fprod.assign(D->nlocal, nullptr);
  VT_CUDA(cudaMalloc(&D->fw, (size_t)K * K * K * sizeof(double)));
  VT_CUDA(cudaMemcpy(D->fw, kernel_host, (size_t)K * K * K * sizeof(double), cudaMemcpyHostToDevice));
  if (!D->opart) VT_CUDA(cudaMalloc(&D->opart, (size_t)D->nlocal * 4 * 4096 * sizeof(double)));
  D->fR = R;
  const long long layer = (long long)D->nx * D->ny;
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    const int nl = G->g.k1 - G->g.k0;
    VT_CUDA(cudaMalloc(&D->fwsum[i], (size_t)G->nel_local() * sizeof(double)));
    VT_CUDA(cudaMalloc(&D->fprod[i], (size_t)(nl + 2 * R) * layer * sizeof(double)));
    VT_CUDA(cudaMemset(D->fprod[i], 0, (size_t)(nl + 2 * R) * layer * sizeof(double)));
    dfilter_kernel<<<G->nsm * 8, DD_THREADS>>>(D->nx, D->ny, D->nz, G->g.k0, nl, R, D->fw, nullptr,
                                               nullptr, nullptr, 0.0, 1, D->fwsum[i]);
    count_launch();
  }
  VT_CUDA(cudaGetLastError());
  VT_CUDA(cudaDeviceSynchronize());
  return VT_OK;
}

// dcf = correlate(rho*dc) / (max(gamma, rho) * wsum) [ref: optimize.py:174-179]
vt_status vt_dist_filter_apply(vt_dist* D, const double* const* dc, const double* const* rho,
                               double gamma, double* const* dcf, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (D->fR < 0) return fail(VT_ESETUP, "filter was not created");
  const long long layer = (long long)D->nx * D->ny;
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    dfilter_prod_kernel<<<G->nsm * 8, DD_THREADS, 0, s>>>(G->nel_local(), layer, D->fR, rho[i], dc[i],
                                                          D->fprod[i]);
    count_launch();
  }
  VT_TRY(halo_prod(D, s));
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    dfilter_kernel<<<G->nsm * 8, DD_THREADS, 0, s>>>(D->nx, D->ny, D->nz, G->g.k0, G->g.k1 - G->g.k0,
                                                     D->fR, D->fw, D->fprod[i], rho[i], D->fwsum[i],
                                                     gamma, 0, dcf[i]);
    count_launch();
  }
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// OC update with bisected multiplier over all ranks [ref: optimize.py:245-302];
// same bracketing / termination as vt_oc_update.  Blocking.
vt_status vt_dist_oc_update(vt_dist* D, const double* const* rho, const int8_t* const* classes,
                            const double* const* dc, const double* const* dv, double volfrac,
                            double move, double eta, double q, double* const* rho_out, double* lam,
                            int* steps, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!D->opart) VT_CUDA(cudaMalloc(&D->opart, (size_t)D->nlocal * 4 * 4096 * sizeof(double)));
  double m3[3];
  VT_TRY(oc_sums(D, 0, rho, classes, dc, dv, 0.0, move, eta, q, s, m3));
  const double n = m3[0], mlo = m3[1] / n, mhi = m3[2] / n;
  if (mlo > volfrac + 1e-6 || mhi < volfrac - 1e-6) {
    char buf[256];
    snprintf(buf, sizeof(buf),
             "volume target unreachable within the move limits (reachable [%.6f, %.6f], target %g)",
             mlo, mhi, volfrac);
    return fail(VT_EVOLUME, buf);
  }
  auto mean_at = [&](double l, double* m) -> vt_status {
    double t[3];
    VT_TRY(oc_sums(D, 1, rho, classes, dc, dv, l, move, eta, q, s, t));
    *m = t[0] / n;
    return VT_OK;
  };
  double l1 = 0.0, l2 = 1e9, m = 0.0;
  for (int it = 0; it < 200; ++it) {  // [ref: optimize.py:279-282]
    VT_TRY(mean_at(l2, &m));
    if (m <= volfrac) break;
    l2 *= 16.0;
  }
  double lm = 0.5 * (l1 + l2);
  int nst = 0;
  VT_TRY(mean_at(lm, &m));
  while (fabs(m - volfrac) > 1e-6) {  // [ref: optimize.py:283-298]
    ++nst;
    if (nst > 200) return fail(VT_EVOLUME, "bisection failed to reach the volume target after 200 halvings");
    if (m > volfrac) l1 = lm; else l2 = lm;
    lm = 0.5 * (l1 + l2);
    VT_TRY(mean_at(lm, &m));
  }
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    doc_kernel<<<doc_grid(G), DD_THREADS, 0, s>>>(2, G->nel_local(), rho[i], classes[i], dc[i], dv[i],
                                                  lm, move, eta, q, rho_out[i], nullptr);
    count_launch();
  }
  VT_CUDA(cudaGetLastError());
  VT_CUDA(cudaStreamSynchronize(s));
  if (lam) *lam = lm;
  if (steps) *steps = nst;
  return VT_OK;
}

// max |a - b| over all elements and the mean of a over active elements (all ranks)
vt_status vt_dist_change_volume(vt_dist* D, const double* const* a, const double* const* b,
                                const int8_t* const* classes, double* max_abs_diff,
                                double* active_mean, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!D->opart) VT_CUDA(cudaMalloc(&D->opart, (size_t)D->nlocal * 4 * 4096 * sizeof(double)));
  double t[3];
  VT_TRY(oc_sums(D, 3, a, classes, b, nullptr, 0.0, 0.0, 0.0, 0.0, s, t));
  if (max_abs_diff) *max_abs_diff = t[0];
  if (active_mean) *active_mean = t[2] > 0 ? t[1] / t[2] : 0.0;
  return VT_OK;
}

}  // extern "C"
