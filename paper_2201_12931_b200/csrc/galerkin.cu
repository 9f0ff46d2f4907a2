// Galerkin coarse operators on B200 -- the reference's default multigrid
// scheme [ref: multigrid.py:59-81, 201-278, 280-316; operator.py:58-105].
//
//  * Level 1 stores, per coarse element E, K_E = sum_c s_c G_c (+ the fine
//    fixed-dof corrections s_c W_c^T (K0 o mm^T - K0) W_c of children that
//    touch a fixed dof), G_c = W_c^T K0 W_c precomputed once: one thread per
//    (E, entry), 8 FMAs.
//  * Level l+1 from level l: K_E = sum_c W_c^T (K_child o mm^T) W_c.  W_c is
//    the octant's trilinear weight table T_c applied per displacement
//    component, so each triple product is 9 component blocks of T^T A T
//    (8x8): one CTA per coarse element, the child's projected matrix staged in
//    shared memory.
//  * The stored-matrix operator: a warp per element forms K_e u_e (24 lanes,
//    one row each, coalesced 4.6 KB matrix read), then one thread per node
//    adds its 8 corner contributions in the reference's corner order c = 0..7
//    and applies the mode's epilogue (apply / residual / damped Jacobi).
//  * Diagonal: the stored diagonals summed per node in corner order.
#include <algorithm>
#include <map>
#include <vector>

#include "vt_internal.h"

namespace vt {

constexpr int GL_THREADS = 256;

__constant__ double c_T[8][8][8];  // T_c[a][b]: weight of coarse corner b at fine corner a of octant c

static void octant_T(double T[8][8][8]) {
  for (int c = 0; c < 8; ++c)
    for (int a = 0; a < 8; ++a)
      for (int b = 0; b < 8; ++b) {
        double w = 1.0;
        for (int d = 0; d < 3; ++d) {
          const double pos = (((c >> d) & 1) + ((a >> d) & 1)) / 2.0;
          w *= ((b >> d) & 1) ? pos : 1.0 - pos;
        }
        T[c][a][b] = w;
      }
}

// W_c (24x24): W[3a+p][3b+q] = T_c[a][b] * (p == q)
static void W_of(const double T[8][8], double W[24][24]) {
  for (int x = 0; x < 24; ++x)
    for (int y = 0; y < 24; ++y) W[x][y] = (x % 3 == y % 3) ? T[x / 3][y / 3] : 0.0;
}

static void wt_a_w(const double W[24][24], const double A[24][24], double R[24][24]) {
  double P[24][24];
  for (int a = 0; a < 24; ++a)
    for (int b = 0; b < 24; ++b) {
      double s = 0.0;
      for (int x = 0; x < 24; ++x) s += A[a][x] * W[x][b];
      P[a][b] = s;
    }
  for (int a = 0; a < 24; ++a)
    for (int b = 0; b < 24; ++b) {
      double s = 0.0;
      for (int x = 0; x < 24; ++x) s += W[x][a] * P[x][b];
      R[a][b] = s;
    }
}

// ------------------------------------------------------------------ kernels
// entry `entry` of the level-1 element matrix of coarse element E = (I, J, K):
// sum_c s_c G_c + corrections (what gal_level1_kernel stores)
struct K1Src {
  Geom gf;
  const double* scale;
  const double* G;
  const double* corr;
  const int* corr_of;
};
__device__ __forceinline__ double k1_entry(const K1Src& k, long long E, int I, int J, int K, int entry) {
  double acc = 0.0;
  double s[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    s[c] = k.scale[elem_off(k.gf, 2 * K + (c >> 2) + 1, 2 * J + ((c >> 1) & 1), 2 * I + (c & 1))];
    acc = fma(s[c], k.G[c * 576 + entry], acc);
  }
  if (k.corr_of) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int q = k.corr_of[E * 8 + c];
      if (q >= 0) acc = __dadd_rn(acc, __dmul_rn(s[c], k.corr[(long long)q * 576 + entry]));
    }
  }
  return acc;
}

// level-1 matrices from the fine scale field (vt element layout of the fine grid)
__global__ void gal_level1_kernel(Geom gf, int cnx, int cny, int cnz, const double* __restrict__ scale,
                                  const double* __restrict__ G, const double* __restrict__ corr,
                                  const int* __restrict__ corr_of, double* __restrict__ mats) {
  griddep_wait();
  const long long total = (long long)cnx * cny * cnz * 576;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const long long E = t / 576;
    const int entry = (int)(t - E * 576);
    const int I = (int)(E % cnx), J = (int)((E / cnx) % cny), K = (int)(E / ((long long)cnx * cny));
    double s[8];
#pragma unroll
    for (int c = 0; c < 8; ++c)
      s[c] = scale[elem_off(gf, 2 * K + (c >> 2) + 1, 2 * J + ((c >> 1) & 1), 2 * I + (c & 1))];
    double acc = 0.0;
#pragma unroll
    for (int c = 0; c < 8; ++c) acc = fma(s[c], G[c * 576 + entry], acc);
    if (corr_of) {
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const int k = corr_of[E * 8 + c];
        if (k >= 0) acc = __dadd_rn(acc, __dmul_rn(s[c], corr[(long long)k * 576 + entry]));
      }
    }
    const int a = entry / 24, b = entry % 24;
    if (a <= b) mats[E * GAL_PACK + gal_sym(a, b)] = acc;
  }
}

// level l -> l+1: one CTA (192 threads, 3 entries each) per coarse element
// (FROM_SCALE: the children are level-1 elements, formed on the fly from the
// fine scales instead of read from storage -- level 1 stays matrix-free)
template <bool FROM_SCALE>
__global__ void __launch_bounds__(192) gal_coarsen_kernel(Geom gl, const uint8_t* __restrict__ mask,
                                                          const double* __restrict__ mats_l,
                                                          K1Src k1, int cnx, int cny, int cnz,
                                                          double* __restrict__ mats_c) {
  griddep_wait();
  __shared__ double A[576], P[576];
  __shared__ double m[24];
  // the octant tables in shared memory (threads of a warp index different
  // columns: the constant cache would serialize them)
  __shared__ double Ts[8 * 8 * 8];
  // FROM_SCALE: the current child's 8 fine scales and correction ids, loaded
  // once per child instead of once per matrix entry
  __shared__ double s8[8];
  __shared__ int c8[8];
  for (int t = threadIdx.x; t < 512; t += blockDim.x) Ts[t] = (&c_T[0][0][0])[t];
  const long long nelc = (long long)cnx * cny * cnz;
  for (long long E = blockIdx.x; E < nelc; E += gridDim.x) {
    const int I = (int)(E % cnx), J = (int)((E / cnx) % cny), K = (int)(E / ((long long)cnx * cny));
    double acc[3] = {0.0, 0.0, 0.0};
    for (int c = 0; c < 8; ++c) {
      const int fi = 2 * I + (c & 1), fj = 2 * J + ((c >> 1) & 1), fk = 2 * K + (c >> 2);
      const long long e = ((long long)fk * gl.ny + fj) * gl.nx + fi;
      __syncthreads();
      if (threadIdx.x < 24) {
        const int corner = threadIdx.x / 3, comp = threadIdx.x % 3;
        const unsigned mk = mask[mask_off(gl, fk + ((corner >> 2) & 1) + 1, fj + ((corner >> 1) & 1),
                                          fi + (corner & 1))];
        m[threadIdx.x] = ((mk >> comp) & 1u) ? 0.0 : 1.0;
      } else if (FROM_SCALE && threadIdx.x < 32) {
        const int cc = threadIdx.x - 24;
        s8[cc] = k1.scale[elem_off(k1.gf, 2 * fk + (cc >> 2) + 1, 2 * fj + ((cc >> 1) & 1), 2 * fi + (cc & 1))];
        c8[cc] = k1.corr_of ? k1.corr_of[e * 8 + cc] : -1;
      }
      __syncthreads();
      for (int q = threadIdx.x; q < 576; q += blockDim.x) {
        double kq;
        if (FROM_SCALE) {  // k1_entry with the child's invariants hoisted (same order)
          kq = 0.0;
#pragma unroll
          for (int cc = 0; cc < 8; ++cc) kq = fma(s8[cc], k1.G[cc * 576 + q], kq);
#pragma unroll
          for (int cc = 0; cc < 8; ++cc)
            if (c8[cc] >= 0) kq = __dadd_rn(kq, __dmul_rn(s8[cc], k1.corr[(long long)c8[cc] * 576 + q]));
        } else {
          kq = mats_l[e * GAL_PACK + gal_sym(q / 24, q % 24)];
        }
        A[q] = kq * (m[q / 24] * m[q % 24]);
      }
      __syncthreads();
      const double* Tc = Ts + c * 64;
      // P = A W_c: P[a][b] = sum_x A[a][3x + b%3] T_c[x][b/3]
      for (int q = threadIdx.x; q < 576; q += blockDim.x) {
        const int a = q / 24, b = q % 24;
        double s = 0.0;
#pragma unroll
        for (int x = 0; x < 8; ++x) s = fma(A[a * 24 + 3 * x + b % 3], Tc[x * 8 + b / 3], s);
        P[q] = s;
      }
      __syncthreads();
      // R = W_c^T P: R[a][b] = sum_x T_c[x][a/3] P[3x + a%3][b]
#pragma unroll
      for (int r = 0; r < 3; ++r) {
        const int q = threadIdx.x + r * 192;
        const int a = q / 24, b = q % 24;
        double s = 0.0;
#pragma unroll
        for (int x = 0; x < 8; ++x) s = fma(Tc[x * 8 + a / 3], P[(3 * x + a % 3) * 24 + b], s);
        acc[r] = __dadd_rn(acc[r], s);
      }
    }
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int q = threadIdx.x + r * 192, a = q / 24, b = q % 24;
      if (a <= b) mats_c[E * GAL_PACK + gal_sym(a, b)] = acc[r];  // upper triangle stored
    }
  }
}

// ve[e][r] = sum_b K_e[r][b] u_e[b], u projected to zero on fixed dofs; a warp
// per element stages the packed upper triangle (2400 B, 16-byte vector loads
// by all 32 lanes) and u_e in its shared-memory slots, then lane r < 24 forms
// row r with two accumulator chains (even / odd columns).  Half the matrix
// bytes of full storage (cfg2 level 2: 157 MB instead of 302 MB; 51 vs 70 us).
// Measured and not kept: a register-prefetched next element (54 us) and an
// expanded, row-padded copy in shared memory (64 us).
constexpr int GE_WARPS = GL_THREADS / 32;
__global__ void __launch_bounds__(GL_THREADS) gal_elem_kernel(Geom g, const uint8_t* __restrict__ mask,
                                                              const double* __restrict__ mats,
                                                              const double* __restrict__ u,
                                                              double* __restrict__ ve, const int* stop) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  __shared__ double us[GE_WARPS][24];
  __shared__ __align__(16) double ms[GE_WARPS][GAL_PACK];
  const long long nel = (long long)g.nx * g.ny * g.nz;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  double* m = ms[wib];
  for (long long e = warp; e < nel; e += nw) {
    const int i = (int)(e % g.nx), j = (int)((e / g.nx) % g.ny), k = (int)(e / ((long long)g.nx * g.ny));
    __syncwarp();
    const double2* src = reinterpret_cast<const double2*>(mats + e * GAL_PACK);
#pragma unroll
    for (int q = lane; q < GAL_PACK / 2; q += 32) reinterpret_cast<double2*>(m)[q] = src[q];
    if (lane < 24) {
      const int corner = lane / 3, comp = lane % 3;
      const int p = k + ((corner >> 2) & 1) + 1, jj = j + ((corner >> 1) & 1), ii = i + (corner & 1);
      const unsigned mk = mask[mask_off(g, p, jj, ii)];
      us[wib][lane] = ((mk >> comp) & 1u) ? 0.0 : u[node_off(g, p, jj, ii) * 3 + comp];
    }
    __syncwarp();
    if (lane < 24) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int b2 = 0; b2 < 12; ++b2) {
        s0 = fma(m[gal_sym(lane, 2 * b2)], us[wib][2 * b2], s0);
        s1 = fma(m[gal_sym(lane, 2 * b2 + 1)], us[wib][2 * b2 + 1], s1);
      }
      ve[e * 24 + lane] = s0 + s1;
    }
  }
}

// node epilogue: v = sum over the node's element corners (c = 0..7) of ve, then
//   MODE 0: out = v (fixed: u)        apply_level  [ref: operator.py:58-81]
//   MODE 1: out = f - v (fixed: 0)    residual     [ref: multigrid.py:387-393]
//   MODE 2: out = u + omega (f - v)/d (fixed: u)   damped Jacobi sweep
template <int MODE>
__global__ void gal_node_kernel(Geom g, const uint8_t* __restrict__ mask, const double* __restrict__ ve,
                                const double* __restrict__ u, const double* __restrict__ f,
                                const double* __restrict__ d, double omega, double* __restrict__ out,
                                const int* stop) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (g.nx + 1));
    const long long r = t / (g.nx + 1);
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const int k = p - 1;
    double v[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int ei = i - (c & 1), ej = j - ((c >> 1) & 1), ek = k - ((c >> 2) & 1);
      if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek >= g.nz) continue;
      const long long e = ((long long)ek * g.ny + ej) * g.nx + ei;
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) v[comp] = __dadd_rn(v[comp], ve[e * 24 + 3 * c + comp]);
    }
    const long long node = node_off(g, p, j, i);
    const unsigned m = mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      const long long o = node * 3 + comp;
      const bool fx = (m >> comp) & 1u;
      double val;
      if (MODE == 0) {
        val = fx ? u[o] : v[comp];
      } else if (MODE == 1) {
        val = fx ? 0.0 : __dsub_rn(f[o], v[comp]);
      } else {
        val = fx ? u[o] : __dadd_rn(u[o], __dmul_rn(omega, ddiv_nr(__dsub_rn(f[o], v[comp]), d[o])));
      }
      out[o] = val;
    }
  }
}

// level-1 epilogue of the matrix-free Galerkin operator (v = P^T Pi K0 Pi P x
// already restricted, coarse fixed dofs zero): same modes as gal_node_kernel
template <int MODE>
__global__ void gal_vec_epilogue_kernel(Geom g, const uint8_t* __restrict__ mask,
                                        const double* __restrict__ v, const double* __restrict__ u,
                                        const double* __restrict__ f, const double* __restrict__ d,
                                        double omega, double* __restrict__ out, const int* stop) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (g.nx + 1));
    const long long r = t / (g.nx + 1);
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const long long node = node_off(g, p, j, i);
    const unsigned m = mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      const long long o = node * 3 + comp;
      const bool fx = (m >> comp) & 1u;
      double val;
      if (MODE == 0)
        val = fx ? u[o] : v[o];
      else if (MODE == 1)
        val = fx ? 0.0 : __dsub_rn(f[o], v[o]);
      else
        val = fx ? u[o] : __dadd_rn(u[o], __dmul_rn(omega, ddiv_nr(__dsub_rn(f[o], v[o]), d[o])));
      out[o] = val;
    }
  }
}

// per-dof diagonal: stored element diagonals summed in corner order; 1 on fixed
template <bool FROM_SCALE>
__global__ void gal_diag_kernel(Geom g, const uint8_t* __restrict__ mask, const double* __restrict__ mats,
                                K1Src k1, double* __restrict__ d) {
  griddep_wait();
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (g.nx + 1));
    const long long r = t / (g.nx + 1);
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const int k = p - 1;
    double v[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int ei = i - (c & 1), ej = j - ((c >> 1) & 1), ek = k - ((c >> 2) & 1);
      if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek >= g.nz) continue;
      const long long e = ((long long)ek * g.ny + ej) * g.nx + ei;
#pragma unroll
      for (int comp = 0; comp < 3; ++comp)
        v[comp] = __dadd_rn(v[comp], FROM_SCALE ? k1_entry(k1, e, ei, ej, ek, (3 * c + comp) * 25)
                                                : mats[e * GAL_PACK + gal_sym(3 * c + comp, 3 * c + comp)]);
    }
    const long long node = node_off(g, p, j, i);
    const unsigned m = mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) d[node * 3 + comp] = ((m >> comp) & 1u) ? 1.0 : v[comp];
  }
}

// u = omega * (f / d) on free dofs (first pre-smooth from zero)
__global__ void gal_jacobi0_kernel(Geom g, const uint8_t* __restrict__ mask, const double* __restrict__ f,
                                   const double* __restrict__ d, double omega, double* __restrict__ u,
                                   const int* stop) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  const long long nn = (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t % (g.nx + 1));
    const long long r = t / (g.nx + 1);
    const int j = (int)(r % (g.ny + 1));
    const int p = (int)(r / (g.ny + 1)) + g.pA;
    const long long node = node_off(g, p, j, i);
    const unsigned m = mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      const long long o = node * 3 + comp;
      u[o] = ((m >> comp) & 1u) ? 0.0 : __dmul_rn(omega, ddiv_nr(f[o], d[o]));
    }
  }
}

// ------------------------------------------------------------------ host side
vt_status gal_setup(vt_hier* H) {
  if (H->lv.size() < 2) return VT_OK;
  vt_grid* F = H->lv[0];
  vt_grid* C1 = H->lv[1];
  double T[8][8][8];
  octant_T(T);
  VT_CUDA(cudaMemcpyToSymbol(c_T, T, sizeof(T)));
  double K0[24][24];
  hex8_k0_host(F->nu, F->h, &K0[0][0]);
  std::vector<double> G(8 * 576);
  double W[24][24], R[24][24];
  for (int c = 0; c < 8; ++c) {
    W_of(T[c], W);
    wt_a_w(W, K0, R);
    for (int q = 0; q < 576; ++q) G[c * 576 + q] = R[q / 24][q % 24];
  }
  VT_CUDA(cudaMalloc(&H->gG, G.size() * sizeof(double)));
  VT_CUDA(cudaMemcpy(H->gG, G.data(), G.size() * sizeof(double), cudaMemcpyHostToDevice));
  // fine fixed-dof corrections, deduplicated by (octant, free pattern)
  const Geom& g = F->g;
  std::vector<uint8_t> hm((size_t)g.P * g.mplane);
  VT_CUDA(cudaMemcpy(hm.data(), F->mask, hm.size(), cudaMemcpyDeviceToHost));
  const long long nel1 = (long long)C1->g.nx * C1->g.ny * C1->g.nz;
  std::vector<int> corr_of((size_t)nel1 * 8, -1);
  std::map<std::pair<int, unsigned>, int> uniq;
  std::vector<double> corr;
  bool any = false;
  for (int k = 0; k < g.nz; ++k)
    for (int j = 0; j < g.ny; ++j)
      for (int i = 0; i < g.nx; ++i) {
        unsigned fixedbits = 0;
        for (int corner = 0; corner < 8; ++corner) {
          const uint8_t mk = hm[((size_t)(k + ((corner >> 2) & 1) + 1) * (g.ny + 1) + j + ((corner >> 1) & 1)) *
                                    g.mp + i + (corner & 1)];
          fixedbits |= (unsigned)(mk & 7u) << (3 * corner);
        }
        if (!fixedbits) continue;
        any = true;
        const int oct = (i & 1) + 2 * (j & 1) + 4 * (k & 1);
        auto key = std::make_pair(oct, fixedbits);
        auto it = uniq.find(key);
        int idx;
        if (it == uniq.end()) {
          idx = (int)uniq.size();
          uniq[key] = idx;
          double Dl[24][24];
          for (int a = 0; a < 24; ++a)
            for (int b = 0; b < 24; ++b) {
              const double ma = ((fixedbits >> a) & 1u) ? 0.0 : 1.0;
              const double mb = ((fixedbits >> b) & 1u) ? 0.0 : 1.0;
              Dl[a][b] = K0[a][b] * (ma * mb) - K0[a][b];
            }
          W_of(T[oct], W);
          wt_a_w(W, Dl, R);
          for (int q = 0; q < 576; ++q) corr.push_back(R[q / 24][q % 24]);
        } else {
          idx = it->second;
        }
        const long long E = ((long long)(k / 2) * C1->g.ny + j / 2) * C1->g.nx + i / 2;
        corr_of[E * 8 + oct] = idx;
      }
  if (any) {
    VT_CUDA(cudaMalloc(&H->gcorr, corr.size() * sizeof(double)));
    VT_CUDA(cudaMemcpy(H->gcorr, corr.data(), corr.size() * sizeof(double), cudaMemcpyHostToDevice));
    VT_CUDA(cudaMalloc(&H->gcorr_of, corr_of.size() * sizeof(int)));
    VT_CUDA(cudaMemcpy(H->gcorr_of, corr_of.data(), corr_of.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  const int L = (int)H->lv.size();
  H->mats.assign(L, nullptr);
  H->gdiag.assign(L, nullptr);
  // Level 1 is applied matrix-free as P^T (Pi K0 Pi) P through the fine kernels
  // when it is not the coarsest level (its 576 doubles per element would be
  // the largest array of the solver: 2.4 GB at cfg2, 65 GB at cfg5);
  // levels >= 2 store their matrices.
  H->gal_mf = L >= 3;
  for (int l = 1; l < L; ++l) {
    vt_grid* G2 = H->lv[l];
    const long long nel = (long long)G2->g.nx * G2->g.ny * G2->g.nz;
    if (!(l == 1 && H->gal_mf)) VT_CUDA(cudaMalloc(&H->mats[l], (size_t)nel * GAL_PACK * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->gdiag[l], G2->vec_len() * sizeof(double)));
    VT_CUDA(cudaMemset(H->gdiag[l], 0, G2->vec_len() * sizeof(double)));
  }
  if (H->gal_mf) {
    VT_CUDA(cudaMalloc(&H->gfa, F->vec_len() * sizeof(double)));
    VT_CUDA(cudaMemset(H->gfa, 0, F->vec_len() * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->gfb, F->vec_len() * sizeof(double)));
    VT_CUDA(cudaMemset(H->gfb, 0, F->vec_len() * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->gc1, C1->vec_len() * sizeof(double)));
    VT_CUDA(cudaMemset(H->gc1, 0, C1->vec_len() * sizeof(double)));
    const long long nel2 = L >= 3 ? (long long)H->lv[2]->g.nx * H->lv[2]->g.ny * H->lv[2]->g.nz : 0;
    VT_CUDA(cudaMalloc(&H->gve, (size_t)(nel2 > 0 ? nel2 : 1) * 24 * sizeof(double)));
  } else {
    VT_CUDA(cudaMalloc(&H->gve, (size_t)nel1 * 24 * sizeof(double)));
  }
  return VT_OK;
}

void gal_free(vt_hier* H) {
  cudaFree(H->gfa);
  cudaFree(H->gfb);
  cudaFree(H->gc1);
  cudaFree(H->gG);
  cudaFree(H->gcorr);
  cudaFree(H->gcorr_of);
  cudaFree(H->gve);
  for (double* p : H->mats) cudaFree(p);
  for (double* p : H->gdiag) cudaFree(p);
  cudaFree(H->mats_full);
}

// full 24x24 matrices of level l from the packed storage (API / tests)
__global__ void gal_expand_kernel(const double* __restrict__ packed, long long nel, double* __restrict__ full) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nel * 576;
       t += (long long)gridDim.x * blockDim.x) {
    const long long e = t / 576;
    const int q = (int)(t - e * 576);
    full[t] = packed[e * GAL_PACK + gal_sym(q / 24, q % 24)];
  }
}

vt_status gal_expand(vt_hier* H, int l, cudaStream_t s) {
  vt_grid* G = H->lv[l];
  const long long nel = (long long)G->g.nx * G->g.ny * G->g.nz;
  if (H->mats_full_n < nel * 576) {
    cudaFree(H->mats_full);
    H->mats_full = nullptr;
    H->mats_full_n = 0;
    VT_CUDA(cudaMalloc(&H->mats_full, (size_t)nel * 576 * sizeof(double)));
    H->mats_full_n = nel * 576;
  }
  launch_pdl(gal_expand_kernel, G->nsm * 8, GL_THREADS, 0, s, (const double*)H->mats[l], nel, H->mats_full);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

static K1Src k1src(vt_hier* H) {
  return K1Src{H->lv[0]->g, H->scale[0], H->gG, H->gcorr, H->gcorr_of};
}

vt_status gal_materialize_level1(vt_hier* H, cudaStream_t s) {
  vt_grid* F = H->lv[0];
  vt_grid* C1 = H->lv[1];
  const long long nel1 = (long long)C1->g.nx * C1->g.ny * C1->g.nz;
  const long long tot1 = nel1 * 576;
  if (!H->mats[1]) VT_CUDA(cudaMalloc(&H->mats[1], (size_t)nel1 * GAL_PACK * sizeof(double)));
  const int grid1 = (int)std::min<long long>((tot1 + GL_THREADS - 1) / GL_THREADS, (long long)F->nsm * 16);
  launch_pdl(gal_level1_kernel, grid1, GL_THREADS, 0, s, F->g, C1->g.nx, C1->g.ny, C1->g.nz, H->scale[0], H->gG,
                                                 H->gcorr, H->gcorr_of, H->mats[1]);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status gal_refresh(vt_hier* H, cudaStream_t s) {
  const int L = (int)H->lv.size();
  if (L < 2) return VT_OK;
  const K1Src k1 = k1src(H);
  if (!H->gal_mf) VT_TRY(gal_materialize_level1(H, s));
  H->mats1_fresh = !H->gal_mf;
  for (int l = 1; l + 1 < L; ++l) {
    vt_grid* Gl = H->lv[l];
    vt_grid* Gc = H->lv[l + 1];
    const long long nelc = (long long)Gc->g.nx * Gc->g.ny * Gc->g.nz;
    const int grid = (int)std::min<long long>(nelc, (long long)Gl->nsm * 32);
    if (l == 1 && H->gal_mf)
      launch_pdl(gal_coarsen_kernel<true>, grid, 192, 0, s, Gl->g, Gl->mask, nullptr, k1, Gc->g.nx, Gc->g.ny,
                                                    Gc->g.nz, H->mats[l + 1]);
    else
      launch_pdl(gal_coarsen_kernel<false>, grid, 192, 0, s, Gl->g, Gl->mask, H->mats[l], k1, Gc->g.nx, Gc->g.ny,
                                                     Gc->g.nz, H->mats[l + 1]);
    count_launch();
  }
  for (int l = 1; l < L; ++l) {
    vt_grid* Gl = H->lv[l];
    if (l == 1 && H->gal_mf)
      launch_pdl(gal_diag_kernel<true>, Gl->nsm * 4, GL_THREADS, 0, s, Gl->g, Gl->mask, nullptr, k1, H->gdiag[l]);
    else
      launch_pdl(gal_diag_kernel<false>, Gl->nsm * 4, GL_THREADS, 0, s, Gl->g, Gl->mask, H->mats[l], k1, H->gdiag[l]);
    count_launch();
  }
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// mode 0 apply, 1 residual, 2 damped Jacobi sweep on galerkin level l >= 1
vt_status gal_level_op(vt_hier* H, int l, int mode, const double* u, const double* f, double* out,
                       const int* stop, cudaStream_t s) {
  vt_grid* G = H->lv[l];
  if (l == 1 && H->gal_mf) {
    // K1 x = Pi1 P^T Pi0 K0 Pi0 P Pi1 x through the fine-level kernels
    vt_grid* F = H->lv[0];
    const double* x = u;
    if (mode == 0) {  // API apply: the input may be non-zero on fixed dofs
      VT_TRY(launch_project(G, u, G->scratch, s));
      x = G->scratch;
    }
    VT_TRY(launch_prolong_set(G, F, x, H->gfa, stop, s));
    VT_TRY(launch_hex8(F, H8_APPLY, false, H->scale[0], H->gfa, nullptr, nullptr, H->gfb, 0.0,
                       nullptr, stop, s));
    VT_TRY(launch_restrict(F, G, H->gfb, H->gc1, stop, -1, -1, s));
    const int grid_n = fit_grid((long long)(G->g.pB - G->g.pA) * (G->g.ny + 1) * (G->g.nx + 1), GL_THREADS, G->nsm * 4);
    if (mode == 0)
      launch_pdl(gal_vec_epilogue_kernel<0>, grid_n, GL_THREADS, 0, s, G->g, G->mask, H->gc1, u, f, H->gdiag[l], H->omega, out, stop);
    else if (mode == 1)
      launch_pdl(gal_vec_epilogue_kernel<1>, grid_n, GL_THREADS, 0, s, G->g, G->mask, H->gc1, u, f, H->gdiag[l], H->omega, out, stop);
    else
      launch_pdl(gal_vec_epilogue_kernel<2>, grid_n, GL_THREADS, 0, s, G->g, G->mask, H->gc1, u, f, H->gdiag[l], H->omega, out, stop);
    count_launch();
    VT_CUDA(cudaGetLastError());
    return VT_OK;
  }
  const long long nel = (long long)G->g.nx * G->g.ny * G->g.nz;
  const int grid_e = (int)std::min<long long>((nel * 32 + GL_THREADS - 1) / GL_THREADS, (long long)G->nsm * 16);
  launch_pdl(gal_elem_kernel, grid_e, GL_THREADS, 0, s, G->g, G->mask, H->mats[l], u, H->gve, stop);
  const int grid_n = fit_grid((long long)(G->g.pB - G->g.pA) * (G->g.ny + 1) * (G->g.nx + 1), GL_THREADS, G->nsm * 4);
  if (mode == 0)
    launch_pdl(gal_node_kernel<0>, grid_n, GL_THREADS, 0, s, G->g, G->mask, H->gve, u, f, H->gdiag[l], H->omega, out, stop);
  else if (mode == 1)
    launch_pdl(gal_node_kernel<1>, grid_n, GL_THREADS, 0, s, G->g, G->mask, H->gve, u, f, H->gdiag[l], H->omega, out, stop);
  else
    launch_pdl(gal_node_kernel<2>, grid_n, GL_THREADS, 0, s, G->g, G->mask, H->gve, u, f, H->gdiag[l], H->omega, out, stop);
  count_launch(2);
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// the same passes on a grid that is not a hierarchy level (a z-slab of level 1)
vt_status launch_gal_jacobi0(vt_grid* G, const double* f, const double* d, double omega, double* u,
                             const int* stop, cudaStream_t s) {
  launch_pdl(gal_jacobi0_kernel, fit_grid((long long)(G->g.pB - G->g.pA) * (G->g.ny + 1) * (G->g.nx + 1), GL_THREADS, G->nsm * 4), GL_THREADS, 0, s, G->g, G->mask, f, d, omega, u, stop);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status launch_gal_vec_epilogue(vt_grid* G, int mode, const double* v, const double* u, const double* f,
                                  const double* d, double omega, double* out, const int* stop,
                                  cudaStream_t s) {
  const int grid_n = fit_grid((long long)(G->g.pB - G->g.pA) * (G->g.ny + 1) * (G->g.nx + 1), GL_THREADS, G->nsm * 4);
  if (mode == 0)
    launch_pdl(gal_vec_epilogue_kernel<0>, grid_n, GL_THREADS, 0, s, G->g, G->mask, v, u, f, d, omega, out, stop);
  else if (mode == 1)
    launch_pdl(gal_vec_epilogue_kernel<1>, grid_n, GL_THREADS, 0, s, G->g, G->mask, v, u, f, d, omega, out, stop);
  else
    launch_pdl(gal_vec_epilogue_kernel<2>, grid_n, GL_THREADS, 0, s, G->g, G->mask, v, u, f, d, omega, out, stop);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status gal_jacobi0(vt_hier* H, int l, const double* f, double* u, const int* stop, cudaStream_t s) {
  vt_grid* G = H->lv[l];
  launch_pdl(gal_jacobi0_kernel, fit_grid((long long)(G->g.pB - G->g.pA) * (G->g.ny + 1) * (G->g.nx + 1), GL_THREADS, G->nsm * 4), GL_THREADS, 0, s, G->g, G->mask, f, H->gdiag[l], H->omega, u, stop);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

}  // namespace vt
