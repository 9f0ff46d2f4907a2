// The coarse tail of the homogenized V-cycle in ONE launch (one thread-block
// cluster).
//
// Below a few ten thousand dofs every V-cycle kernel is launch- and
// latency-bound: the five passes per level (first Jacobi sweep, residual,
// restriction, prolongation, smoother) and the three coarsest mat-vecs cost
// ~5-8 us each at any size, ~30 launches per V-cycle.  Here the levels
// T..L-1 (T = the first level with at most TAIL_MAX_EL elements) run inside
// one cluster of CTAs; every dependent pass is separated by a hardware
// cluster barrier (release / acquire: global writes of one CTA are visible to
// the others) instead of a kernel boundary.  All vectors stay in global
// memory (L2-resident at these sizes); values written inside the launch are
// read with ld.global.cg.
//
// The arithmetic is the multi-kernel V-cycle's, operation for operation:
//  * the operator is the factorized hex8 product of hex8_apply.cu split in
//    two deterministic phases: an element phase stores each element's top /
//    bottom contributions in the (S,D)_xy basis (exactly the arrays the tile
//    kernel carries in registers: Top = its Tn, Bot = the part it adds to the
//    carried Tp), then a node phase forms Ft = Top(below) + Bot(above) for
//    the 4 element columns of the node and the same y / x transposed-butterfly
//    sums (lowy + xb, then (e0 - e1) + (e0 + e1) of the left column) and
//    epilogues (residual / damped Jacobi with the on-the-fly diagonal);
//  * restriction / prolongation per dof with the z -> y -> x pass order of
//    restrict_kernel / prolong_kernel; the coarsest solve as coarse_mv_kernel
//    (one warp per row, lane-strided FMAs, xor tree);
// so the V-cycle output is the same as the kernel-per-pass sequence (up to
// the sign of exact zeros).
#include <stdlib.h>

#include "vt_internal.h"

namespace vt {

constexpr int TAIL_THREADS = 512;
constexpr int TAIL_MAX_LEV = 8;

struct TailLevel {
  Geom g;
  const uint8_t* mask;
  const double* scale;  // vt element layout
  const double* wd;     // omega / diag per dof (0 on fixed)
  double* u;
  double* f;
  double* r;
  double* ev;           // element scratch: 24 doubles per element (Top[12], Bot[12])
  double kc[6];
  double kd;
};

struct TailArgs {
  int nlev;             // levels T .. L-1 (entry nlev-1 is the coarsest)
  TailLevel lv[TAIL_MAX_LEV];
  int nL;               // coarsest dofs
  const double* Kinv;
  const double* A0;
  double* cvec;         // fc, x0, cr
  double omega;
  const int* stop;
};

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned cluster_ncta() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}

// the tile kernel's face_coeffs on four gathered corner nodes (rows j, j+1)
__device__ __forceinline__ void face4(const double* n00, const double* n10, const double* n01,
                                      const double* n11, double F[12]) {
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double a00 = __ldcg(n00 + c), a10 = __ldcg(n10 + c), a01 = __ldcg(n01 + c), a11 = __ldcg(n11 + c);
    const double sx0 = a10 + a00, dx0 = a10 - a00, sx1 = a11 + a01, dx1 = a11 - a01;
    F[c * 4 + 0] = sx1 + sx0;
    F[c * 4 + 1] = dx1 + dx0;
    F[c * 4 + 2] = sx1 - sx0;
    F[c * 4 + 3] = dx1 - dx0;
  }
}

// sparse (S,D)^3 coupling of hex8_apply.cu (same operation order)
__device__ __forceinline__ void tail_couple(const double C[3][8], double s, const double* kc,
                                            double O[3][8]) {
  const double a1 = s * kc[0], a2 = s * kc[1], a3 = s * kc[2], a4 = s * kc[3], a5 = s * kc[4],
               a6 = s * kc[5];
  const double d0 = C[0][1] + C[1][2] + C[2][4];
  const double ld = a1 * d0;
  O[0][1] = fma(a2, C[0][1], ld);
  O[1][2] = fma(a2, C[1][2], ld);
  O[2][4] = fma(a2, C[2][4], ld);
  const double t01 = a3 * (C[0][2] + C[1][1]);
  const double t02 = a3 * (C[0][4] + C[2][1]);
  const double t12 = a3 * (C[1][4] + C[2][2]);
  O[0][2] = t01; O[1][1] = t01;
  O[0][4] = t02; O[2][1] = t02;
  O[1][4] = t12; O[2][2] = t12;
  double w = a4 * (C[0][3] + C[2][6]);
  O[0][3] = fma(a3, C[0][3], w);
  O[2][6] = fma(a3, C[2][6], w);
  w = a4 * (C[0][5] + C[1][6]);
  O[0][5] = fma(a3, C[0][5], w);
  O[1][6] = fma(a3, C[1][6], w);
  w = a4 * (C[1][3] + C[2][5]);
  O[1][3] = fma(a3, C[1][3], w);
  O[2][5] = fma(a3, C[2][5], w);
  const double tt = C[0][6] + C[1][5] + C[2][3];
  O[0][6] = a5 * (tt + C[0][6]);
  O[1][5] = a5 * (tt + C[1][5]);
  O[2][3] = a5 * (tt + C[2][3]);
  O[0][7] = a6 * C[0][7];
  O[1][7] = a6 * C[1][7];
  O[2][7] = a6 * C[2][7];
}

// element phase: ev[e] = {Top[12], Bot[12]} of K_e u_e
__device__ void tail_elements(const TailLevel& L, const double* u, long long tid, long long nth) {
  const Geom& g = L.g;
  const long long nel = (long long)g.nx * g.ny * g.nz;
  for (long long e = tid; e < nel; e += nth) {
    const int i = (int)(e % g.nx);
    const long long r = e / g.nx;
    const int j = (int)(r % g.ny), k = (int)(r / g.ny);
    const double* b00 = u + node_off(g, k + 1, j, i) * 3;
    const double* b01 = u + node_off(g, k + 1, j + 1, i) * 3;
    const double* t00 = u + node_off(g, k + 2, j, i) * 3;
    const double* t01 = u + node_off(g, k + 2, j + 1, i) * 3;
    double Fp[12], Fn[12];
    face4(b00, b00 + 3, b01, b01 + 3, Fp);
    face4(t00, t00 + 3, t01, t01 + 3, Fn);
    double C[3][8], O[3][8];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      C[c][0] = 0.0;
#pragma unroll
      for (int xy = 0; xy < 4; ++xy) {
        if (xy) C[c][xy] = Fn[c * 4 + xy] + Fp[c * 4 + xy];
        C[c][xy | 4] = Fn[c * 4 + xy] - Fp[c * 4 + xy];
      }
    }
    tail_couple(C, L.scale[elem_off(g, k + 1, j, i)], L.kc, O);
    double* out = L.ev + e * 24;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[c * 4 + 0] = O[c][4];          // Top
      out[12 + c * 4 + 0] = -O[c][4];    // Bot (the tile kernel's Tp - O4)
#pragma unroll
      for (int xy = 1; xy < 4; ++xy) {
        const double lo = O[c][xy], hi = O[c][xy | 4];
        out[c * 4 + xy] = lo + hi;
        out[12 + c * 4 + xy] = lo - hi;
      }
    }
  }
}

// Ft of element column (ex, ey) for node plane k: Top(layer k-1) + Bot(layer k)
__device__ __forceinline__ void tail_ft(const TailLevel& L, int ex, int ey, int k, int c, double ft[4]) {
  const Geom& g = L.g;
  if (ex < 0 || ex >= g.nx || ey < 0 || ey >= g.ny) {
    ft[0] = ft[1] = ft[2] = ft[3] = 0.0;
    return;
  }
  const long long base = ((long long)ey * g.nx + ex);
  const long long lay = (long long)g.nx * g.ny;
#pragma unroll
  for (int xy = 0; xy < 4; ++xy) {
    const double top = k >= 1 ? __ldcg(L.ev + (base + (k - 1) * lay) * 24 + c * 4 + xy) : 0.0;
    const double bot = k < g.nz ? __ldcg(L.ev + (base + k * lay) * 24 + 12 + c * 4 + xy) : 0.0;
    ft[xy] = top + bot;
  }
}

// node phase.  MODE 1: r = f - K u (fixed 0);  MODE 2: damped Jacobi in place
template <int MODE>
__device__ void tail_nodes(const TailLevel& L, double omega, long long tid, long long nth) {
  const Geom& g = L.g;
  const int nx1 = g.nx + 1, ny1 = g.ny + 1;
  const long long nn = (long long)nx1 * ny1 * (g.nz + 1);
  for (long long t = tid; t < nn; t += nth) {
    const int i = (int)(t % nx1);
    const long long r0 = t / nx1;
    const int j = (int)(r0 % ny1), k = (int)(r0 / ny1);
    const long long node = node_off(g, k + 1, j, i);
    const unsigned fm = L.mask[mask_off(g, k + 1, j, i)];
    double v[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      double E[2][2];  // [column i-1, i][tau]
#pragma unroll
      for (int col = 0; col < 2; ++col) {
        double lo[4], hiy[4];
        tail_ft(L, i - 1 + col, j, k, c, lo);       // element row j: low-y halves
        tail_ft(L, i - 1 + col, j - 1, k, c, hiy);  // element row j-1: high-y halves
#pragma unroll
        for (int tau = 0; tau < 2; ++tau) {
          const double lowy = lo[tau] - lo[tau + 2];
          const double xb = hiy[tau] + hiy[tau + 2];
          E[col][tau] = lowy + xb;
        }
      }
      v[c] = (E[1][0] - E[1][1]) + (E[0][0] + E[0][1]);
    }
    const double* f = L.f + node * 3;
    double* out = (MODE == 1 ? L.r : L.u) + node * 3;
    if (MODE == 1) {
#pragma unroll
      for (int c = 0; c < 3; ++c) out[c] = ((fm >> c) & 1u) ? 0.0 : __dsub_rn(__ldcg(f + c), v[c]);
    } else {
      // the SMOOTH epilogue: w = omega / (kd * sum of the 8 incident scales)
      auto sc = [&](int ex, int ey, int q) -> double {
        if (ex < 0 || ex >= g.nx || ey < 0 || ey >= g.ny || q < 0 || q >= g.Q) return 0.0;
        return L.scale[elem_off(g, q, ey, ex)];
      };
      const double s0 = sc(i, j, k + 1), s1 = sc(i - 1, j, k + 1), s2 = sc(i, j - 1, k + 1),
                   s3 = sc(i - 1, j - 1, k + 1), s4 = sc(i, j, k), s5 = sc(i - 1, j, k),
                   s6 = sc(i, j - 1, k), s7 = sc(i - 1, j - 1, k);
      const double ssum = ((s0 + s1) + (s2 + s3)) + ((s4 + s5) + (s6 + s7));
      const double w = __ddiv_rn(omega, __dmul_rn(ssum, L.kd));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double uo = __ldcg(out + c);
        out[c] = ((fm >> c) & 1u) ? 0.0 : fma(__dsub_rn(__ldcg(f + c), v[c]), w, uo);
      }
    }
  }
}

// u = w f (first Jacobi sweep from zero) over the owned planes (pads: w = 0)
__device__ void tail_jacobi0(const TailLevel& L, long long tid, long long nth) {
  const Geom& g = L.g;
  const long long a = (long long)g.pA * g.nplane, n = (long long)(g.pB - g.pA) * g.nplane;
  for (long long t = tid; t < n; t += nth) {
    const double w = L.wd[a + t];
    L.u[a + t] = w == 0.0 ? 0.0 : __dmul_rn(w, __ldcg(L.f + a + t));
  }
}

// f_c = P^T r_f (restrict_kernel's pass order)
__device__ void tail_restrict(const TailLevel& F, const TailLevel& Cl, long long tid, long long nth) {
  const Geom& gf = F.g;
  const Geom& gc = Cl.g;
  const int cx1 = gc.nx + 1, cy1 = gc.ny + 1;
  const long long n = (long long)cx1 * cy1 * (gc.nz + 1) * 3;
  for (long long t = tid; t < n; t += nth) {
    const int c = (int)(t % 3);
    const long long nd = t / 3;
    const int I = (int)(nd % cx1);
    const long long r0 = nd / cx1;
    const int J = (int)(r0 % cy1), K = (int)(r0 / cy1);
    const bool ok1 = 2 * K + 1 <= gf.nz, ok2 = K >= 1;
    const bool okj1 = 2 * J + 1 <= gf.ny, okj2 = J >= 1;
    const bool oki1 = 2 * I + 1 <= gf.nx, oki2 = I >= 1;
    auto tz = [&](int y, int x) -> double {
      const double* p0 = F.r + node_off(gf, 2 * K + 1, y, x) * 3 + c;
      double v = __ldcg(p0);
      if (ok1) v = __dadd_rn(v, 0.5 * __ldcg(p0 + gf.nplane));
      if (ok2) v = __dadd_rn(v, 0.5 * __ldcg(p0 - gf.nplane));
      return v;
    };
    double ty[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const int dx = b == 0 ? 0 : (b == 1 ? 1 : -1);
      if ((b == 1 && !oki1) || (b == 2 && !oki2)) {
        ty[b] = 0.0;
        continue;
      }
      const int x = 2 * I + dx;
      double v = tz(2 * J, x);
      if (okj1) v = __dadd_rn(v, 0.5 * tz(2 * J + 1, x));
      if (okj2) v = __dadd_rn(v, 0.5 * tz(2 * J - 1, x));
      ty[b] = v;
    }
    double v = ty[0];
    if (oki1) v = __dadd_rn(v, 0.5 * ty[1]);
    if (oki2) v = __dadd_rn(v, 0.5 * ty[2]);
    const unsigned m = Cl.mask[mask_off(gc, K + 1, J, I)];
    Cl.f[node_off(gc, K + 1, J, I) * 3 + c] = ((m >> c) & 1u) ? 0.0 : v;
  }
}

// u_f += P u_c (prolong_kernel<true>'s pass order)
__device__ void tail_prolong_add(const TailLevel& Cl, const TailLevel& F, long long tid, long long nth) {
  const Geom& gf = F.g;
  const Geom& gc = Cl.g;
  const int fx1 = gf.nx + 1, fy1 = gf.ny + 1;
  const long long n = (long long)fx1 * fy1 * (gf.nz + 1) * 3;
  for (long long t = tid; t < n; t += nth) {
    const int comp = (int)(t % 3);
    const long long nd = t / 3;
    const int ix = (int)(nd % fx1);
    const long long r0 = nd / fx1;
    const int fy = (int)(r0 % fy1), fz = (int)(r0 / fy1);
    const int K = fz >> 1, cz = fz & 1, J = fy >> 1, I = ix >> 1;
    const bool ox = ix & 1;
    const int Kp = K + 1 <= gc.nz ? K + 1 : K;
    auto q = [&](int kk, int jj, int ii) -> double {
      return __ldcg(Cl.u + node_off(gc, kk + 1, jj, ii) * 3 + comp);
    };
    auto zrow = [&](int jy, double& z0, double& z1) {
      z0 = cz ? 0.5 * __dadd_rn(q(K, jy, I), q(Kp, jy, I)) : q(K, jy, I);
      z1 = ox ? (cz ? 0.5 * __dadd_rn(q(K, jy, I + 1), q(Kp, jy, I + 1)) : q(K, jy, I + 1)) : 0.0;
    };
    double za0, za1, v;
    zrow(J, za0, za1);
    if ((fy & 1) == 0) {
      v = ox ? 0.5 * __dadd_rn(za0, za1) : za0;
    } else {
      double zb0, zb1;
      zrow(J + 1, zb0, zb1);
      const double y0 = 0.5 * __dadd_rn(za0, zb0);
      v = ox ? 0.5 * __dadd_rn(y0, 0.5 * __dadd_rn(za1, zb1)) : y0;
    }
    const unsigned m = F.mask[mask_off(gf, fz + 1, fy, ix)];
    if ((m >> comp) & 1u) v = 0.0;
    double* uf = F.u + node_off(gf, fz + 1, fy, ix) * 3 + comp;
    *uf = __dadd_rn(__ldcg(uf), v);
  }
}

__device__ __forceinline__ void coarse_dof(const Geom& g, int d, long long* nd, int* c, long long* mo) {
  const int nx1 = g.nx + 1, ny1 = g.ny + 1;
  const int node = d / 3;
  *c = d % 3;
  const int i = node % nx1, j = (node / nx1) % ny1, k = node / (nx1 * ny1);
  *nd = node_off(g, k + 1, j, i);
  *mo = mask_off(g, k + 1, j, i);
}

// coarse_mv_kernel<MODE> with the cluster's warps as rows:
//   0: fc = gather(f), x0 = Kinv fc;  1: cr = fc - A0 x0;  2: u = scatter(x0 + Kinv cr)
template <int MODE>
__device__ void tail_coarse_mv(const TailArgs& a, const TailLevel& L, double* vs, long long wid,
                               long long nwarp) {
  const int n = a.nL;
  double *cf = a.cvec, *x0 = a.cvec + n, *cr = a.cvec + 2 * n;
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    double v;
    if (MODE == 0) {
      long long nd, mo;
      int c;
      coarse_dof(L.g, d, &nd, &c, &mo);
      v = __ldcg(L.f + nd * 3 + c);
    } else {
      v = __ldcg((MODE == 1 ? x0 : cr) + d);
    }
    vs[d] = v;
  }
  __syncthreads();
  const int lane = threadIdx.x % 32;
  const double* M = MODE == 1 ? a.A0 : a.Kinv;
  for (long long r = wid; r < n; r += nwarp) {
    double s = 0.0;
    for (int e = lane; e < n; e += 32) s = fma(M[(long long)r * n + e], vs[e], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (MODE == 0) {
        cf[r] = vs[r];
        x0[r] = s;
      } else if (MODE == 1) {
        cr[r] = __ldcg(cf + r) - s;
      } else {
        long long nd, mo;
        int c;
        coarse_dof(L.g, (int)r, &nd, &c, &mo);
        L.u[nd * 3 + c] = ((L.mask[mo] >> c) & 1u) ? 0.0 : __ldcg(x0 + r) + s;
      }
    }
  }
}

// One V(1,1) cycle of the homogenized tail: f of level T given (already
// restricted), u of level T returned in place.  Launched as one cluster.
__global__ void __launch_bounds__(TAIL_THREADS, 1) tail_vcycle_kernel(const __grid_constant__ TailArgs a) {
  griddep_wait();
  if (a.stop != nullptr && *(volatile const int*)a.stop) return;
  extern __shared__ double vs[];
  const long long ncta = cluster_ncta();
  const long long tid = (long long)cluster_rank() * blockDim.x + threadIdx.x;
  const long long nth = ncta * blockDim.x;
  const long long wid = tid / 32, nwarp = nth / 32;
  const int last = a.nlev - 1;
  for (int l = 0; l < last; ++l) {
    const TailLevel& L = a.lv[l];
    tail_jacobi0(L, tid, nth);
    cluster_sync_all();
    tail_elements(L, L.u, tid, nth);
    cluster_sync_all();
    tail_nodes<1>(L, a.omega, tid, nth);
    cluster_sync_all();
    tail_restrict(L, a.lv[l + 1], tid, nth);
    cluster_sync_all();
  }
  tail_coarse_mv<0>(a, a.lv[last], vs, wid, nwarp);
  cluster_sync_all();
  tail_coarse_mv<1>(a, a.lv[last], vs, wid, nwarp);
  cluster_sync_all();
  tail_coarse_mv<2>(a, a.lv[last], vs, wid, nwarp);
  cluster_sync_all();
  for (int l = last - 1; l >= 0; --l) {
    const TailLevel& L = a.lv[l];
    tail_prolong_add(a.lv[l + 1], L, tid, nth);
    cluster_sync_all();
    tail_elements(L, L.u, tid, nth);
    cluster_sync_all();
    tail_nodes<2>(L, a.omega, tid, nth);
    if (l > 0) cluster_sync_all();
  }
}

// ------------------------------------------------------------------ host
static int g_tail_cluster = 0;  // CTAs per cluster (0: not probed yet, -1: unavailable)

static int tail_cluster_size(int smem) {
  if (g_tail_cluster != 0) return g_tail_cluster;
  g_tail_cluster = -1;
  if (cudaFuncSetAttribute(tail_vcycle_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
      cudaFuncSetAttribute(tail_vcycle_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
    cudaGetLastError();
    return g_tail_cluster;
  }
  const char* force = getenv("VT_TAIL_CLUSTER");  // dev: force a cluster size
  const int sizes_all[3] = {16, 8, 4};
  for (int cs : sizes_all) {
    if (force && atoi(force) > 0 && cs != atoi(force)) continue;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(TAIL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, tail_vcycle_kernel, &cfg) == cudaSuccess && n >= 1) {
      g_tail_cluster = cs;
      break;
    }
    cudaGetLastError();
  }
  return g_tail_cluster;
}

// first level of the one-launch tail, or -1 (galerkin levels, several sweeps,
// a large coarsest system, or VT_TAIL=0)
int tail_start(vt_hier* H, int top) {
  const char* e = getenv("VT_TAIL");  // VT_TAIL=0: the kernel-per-pass tail (A/B, tests)
  const int env = e ? atoi(e) : 1;
  const int L = (int)H->lv.size();
  if (!env || H->scheme != 0 || H->sweeps != 1 || L < 2 || H->nL > TAIL_MAX_NL || !H->tail_ev) return -1;
  const int T = H->tail_T;
  if (T < top + 1 || T > L - 2) return -1;  // the tail must have a smoothed level and a coarser one
  if (L - T > TAIL_MAX_LEV || g_tail_cluster <= 0) return -1;
  return T;
}

vt_status tail_alloc(vt_hier* H) {
  const int L = (int)H->lv.size();
  H->tail_T = -1;
  if (H->scheme != 0 || L < 3) return VT_OK;
  int T = -1;
  for (int l = 1; l <= L - 2; ++l) {
    const long long nel = H->lv[l]->nel_local();
    if (nel <= TAIL_MAX_EL) { T = l; break; }
  }
  if (T < 1) return VT_OK;
  // probe the cluster launch here, outside any stream capture
  if (tail_cluster_size((int)(TAIL_MAX_NL * sizeof(double))) <= 0) return VT_OK;
  long long tot = 0;
  for (int l = T; l < L - 1; ++l) tot += H->lv[l]->nel_local() * 24;
  VT_CUDA(cudaMalloc(&H->tail_ev, tot * sizeof(double)));
  H->tail_T = T;
  return VT_OK;
}

vt_status launch_tail_vcycle(vt_hier* H, int T, const double* fT, const int* stop, cudaStream_t s) {
  const int L = (int)H->lv.size();
  TailArgs a = {};
  a.nlev = L - T;
  a.nL = H->nL;
  a.Kinv = H->Kinv;
  a.A0 = H->A0;
  a.cvec = H->cvec;
  a.omega = H->omega;
  a.stop = stop;
  double* ev = H->tail_ev;
  for (int l = T; l < L; ++l) {
    vt_grid* G = H->lv[l];
    TailLevel& t = a.lv[l - T];
    t.g = G->g;
    t.mask = G->mask;
    t.scale = H->scale[l];
    t.wd = H->wd[l];
    t.u = H->u[l];
    t.f = (l == T) ? const_cast<double*>(fT) : H->f[l];
    t.r = H->r[l];
    t.ev = (l < L - 1) ? ev : nullptr;
    if (l < L - 1) ev += G->nel_local() * 24;
    for (int i = 0; i < 6; ++i) t.kc[i] = G->coef.kc[i];
    t.kd = G->coef.kd;
  }
  const int cs = g_tail_cluster;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(TAIL_THREADS);
  cfg.dynamicSmemBytes = TAIL_MAX_NL * sizeof(double);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  VT_CUDA(cudaLaunchKernelEx(&cfg, tail_vcycle_kernel, a));
  count_launch();
  return VT_OK;
}

}  // namespace vt
