// Homogenized geometric multigrid on B200 [ref: multigrid.py:84-499].
//
//  * restriction / prolongation reproduce the reference's separable axis
//    passes (z, then y, then x) operation for operation, so the transfers
//    are bit-identical to numpy [ref: multigrid.py:341-371, 433-459];
//  * coarse densities are the pairwise mean of the 8 children exactly as
//    numpy's mean(axis=1) rounds it [ref: multigrid.py:94-104, 209-215];
//  * the coarsest level is factored on the device (dense Cholesky) and
//    inverted once per refresh, so each V-cycle's coarse solve is one
//    deterministic dense mat-vec [ref: multigrid.py:280-316, 395-402].
#include <math.h>

#include <vector>

#include <atomic>

#include <stdlib.h>

#include "vt_internal.h"
#include "vt_pcg.cuh"

namespace vt {

constexpr int MG_THREADS = 256;
#ifndef VT_MG_R
#define VT_MG_R 6
#endif
constexpr int MG_R = VT_MG_R;  // rows in flight per thread in the transfer kernels
#ifndef VT_MG_CPS
#define VT_MG_CPS 8
#endif
constexpr int MG_CPS = VT_MG_CPS;  // transfer-kernel CTAs per SM (grid cap)

__device__ __forceinline__ bool node_coords(const Geom& g, long long t, int& p, int& j, int& i) {
  i = (int)(t % (g.nx + 1));
  const long long r = t / (g.nx + 1);
  j = (int)(r % (g.ny + 1));
  p = (int)(r / (g.ny + 1)) + g.pA;
  return true;
}
__device__ __forceinline__ long long owned_nodes(const Geom& g) {
  return (long long)(g.pB - g.pA) * (g.ny + 1) * (g.nx + 1);
}

// ---------------------------------------------------------------- SIMP scale

__global__ void scale_kernel(Geom g, const double* rho, double p, double kmin, double E,
                             double* scale, int* bad) {
  griddep_wait();
  const long long nel = (long long)g.nx * g.ny * (g.k1 - g.k0);
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % g.nx);
    const long long r = e / g.nx;
    const int j = (int)(r % g.ny);
    const int q = (int)(r / g.ny) + 1;
    const double x = rho[e];
    if (!(x >= 0.0 && x <= 1.0)) *bad = 1;
    // E * (kmin + r**p * (1 - kmin))  [ref: element.py:107, operator.py:142]
    const double s = __dmul_rn(E, __dadd_rn(kmin, __dmul_rn(simp_pow(x, p), 1.0 - kmin)));
    scale[elem_off(g, q, j, i)] = s;
  }
}

vt_status launch_scale(vt_grid* G, const double* rho, double p, double kmin, double E,
                       double* scale, int* bad, cudaStream_t s) {
  launch_pdl(scale_kernel, G->nsm * 8, MG_THREADS, 0, s, G->g, rho, p, kmin, E, scale, bad);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// ---------------------------------------------------------------- coarsening
// rho_c = mean of the 8 children, numpy pairwise order
__global__ void coarsen_rho_kernel(int fnx, int fny, int cnx, int cny, int cnz,
                                   const double* __restrict__ rf, double* __restrict__ rc) {
  griddep_wait();
  const long long nel = (long long)cnx * cny * cnz;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nel;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e % cnx);
    const long long r = e / cnx;
    const int j = (int)(r % cny);
    const int k = (int)(r / cny);
    double ch[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const long long fi = 2 * i + (c & 1), fj = 2 * j + ((c >> 1) & 1), fk = 2 * k + (c >> 2);
      ch[c] = rf[(fk * fny + fj) * fnx + fi];
    }
    const double s = __dadd_rn(__dadd_rn(__dadd_rn(ch[0], ch[1]), __dadd_rn(ch[2], ch[3])),
                               __dadd_rn(__dadd_rn(ch[4], ch[5]), __dadd_rn(ch[6], ch[7])));
    rc[e] = s / 8.0;
  }
}

// coarse dof fixed <=> coincident fine dof fixed [ref: multigrid.py:137-141]
__global__ void coarsen_mask_kernel(Geom gf, Geom gc, const uint8_t* mf, uint8_t* mc) {
  griddep_wait();
  const long long nn = owned_nodes(gc);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    int p, j, i;
    node_coords(gc, t, p, j, i);
    const int K = p - 1 + gc.k0;
    const int pf = 2 * K - gf.k0 + 1;
    mc[mask_off(gc, p, j, i)] = mf[mask_off(gf, pf, 2 * j, 2 * i)];
  }
}

__global__ void count_fixed_kernel(Geom g, const uint8_t* m, unsigned long long* out) {
  griddep_wait();
  const long long nn = owned_nodes(g);
  unsigned long long c = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    int p, j, i;
    node_coords(g, t, p, j, i);
    c += __popc((unsigned)m[mask_off(g, p, j, i)] & 7u);
  }
  atomicAdd(out, c);  // integer: order-independent
}

// ---------------------------------------------------------------- transfers
// f_c = P^T r_f, coarse fixed zeroed.  Per axis (z, y, x):
//   dst[i] = (src[2i] + 0.5 src[2i+1]) + 0.5 src[2i-1]   (missing terms skipped)
// Coarse node planes [kb, ke) (global); a z-slab of the fine level restricts
// into the planes whose centre fine plane 2K it owns (its ghost planes hold
// the neighbours' residual planes 2K0-1 and 2K1-1+1).
//
// A CTA takes a block of RJ coarse rows x RI coarse nodes of one coarse plane
// K.  Phase 1 streams the (2 RJ + 1) fine rows x (2 RI + 1) fine nodes of the
// three fine planes 2K, 2K+1, 2K-1 with coalesced row loads and keeps their
// z-pass combination in shared memory; phase 2 computes each coarse dof from
// 9 staged values (y pass, then x pass).  Every fine value is read from L2
// ~1.6 times (the plane 2K+1 is shared with K+1) instead of through 16-byte
// gathers at a 48-byte stride (3 L1 wavefronts per useful sector).  Same pass
// order and rounding as the reference: bit-identical.
constexpr int RJ_MAX = 8, RI_MAX = 42;  // 3 (2 RI + 1) <= 256 staged dofs per row: one per thread

struct RestrictBlk {
  int nJb, nIb, RI, RJ;  // blocks per plane in y / x, coarse nodes per x block, rows per block
};
// row blocks as tall as possible while the launch still has ~4 units per SM
// (small coarse levels would otherwise walk rows serially in a few CTAs)
static int transfer_rows(int planes, int rows, int nIb, int nsm) {
  int r = RJ_MAX;
  while (r > 1 && (long long)planes * ((rows + r - 1) / r) * nIb < 4LL * nsm) r /= 2;
  return r;
}
static RestrictBlk restrict_blocks(const Geom& gc, int kb, int ke, int nsm) {
  RestrictBlk b;
  b.nIb = (gc.nx + 1 + RI_MAX - 1) / RI_MAX;
  b.RI = (gc.nx + 1 + b.nIb - 1) / b.nIb;
  b.RJ = transfer_rows(ke - kb, gc.ny + 1, b.nIb, nsm);
  b.nJb = (gc.ny + 1 + b.RJ - 1) / b.RJ;
  return b;
}
static size_t restrict_smem(const RestrictBlk& b) { return (size_t)(2 * b.RJ + 1) * (2 * b.RI + 1) * 3 * sizeof(double); }

// Threads own row positions (a fine dof column of the staged block, then a
// coarse dof column) and walk the rows, so the index arithmetic is per column
// and every row step is one coalesced load per plane.
__global__ void __launch_bounds__(MG_THREADS)
    restrict_kernel(Geom gf, Geom gc, const uint8_t* __restrict__ mc, const double* __restrict__ rf,
                    double* __restrict__ fc, const int* stop, int kb, int ke, RestrictBlk blk) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  extern __shared__ double tzs[];  // [2 RJ + 1][3 (2 RI + 1)]
  const int W = 3 * (2 * blk.RI + 1);
  const long long units = (long long)(ke - kb) * blk.nJb * blk.nIb;
  const long long rowpitch = (long long)gf.rp * 3;
  for (long long unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int ib = (int)(unit % blk.nIb);
    const long long r0 = unit / blk.nIb;
    const int jb = (int)(r0 % blk.nJb);
    const int K = (int)(r0 / blk.nJb) + kb;
    const int J0 = jb * blk.RJ, I0 = ib * blk.RI;
    const int nJ = min(blk.RJ, gc.ny + 1 - J0), nI = min(blk.RI, gc.nx + 1 - I0);
    // staged fine rows y0 .. y0 + nrow - 1, clipped to [0, ny]
    const int y0 = 2 * J0 - 1;
    const int ya = max(y0, 0), yb = min(y0 + 2 * nJ + 1, gf.ny + 1);
    const bool ok1 = 2 * K + 1 <= gf.nz, ok2 = K >= 1;
    const double* pl0 = rf + node_off(gf, 2 * K - gf.k0 + 1, 0, 0) * 3;
    const double* pl1 = ok1 ? pl0 + gf.nplane : pl0;
    const double* pl2 = ok2 ? pl0 - gf.nplane : pl0;
    __syncthreads();
    // phase 1: z pass of the staged fine rows
    const int wn = 3 * (2 * nI + 1);
    for (int e = threadIdx.x; e < wn; e += blockDim.x) {
      const int xd = 3 * (2 * I0 - 1) + e;  // fine dof index within the row
      if (xd < 0 || xd >= 3 * (gf.nx + 1)) continue;
      for (int y = ya; y < yb; y += MG_R) {
        double a0[MG_R], a1[MG_R], a2[MG_R];
#pragma unroll
        for (int k = 0; k < MG_R; ++k) {
          if (y + k >= yb) break;
          const long long o = (y + k) * rowpitch + xd;
          a0[k] = pl0[o];
          a1[k] = pl1[o];
          a2[k] = pl2[o];
        }
#pragma unroll
        for (int k = 0; k < MG_R; ++k) {
          if (y + k >= yb) break;
          double v = a0[k];
          if (ok1) v = __dadd_rn(v, 0.5 * a1[k]);
          if (ok2) v = __dadd_rn(v, 0.5 * a2[k]);
          tzs[(y + k - y0) * W + e] = v;
        }
      }
    }
    __syncthreads();
    // phase 2: y pass then x pass per coarse dof
    const int p = K - gc.k0 + 1;
    const int cw = 3 * nI;
    for (int e = threadIdx.x; e < cw; e += blockDim.x) {
      const int ii = e / 3, c = e - 3 * ii;
      const int I = I0 + ii;
      const bool oki1 = 2 * I + 1 <= gf.nx, oki2 = I >= 1;
      double* out = fc + node_off(gc, p, J0, I) * 3 + c;
      const uint8_t* mrow = mc + mask_off(gc, p, J0, I);
#pragma unroll 2
      for (int jj = 0; jj < nJ; ++jj) {
        const int J = J0 + jj;
        const bool okj1 = 2 * J + 1 <= gf.ny, okj2 = J >= 1;
        // staged row of fine y = 2J + d is 2 jj + 1 + d; node x = 2I + d is 2 ii + 1 + d
        const double* rw = tzs + (2 * jj + 1) * W + 3 * (2 * ii + 1) + c;
        double ty[3];
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          const int dx = b == 0 ? 0 : (b == 1 ? 3 : -3);
          if ((b == 1 && !oki1) || (b == 2 && !oki2)) {
            ty[b] = 0.0;
            continue;
          }
          double v = rw[dx];
          if (okj1) v = __dadd_rn(v, 0.5 * rw[W + dx]);
          if (okj2) v = __dadd_rn(v, 0.5 * rw[-W + dx]);
          ty[b] = v;
        }
        double v = ty[0];
        if (oki1) v = __dadd_rn(v, 0.5 * ty[1]);
        if (oki2) v = __dadd_rn(v, 0.5 * ty[2]);
        const unsigned m = mrow[(long long)jj * gc.mp];
        out[(long long)jj * gc.rp * 3] = ((m >> c) & 1u) ? 0.0 : v;
      }
    }
  }
}

// ---- TMA-streamed restriction (large levels).  Same units and the same
// arithmetic as restrict_kernel (bit-identical), but each unit's three fine
// planes x (2 XR_RJ + 1) rows x (2 XR_RI + 1) nodes arrive by three TMA loads
// into a ring of XR_NS stages, issued XR_NS units ahead by one thread: the
// row walk of restrict_kernel waits on its own loads unit by unit (ncu:
// long-scoreboard + barrier stalls, ~3 TB/s); here the loads of the next
// units are in flight while this unit's z / y / x passes run.
#ifndef VT_XR_NS
#define VT_XR_NS 2
#endif
#ifndef VT_XR_RJ
#define VT_XR_RJ 4
#endif
constexpr int XR_RI = 33, XR_RJ = VT_XR_RJ, XR_NS = VT_XR_NS;
constexpr int XR_IT = (XR_RJ * 3 * XR_RI + MG_THREADS - 1) / MG_THREADS;  // phase-2 items per thread
constexpr int XR_W = 3 * (2 * XR_RI + 1);      // fine dofs of a staged row (201)
constexpr int XR_BW = XR_W + 1;                // TMA box width (even start one dof early)
constexpr int XR_BR = 2 * XR_RJ + 1;           // staged fine rows
constexpr int XR_PLANE_B = ((XR_BW * XR_BR * 8 + 127) / 128) * 128;
constexpr int XR_STAGE_B = 3 * XR_PLANE_B;
constexpr int XR_SMEM = XR_NS * XR_STAGE_B + XR_BR * XR_W * 8 + XR_NS * 8 + 128;
constexpr int XR_CPS = (220 * 1024) / XR_SMEM < 4 ? (220 * 1024) / XR_SMEM : 4;  // resident CTAs per SM

struct XrUnits {
  int kb, ke, nJb, nIb;
};

__device__ __forceinline__ void xr_issue(const CUtensorMap* m, const Geom& gf, const XrUnits& U, long long unit,
                                         unsigned char* stage, uint64_t* bar) {
  const int ib = (int)(unit % U.nIb);
  const long long r0 = unit / U.nIb;
  const int jb = (int)(r0 % U.nJb);
  const int K = (int)(r0 / U.nJb) + U.kb;
  const int x0 = 3 * (2 * ib * XR_RI - 1) - 1;  // one dof early: even (16-byte) start
  const int y0 = 2 * jb * XR_RJ - 1;
  const int p0 = 2 * K - gf.k0 + 1;
  mbar_expect_tx(bar, 3 * XR_BW * XR_BR * 8);
  tma_load_3d(stage, m, bar, x0, y0, p0);                        // plane 2K
  tma_load_3d(stage + XR_PLANE_B, m, bar, x0, y0, p0 + 1);       // plane 2K + 1
  tma_load_3d(stage + 2 * XR_PLANE_B, m, bar, x0, y0, p0 - 1);   // plane 2K - 1
}

__global__ void __launch_bounds__(MG_THREADS)
    restrict_tma_kernel(const __grid_constant__ CUtensorMap mf, Geom gf, Geom gc, const uint8_t* __restrict__ mc,
                        double* __restrict__ fc, const int* stop, XrUnits U) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  extern __shared__ __align__(128) unsigned char xsm[];
  double* tzs = reinterpret_cast<double*>(xsm + XR_NS * XR_STAGE_B);
  uint64_t* bars = reinterpret_cast<uint64_t*>(tzs + XR_BR * XR_W);
  const long long units = (long long)(U.ke - U.kb) * U.nJb * U.nIb;
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&mf);
    for (int i = 0; i < XR_NS; ++i) mbar_init(&bars[i], 1);
    mbar_fence_init();
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int i = 0; i < XR_NS; ++i) {
      const long long u = blockIdx.x + (long long)i * gridDim.x;
      if (u < units) xr_issue(&mf, gf, U, u, xsm + i * XR_STAGE_B, &bars[i]);
    }
  int it = 0;
  for (long long unit = blockIdx.x; unit < units; unit += gridDim.x, ++it) {
    const int slot = it % XR_NS;
    const int ib = (int)(unit % U.nIb);
    const long long r0 = unit / U.nIb;
    const int jb = (int)(r0 % U.nJb);
    const int K = (int)(r0 / U.nJb) + U.kb;
    const int J0 = jb * XR_RJ, I0 = ib * XR_RI;
    const int nJ = min(XR_RJ, gc.ny + 1 - J0), nI = min(XR_RI, gc.nx + 1 - I0);
    const bool ok1 = 2 * K + 1 <= gf.nz, ok2 = K >= 1;
    const int p = K - gc.k0 + 1;
    const int cw = 3 * nI, nit = nJ * cw;
    // phase-2 items of this thread (at most XR_IT): their coarse masks are
    // loaded now, so the global-load latency overlaps the wait and phase 1
    unsigned mk[XR_IT];
#pragma unroll
    for (int q = 0; q < XR_IT; ++q) {
      const int t = threadIdx.x + q * MG_THREADS;
      mk[q] = 0;
      if (t < nit) {
        const int jj = t / cw, e = t - jj * cw;
        mk[q] = mc[mask_off(gc, p, J0 + jj, I0 + e / 3)];
      }
    }
    mbar_wait(&bars[slot], (uint32_t)((it / XR_NS) & 1));
    const double* st = reinterpret_cast<const double*>(xsm + slot * XR_STAGE_B);
    const double* s1 = st + XR_PLANE_B / 8;
    const double* s2 = st + 2 * XR_PLANE_B / 8;
    // phase 1: z pass of the staged rows (out-of-grid rows / dofs arrive as 0 and are never read)
    for (int e = threadIdx.x; e < XR_BR * XR_W; e += blockDim.x) {
      const int r = e / XR_W, c = e - r * XR_W;
      const int o = r * XR_BW + c + 1;
      double v = st[o];
      if (ok1) v = __dadd_rn(v, 0.5 * s1[o]);
      if (ok2) v = __dadd_rn(v, 0.5 * s2[o]);
      tzs[e] = v;
    }
    __syncthreads();
    // the stage is free: refill it XR_NS units ahead
    if (threadIdx.x == 0) {
      const long long nu = unit + (long long)XR_NS * gridDim.x;
      if (nu < units) xr_issue(&mf, gf, U, nu, xsm + slot * XR_STAGE_B, &bars[slot]);
    }
    // phase 2: y pass then x pass per coarse dof (restrict_kernel's arithmetic),
    // every (row, dof) of the unit an independent item
#pragma unroll
    for (int q = 0; q < XR_IT; ++q) {
      const int t = threadIdx.x + q * MG_THREADS;
      if (t >= nit) break;
      const int jj = t / cw, e = t - jj * cw;
      const int ii = e / 3, c = e - 3 * ii;
      const int I = I0 + ii, J = J0 + jj;
      const bool oki1 = 2 * I + 1 <= gf.nx, oki2 = I >= 1;
      const bool okj1 = 2 * J + 1 <= gf.ny, okj2 = J >= 1;
      const double* rw = tzs + (2 * jj + 1) * XR_W + 3 * (2 * ii + 1) + c;
      double ty[3];
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int dx = b == 0 ? 0 : (b == 1 ? 3 : -3);
        if ((b == 1 && !oki1) || (b == 2 && !oki2)) {
          ty[b] = 0.0;
          continue;
        }
        double v = rw[dx];
        if (okj1) v = __dadd_rn(v, 0.5 * rw[XR_W + dx]);
        if (okj2) v = __dadd_rn(v, 0.5 * rw[-XR_W + dx]);
        ty[b] = v;
      }
      double v = ty[0];
      if (oki1) v = __dadd_rn(v, 0.5 * ty[1]);
      if (oki2) v = __dadd_rn(v, 0.5 * ty[2]);
      fc[node_off(gc, p, J, I) * 3 + c] = ((mk[q] >> c) & 1u) ? 0.0 : v;
    }
    __syncthreads();  // tzs is rewritten by the next unit
  }
}

static bool g_xr_tma = true;  // VT_XR_TMA=0: always the row-walk kernel (A/B)

// kb < 0: every coarse plane the coarse grid owns
vt_status launch_restrict(vt_grid* F, vt_grid* C, const double* rf, double* fc, const int* stop,
                          int kb, int ke, cudaStream_t s) {
  if (kb < 0) {
    kb = C->g.k0;
    ke = C->g.k1 + C->g.last;
  }
  if (ke <= kb) return VT_OK;
  // large fine levels: the TMA-streamed kernel (one CTA per 8 fine dof rows
  // of staging is not worth it below ~1M fine dofs)
  static int xr_env = -1;
  if (xr_env < 0) {
    const char* e = getenv("VT_XR_TMA");
    xr_env = e ? atoi(e) : 1;
    g_xr_tma = xr_env != 0;
  }
  if (g_xr_tma && (long long)F->g.nplane * (F->g.pB - F->g.pA) >= (1LL << 20)) {
    const CUtensorMap* m = xfer_map(F, rf, XR_BW, XR_BR);
    if (m) {
      static bool attr = false;
      if (!attr) {
        VT_CUDA(cudaFuncSetAttribute(restrict_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, XR_SMEM));
        attr = true;
      }
      XrUnits U{kb, ke, (C->g.ny + 1 + XR_RJ - 1) / XR_RJ, (C->g.nx + 1 + XR_RI - 1) / XR_RI};
      const long long units = (long long)(ke - kb) * U.nJb * U.nIb;
      const CUtensorMap mv = *m;
      launch_pdl(restrict_tma_kernel, fit_grid(units, 1, C->nsm * XR_CPS), MG_THREADS, XR_SMEM, s,
                 mv, F->g, C->g, (const uint8_t*)C->mask, fc, stop, U);
      count_launch();
      VT_CUDA(cudaGetLastError());
      return VT_OK;
    }
  }
  const RestrictBlk blk = restrict_blocks(C->g, kb, ke, C->nsm);
  const size_t sm = restrict_smem(blk);
  static bool attr = false;
  if (!attr) {
    VT_CUDA(cudaFuncSetAttribute(restrict_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)((2 * RJ_MAX + 1) * (2 * RI_MAX + 1) * 3 * sizeof(double))));
    attr = true;
  }
  const long long units = (long long)(ke - kb) * blk.nJb * blk.nIb;
  launch_pdl(restrict_kernel, fit_grid(units, 1, C->nsm * MG_CPS), MG_THREADS, sm, s, F->g, C->g,
             (const uint8_t*)C->mask, rf, fc, stop, kb, ke, blk);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// u_f (+)= P u_c with fine fixed dofs zeroed in P u_c.  Per axis (z, y, x):
//   even: dst = src[i/2];  odd: dst = 0.5 * (src[(i-1)/2] + src[(i+1)/2])
// A CTA takes a block of PJ coarse rows x PI coarse nodes of one coarse plane
// K: it stages the coarse values of planes K, K+1, rows J0..J0+PJ, nodes
// I0..I0+PI in shared memory, then updates the fine dofs of planes 2K, 2K+1,
// rows 2J0.., nodes 2I0..  A thread owns one fine dof column and walks the
// coarse rows: the z pass of coarse row jy+1 is formed once and serves fine
// rows 2jy (even) and 2jy+1 (odd, with row jy's carried value); every global
// access is contiguous along the row, read-modify-writes batched.  Same
// z -> y -> x pass order and rounding as the reference: bit-identical.  A
// slab produces exactly the fine planes it owns.
constexpr int PJ_MAX = 8, PI_MAX = 42;  // 6 PI <= 256 fine dofs per row: one per thread
#ifndef VT_PR_B
#define VT_PR_B 4
#endif
constexpr int PR_B = VT_PR_B;  // coarse rows (2 PR_B fine rows) per batch of read-modify-writes

struct ProlongBlk {
  int K0, K1;            // coarse planes covering the fine slab's owned planes
  int nJb, nIb, PI, PJ;  // blocks per plane in y / x, coarse nodes per x block, rows per block
};
static ProlongBlk prolong_blocks(const Geom& gc, const Geom& gf, int nsm) {
  ProlongBlk b;
  const int fk0 = gf.k0 + gf.pA - 1, fk1 = gf.k0 + gf.pB - 1;
  b.K0 = fk0 >> 1;
  b.K1 = ((fk1 - 1) >> 1) + 1;
  b.nIb = (gc.nx + 1 + PI_MAX - 1) / PI_MAX;
  b.PI = (gc.nx + 1 + b.nIb - 1) / b.nIb;
  b.PJ = transfer_rows(b.K1 - b.K0, gc.ny + 1, b.nIb, nsm);
  b.nJb = (gc.ny + 1 + b.PJ - 1) / b.PJ;
  return b;
}
static size_t prolong_smem(const ProlongBlk& b) { return (size_t)2 * (b.PJ + 1) * (b.PI + 1) * 3 * sizeof(double); }

template <bool ADD>
__global__ void __launch_bounds__(MG_THREADS)
    prolong_kernel(Geom gc, Geom gf, const uint8_t* __restrict__ mf, const double* __restrict__ uc,
                   double* __restrict__ uf, const int* stop, ProlongBlk blk) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  extern __shared__ double sc[];  // [kz 2][PJ + 1][3 (PI + 1)]
  const int fk0 = gf.k0 + gf.pA - 1, fk1 = gf.k0 + gf.pB - 1;
  const int SW = 3 * (blk.PI + 1), SP = (blk.PJ + 1) * SW;
  const long long units = (long long)(blk.K1 - blk.K0) * blk.nJb * blk.nIb;
  const long long rowpitch = (long long)gf.rp * 3;
  for (long long unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int ib = (int)(unit % blk.nIb);
    const long long r0 = unit / blk.nIb;
    const int jb = (int)(r0 % blk.nJb);
    const int K = (int)(r0 / blk.nJb) + blk.K0;
    const int J0 = jb * blk.PJ, I0 = ib * blk.PI;
    const int nJ = min(blk.PJ, gc.ny + 1 - J0), nI = min(blk.PI, gc.nx + 1 - I0);
    // staged coarse rows J0..J0+nJ, nodes I0..I0+nI (clipped to the grid)
    const int sJ = min(nJ + 1, gc.ny + 1 - J0), sw = 3 * min(nI + 1, gc.nx + 1 - I0);
    const int Kp = K + 1 <= gc.nz ? K + 1 : K;
    __syncthreads();
    for (int t = threadIdx.x; t < 2 * sJ * sw; t += blockDim.x) {
      const int r = t / sw, e = t - r * sw;
      const int kz = r / sJ, jj = r - kz * sJ;
      sc[kz * SP + jj * SW + e] = uc[node_off(gc, (kz ? Kp : K) - gc.k0 + 1, J0 + jj, I0) * 3 + e];
    }
    __syncthreads();
    // fine planes 2K + cz (owned), rows 2 J0 + ry (<= ny), dofs 3 (2 I0) + e
    const int fy0 = 2 * J0, fx0 = 2 * I0;
    const int nfy = min(2 * nJ, gf.ny + 1 - fy0), nfx = min(2 * nI, gf.nx + 1 - fx0);
    const int czb = (2 * K >= fk0) ? 0 : 1;
    const int cze = (2 * K + 1 < fk1 && 2 * K + 1 <= gf.nz) ? 2 : 1;
    for (int e = threadIdx.x; e < 3 * nfx; e += blockDim.x) {
      const int ix = e / 3, comp = e - 3 * ix;
      const bool ox = ix & 1;
      const double* col = sc + 3 * (ix >> 1) + comp;
      for (int cz = czb; cz < cze; ++cz) {
        const int pf = 2 * K + cz - gf.k0 + 1;
        double* urow = uf + node_off(gf, pf, fy0, fx0) * 3 + e;
        const uint8_t* mrow = mf + mask_off(gf, pf, fy0, fx0 + ix);
        // z pass of coarse row jy at x offsets 0 and +1 (the latter for odd columns)
        auto zrow = [&](int jy, double& z0, double& z1) {
          const double* q = col + jy * SW;
          z0 = cz ? 0.5 * __dadd_rn(q[0], q[SP]) : q[0];
          z1 = ox ? (cz ? 0.5 * __dadd_rn(q[3], q[SP + 3]) : q[3]) : 0.0;
        };
        double za0, za1;  // row jy (carried)
        zrow(0, za0, za1);
        for (int jy0 = 0; 2 * jy0 < nfy; jy0 += PR_B) {
          double old[2 * PR_B];
          unsigned mk[2 * PR_B];
#pragma unroll
          for (int k = 0; k < 2 * PR_B; ++k) {
            const int ry = 2 * jy0 + k;
            if (ry >= nfy) break;
            old[k] = ADD ? urow[ry * rowpitch] : 0.0;
            mk[k] = mrow[(long long)ry * gf.mp];
          }
#pragma unroll
          for (int k = 0; k < PR_B; ++k) {
            const int jy = jy0 + k;
            if (2 * jy >= nfy) break;
            // even fine row 2 jy: y = z(jy)
            double v = ox ? 0.5 * __dadd_rn(za0, za1) : za0;
            if ((mk[2 * k] >> comp) & 1u) v = 0.0;
            urow[(2 * jy) * rowpitch] = ADD ? __dadd_rn(old[2 * k], v) : v;
            if (2 * jy + 1 >= nfy) break;
            // odd fine row 2 jy + 1: y = 0.5 (z(jy) + z(jy + 1))
            double zb0, zb1;
            zrow(jy + 1, zb0, zb1);
            const double y0 = 0.5 * __dadd_rn(za0, zb0);
            v = ox ? 0.5 * __dadd_rn(y0, 0.5 * __dadd_rn(za1, zb1)) : y0;
            if ((mk[2 * k + 1] >> comp) & 1u) v = 0.0;
            urow[(2 * jy + 1) * rowpitch] = ADD ? __dadd_rn(old[2 * k + 1], v) : v;
            za0 = zb0;
            za1 = zb1;
          }
        }
      }
    }
  }
}

// one CTA per coarse (plane, row block, node block) unit covering the fine slab's owned planes
static int prolong_grid(const ProlongBlk& b, int cap) {  // (cap: CTAs)
  return fit_grid((long long)(b.K1 - b.K0) * b.nJb * b.nIb, 1, cap);
}

vt_status launch_prolong_add(vt_grid* C, vt_grid* F, const double* uc, double* uf,
                             const int* stop, cudaStream_t s) {
  const ProlongBlk b = prolong_blocks(C->g, F->g, F->nsm);
  launch_pdl(prolong_kernel<true>, prolong_grid(b, F->nsm * MG_CPS), MG_THREADS, prolong_smem(b), s, C->g,
             F->g, (const uint8_t*)F->mask, uc, uf, stop, b);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status launch_prolong_set(vt_grid* C, vt_grid* F, const double* uc, double* uf, const int* stop,
                             cudaStream_t s) {
  const ProlongBlk b = prolong_blocks(C->g, F->g, F->nsm);
  launch_pdl(prolong_kernel<false>, prolong_grid(b, F->nsm * MG_CPS), MG_THREADS, prolong_smem(b), s, C->g,
             F->g, (const uint8_t*)F->mask, uc, uf, stop, b);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status launch_coarsen_mask(vt_grid* F, vt_grid* C, cudaStream_t s) {
  launch_pdl(coarsen_mask_kernel, C->nsm * 4, MG_THREADS, 0, s, F->g, C->g, F->mask, C->mask);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

vt_status launch_coarsen_rho(vt_grid* F, vt_grid* C, const double* rf, double* rc, cudaStream_t s) {
  launch_pdl(coarsen_rho_kernel, C->nsm * 4, MG_THREADS, 0, s, F->g.nx, F->g.ny, C->g.nx, C->g.ny,
                                                      C->g.k1 - C->g.k0, rf, rc);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// ---------------------------------------------------------------- coarsest level
// Dense assembly (identity on fixed), in-place Cholesky; one CTA.
// [ref: multigrid.py:280-316]
__global__ void __launch_bounds__(1024, 1)
    coarse_factor_kernel(Geom g, const double* scale, const double* k0l, const double* mats,
                         const uint8_t* mask, int n, double* A, double* A0, int* status) {
  griddep_wait();
  const int nx1 = g.nx + 1, ny1 = g.ny + 1;
  for (long long t = threadIdx.x; t < (long long)n * n; t += blockDim.x) A[t] = 0.0;
  __syncthreads();
  const int nel = g.nx * g.ny * g.nz;
  for (int e = 0; e < nel; ++e) {
    const int i = e % g.nx, j = (e / g.nx) % g.ny, k = e / (g.nx * g.ny);
    const double s = mats ? 0.0 : scale[elem_off(g, k + 1, j, i)];
    for (int t = threadIdx.x; t < 576; t += blockDim.x) {
      const int a = t / 24, b = t % 24;
      const int ca = a / 3, cb = b / 3;
      const int na = (i + (ca & 1)) + (j + ((ca >> 1) & 1)) * nx1 + (k + (ca >> 2)) * nx1 * ny1;
      const int nb = (i + (cb & 1)) + (j + ((cb >> 1) & 1)) * nx1 + (k + (cb >> 2)) * nx1 * ny1;
      const int da = 3 * na + a % 3, db = 3 * nb + b % 3;
      A[(long long)da * n + db] += mats ? mats[(long long)e * GAL_PACK + gal_sym(a, b)] : s * k0l[t];
    }
    __syncthreads();
  }
  // identity rows / columns on fixed dofs
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    const int node = d / 3, c = d % 3;
    const int i = node % nx1, j = (node / nx1) % ny1, k = node / (nx1 * ny1);
    if ((mask[mask_off(g, k + 1, j, i)] >> c) & 1u) {
      for (int e = 0; e < n; ++e) A[(long long)d * n + e] = 0.0;
    }
  }
  __syncthreads();
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    for (int e = 0; e < n; ++e) {
      const int node = e / 3, c = e % 3;
      const int i = node % nx1, j = (node / nx1) % ny1, k = node / (nx1 * ny1);
      if ((mask[mask_off(g, k + 1, j, i)] >> c) & 1u) A[(long long)d * n + e] = (d == e) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  for (long long t = threadIdx.x; t < (long long)n * n; t += blockDim.x) A0[t] = A[t];
  // right-looking Cholesky, lower triangle
  __shared__ double piv;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int j = 0; j < n; ++j) {
    if (threadIdx.x == 0) {
      const double d = A[(long long)j * n + j];
      if (!(d > 0.0) || !isfinite(d)) {
        bad = 1;
        piv = 1.0;
      } else {
        piv = sqrt(d);
      }
      A[(long long)j * n + j] = piv;
    }
    __syncthreads();
    if (bad) break;
    const double lj = piv;
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) A[(long long)i * n + j] /= lj;
    __syncthreads();
    const long long m = n - j - 1;
    for (long long t = threadIdx.x; t < m * m; t += blockDim.x) {
      const int ii = j + 1 + (int)(t / m), kk = j + 1 + (int)(t % m);
      if (kk <= ii) A[(long long)ii * n + kk] -= A[(long long)ii * n + j] * A[(long long)kk * n + j];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *status = bad;
}

// Small coarsest systems (n^2 doubles fit in shared memory: n <= 160, e.g.
// 135 dofs at cfg2/cfg3): assembly, Cholesky, in-place triangular inverse
// and Kinv = L^-T L^-1 in ONE CTA entirely in shared memory -- the global-
// memory version pays a memory round trip on every one of its ~3n dependent
// steps (0.85 ms per refresh at cfg2).  Same assembly order and the same
// right-looking Cholesky recurrence; the inverse follows LAPACK dtrti2
// (lower, non-unit).  A0 (the assembled matrix) goes to global for the
// refinement step of the coarse solve.
constexpr int COARSE_SMEM_N = 160;
__global__ void __launch_bounds__(1024, 1)
    coarse_factor_smem_kernel(Geom g, const double* scale, const double* k0l, const double* mats,
                              const uint8_t* mask, int n, double* A0, double* Kinv, int* status) {
  griddep_wait();
  extern __shared__ double As[];  // n x n, then n scratch
  double* tmp = As + (size_t)n * n;
  const int nx1 = g.nx + 1, ny1 = g.ny + 1;
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) As[t] = 0.0;
  __syncthreads();
  const int nel = g.nx * g.ny * g.nz;
  for (int e = 0; e < nel; ++e) {
    const int i = e % g.nx, j = (e / g.nx) % g.ny, k = e / (g.nx * g.ny);
    const double sc = mats ? 0.0 : scale[elem_off(g, k + 1, j, i)];
    for (int t = threadIdx.x; t < 576; t += blockDim.x) {
      const int a = t / 24, b = t % 24;
      const int ca = a / 3, cb = b / 3;
      const int na = (i + (ca & 1)) + (j + ((ca >> 1) & 1)) * nx1 + (k + (ca >> 2)) * nx1 * ny1;
      const int nb = (i + (cb & 1)) + (j + ((cb >> 1) & 1)) * nx1 + (k + (cb >> 2)) * nx1 * ny1;
      As[(3 * na + a % 3) * n + 3 * nb + b % 3] += mats ? mats[(long long)e * GAL_PACK + gal_sym(a, b)] : sc * k0l[t];
    }
    __syncthreads();
  }
  // identity rows / columns on fixed dofs
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    const int node = d / 3, c = d % 3;
    const int i = node % nx1, j = (node / nx1) % ny1, k = node / (nx1 * ny1);
    tmp[d] = ((mask[mask_off(g, k + 1, j, i)] >> c) & 1u) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int r = t / n, c = t % n;
    if (tmp[r] != 0.0 || tmp[c] != 0.0) As[t] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) A0[t] = As[t];
  // right-looking Cholesky, lower triangle
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    const double d = As[j * n + j];
    const double piv = (d > 0.0 && isfinite(d)) ? sqrt(d) : 1.0;
    if (!(d > 0.0) || !isfinite(d)) {
      if (threadIdx.x == 0) bad = 1;
    }
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) As[i * n + j] /= piv;
    __syncthreads();
    if (threadIdx.x == 0) As[j * n + j] = piv;
    const int m = n - j - 1;
    for (int t = threadIdx.x; t < m * m; t += blockDim.x) {
      const int ii = j + 1 + t / m, kk = j + 1 + t % m;
      if (kk <= ii) As[ii * n + kk] -= As[ii * n + j] * As[kk * n + j];
    }
    __syncthreads();
  }
  if (bad) {
    if (threadIdx.x == 0) *status = 1;
    return;
  }
  // in-place inverse of the lower-triangular factor (LAPACK dtrti2, 'L', 'N')
  for (int j = n - 1; j >= 0; --j) {
    const double ajj = -1.0 / As[j * n + j];
    // tmp = T x with T the inverted trailing block, x = column j below the diagonal
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double acc = 0.0;
      for (int k = j + 1; k <= i; ++k) acc = fma(As[i * n + k], As[k * n + j], acc);
      tmp[i] = acc;
    }
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) As[i * n + j] = ajj * tmp[i];
    if (threadIdx.x == 0) As[j * n + j] = -ajj;
    __syncthreads();
  }
  // Kinv = W^T W with W = L^-1 (lower): Kinv[i][j] = sum_{k >= max(i,j)} W[k][i] W[k][j]
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int i = t / n, j = t % n;
    double acc = 0.0;
    for (int k = max(i, j); k < n; ++k) acc = fma(As[k * n + i], As[k * n + j], acc);
    Kinv[t] = acc;
  }
  if (threadIdx.x == 0) *status = 0;
}

// W = L^{-1}: one thread per column
__global__ void tri_inverse_kernel(int n, const double* A, double* W) {
  griddep_wait();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  for (int i = 0; i < c; ++i) W[(long long)i * n + c] = 0.0;
  for (int i = c; i < n; ++i) {
    double s = (i == c) ? 1.0 : 0.0;
    for (int k = c; k < i; ++k) s -= A[(long long)i * n + k] * W[(long long)k * n + c];
    W[(long long)i * n + c] = s / A[(long long)i * n + i];
  }
}

// Kinv = W^T W
__global__ void gram_kernel(int n, const double* W, double* Kinv) {
  griddep_wait();
  const long long nn = (long long)n * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < nn;
       t += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(t / n), j = (int)(t % n);
    double s = 0.0;
    for (int k = max(i, j); k < n; ++k) s = fma(W[(long long)k * n + i], W[(long long)k * n + j], s);
    Kinv[t] = s;
  }
}

// Coarsest solve u = A^{-1} f [ref: multigrid.py:395-402, cho_solve].  The
// explicit inverse alone (one mat-vec) is not accurate enough: its error is
// relative to |A^{-1}|, which at SIMP contrasts (kmin = 1e-9) perturbs the
// preconditioner far more than LAPACK's backward-stable dpotrs does (measured:
// 3e-5 vs 2e-7 compliance drift over the 40 cfg1 iterations).  One step of
// iterative refinement with the assembled matrix, x = x0 + Kinv (f - A x0),
// restores backward stability at the cost of two more dense mat-vecs:
//   mode 0: fc = gather(f); x0 = Kinv fc          (fc, x0 -> dense scratch)
//   mode 1: r  = fc - A x0                        (dense scratch)
//   mode 2: u  = scatter(x0 + Kinv r), fixed -> 0 (vt layout)
// One warp per row: lane-strided FMAs then the xor tree (fixed order).
__device__ __forceinline__ void coarse_node(const Geom& g, int d, long long* nd, int* c, int* fixed,
                                            const uint8_t* mask) {
  const int nx1 = g.nx + 1, ny1 = g.ny + 1;
  const int node = d / 3;
  *c = d % 3;
  const int i = node % nx1, j = (node / nx1) % ny1, k = node / (nx1 * ny1);
  *nd = node_off(g, k + 1, j, i);
  if (fixed) *fixed = (mask[mask_off(g, k + 1, j, i)] >> *c) & 1u;
}

template <int MODE>
__global__ void coarse_mv_kernel(Geom g, const uint8_t* mask, int n, const double* M,
                                 const double* f, double* cf, double* x0, double* cr, double* u,
                                 const int* stop) {
  griddep_wait();
  if (stop && *(volatile const int*)stop) return;
  extern __shared__ double vs[];
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    double v;
    if (MODE == 0) {
      long long nd;
      int c;
      coarse_node(g, d, &nd, &c, nullptr, mask);
      v = f[nd * 3 + c];
      if (blockIdx.x == 0) cf[d] = v;
    } else {
      v = (MODE == 1) ? x0[d] : cr[d];
    }
    vs[d] = v;
  }
  __syncthreads();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int r = blockIdx.x * nw + warp; r < n; r += gridDim.x * nw) {
    double s = 0.0;
    for (int e = lane; e < n; e += 32) s = fma(M[(long long)r * n + e], vs[e], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (MODE == 0) {
        x0[r] = s;
      } else if (MODE == 1) {
        cr[r] = cf[r] - s;
      } else {
        long long nd;
        int c, fx;
        coarse_node(g, r, &nd, &c, &fx, mask);
        u[nd * 3 + c] = fx ? 0.0 : x0[r] + s;
      }
    }
  }
}

}  // namespace vt

// (struct vt_hier lives in vt_internal.h)

namespace vt {

vt_status hier_alloc_vec(vt_grid* G, double** p) {
  VT_CUDA(cudaMalloc(p, G->vec_len() * sizeof(double)));
  VT_CUDA(cudaMemset(*p, 0, G->vec_len() * sizeof(double)));
  return VT_OK;
}


// coarsest solve with one refinement step (3 launches, capturable)
vt_status launch_coarse_solve(vt_hier* H, const double* f, double* u, const int* stop,
                              cudaStream_t s) {
  vt_grid* G = H->lv.back();
  const int n = H->nL;
  const size_t sm = (size_t)n * sizeof(double);
  const int grid = (n + 7) / 8;  // one warp per row, 8 warps per CTA
  double *cf = H->cvec, *x0 = H->cvec + n, *cr = H->cvec + 2 * n;
  launch_pdl(coarse_mv_kernel<0>, grid, 256, sm, s, G->g, G->mask, n, H->Kinv, f, cf, x0, cr, u, stop);
  launch_pdl(coarse_mv_kernel<1>, grid, 256, sm, s, G->g, G->mask, n, H->A0, f, cf, x0, cr, u, stop);
  launch_pdl(coarse_mv_kernel<2>, grid, 256, sm, s, G->g, G->mask, n, H->Kinv, f, cf, x0, cr, u, stop);
  count_launch(3);
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// Build the level sequence of one V-cycle on `s` (capturable), entered at
// level `top` with right-hand side f0 (top > 0: the replicated coarse tail of a
// z-slab hierarchy, whose level-`top` residual the slabs restricted into
// H->f[top]; see dist.cu).
// fused_j0: the PCG control block when pcg_update already wrote the level-0
// first Jacobi sweep into H->u[0] (see pcg_update_kernel)
vt_status hier_vcycle_launch(vt_hier* H, const double* f0, const int* stop, double* rz_partial,
                             bool want_rz, cudaStream_t s, const double** z_out, int top,
                             const PcgCtl* fused_j0) {
  const int L = (int)H->lv.size();
  std::vector<const double*> fl(L);
  std::vector<double*> ucur(L);
  for (int l = 1; l < L; ++l) fl[l] = H->f[l];
  fl[top] = f0;
  const auto gal = [&](int l) { return H->scheme == 1 && l >= 1; };  // stored-matrix level
  auto smooth = [&](int l, bool dot) -> vt_status {
    vt_grid* G = H->lv[l];
    double* dst = (ucur[l] == H->u[l]) ? H->u2[l] : H->u[l];
    if (gal(l)) {
      VT_TRY(gal_level_op(H, l, 2, ucur[l], fl[l], dst, stop, s));
    } else {
      VT_TRY(launch_hex8(G, H8_SMOOTH, dot, H->scale[l], ucur[l], nullptr, fl[l], dst, H->omega,
                         rz_partial, stop, s));
    }
    ucur[l] = dst;
    return VT_OK;
  };
  // levels >= t run as one fused cluster kernel (tail.cu); t == L: none
  const int t = hier_tail_start(H, top);
  for (int l = top; l < L - 1 && l < t; ++l) {
    vt_grid* G = H->lv[l];
    ucur[l] = H->u[l];
    if (H->sweeps >= 1) {
      if (gal(l))
        VT_TRY(gal_jacobi0(H, l, fl[l], H->u[l], stop, s));
      else
        VT_TRY(launch_jacobi0w(G, H->wd[l], fl[l], H->u[l], stop, s, l == 0 ? fused_j0 : nullptr));
      for (int k = 1; k < H->sweeps; ++k) VT_TRY(smooth(l, false));
      if (gal(l))
        VT_TRY(gal_level_op(H, l, 1, ucur[l], fl[l], H->r[l], stop, s));
      else
        VT_TRY(launch_hex8(G, H8_RESID, false, H->scale[l], ucur[l], ucur[l], fl[l], H->r[l], 0.0,
                           nullptr, stop, s));
      VT_TRY(launch_restrict(G, H->lv[l + 1], H->r[l], H->f[l + 1], stop, -1, -1, s));
    } else {
      VT_TRY(launch_zero_owned(G, H->u[l], s));
      VT_TRY(launch_restrict(G, H->lv[l + 1], fl[l], H->f[l + 1], stop, -1, -1, s));
    }
  }
  if (t < L) {
    const double* zt = nullptr;
    VT_TRY(launch_tail(H, t, fl[t], stop, s, &zt));
    ucur[t] = const_cast<double*>(zt);
  } else {
    VT_TRY(launch_coarse_solve(H, fl[L - 1], H->u[L - 1], stop, s));
    ucur[L - 1] = H->u[L - 1];
  }
  for (int l = std::min(L - 2, t - 1); l >= top; --l) {
    vt_grid* G = H->lv[l];
    VT_TRY(launch_prolong_add(H->lv[l + 1], G, ucur[l + 1], ucur[l], stop, s));
    for (int k = 0; k < H->sweeps; ++k) VT_TRY(smooth(l, want_rz && l == 0 && k == H->sweeps - 1));
  }
  *z_out = ucur[top];
  if (top == 0) H->last_z = ucur[0];
  return VT_OK;
}

// number of partials the V-cycle's rz dot leaves (0 if it cannot fuse it)
int hier_rz_parts(vt_hier* H) {
  if (H->lv.size() < 2 || H->sweeps < 1) return 0;
  return H->lv[0]->h8.grid;
}

}  // namespace vt

using namespace vt;

extern "C" {

vt_status vt_hier_create(vt_hier** out, vt_grid* fine, int n_levels, double omega, int sweeps) {
  return vt_hier_create_ex(out, fine, n_levels, omega, sweeps, 0);
}

vt_status vt_hier_create_ex(vt_hier** out, vt_grid* fine, int n_levels, double omega, int sweeps,
                            int scheme) {
  if (scheme != 0 && scheme != 1) return fail(VT_EINVAL, "scheme must be 0 (homogenized) or 1 (galerkin)");
  if (!out || !fine) return fail(VT_EINVAL, "null argument");
  if (n_levels < 1) return fail(VT_EINVAL, "max_levels must be at least 1");
  if (!(omega > 0.0 && omega <= 1.0))
    return fail(VT_EINVAL, "jacobi damping must lie in (0, 1]");
  if (sweeps < 0) return fail(VT_EINVAL, "sweeps must be non-negative");
  if (fine->g.k0 != 0 || fine->g.k1 != fine->g.nz)
    return fail(VT_EINVAL, "multi-slab hierarchies are built by the distributed runtime");
  VT_CUDA(cudaSetDevice(fine->device));
  static std::atomic<unsigned long long> next_uid{1};
  vt_hier* H = new vt_hier();
  H->uid = next_uid++;
  H->omega = omega;
  H->sweeps = sweeps;
  H->lv.push_back(fine);
  int nx = fine->g.nx, ny = fine->g.ny, nz = fine->g.nz;
  double h = fine->h;
  for (int l = 1; l < n_levels; ++l) {
    nx /= 2; ny /= 2; nz /= 2; h *= 2.0;
    vt_grid* c = nullptr;
    vt_status st = vt_grid_create(&c, nx, ny, nz, h, fine->nu, nullptr, 0, nz, fine->device);
    if (st != VT_OK) { vt_hier_destroy(H); return st; }
    vt_grid* f = H->lv.back();
    coarsen_mask_kernel<<<c->nsm * 4, MG_THREADS>>>(f->g, c->g, f->mask, c->mask);
    count_launch();
    unsigned long long* cnt;
    VT_CUDA(cudaMalloc(&cnt, sizeof(unsigned long long)));
    VT_CUDA(cudaMemset(cnt, 0, sizeof(unsigned long long)));
    count_fixed_kernel<<<c->nsm, MG_THREADS>>>(c->g, c->mask, cnt);
    count_launch();
    unsigned long long hc = 0;
    VT_CUDA(cudaMemcpy(&hc, cnt, sizeof(hc), cudaMemcpyDeviceToHost));
    VT_CUDA(cudaFree(cnt));
    c->n_fixed = (long long)hc;
    H->lv.push_back(c);
  }
  const int L = (int)H->lv.size();
  H->u.assign(L, nullptr); H->u2.assign(L, nullptr); H->r.assign(L, nullptr);
  H->f.assign(L, nullptr); H->scale.assign(L, nullptr); H->rho.assign(L, nullptr);
  for (int l = 0; l < L; ++l) {
    vt_grid* G = H->lv[l];
    VT_TRY(hier_alloc_vec(G, &H->u[l]));
    VT_TRY(hier_alloc_vec(G, &H->u2[l]));
    VT_TRY(hier_alloc_vec(G, &H->r[l]));
    if (l > 0) VT_TRY(hier_alloc_vec(G, &H->f[l]));
    VT_CUDA(cudaMalloc(&H->scale[l], G->elem_len() * sizeof(double)));
    VT_CUDA(cudaMemset(H->scale[l], 0, G->elem_len() * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->rho[l], (size_t)G->nel_local() * sizeof(double)));
  }
  // damped inverse diagonals of the smoothed homogenized-operator levels
  H->wd.assign(L, nullptr);
  for (int l = 0; l + 1 < L; ++l)
    if (l == 0 || H->scheme == 0) VT_TRY(hier_alloc_vec(H->lv[l], &H->wd[l]));
  vt_grid* C = H->lv.back();
  H->nL = (int)(3LL * (C->g.nx + 1) * (C->g.ny + 1) * (C->g.nz + 1));
  H->scheme = scheme;
  if (scheme == 1) {
    cudaDeviceSynchronize();  // coarse masks are built on the legacy stream
    vt_status st = gal_setup(H);
    if (st != VT_OK) { vt_hier_destroy(H); return st; }
  }
  {
    vt_status st = tail_setup(H);
    if (st != VT_OK) { vt_hier_destroy(H); return st; }
  }
  *out = H;
  return VT_OK;
}

vt_status vt_hier_destroy(vt_hier* H) {
  if (!H) return VT_OK;
  for (size_t l = 0; l < H->lv.size(); ++l) {
    cudaFree(H->u[l]); cudaFree(H->u2[l]); cudaFree(H->r[l]);
    if (l > 0) cudaFree(H->f[l]);
    cudaFree(H->scale[l]); cudaFree(H->rho[l]);
    if (l < H->wd.size()) cudaFree(H->wd[l]);
    if (l > 0) vt_grid_destroy(H->lv[l]);
  }
  gal_free(H);
  cudaFree(H->tail_ve);
  cudaFree(H->tail_bar);
  cudaFree(H->A); cudaFree(H->A0); cudaFree(H->cvec); cudaFree(H->W); cudaFree(H->Kinv); cudaFree(H->k0l); cudaFree(H->status);
  delete H;
  return VT_OK;
}

int vt_hier_levels(const vt_hier* H) { return H ? (int)H->lv.size() : 0; }
vt_grid* vt_hier_grid(vt_hier* H, int l) {
  return (H && l >= 0 && l < (int)H->lv.size()) ? H->lv[l] : nullptr;
}
const double* vt_hier_level_scale(vt_hier* H, int l) { return H->scale[l]; }
const double* vt_hier_level_mats(vt_hier* H, int l) {
  if (!H || H->scheme != 1 || l < 1 || l >= (int)H->lv.size()) return nullptr;
  if (l == 1 && H->gal_mf && !H->mats1_fresh) {  // matrix-free level 1: materialize on demand
    if (gal_materialize_level1(H, 0) != VT_OK || cudaDeviceSynchronize() != cudaSuccess) return nullptr;
    H->mats1_fresh = true;
  }
  // stored as the packed upper triangle: expand into the hierarchy's scratch
  if (!H->mats[l] || gal_expand(H, l, 0) != VT_OK || cudaDeviceSynchronize() != cudaSuccess) return nullptr;
  return H->mats_full;
}
int vt_hier_scheme(const vt_hier* H) { return H ? H->scheme : -1; }
const double* vt_hier_level_rho(vt_hier* H, int l) { return H->rho[l]; }

vt_status vt_hier_refresh(vt_hier* H, const double* rho, const double* scale0, double p,
                          double kmin, double E, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  const int L = (int)H->lv.size();
  vt_grid* F = H->lv[0];
  VT_CUDA(cudaMemcpyAsync(H->scale[0], scale0, F->elem_len() * sizeof(double),
                          cudaMemcpyDeviceToDevice, s));
  VT_CUDA(cudaMemcpyAsync(H->rho[0], rho, F->nel_local() * sizeof(double),
                          cudaMemcpyDeviceToDevice, s));
  return hier_refresh_levels(H, p, kmin, E, s);
}

}  // extern "C"

namespace vt {
// everything of a refresh after the level-0 scale (and densities) are in
// place: coarse operators, damped inverse diagonals, the coarsest factor
vt_status hier_refresh_levels(vt_hier* H, double p, double kmin, double E, cudaStream_t s) {
  const int L = (int)H->lv.size();
  vt_grid* F = H->lv[0];
  int* bad = reinterpret_cast<int*>(F->scalars);
  VT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  if (H->scheme == 1) {
    VT_TRY(gal_refresh(H, s));  // [ref: multigrid.py:216-223, 262-278]
  } else {
    for (int l = 1; l < L; ++l) {
      vt_grid* f = H->lv[l - 1];
      vt_grid* c = H->lv[l];
      launch_pdl(coarsen_rho_kernel, c->nsm * 4, MG_THREADS, 0, s, f->g.nx, f->g.ny, c->g.nx, c->g.ny,
                                                           c->g.nz, H->rho[l - 1], H->rho[l]);
      count_launch();
      VT_TRY(launch_scale(c, H->rho[l], p, kmin, E, H->scale[l], bad, s));
    }
  }
  for (int l = 0; l < L; ++l)
    if (H->wd[l]) VT_TRY(launch_wdiag(H->lv[l], H->scale[l], H->omega, H->wd[l], s));
  // coarsest direct factor
  vt_grid* C = H->lv.back();
  const int n = H->nL;
  if (n > 20000)
    return fail(VT_ESETUP, "coarsest level has " + std::to_string(n) +
                               " dofs, above the direct-solve guard 20000; increase the level count");
  if (H->scheme == 0 && L > 1 && C->n_fixed < 6)
    return fail(VT_ESETUP, "only " + std::to_string(C->n_fixed) +
                               " fixed dofs survive on the coarsest level; rigid modes are "
                               "unconstrained (bad fixed-dof coarsening)");
  if (!H->A) {
    VT_CUDA(cudaMalloc(&H->A, (size_t)n * n * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->W, (size_t)n * n * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->Kinv, (size_t)n * n * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->A0, (size_t)n * n * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->cvec, 3 * (size_t)n * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->k0l, 576 * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->status, sizeof(int)));
    double K[576];
    hex8_k0_host(C->nu, C->h, K);
    VT_CUDA(cudaMemcpy(H->k0l, K, sizeof(K), cudaMemcpyHostToDevice));
    if ((size_t)n * sizeof(double) > 48 * 1024)
    {
      VT_CUDA(cudaFuncSetAttribute(coarse_mv_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(n * sizeof(double))));
      VT_CUDA(cudaFuncSetAttribute(coarse_mv_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(n * sizeof(double))));
      VT_CUDA(cudaFuncSetAttribute(coarse_mv_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(n * sizeof(double))));
    }
  }
  const double* cmats = (H->scheme == 1 && L > 1) ? H->mats[L - 1] : nullptr;
  if (n <= COARSE_SMEM_N) {
    const size_t sm = ((size_t)n * n + n) * sizeof(double);
    static bool attr = false;
    if (!attr) {
      VT_CUDA(cudaFuncSetAttribute(coarse_factor_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(((size_t)COARSE_SMEM_N * COARSE_SMEM_N + COARSE_SMEM_N) * sizeof(double))));
      attr = true;
    }
    launch_pdl(coarse_factor_smem_kernel, 1, 1024, sm, s, C->g, H->scale[L - 1], H->k0l, cmats,
               C->mask, n, H->A0, H->Kinv, H->status);
    count_launch(1);
  } else {
    launch_pdl(coarse_factor_kernel, 1, 1024, 0, s, C->g, H->scale[L - 1], H->k0l, cmats, C->mask, n,
               H->A, H->A0, H->status);
    launch_pdl(tri_inverse_kernel, (n + 127) / 128, 128, 0, s, n, H->A, H->W);
    launch_pdl(gram_kernel, C->nsm * 4, 256, 0, s, n, H->W, H->Kinv);
    count_launch(3);
  }
  VT_CUDA(cudaGetLastError());
  int hb[2] = {0, 0};
  VT_CUDA(cudaMemcpyAsync(&hb[0], bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaMemcpyAsync(&hb[1], H->status, sizeof(int), cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  if (hb[0]) return fail(VT_EDENSITY, "density outside [0, 1]");
  if (hb[1])
    return fail(VT_ESETUP,
                "coarsest-level matrix is not positive definite; the fixed dof set may vanish "
                "under coarsening");
  H->factored = true;
  return VT_OK;
}
}  // namespace vt

extern "C" {

vt_status vt_hier_vcycle(vt_hier* H, const double* f, double* z, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!H->factored) return fail(VT_ESETUP, "hierarchy was not refreshed before use");
  vt_grid* F = H->lv[0];
  // fine.f = f with fixed dofs zeroed [ref: multigrid.py:413-414]
  VT_TRY(launch_project(F, f, F->scratch, s));
  const double* zb = nullptr;
  VT_TRY(hier_vcycle_launch(H, F->scratch, nullptr, nullptr, false, s, &zb));
  VT_CUDA(cudaMemcpyAsync(z, zb, F->vec_len() * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return VT_OK;
}

vt_status vt_hier_restrict(vt_hier* H, int l, const double* fine, double* coarse, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (l < 0 || l + 1 >= (int)H->lv.size()) return fail(VT_EINVAL, "level out of range");
  vt_grid* F = H->lv[l];
  VT_TRY(launch_project(F, fine, F->scratch, s));
  VT_TRY(launch_restrict(F, H->lv[l + 1], F->scratch, coarse, nullptr, -1, -1, s));
  return VT_OK;
}

vt_status vt_hier_prolong(vt_hier* H, int l, const double* coarse, double* fine, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (l < 0 || l + 1 >= (int)H->lv.size()) return fail(VT_EINVAL, "level out of range");
  vt_grid* F = H->lv[l];
  return launch_prolong_set(H->lv[l + 1], F, coarse, fine, nullptr, s);
}

vt_status vt_hier_jacobi(vt_hier* H, int l, const double* u, const double* f, int sweeps,
                         double* out, void* stream) {
  // out-of-place sweeps; fixed dofs keep the input values [ref: multigrid.py:375-385]
  cudaStream_t s = (cudaStream_t)stream;
  if (l < 0 || l >= (int)H->lv.size()) return fail(VT_EINVAL, "level out of range");
  vt_grid* G = H->lv[l];
  const size_t bytes = G->vec_len() * sizeof(double);
  VT_CUDA(cudaMemcpyAsync(out, u, bytes, cudaMemcpyDeviceToDevice, s));
  for (int k = 0; k < sweeps; ++k) {
    if (H->scheme == 1 && l >= 1) {
      VT_TRY(gal_level_op(H, l, 2, out, f, G->scratch2, nullptr, s));
      VT_CUDA(cudaMemcpyAsync(out, G->scratch2, bytes, cudaMemcpyDeviceToDevice, s));
      continue;
    }
    VT_TRY(launch_project(G, out, G->scratch, s));
    VT_TRY(launch_hex8(G, H8_SMOOTH, false, H->scale[l], G->scratch, out, f, G->scratch2,
                       H->omega, nullptr, nullptr, s));
    VT_CUDA(cudaMemcpyAsync(out, G->scratch2, bytes, cudaMemcpyDeviceToDevice, s));
  }
  return VT_OK;
}

vt_status vt_hier_level_apply(vt_hier* H, int l, const double* u, double* v, void* stream) {
  if (l < 0 || l >= (int)H->lv.size()) return fail(VT_EINVAL, "level out of range");
  if (H->scheme == 1 && l >= 1) {
    if (!H->factored) return fail(VT_ESETUP, "hierarchy was not refreshed before use");
    return gal_level_op(H, l, 0, u, nullptr, v, nullptr, (cudaStream_t)stream);
  }
  return vt_apply(H->lv[l], H->scale[l], u, v, stream);
}

vt_status vt_hier_level_diag(vt_hier* H, int l, double* d, void* stream) {
  if (l < 0 || l >= (int)H->lv.size()) return fail(VT_EINVAL, "level out of range");
  if (H->scheme == 1 && l >= 1) {
    VT_CUDA(cudaMemcpyAsync(d, H->gdiag[l], H->lv[l]->vec_len() * sizeof(double),
                            cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return VT_OK;
  }
  return vt_diagonal(H->lv[l], H->scale[l], d, stream);
}

vt_status vt_hier_coarse_solve(vt_hier* H, const double* f, double* u, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!H->factored) return fail(VT_ESETUP, "hierarchy was not refreshed before use");
  return launch_coarse_solve(H, f, u, nullptr, s);
}

}  // extern "C"
