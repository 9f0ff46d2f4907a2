// Fused coarse tail of the V-cycle: every level from the first one with at
// most VT_TAIL_NODES nodes down to the coarsest direct solve and back up, in
// ONE launch of one thread-block cluster [ref: multigrid.py:404-430 (_cycle)].
// OFF by default (vt_tail_config): measured slower than the kernel chain, see
// tail_nodes_limit() below and DESIGN.md 3.1.
//
// Below ~10K nodes a level's kernels are pure latency: each of the ~30
// launches of the multi-kernel tail (jacobi sweep, residual, restriction per
// level on the way down, three coarse mat-vecs, prolongation + smoother on the
// way up) costs 4-7 us whatever its size.  Here the same passes run as phases
// of one kernel separated by cluster barriers (barrier.cluster arrive.release /
// wait.acquire), with the level vectors in L2 and every vector produced inside
// the kernel read with ld.global.cg, so no CTA can see a stale L1 line.
//
// Phases (level l, sweeps nu):
//   down:   E0  element products of u0 = jacobi0(f) (computed on the fly)
//           N0  node sums: r = f - K u0 (fixed 0) and u = u0 written
//           (nu > 1: E + N smoothing sweeps in between)
//           R   r -> f_{l+1} (restriction)
//   coarse: three warp-per-row mat-vecs (x0 = Kinv f, r = f - A0 x0, u = x0 + Kinv r)
//   up:     P   u_l += P u_{l+1}
//           E + N smoothing sweeps
// Element products: homogenized levels use the factorized hex8 element
// operator (Walsh butterflies around couple(), vt_couple.cuh) with the level's
// scale; Galerkin levels the stored 24x24 matrices with the same lane order and
// accumulator split as gal_elem_kernel.  Node sums run over the incident
// elements in the reference's corner order c = 0..7.  The transfers and the
// coarse mat-vecs use the operation order of restrict_kernel, prolong_kernel
// and coarse_mv_kernel: bit-identical to them.  The Galerkin tail is
// bit-identical to the multi-kernel Galerkin path; the homogenized smoothers
// round differently from the tile kernel (another summation order), within
// the V-cycle's 1e-10 parity bar.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "vt_couple.cuh"
#include "vt_internal.h"

namespace cg = cooperative_groups;

namespace vt {

constexpr int TL_THREADS = 512;
constexpr int TL_WARPS = TL_THREADS / 32;
constexpr int TL_MAXL = 12;
constexpr int TL_MAX_COARSE = 4096;  // coarsest dofs staged in shared memory

struct TailLevel {
  Geom g;
  const uint8_t* mask;
  const double* scale;  // homogenized: element scales (vt element layout)
  const double* mats;   // galerkin: element matrices (dense element order)
  const double* wd;     // homogenized: omega / diag (0 on fixed)
  const double* d;      // galerkin: stored diagonal
  double *u, *u2, *r, *f;
  double kc[6];
};

struct TailArgs {
  int nlev;  // tail levels; lv[nlev - 1] is the coarsest
  int scheme, sweeps;
  double omega;
  const double* f0;  // right-hand side of lv[0]
  double* ve;        // element products, 24 per element
  int n;             // coarsest dofs
  const double *Kinv, *A0;
  double *cf, *x0, *cr;
  const int* stop;
  unsigned long long* trace;  // optional: %globaltimer after every phase (vt_tail_trace)
  unsigned* gbar;             // grid-barrier mode: {arrivals, generation}; nullptr = one cluster
  TailLevel lv[TL_MAXL];
};

__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// (tail levels are small: 32-bit item indices)
__device__ __forceinline__ void node_ijk(const Geom& g, int t, int& p, int& j, int& i) {
  i = t % (g.nx + 1);
  const int r = t / (g.nx + 1);
  j = r % (g.ny + 1);
  p = r / (g.ny + 1) + g.pA;
}

__device__ __forceinline__ int n_nodes(const Geom& g) { return (g.pB - g.pA) * (g.ny + 1) * (g.nx + 1); }

__device__ __forceinline__ int gtid() { return blockIdx.x * blockDim.x + threadIdx.x; }
__device__ __forceinline__ int gnt() { return gridDim.x * blockDim.x; }

// first damped-Jacobi sweep from zero (jacobi0w_kernel / gal_jacobi0_kernel)
__device__ __forceinline__ double jac0(const TailArgs& a, const TailLevel& L, const double* f, long long o,
                                       bool fx) {
  if (a.scheme == 0) {
    const double w = L.wd[o];
    return w == 0.0 ? 0.0 : __dmul_rn(w, ldcg(f + o));
  }
  return fx ? 0.0 : __dmul_rn(a.omega, ddiv_nr(ldcg(f + o), L.d[o]));
}

// ---- element phase: ve[e] = K_e x_e.  J0: x = jacobi0(f) on the fly.
template <bool J0>
__device__ void elem_phase(const TailArgs& a, const TailLevel& L, const double* x, const double* f,
                           double* us_all) {
  const Geom& g = L.g;
  const int nel = g.nx * g.ny * g.nz;
  if (a.scheme == 0) {
    for (int e = gtid(); e < nel; e += gnt()) {
      const int i = e % g.nx, j = (e / g.nx) % g.ny, k = e / (g.nx * g.ny);
      double C[3][8];
#pragma unroll
      for (int corner = 0; corner < 8; ++corner) {
        const int p = k + (corner >> 2) + 1, jj = j + ((corner >> 1) & 1), ii = i + (corner & 1);
        const long long o = node_off(g, p, jj, ii) * 3;
        if (J0) {
          const unsigned mk = L.mask[mask_off(g, p, jj, ii)];
#pragma unroll
          for (int c = 0; c < 3; ++c) C[c][corner] = jac0(a, L, f, o + c, (mk >> c) & 1u);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) C[c][corner] = ldcg(x + o + c);
        }
      }
      // forward butterflies x, y, z: index bit set = difference along that axis
#pragma unroll
      for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
#pragma unroll
          for (int lo = 0; lo < 8; ++lo) {
            if (lo & (1 << ax)) continue;
            const int hi = lo | (1 << ax);
            const double s = C[c][hi] + C[c][lo], dd = C[c][hi] - C[c][lo];
            C[c][lo] = s;
            C[c][hi] = dd;
          }
        }
      }
      double O[3][8];
      couple(C, L.scale[elem_off(g, k + 1, j, i)], L.kc, O);
      // transposed butterflies z, y, x (O[.][0] -- the rigid translation -- is 0)
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        O[c][0] = 0.0;
#pragma unroll
        for (int ax = 2; ax >= 0; --ax) {
#pragma unroll
          for (int lo = 0; lo < 8; ++lo) {
            if (lo & (1 << ax)) continue;
            const int hi = lo | (1 << ax);
            const double s = O[c][lo], w = O[c][hi];
            O[c][lo] = s - w;
            O[c][hi] = s + w;
          }
        }
      }
      // component-major (SoA) products: coalesced here and in the node sums
#pragma unroll
      for (int corner = 0; corner < 8; ++corner)
#pragma unroll
        for (int c = 0; c < 3; ++c) a.ve[(long long)(3 * corner + c) * nel + e] = O[c][corner];
    }
  } else {
    // warp per element, lane r < 24 owns row r (gal_elem_kernel's arithmetic)
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    double* us = us_all + wib * 24;
    const int warp = gtid() >> 5, nw = gnt() >> 5;
    for (int e = warp; e < nel; e += nw) {
      const int i = e % g.nx, j = (e / g.nx) % g.ny, k = e / (g.nx * g.ny);
      __syncwarp();
      if (lane < 24) {
        const int corner = lane / 3, comp = lane % 3;
        const int p = k + ((corner >> 2) & 1) + 1, jj = j + ((corner >> 1) & 1), ii = i + (corner & 1);
        const unsigned mk = L.mask[mask_off(g, p, jj, ii)];
        const long long o = node_off(g, p, jj, ii) * 3 + comp;
        const bool fx = (mk >> comp) & 1u;
        us[lane] = J0 ? jac0(a, L, f, o, fx) : (fx ? 0.0 : ldcg(x + o));
      }
      __syncwarp();
      if (lane < 24) {
        const double* m = L.mats + (long long)e * GAL_PACK;  // packed upper triangle
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int b2 = 0; b2 < 12; ++b2) {
          s0 = fma(m[gal_sym(lane, 2 * b2)], us[2 * b2], s0);
          s1 = fma(m[gal_sym(lane, 2 * b2 + 1)], us[2 * b2 + 1], s1);
        }
        a.ve[(long long)e * 24 + lane] = s0 + s1;
      }
    }
  }
}

// ---- node phase: v = sum of the incident element products (corner order), then
//   RESID: r = f - v (fixed 0); with J0 also u = jacobi0(f) (the sweep E0 used)
//   SMOOTH: out = x + smoother(f - v); with J0, x = jacobi0(f) on the fly
template <bool RESID, bool J0>
__device__ void node_phase(const TailArgs& a, const TailLevel& L, const double* x, const double* f,
                           double* out, double* u_out) {
  const Geom& g = L.g;
  const int nn = n_nodes(g), nel = g.nx * g.ny * g.nz;
  // element products: SoA (homogenized) or per-element rows (galerkin)
  const long long es = a.scheme == 0 ? 1 : 24, cs = a.scheme == 0 ? nel : 1;
  for (int t = gtid(); t < nn; t += gnt()) {
    int p, j, i;
    node_ijk(g, t, p, j, i);
    const int k = p - 1;
    double v[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int ei = i - (c & 1), ej = j - ((c >> 1) & 1), ek = k - ((c >> 2) & 1);
      if (ei < 0 || ei >= g.nx || ej < 0 || ej >= g.ny || ek < 0 || ek >= g.nz) continue;
      const int e = (ek * g.ny + ej) * g.nx + ei;
#pragma unroll
      for (int comp = 0; comp < 3; ++comp)
        v[comp] = __dadd_rn(v[comp], ldcg(a.ve + e * es + (3 * c + comp) * cs));
    }
    const long long node = node_off(g, p, j, i);
    const unsigned m = L.mask[mask_off(g, p, j, i)];
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      const long long o = node * 3 + comp;
      const bool fx = (m >> comp) & 1u;
      const double fo = ldcg(f + o);
      if (RESID) {
        out[o] = fx ? 0.0 : __dsub_rn(fo, v[comp]);
        if (J0) u_out[o] = jac0(a, L, f, o, fx);
      } else {
        const double xo = J0 ? jac0(a, L, f, o, fx) : ldcg(x + o);
        if (a.scheme == 0)  // hex8 SMOOTH: fixed dofs stay 0 (solver-internal vectors)
          out[o] = fx ? 0.0 : fma(__dsub_rn(fo, v[comp]), L.wd[o], xo);
        else                // gal_node_kernel<2>
          out[o] = fx ? xo : __dadd_rn(xo, __dmul_rn(a.omega, ddiv_nr(__dsub_rn(fo, v[comp]), L.d[o])));
      }
    }
  }
}

// ---- restriction f_c = P^T r_f (restrict_kernel's pass order: z, y, x)
__device__ void restrict_phase(const TailLevel& F, const TailLevel& C, const double* rf, double* fc) {
  const Geom &gf = F.g, &gc = C.g;
  const int nn = n_nodes(gc) * 3;
  for (int t = gtid(); t < nn; t += gnt()) {
    const int c = t % 3;
    int p, J, I;
    node_ijk(gc, t / 3, p, J, I);
    const int K = p - 1;
    const bool ok1 = 2 * K + 1 <= gf.nz, ok2 = K >= 1;
    const bool okj1 = 2 * J + 1 <= gf.ny, okj2 = J >= 1;
    const bool oki1 = 2 * I + 1 <= gf.nx, oki2 = I >= 1;
    const int pf = 2 * K + 1;
    auto tz = [&](int y, int x) {
      const long long o = node_off(gf, pf, y, x) * 3 + c;
      double v = ldcg(rf + o);
      if (ok1) v = __dadd_rn(v, 0.5 * ldcg(rf + o + gf.nplane));
      if (ok2) v = __dadd_rn(v, 0.5 * ldcg(rf + o - gf.nplane));
      return v;
    };
    double ty[3];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      if ((b == 1 && !oki1) || (b == 2 && !oki2)) {
        ty[b] = 0.0;
        continue;
      }
      const int x = 2 * I + (b == 0 ? 0 : (b == 1 ? 1 : -1));
      double v = tz(2 * J, x);
      if (okj1) v = __dadd_rn(v, 0.5 * tz(2 * J + 1, x));
      if (okj2) v = __dadd_rn(v, 0.5 * tz(2 * J - 1, x));
      ty[b] = v;
    }
    double v = ty[0];
    if (oki1) v = __dadd_rn(v, 0.5 * ty[1]);
    if (oki2) v = __dadd_rn(v, 0.5 * ty[2]);
    const unsigned m = C.mask[mask_off(gc, p, J, I)];
    fc[node_off(gc, p, J, I) * 3 + c] = ((m >> c) & 1u) ? 0.0 : v;
  }
}

// ---- prolongation u_f += P u_c, fine fixed 0 (prolong_kernel<true>'s pass order)
__device__ void prolong_phase(const TailLevel& C, const TailLevel& F, const double* uc, double* uf) {
  const Geom &gc = C.g, &gf = F.g;
  const int nn = n_nodes(gf) * 3;
  for (int t = gtid(); t < nn; t += gnt()) {
    const int comp = t % 3;
    int p, fy, fx;
    node_ijk(gf, t / 3, p, fy, fx);
    const int fz = p - 1;
    const int I = fx >> 1, J = fy >> 1, K = fz >> 1;
    const bool ox = fx & 1, oy = fy & 1, cz = fz & 1;
    auto zval = [&](int jj, int ii) {
      const long long o = node_off(gc, K + 1, jj, ii) * 3 + comp;
      const double q0 = ldcg(uc + o);
      return cz ? 0.5 * __dadd_rn(q0, ldcg(uc + o + gc.nplane)) : q0;
    };
    const double za0 = zval(J, I), za1 = ox ? zval(J, I + 1) : 0.0;
    double v;
    if (!oy) {
      v = ox ? 0.5 * __dadd_rn(za0, za1) : za0;
    } else {
      const double zb0 = zval(J + 1, I), zb1 = ox ? zval(J + 1, I + 1) : 0.0;
      const double y0 = 0.5 * __dadd_rn(za0, zb0);
      v = ox ? 0.5 * __dadd_rn(y0, 0.5 * __dadd_rn(za1, zb1)) : y0;
    }
    const unsigned m = F.mask[mask_off(gf, p, fy, fx)];
    if ((m >> comp) & 1u) v = 0.0;
    const long long o = node_off(gf, p, fy, fx) * 3 + comp;
    uf[o] = __dadd_rn(ldcg(uf + o), v);
  }
}

// ---- coarsest solve, coarse_mv_kernel's three passes (warp per row over the cluster)
template <int MODE>
__device__ void coarse_phase(const TailArgs& a, const TailLevel& Lc, const double* f, double* u, double* vs) {
  const Geom& g = Lc.g;
  const int n = a.n;
  const int nx1 = g.nx + 1, ny1 = g.ny + 1;
  auto dof = [&](int d, long long& o, bool& fx) {
    const int node = d / 3, c = d % 3;
    const int i = node % nx1, j = (node / nx1) % ny1, k = node / (nx1 * ny1);
    o = node_off(g, k + 1, j, i) * 3 + c;
    fx = (Lc.mask[mask_off(g, k + 1, j, i)] >> c) & 1u;
  };
  __syncthreads();
  for (int d = threadIdx.x; d < n; d += blockDim.x) {
    double v;
    if (MODE == 0) {
      long long o;
      bool fx;
      dof(d, o, fx);
      v = ldcg(f + o);
      if (blockIdx.x == 0) a.cf[d] = v;
    } else {
      v = ldcg((MODE == 1 ? a.x0 : a.cr) + d);
    }
    vs[d] = v;
  }
  __syncthreads();
  const double* M = MODE == 1 ? a.A0 : a.Kinv;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int r = blockIdx.x * TL_WARPS + warp; r < n; r += gridDim.x * TL_WARPS) {
    double s = 0.0;
    for (int e = lane; e < n; e += 32) s = fma(M[(long long)r * n + e], vs[e], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) {
      if (MODE == 0) {
        a.x0[r] = s;
      } else if (MODE == 1) {
        a.cr[r] = ldcg(a.cf + r) - s;
      } else {
        long long o;
        bool fx;
        dof(r, o, fx);
        u[o] = fx ? 0.0 : ldcg(a.x0 + r) + s;
      }
    }
  }
}

// Software grid barrier (one CTA per SM, all co-resident): arrivals counted
// with an atomic, the last arriver resets the count and bumps the generation
// the others spin on.  The gpu-scope fences make every CTA's writes of the
// phase visible (and invalidate L1) before anyone proceeds.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned g = gen;
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0;
      __threadfence();
      atomicExch(&bar[1], g + 1);
    } else {
      unsigned v;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
      } while (v == g);
    }
    __threadfence();
    gen = g + 1;
  }
  __syncthreads();
}

// L2 prefetch with the evict_last priority: the tail's read-only level data
// (masks, scales / diagonals, the coarse inverse) would otherwise be evicted by
// the fine levels' ~1 GB of streams between two V-cycles, and every phase would
// wait on HBM latency; marked evict_last they stay resident from cycle to cycle.
__device__ __forceinline__ void l2_keep(const void* p, long long bytes) {
  const char* c = static_cast<const char*>(p);
  for (long long o = (long long)gtid() * 128; o < bytes; o += (long long)gnt() * 128)
    asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(c + o));
}

__global__ void __launch_bounds__(TL_THREADS, 1) tail_vcycle_kernel(const __grid_constant__ TailArgs a) {
  {  // read-only level data: resident in L2 before the phases need it
    for (int l = 0; l < a.nlev; ++l) {
      const TailLevel& L = a.lv[l];
      const Geom& g = L.g;
      const long long nv = (long long)g.P * g.nplane * 8;
      l2_keep(L.mask, (long long)g.P * g.mplane);
      if (a.scheme == 0) {
        l2_keep(L.scale, (long long)g.Q * g.eplane * 8);
        if (L.wd) l2_keep(L.wd, nv);
      } else if (L.d) {
        l2_keep(L.d, nv);
        if (L.mats && (long long)g.nx * g.ny * g.nz * 4608 <= (4 << 20)) l2_keep(L.mats, (long long)g.nx * g.ny * g.nz * 4608);
      }
    }
    l2_keep(a.Kinv, (long long)a.n * a.n * 8);
    l2_keep(a.A0, (long long)a.n * a.n * 8);
  }
  griddep_wait();
  if (a.stop && *(volatile const int*)a.stop) return;
  cg::cluster_group cl = cg::this_cluster();
  unsigned gen = 0;
  if (a.gbar && threadIdx.x == 0) gen = *(volatile unsigned*)(a.gbar + 1);
  int nph = 0;
  auto sync = [&]() {
    if (a.gbar)
      grid_barrier(a.gbar, gen);
    else
      cl.sync();
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
      unsigned long long g;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
      a.trace[nph] = g;
    }
    ++nph;
  };
  if (a.trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    a.trace[63] = g;
  }
  extern __shared__ double tl_smem[];
  double* us = tl_smem;                     // galerkin: TL_WARPS x 24
  double* vs = tl_smem + TL_WARPS * 24;     // coarse vector
  const int nl = a.nlev;
  double* cur[TL_MAXL];
  // ---- down (the buffer sequence of hier_vcycle_launch: u, then alternating u2 / u)
  for (int l = 0; l + 1 < nl; ++l) {
    const TailLevel& L = a.lv[l];
    const double* f = l == 0 ? a.f0 : L.f;
    elem_phase<true>(a, L, nullptr, f, us);
    sync();
    if (a.sweeps == 1) {
      node_phase<true, true>(a, L, nullptr, f, L.r, L.u);
      sync();
      cur[l] = L.u;
    } else {
      node_phase<false, true>(a, L, nullptr, f, L.u2, nullptr);
      sync();
      cur[l] = L.u2;
      for (int k = 2; k < a.sweeps; ++k) {
        elem_phase<false>(a, L, cur[l], nullptr, us);
        sync();
        double* dst = cur[l] == L.u ? L.u2 : L.u;
        node_phase<false, false>(a, L, cur[l], f, dst, nullptr);
        sync();
        cur[l] = dst;
      }
      elem_phase<false>(a, L, cur[l], nullptr, us);
      sync();
      node_phase<true, false>(a, L, cur[l], f, L.r, nullptr);
      sync();
    }
    restrict_phase(L, a.lv[l + 1], L.r, a.lv[l + 1].f);
    sync();
  }
  // ---- coarsest
  const TailLevel& Lc = a.lv[nl - 1];
  const double* fcst = nl == 1 ? a.f0 : Lc.f;
  coarse_phase<0>(a, Lc, fcst, Lc.u, vs);
  sync();
  coarse_phase<1>(a, Lc, fcst, Lc.u, vs);
  sync();
  coarse_phase<2>(a, Lc, fcst, Lc.u, vs);
  sync();
  cur[nl - 1] = Lc.u;
  // ---- up
  for (int l = nl - 2; l >= 0; --l) {
    const TailLevel& L = a.lv[l];
    const double* f = l == 0 ? a.f0 : L.f;
    prolong_phase(a.lv[l + 1], L, cur[l + 1], cur[l]);
    sync();
    for (int k = 0; k < a.sweeps; ++k) {
      elem_phase<false>(a, L, cur[l], nullptr, us);
      sync();
      double* dst = cur[l] == L.u ? L.u2 : L.u;
      node_phase<false, false>(a, L, cur[l], f, dst, nullptr);
      sync();
      cur[l] = dst;
    }
  }
}

}  // namespace vt

// ------------------------------------------------------------------ host side
namespace vt {

// node budget of the fused tail's first level (VT_TAIL_NODES / vt_tail_config).
// Default 0 = off: measured on B200 at cfg2 the fused tail is 10-55 us SLOWER
// per V-cycle than the PDL-chained kernels at every budget:
// a phase costs a dependent load -> store -> barrier round trip (~1.2 us even
// when empty of work) plus the scattered-access throughput of 16 SMs, i.e.
// about what a PDL-overlapped kernel costs on all 148.
static long long g_tail_nodes = -1;
static long long tail_nodes_limit() {
  if (g_tail_nodes < 0) g_tail_nodes = getenv("VT_TAIL_NODES") ? atoll(getenv("VT_TAIL_NODES")) : 0;
  return g_tail_nodes;
}

static long long level_nodes(const vt_grid* G) {
  return (long long)(G->g.nx + 1) * (G->g.ny + 1) * (G->g.nz + 1);
}

static unsigned long long* g_tail_trace_buf = nullptr;  // device, 64 slots
static unsigned long long* g_tail_trace = nullptr;      // = the buffer while tracing

// VT_TAIL_MODE=grid: one CTA per SM with a software grid barrier instead of a cluster
static bool tail_grid_mode() {
  static const bool g = getenv("VT_TAIL_MODE") && strcmp(getenv("VT_TAIL_MODE"), "grid") == 0;
  return g;
}

static size_t tail_smem() { return (size_t)(TL_WARPS * 24 + TL_MAX_COARSE) * sizeof(double); }

// cluster size of the tail launch: 16 CTAs when the part can co-schedule a
// non-portable cluster of that size, else the portable 8 (0: unavailable)
static int tail_cluster() {
  static int cs = -1;
  if (cs >= 0) return cs;
  cs = 0;
  if (cudaFuncSetAttribute(tail_vcycle_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
    cudaGetLastError();
    return cs;
  }
  const int want = getenv("VT_TAIL_CLUSTER") ? atoi(getenv("VT_TAIL_CLUSTER")) : 16;
  for (int c = want; c >= 8; c /= 2) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c);
    cfg.blockDim = dim3(TL_THREADS);
    cfg.dynamicSmemBytes = tail_smem();
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = c;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, tail_vcycle_kernel, &cfg) == cudaSuccess && n >= 1) {
      cs = c;
      break;
    }
    cudaGetLastError();
  }
  return cs;
}

vt_status tail_setup(vt_hier* H) {
  const int L = (int)H->lv.size();
  const long long lim = tail_nodes_limit();
  if (lim <= 0 || H->nL > TL_MAX_COARSE) return VT_OK;
  for (int l = 1; l < L; ++l) {
    const vt_grid* G = H->lv[l];
    if (level_nodes(G) > lim) continue;
    if (L - l > TL_MAXL) return VT_OK;
    const long long nel = (long long)G->g.nx * G->g.ny * G->g.nz;
    VT_CUDA(cudaMalloc(&H->tail_ve, (size_t)(nel > 0 ? nel : 1) * 24 * sizeof(double)));
    VT_CUDA(cudaMalloc(&H->tail_bar, 2 * sizeof(unsigned)));
    VT_CUDA(cudaMemset(H->tail_bar, 0, 2 * sizeof(unsigned)));
    H->tail_first = l;
    return VT_OK;
  }
  return VT_OK;
}

int hier_tail_start(vt_hier* H, int top) {
  const int L = (int)H->lv.size();
  if (!H->tail_ve || H->sweeps < 1 || H->tail_first < 1) return L;
  int t = std::max(top, H->tail_first);
  if (H->scheme == 1 && H->gal_mf) t = std::max(t, 2);  // level 1 is matrix-free
  if (t >= L || t < 1) return L;
  if (!tail_grid_mode() && tail_cluster() == 0) return L;
  return t;
}

vt_status launch_tail(vt_hier* H, int t, const double* ft, const int* stop, cudaStream_t s,
                      const double** z_out) {
  const int L = (int)H->lv.size();
  const bool gm = tail_grid_mode();
  const int cs = gm ? 0 : tail_cluster();
  if (!gm && cs == 0) return fail(VT_ECUDA, "fused tail: no cluster launch");
  TailArgs a;
  memset(&a, 0, sizeof(a));
  a.nlev = L - t;
  a.scheme = H->scheme;
  a.sweeps = H->sweeps;
  a.omega = H->omega;
  a.f0 = ft;
  a.ve = H->tail_ve;
  a.n = H->nL;
  a.Kinv = H->Kinv;
  a.A0 = H->A0;
  a.cf = H->cvec;
  a.x0 = H->cvec + H->nL;
  a.cr = H->cvec + 2 * H->nL;
  a.stop = stop;
  a.trace = g_tail_trace;
  a.gbar = gm ? reinterpret_cast<unsigned*>(H->tail_bar) : nullptr;
  for (int i = 0; i < a.nlev; ++i) {
    const int l = t + i;
    vt_grid* G = H->lv[l];
    TailLevel& T = a.lv[i];
    T.g = G->g;
    T.mask = G->mask;
    T.scale = H->scale[l];
    T.mats = (H->scheme == 1 && l < (int)H->mats.size()) ? H->mats[l] : nullptr;
    T.wd = l < (int)H->wd.size() ? H->wd[l] : nullptr;
    T.d = (H->scheme == 1 && l < (int)H->gdiag.size()) ? H->gdiag[l] : nullptr;
    T.u = H->u[l];
    T.u2 = H->u2[l];
    T.r = H->r[l];
    T.f = H->f[l];
    for (int k = 0; k < 6; ++k) T.kc[k] = G->coef.kc[k];
    if (i + 1 < a.nlev && ((H->scheme == 0 && !T.wd) || (H->scheme == 1 && (!T.mats || !T.d))))
      return fail(VT_ESETUP, "fused tail: level operator not set up");
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(gm ? H->lv[0]->nsm : cs);
  cfg.blockDim = dim3(TL_THREADS);
  cfg.dynamicSmemBytes = tail_smem();
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  if (gm) {
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
  } else {
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
  }
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 2 : 1;
  VT_CUDA(cudaLaunchKernelEx(&cfg, tail_vcycle_kernel, a));
  count_launch();
  // the level-t buffer the kernel ends in (hier_vcycle_launch's alternation)
  const double* c = H->u[t];
  auto other = [&](const double* b) -> const double* { return b == H->u[t] ? H->u2[t] : H->u[t]; };
  if (t < L - 1) {
    for (int k = 1; k < H->sweeps; ++k) c = other(c);
    for (int k = 0; k < H->sweeps; ++k) c = other(c);
  }
  *z_out = c;
  return VT_OK;
}

}  // namespace vt

extern "C" {

long long vt_tail_config(long long nodes) {
  const long long prev = vt::tail_nodes_limit();
  vt::g_tail_nodes = nodes < 0 ? 0 : nodes;
  return prev;
}

vt_status vt_tail_trace(int enable, uint64_t* host_out, int max_slots) {
  // the buffer is never freed: a graph captured while tracing keeps its address
  if (enable && !vt::g_tail_trace_buf) {
    VT_CUDA(cudaMalloc(&vt::g_tail_trace_buf, 64 * sizeof(unsigned long long)));
    VT_CUDA(cudaMemset(vt::g_tail_trace_buf, 0, 64 * sizeof(unsigned long long)));
  }
  if (host_out && vt::g_tail_trace_buf) {
    VT_CUDA(cudaDeviceSynchronize());
    VT_CUDA(cudaMemcpy(host_out, vt::g_tail_trace_buf, (size_t)std::min(max_slots, 64) * sizeof(uint64_t),
                       cudaMemcpyDeviceToHost));
  }
  vt::g_tail_trace = enable ? vt::g_tail_trace_buf : nullptr;
  return VT_OK;
}

int vt_hier_tail_level(vt_hier* H) {
  if (!H) return -1;
  const int t = vt::hier_tail_start(H, 0);
  return t < (int)H->lv.size() ? t : -1;
}

}  // extern "C"
