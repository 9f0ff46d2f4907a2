// Z-slab decomposition of the MGPCG state-equation solve [SURVEY 8(e)].
//
// The reference is single-process (there is no distributed path to mirror);
// the decomposition keeps its arithmetic per dof and adds the exchange steps
// a partitioned structured grid needs:
//
//  * Rank g owns element layers [k0_g, k1_g) of every distributed level and
//    node planes [k0_g, k1_g) (+ plane nz on the last rank).  Each slab vector
//    carries one ghost node plane below and above and one ghost element layer
//    below (vt layouts, include/voxb200.h), so every stencil kernel of the
//    single-GPU path runs unchanged on a slab: global plane k = p - 1 + k0.
//  * Halo exchanges (one node plane per neighbour) precede every operator
//    application / smoother / residual and the transfers that read across the
//    slab boundary; the element-scale ghost layer is exchanged once per
//    refresh.
//  * Dot products: every slab reduces its CTA partials to one scalar (fixed
//    order), the per-rank scalars are all-gathered and every rank sums them in
//    rank order, so all ranks take identical scalar decisions (alpha, beta,
//    convergence) and launch the same number of iteration graphs.
//  * Multigrid: levels 0..D are distributed (the planner picks D so that every
//    slab's layer count stays integral); level D's residual is restricted
//    slab-by-slab into a replicated full grid of level D+1 (each slab writes
//    the coarse planes whose centre fine plane it owns, then the ranges are
//    broadcast), the coarse tail D+1..L-1 (incl. the dense coarsest solve) runs
//    redundantly on every rank, and its correction is prolongated straight
//    into each slab.
//
// Transport: slabs living in this process exchange with device copies (one GPU
// can host all slabs -- the parity tests run that way); slabs on other ranks
// exchange with NCCL send/recv/broadcast/all-gather on the solver stream (one
// process per GPU, NVLink/NVSwitch), all captured in the per-iteration CUDA
// graph.  NCCL is loaded with dlopen so the single-GPU library has no NCCL
// dependency.  Both transports move the same planes in the same order, so the
// arithmetic is identical.
#include <dlfcn.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "dist_internal.h"

namespace vt {

NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  const char* names[] = {getenv("VT_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
  void* h = nullptr;
  for (const char* n : names) {
    if (!n || !*n) continue;
    h = dlopen(n, RTLD_NOW | RTLD_LOCAL);
    if (h) break;
  }
  if (!h) return api;
#define VT_SYM(f, name) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, name))
  VT_SYM(GetUniqueId, "ncclGetUniqueId");
  VT_SYM(CommInitRank, "ncclCommInitRank");
  VT_SYM(CommDestroy, "ncclCommDestroy");
  VT_SYM(Send, "ncclSend");
  VT_SYM(Recv, "ncclRecv");
  VT_SYM(GroupStart, "ncclGroupStart");
  VT_SYM(GroupEnd, "ncclGroupEnd");
  VT_SYM(AllGather, "ncclAllGather");
  VT_SYM(Broadcast, "ncclBroadcast");
  VT_SYM(GetErrorString, "ncclGetErrorString");
#undef VT_SYM
  api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.Send && api.Recv &&
           api.GroupStart && api.GroupEnd && api.AllGather && api.Broadcast;
  return api;
}


// ------------------------------------------------------------------ kernels
// one slab's CTA partials -> its rank slot (fixed order); `sel` picks the
// partial count from the iteration counter like pcg_s2 does (k % 50 == 0:
// true residual from the hex8 grid, else the recurrence from the dot grid)
__global__ void slab_sum_kernel(const PcgCtl* ctl, const double* partial, int n, int n50,
                                double* out) {
  griddep_wait();
  if (ctl && ctl->stop) return;
  const int cnt = (ctl && n50 > 0 && (ctl->k % 50) == 0) ? n50 : n;
  const double s = warp_sum_partials(partial, cnt);
  if (threadIdx.x == 0) *out = s;
}


}  // namespace vt



namespace vt {

static int lvl_k(int k, int l) { return k >> l; }

// ------------------------------------------------------------------ exchanges
// ghost node planes of level l for one vector per local slab
vt_status halo_nodes(vt_dist* D, int l, const std::vector<double*>& v, cudaStream_t s, const int* skip) {
  if (D->N == 1) return VT_OK;
  if (!D->remote()) {
    for (int i = 0; i < D->N; ++i) {
      const Geom& g = D->sl[i].lv[l]->g;
      const size_t pb = (size_t)g.nplane * sizeof(double);
      if (i > 0) {
        const Geom& gb = D->sl[i - 1].lv[l]->g;
        VT_CUDA(cudaMemcpyAsync(v[i], v[i - 1] + (size_t)(gb.k1 - gb.k0) * gb.nplane, pb,
                                cudaMemcpyDeviceToDevice, s));
      }
      if (i < D->N - 1)
        VT_CUDA(cudaMemcpyAsync(v[i] + (size_t)(g.k1 - g.k0 + 1) * g.nplane,
                                v[i + 1] + (size_t)g.nplane, pb, cudaMemcpyDeviceToDevice, s));
    }
    return VT_OK;
  }
  const DSlab& S = D->sl[0];
  const Geom& g = S.lv[l]->g;
  const int r = S.rank, n = g.k1 - g.k0;
  double* x = v[0];
  if (D->px)
    return peer_halo(D, x + (size_t)g.nplane, x + (size_t)n * g.nplane, x, x + (size_t)(n + 1) * g.nplane,
                     g.nplane, s, skip);
  auto& A = nccl();
  VT_NCCL(A.GroupStart());
  if (r > 0) {
    VT_NCCL(A.Send(x + (size_t)g.nplane, g.nplane, ncclDouble, r - 1, D->comm, s));
    VT_NCCL(A.Recv(x, g.nplane, ncclDouble, r - 1, D->comm, s));
  }
  if (r < D->N - 1) {
    VT_NCCL(A.Send(x + (size_t)n * g.nplane, g.nplane, ncclDouble, r + 1, D->comm, s));
    VT_NCCL(A.Recv(x + (size_t)(n + 1) * g.nplane, g.nplane, ncclDouble, r + 1, D->comm, s));
  }
  VT_NCCL(A.GroupEnd());
  return VT_OK;
}

// ghost element layer (q = 0) of level l: the neighbour below's top layer
vt_status halo_elems(vt_dist* D, int l, const std::vector<double*>& e, cudaStream_t s) {
  if (D->N == 1) return VT_OK;
  if (!D->remote()) {
    for (int i = 1; i < D->N; ++i) {
      const Geom& gb = D->sl[i - 1].lv[l]->g;
      VT_CUDA(cudaMemcpyAsync(e[i], e[i - 1] + (size_t)(gb.k1 - gb.k0) * gb.eplane,
                              (size_t)gb.eplane * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    return VT_OK;
  }
  const DSlab& S = D->sl[0];
  const Geom& g = S.lv[l]->g;
  const int r = S.rank, n = g.k1 - g.k0;
  if (D->px) {  // only the layer below travels (rank+1 pulls my top layer)
    PeerOps o;
    if (r < D->N - 1) {
      o.pack(e[0] + (size_t)n * g.eplane, (long long)D->px->half, g.eplane);
      o.wait(r + 1);
    }
    if (r > 0) {
      o.pull(r - 1, (long long)D->px->half, e[0], g.eplane);
      o.wait(r - 1);
    }
    return peer_exchange(D, o, s);
  }
  auto& A = nccl();
  VT_NCCL(A.GroupStart());
  if (r < D->N - 1) VT_NCCL(A.Send(e[0] + (size_t)n * g.eplane, g.eplane, ncclDouble, r + 1, D->comm, s));
  if (r > 0) VT_NCCL(A.Recv(e[0], g.eplane, ncclDouble, r - 1, D->comm, s));
  VT_NCCL(A.GroupEnd());
  return VT_OK;
}

// per-rank scalar slot -> complete on every rank
vt_status gather_scal(vt_dist* D, int slot, cudaStream_t s) {
  if (!D->remote()) return VT_OK;
  double* base = D->scal + (size_t)slot * D->N;
  if (D->px) {
    PeerOps o = peer_all_but_self(D);
    o.pack(base + D->sl[0].rank, 0, 1);
    for (int i = 0; i < o.nwait; ++i) o.pull(o.wpeer[i], 0, base + o.wpeer[i], 1);
    return peer_exchange(D, o, s);
  }
  VT_NCCL(nccl().AllGather(base + D->sl[0].rank, base, 1, ncclDouble, D->comm, s));
  return VT_OK;
}

vt_status slab_sum(vt_dist* D, int i, const double* partial, int n, int n50, int slot,
                          const PcgCtl* ctl, cudaStream_t s) {
  launch_pdl(slab_sum_kernel, 1, 32, 0, s, ctl, partial, n, n50,
                                   D->scal + (size_t)slot * D->N + D->sl[i].rank);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// host-side sum of a complete slot in rank order (setup scalars only)
vt_status host_slot_sum(vt_dist* D, int slot, cudaStream_t s, double* out) {
  VT_TRY(gather_scal(D, slot, s));
  VT_CUDA(cudaMemcpyAsync(D->host_scal, D->scal + (size_t)slot * D->N, D->N * sizeof(double),
                          cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  VT_TRY(peer_check(D));
  double acc = 0.0;
  for (int g = 0; g < D->N; ++g) acc += D->host_scal[g];
  *out = acc;
  return VT_OK;
}

vt_status host_slot_values(vt_dist* D, int slot, cudaStream_t s, double* out) {
  VT_TRY(gather_scal(D, slot, s));
  VT_CUDA(cudaMemcpyAsync(out, D->scal + (size_t)slot * D->N, D->N * sizeof(double),
                          cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  return peer_check(D);
}

// tail-level rhs ranges written by each rank -> every rank (C / f: the
// replicated grid of level D+1 and its rhs)
vt_status gather_tail_f(vt_dist* D, vt_grid* C, double* f, cudaStream_t s) {
  if (!D->remote()) return VT_OK;
  auto range = [&](int r, int* kb, int* ke) {
    const int a = lvl_k(D->kb[r], D->D), b = lvl_k(D->kb[r + 1], D->D) + (r == D->N - 1 ? 1 : 0);
    *kb = (a + 1) / 2;
    *ke = (b + 1) / 2;
  };
  if (D->px) {
    PeerOps o = peer_all_but_self(D);
    int kb, ke;
    range(D->sl[0].rank, &kb, &ke);
    if (ke > kb) o.pack(f + (size_t)(kb + 1) * C->g.nplane, 0, (long long)(ke - kb) * C->g.nplane);
    for (int i = 0; i < o.nwait; ++i) {
      range(o.wpeer[i], &kb, &ke);
      if (ke > kb)
        o.pull(o.wpeer[i], 0, f + (size_t)(kb + 1) * C->g.nplane, (long long)(ke - kb) * C->g.nplane);
    }
    return peer_exchange(D, o, s);
  }
  auto& A = nccl();
  VT_NCCL(A.GroupStart());
  for (int r = 0; r < D->N; ++r) {
    // each rank's range, recomputed from the plan (identical on all ranks)
    const int a = lvl_k(D->kb[r], D->D), b = lvl_k(D->kb[r + 1], D->D) + (r == D->N - 1 ? 1 : 0);
    const int kb = (a + 1) / 2, ke = (b + 1) / 2;
    if (ke <= kb) continue;
    double* p = f + (size_t)(kb + 1) * C->g.nplane;
    VT_NCCL(A.Broadcast(p, p, (size_t)(ke - kb) * C->g.nplane, ncclDouble, r, D->comm, s));
  }
  VT_NCCL(A.GroupEnd());
  return VT_OK;
}

// ------------------------------------------------------------------ V-cycle
// z = V(1,1) cycle of r (level-0 slab vectors); rz partials of the last fine
// smoother land in each slab's partial + 3*4096.  Capturable.
static vt_status dist_vcycle(vt_dist* D, const std::vector<const double*>& f0, const int* stop,
                             bool want_rz, cudaStream_t s) {
  if (D->scheme == 1) return dist_vcycle_galerkin(D, f0, stop, want_rz, s);
  const int NL = (int)D->sl.size();
  const int Dl = D->D;
  std::vector<std::vector<double*>> ucur(Dl + 1, std::vector<double*>(NL));
  auto fl = [&](int i, int l) -> const double* { return l == 0 ? f0[i] : D->sl[i].f[l]; };
  auto level_vec = [&](int l, std::vector<double*>& v) { return halo_nodes(D, l, v, s); };
  for (int l = 0; l <= Dl; ++l) {
    std::vector<double*> uu(NL), rr(NL);
    for (int i = 0; i < NL; ++i) {
      DSlab& S = D->sl[i];
      VT_TRY(launch_jacobi0w(S.lv[l], S.wd[l], fl(i, l), S.u[l], stop, s));
      ucur[l][i] = S.u[l];
      uu[i] = S.u[l];
      rr[i] = S.r[l];
    }
    VT_TRY(level_vec(l, uu));
    for (int i = 0; i < NL; ++i) {
      DSlab& S = D->sl[i];
      VT_TRY(launch_hex8(S.lv[l], H8_RESID, false, S.scale[l], S.u[l], S.u[l], fl(i, l), S.r[l],
                         0.0, nullptr, stop, s));
    }
    VT_TRY(level_vec(l, rr));
    for (int i = 0; i < NL; ++i) {
      DSlab& S = D->sl[i];
      if (l < Dl) {
        VT_TRY(launch_restrict(S.lv[l], S.lv[l + 1], S.r[l], S.f[l + 1], stop, -1, -1, s));
      } else {
        VT_TRY(launch_restrict(S.lv[l], D->tail->lv[1], S.r[l], D->tail->f[1], stop, S.tkb,
                               S.tke, s));
      }
    }
  }
  VT_TRY(gather_tail_f(D, D->tail->lv[1], D->tail->f[1], s));
  const double* zt = nullptr;
  VT_TRY(hier_vcycle_launch(D->tail, D->tail->f[1], stop, nullptr, false, s, &zt, 1));
  for (int l = Dl; l >= 0; --l) {
    if (l < Dl) VT_TRY(level_vec(l + 1, ucur[l + 1]));
    for (int i = 0; i < NL; ++i) {
      DSlab& S = D->sl[i];
      if (l == Dl)
        VT_TRY(launch_prolong_add(D->tail->lv[1], S.lv[l], zt, ucur[l][i], stop, s));
      else
        VT_TRY(launch_prolong_add(D->sl[i].lv[l + 1], S.lv[l], ucur[l + 1][i], ucur[l][i], stop, s));
    }
    for (int k = 0; k < D->sweeps; ++k) {
      VT_TRY(level_vec(l, ucur[l]));
      const bool dot = want_rz && l == 0 && k == D->sweeps - 1;
      for (int i = 0; i < NL; ++i) {
        DSlab& S = D->sl[i];
        double* dst = (ucur[l][i] == S.u[l]) ? S.u2[l] : S.u[l];
        VT_TRY(launch_hex8(S.lv[l], H8_SMOOTH, dot, S.scale[l], ucur[l][i], nullptr, fl(i, l),
                           dst, D->omega, S.lv[0]->partial + 3 * 4096, stop, s));
        ucur[l][i] = dst;
      }
    }
  }
  for (int i = 0; i < NL; ++i) D->sl[i].z = ucur[0][i];
  return VT_OK;
}

// ------------------------------------------------------------------ PCG graph
static vt_status dist_capture(vt_dist* D, cudaStream_t s) {
  PcgCtl* ctl = D->ctl;
  const int NL = (int)D->sl.size();
  const unsigned long long before = g_launches;
  VT_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  vt_status st = VT_OK;
  auto vecs = [&](double* DSlab::*m) {
    std::vector<double*> v(NL);
    for (int i = 0; i < NL; ++i) v[i] = D->sl[i].*m;
    return v;
  };
  do {
    // q = K p, p.q                                    [ref: solver.py:123-124]
    if ((st = halo_nodes(D, 0, vecs(&DSlab::p), s)) != VT_OK) break;
    for (int i = 0; i < NL && st == VT_OK; ++i) {
      DSlab& S = D->sl[i];
      vt_grid* G = S.lv[0];
      st = launch_hex8(G, H8_APPLY, true, S.scale[0], S.p, nullptr, nullptr, S.q, 0.0, G->partial,
                       &ctl->stop, s);
      if (st == VT_OK) st = slab_sum(D, i, G->partial, G->h8.grid, 0, 0, ctl, s);
    }
    if (st != VT_OK) break;
    if ((st = gather_scal(D, 0, s)) != VT_OK) break;
    if ((st = launch_pcg_s1(ctl, D->scal, D->N, s)) != VT_OK) break;
    // x += alpha p ; r -= alpha q | r = f - K x       [ref: solver.py:131-136]
    for (int i = 0; i < NL && st == VT_OK; ++i) {
      DSlab& S = D->sl[i];
      vt_grid* G = S.lv[0];
      st = launch_pcg_update(G, ctl, S.x, S.p, S.rr, S.q, G->partial + 4096, 1, s);
      if (st == VT_OK) st = launch_pcg_update(G, ctl, S.x, S.p, S.rr, S.q, G->partial + 4096, 0, s);
    }
    if (st != VT_OK) break;
    // x halo for the true residual; the peer transport skips it (and the
    // candidate's below) in the iterations that do not need it
    if ((st = halo_nodes(D, 0, vecs(&DSlab::x), s, &ctl->skip_true50)) != VT_OK) break;
    for (int i = 0; i < NL && st == VT_OK; ++i) {
      DSlab& S = D->sl[i];
      vt_grid* G = S.lv[0];
      st = launch_hex8(G, H8_RESID, true, S.scale[0], S.x, S.x, S.fv, S.rr, 0.0, G->partial + 4096,
                       &ctl->skip_true50, s);
      if (st == VT_OK) st = slab_sum(D, i, G->partial + 4096, dot_grid(G), G->h8.grid, 1, ctl, s);
    }
    if (st != VT_OK) break;
    if ((st = gather_scal(D, 1, s)) != VT_OK) break;
    if ((st = launch_pcg_s2(ctl, D->scal + D->N, D->N, D->N, s)) != VT_OK) break;
    // candidate not on a true-residual iteration: its x halo (peer transport;
    // the others exchanged x unconditionally above)
    if (D->px && (st = halo_nodes(D, 0, vecs(&DSlab::x), s, &ctl->skip_xc)) != VT_OK) break;
    // convergence candidate: true residual          [ref: solver.py:140-149]
    for (int i = 0; i < NL && st == VT_OK; ++i) {
      DSlab& S = D->sl[i];
      vt_grid* G = S.lv[0];
      st = launch_hex8(G, H8_RESID, true, S.scale[0], S.x, S.x, S.fv, S.t, 0.0, G->partial + 2 * 4096,
                       &ctl->skip_cand, s);
      if (st == VT_OK) st = slab_sum(D, i, G->partial + 2 * 4096, G->h8.grid, 0, 2, ctl, s);
    }
    if (st != VT_OK) break;
    if ((st = gather_scal(D, 2, s)) != VT_OK) break;
    if ((st = launch_pcg_s3(ctl, D->scal + 2 * D->N, D->N, s)) != VT_OK) break;
    for (int i = 0; i < NL && st == VT_OK; ++i)
      st = launch_copy(D->sl[i].lv[0], &ctl->skip_swap, D->sl[i].t, D->sl[i].rr, s);
    if (st != VT_OK) break;
    // z = M r ; r.z                                   [ref: solver.py:150-151]
    std::vector<const double*> r0(NL);
    for (int i = 0; i < NL; ++i) r0[i] = D->sl[i].rr;
    if ((st = dist_vcycle(D, r0, &ctl->stop, true, s)) != VT_OK) break;
    for (int i = 0; i < NL && st == VT_OK; ++i) {
      vt_grid* G = D->sl[i].lv[0];
      st = slab_sum(D, i, G->partial + 3 * 4096, G->h8.grid, 0, 3, ctl, s);
    }
    if (st != VT_OK) break;
    if ((st = gather_scal(D, 3, s)) != VT_OK) break;
    if ((st = launch_pcg_s4(ctl, D->scal + 3 * D->N, D->N, 1, s)) != VT_OK) break;
    // p = z + beta p                                  [ref: solver.py:158]
    for (int i = 0; i < NL && st == VT_OK; ++i)
      st = launch_pcg_xpby(D->sl[i].lv[0], ctl, D->sl[i].z, D->sl[i].p, s);
  } while (0);
  cudaGraph_t graph = nullptr;
  cudaError_t ce = cudaStreamEndCapture(s, &graph);
  if (st != VT_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaStreamEndCapture (dist)");
  D->nodes = g_launches - before;
  g_launches = before;
  if (D->graph) cudaGraphExecDestroy(D->graph);
  D->graph = nullptr;
  ce = cudaGraphInstantiate(&D->graph, graph, 0);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess) return cuda_fail(ce, "cudaGraphInstantiate (dist)");
  return VT_OK;
}

static vt_status alloc_zero(double** p, size_t n) {
  VT_CUDA(cudaMalloc(p, n * sizeof(double)));
  VT_CUDA(cudaMemset(*p, 0, n * sizeof(double)));
  return VT_OK;
}

}  // namespace vt

using namespace vt;

extern "C" {

vt_status vt_nccl_unique_id(uint8_t* out, int nbytes) {
  if (!out || nbytes < (int)sizeof(ncclUniqueId)) return fail(VT_EINVAL, "id buffer too small");
  auto& A = nccl();
  if (!A.ok) return fail(VT_ECUDA, "NCCL library not found (set VT_NCCL_LIB)");
  ncclUniqueId id;
  VT_NCCL(A.GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return VT_OK;
}

int vt_nccl_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

}  // extern "C"

static vt_status dist_create(vt_dist** out, int nx, int ny, int nz, double h, double nu,
                             const uint8_t* node_mask, int levels, double omega, int nranks,
                             int rank0, int nlocal, const int* kbounds, int dist_level,
                             const uint8_t* nccl_id, bool peer, int device) {
  if (!out || !node_mask || !kbounds) return fail(VT_EINVAL, "null argument");
  if (nranks < 1 || nlocal < 1 || rank0 < 0 || rank0 + nlocal > nranks)
    return fail(VT_EINVAL, "bad rank layout");
  const bool multi = nccl_id != nullptr || peer;
  if (!multi && nlocal != nranks)
    return fail(VT_EINVAL, "without a transport every slab must live in this process");
  if (multi && nlocal != 1)
    return fail(VT_EINVAL, "with a multi-process transport each process owns exactly one slab");
  if (levels < 2) return fail(VT_EINVAL, "the slab solver needs at least 2 multigrid levels");
  if (dist_level < 0 || dist_level > levels - 2)
    return fail(VT_EINVAL, "distributed levels must leave a replicated coarse tail");
  if (kbounds[0] != 0 || kbounds[nranks] != nz) return fail(VT_EINVAL, "slab bounds must cover [0, nz)");
  const int step = 1 << dist_level;
  for (int r = 0; r < nranks; ++r) {
    if (kbounds[r + 1] <= kbounds[r] || (kbounds[r] % step) != 0)
      return fail(VT_EINVAL, "slab bounds must be increasing multiples of 2^dist_level");
  }
  for (int l = 0; l < levels - 1; ++l) {
    if (((nx >> l) & 1) || ((ny >> l) & 1) || ((nz >> l) & 1))
      return fail(VT_EINVAL, "grid dimensions do not support this many levels");
  }
  VT_CUDA(cudaSetDevice(device));
  vt_dist* D = new vt_dist();
  D->N = nranks; D->rank0 = rank0; D->nlocal = nlocal; D->L = levels; D->D = dist_level;
  D->device = device; D->omega = omega; D->nx = nx; D->ny = ny; D->nz = nz;
  D->kb.assign(kbounds, kbounds + nranks + 1);
  D->h = h;
  D->nu = nu;
  D->node_mask.assign(node_mask, node_mask + (size_t)(nx + 1) * (ny + 1) * (nz + 1));
  vt_status st = VT_OK;
  auto bail = [&](vt_status s2) { vt_dist_destroy(D); return s2; };
  if (nccl_id) {
    auto& A = nccl();
    if (!A.ok) return bail(fail(VT_ECUDA, "NCCL library not found (set VT_NCCL_LIB)"));
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    ncclResult_t r = A.CommInitRank(&D->comm, nranks, id, rank0);
    if (r != ncclSuccess) return bail(fail(VT_ECUDA, "ncclCommInitRank failed"));
  }
  D->sl.resize(nlocal);
  for (int i = 0; i < nlocal; ++i) {
    DSlab& S = D->sl[i];
    S.rank = rank0 + i;
    const int k0 = kbounds[S.rank], k1 = kbounds[S.rank + 1];
    double hl = h;
    for (int l = 0; l <= dist_level; ++l) {
      vt_grid* G = nullptr;
      st = vt_grid_create(&G, nx >> l, ny >> l, nz >> l, hl, nu, l == 0 ? node_mask : nullptr,
                          k0 >> l, k1 >> l, device);
      if (st != VT_OK) return bail(st);
      if (l > 0) {
        st = launch_coarsen_mask(S.lv[l - 1], G, 0);
        if (st != VT_OK) { vt_grid_destroy(G); return bail(st); }
      }
      S.lv.push_back(G);
      hl *= 2.0;
    }
    const int NLv = dist_level + 1;
    S.u.assign(NLv, nullptr); S.u2.assign(NLv, nullptr); S.r.assign(NLv, nullptr);
    S.f.assign(NLv, nullptr); S.scale.assign(NLv, nullptr); S.rho.assign(NLv, nullptr);
    S.wd.assign(NLv, nullptr);
    for (int l = 0; l < NLv; ++l) {
      vt_grid* G = S.lv[l];
      const size_t vl = G->vec_len(), el = G->elem_len();
      if ((st = alloc_zero(&S.u[l], vl)) || (st = alloc_zero(&S.u2[l], vl)) ||
          (st = alloc_zero(&S.wd[l], vl)) ||
          (st = alloc_zero(&S.r[l], vl)) || (st = alloc_zero(&S.f[l], vl)) ||
          (st = alloc_zero(&S.scale[l], el)) || (st = alloc_zero(&S.rho[l], G->nel_local())))
        return bail(st);
    }
    vt_grid* G = S.lv[0];
    const size_t vl = G->vec_len();
    if ((st = alloc_zero(&S.x, vl)) || (st = alloc_zero(&S.fv, vl)) || (st = alloc_zero(&S.rr, vl)) ||
        (st = alloc_zero(&S.p, vl)) || (st = alloc_zero(&S.q, vl)) || (st = alloc_zero(&S.t, vl)))
      return bail(st);
    const int a = k0 >> dist_level, b = (k1 >> dist_level) + (k1 == nz ? 1 : 0);
    S.tkb = (a + 1) / 2;
    S.tke = (b + 1) / 2;
  }
  // replicated full grid of level D (mask = fine mask at nodes that are multiples of 2^D)
  {
    const int fx = nx >> dist_level, fy = ny >> dist_level, fz = nz >> dist_level;
    std::vector<uint8_t> m((size_t)(fx + 1) * (fy + 1) * (fz + 1));
    for (int k = 0; k <= fz; ++k)
      for (int j = 0; j <= fy; ++j)
        for (int i = 0; i <= fx; ++i)
          m[((size_t)k * (fy + 1) + j) * (fx + 1) + i] =
              node_mask[(((size_t)k << dist_level) * (ny + 1) + ((size_t)j << dist_level)) * (nx + 1) +
                        ((size_t)i << dist_level)];
    st = vt_grid_create(&D->full, fx, fy, fz, h * (double)(1 << dist_level), nu, m.data(), 0, fz,
                        device);
    if (st != VT_OK) return bail(st);
    st = vt_hier_create(&D->tail, D->full, levels - dist_level, omega, 1);
    if (st != VT_OK) return bail(st);
    if ((st = alloc_zero(&D->rho_full, D->full->nel_local())) ||
        (st = alloc_zero(&D->scale_full, D->full->elem_len())))
      return bail(st);
  }
  if ((st = alloc_zero(&D->scal, (size_t)NSLOT * nranks))) return bail(st);
  if (cudaMallocHost(&D->host_scal, NSLOT * nranks * sizeof(double)) != cudaSuccess)
    return bail(fail(VT_ENOMEM, "pinned alloc"));
  if (cudaMalloc(&D->ctl, sizeof(PcgCtl)) != cudaSuccess ||
      cudaMallocHost(&D->ctl_host, 2 * sizeof(PcgCtl)) != cudaSuccess)
    return bail(fail(VT_ENOMEM, "control block alloc"));
  if (cudaStreamCreateWithFlags(&D->stream, cudaStreamNonBlocking) != cudaSuccess)
    return bail(fail(VT_ECUDA, "stream create"));
  if (peer) {
    // staging: halves large enough for a level-0 node plane, an element layer
    // and PEER_MAX_R filter layers; the whole area for one rank's share of the
    // tail right-hand side / the level-D densities
    const Geom& g0 = D->sl[0].lv[0]->g;
    const long long layer = (long long)nx * ny;
    long long half = g0.nplane;
    half = half > g0.eplane ? half : g0.eplane;
    half = half > PEER_MAX_R * layer ? half : PEER_MAX_R * layer;
    long long whole = 2 * half;
    vt_grid* C = D->tail->lv[1];
    const long long per_layer = (long long)(nx >> dist_level) * (ny >> dist_level);
    for (int r = 0; r < nranks; ++r) {
      const int a = kbounds[r] >> dist_level, b = (kbounds[r + 1] >> dist_level) + (r == nranks - 1 ? 1 : 0);
      const long long tf = (long long)((b + 1) / 2 - (a + 1) / 2) * C->g.nplane;
      const long long rd = (long long)((kbounds[r + 1] - kbounds[r]) >> dist_level) * per_layer;
      whole = whole > tf ? whole : tf;
      whole = whole > rd ? whole : rd;
    }
    st = peer_init(D, (size_t)(whole + (whole & 1)));
    if (st != VT_OK) return bail(st);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return bail(fail(VT_ECUDA, "dist setup"));
  *out = D;
  return VT_OK;
}

extern "C" {

vt_status vt_dist_create(vt_dist** out, int nx, int ny, int nz, double h, double nu,
                         const uint8_t* node_mask, int levels, double omega, int nranks,
                         int rank0, int nlocal, const int* kbounds, int dist_level,
                         const uint8_t* nccl_id, int device) {
  return dist_create(out, nx, ny, nz, h, nu, node_mask, levels, omega, nranks, rank0, nlocal, kbounds,
                     dist_level, nccl_id, false, device);
}

vt_status vt_dist_create_peer(vt_dist** out, int nx, int ny, int nz, double h, double nu,
                              const uint8_t* node_mask, int levels, double omega, int nranks,
                              int rank, const int* kbounds, int dist_level, int device) {
  return dist_create(out, nx, ny, nz, h, nu, node_mask, levels, omega, nranks, rank, 1, kbounds,
                     dist_level, nullptr, true, device);
}

vt_status vt_dist_destroy(vt_dist* D) {
  if (!D) return VT_OK;
  cudaSetDevice(D->device);
  if (D->graph) cudaGraphExecDestroy(D->graph);
  if (D->stream) cudaStreamDestroy(D->stream);
  for (DSlab& S : D->sl) {
    for (size_t l = 0; l < S.lv.size(); ++l) {
      if (l < S.u.size()) {
        cudaFree(S.u[l]); cudaFree(S.u2[l]); cudaFree(S.r[l]); cudaFree(S.f[l]);
        cudaFree(S.scale[l]); cudaFree(S.rho[l]); cudaFree(S.wd[l]);
      }
      vt_grid_destroy(S.lv[l]);
    }
    double* w[] = {S.x, S.fv, S.rr, S.p, S.q, S.t};
    for (double* p : w) cudaFree(p);
  }
  if (D->tail) vt_hier_destroy(D->tail);
  if (D->full) vt_grid_destroy(D->full);
  cudaFree(D->rho_full); cudaFree(D->scale_full); cudaFree(D->scal); cudaFreeHost(D->host_scal);
  cudaFree(D->ctl); cudaFreeHost(D->ctl_host);
  cudaFree(D->fw); cudaFree(D->opart);
  for (double* p : D->fwsum) cudaFree(p);
  for (double* p : D->fprod) cudaFree(p);
  for (double* p : D->gpad) cudaFree(p);
  if (D->comm) nccl().CommDestroy(D->comm);
  dist_galerkin_free(D);
  peer_free(D);
  delete D;
  return VT_OK;
}

int vt_dist_levels(const vt_dist* D) { return D ? D->L : 0; }
int vt_dist_dist_level(const vt_dist* D) { return D ? D->D : -1; }
int vt_dist_nlocal(const vt_dist* D) { return D ? D->nlocal : 0; }
vt_grid* vt_dist_grid(vt_dist* D, int i, int level) {
  if (!D || i < 0 || i >= D->nlocal || level < 0 || level > D->D) return nullptr;
  return D->sl[i].lv[level];
}
vt_hier* vt_dist_tail(vt_dist* D) { return D ? D->tail : nullptr; }
uint64_t vt_dist_graph_nodes(const vt_dist* D) { return D ? D->nodes : 0; }

// level-0 scale of every local slab (vt element layout of the slab grid); the
// ghost element layer is filled from the neighbour below.
vt_status vt_dist_set_scale(vt_dist* D, const double* const* scale0, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double*> e(D->nlocal);
  for (int i = 0; i < D->nlocal; ++i) {
    DSlab& S = D->sl[i];
    VT_CUDA(cudaMemcpyAsync(S.scale[0], scale0[i], S.lv[0]->elem_len() * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
    e[i] = S.scale[0];
  }
  return halo_elems(D, 0, e, s);
}

// homogenized coarse levels of every slab, the replicated tail and its
// coarsest factor [ref: multigrid.py:201-233, 280-316]; rho: plain slab
// densities (n_elements of the slab), scale0: level-0 slab scales.  Blocking.
vt_status vt_dist_refresh(vt_dist* D, const double* const* rho, const double* const* scale0,
                          double p, double kmin, double E, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  VT_CUDA(cudaSetDevice(D->device));
  VT_TRY(vt_dist_set_scale(D, scale0, stream));
  if (D->scheme == 1) {
    VT_TRY(dist_refresh_galerkin(D, p, kmin, E, s));
    D->refreshed = true;
    return VT_OK;
  }
  int* bad = reinterpret_cast<int*>(D->sl[0].lv[0]->scalars);
  VT_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  for (int i = 0; i < D->nlocal; ++i) {
    DSlab& S = D->sl[i];
    VT_CUDA(cudaMemcpyAsync(S.rho[0], rho[i], S.lv[0]->nel_local() * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
  }
  for (int l = 1; l <= D->D; ++l) {
    std::vector<double*> e(D->nlocal);
    for (int i = 0; i < D->nlocal; ++i) {
      DSlab& S = D->sl[i];
      VT_TRY(launch_coarsen_rho(S.lv[l - 1], S.lv[l], S.rho[l - 1], S.rho[l], s));
      VT_TRY(launch_scale(S.lv[l], S.rho[l], p, kmin, E, S.scale[l], bad, s));
      e[i] = S.scale[l];
    }
    VT_TRY(halo_elems(D, l, e, s));
  }
  for (int l = 0; l <= D->D; ++l)
    for (DSlab& S : D->sl) VT_TRY(launch_wdiag(S.lv[l], S.scale[l], D->omega, S.wd[l], s));
  // gather level-D densities into the replicated full grid (slab = contiguous range)
  const long long per_layer = (long long)(D->nx >> D->D) * (D->ny >> D->D);
  if (!D->remote()) {
    for (int i = 0; i < D->nlocal; ++i) {
      DSlab& S = D->sl[i];
      vt_grid* G = S.lv[D->D];
      VT_CUDA(cudaMemcpyAsync(D->rho_full + (long long)G->g.k0 * per_layer, S.rho[D->D],
                              G->nel_local() * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
  } else if (D->px) {
    PeerOps o = peer_all_but_self(D);
    const DSlab& S = D->sl[0];
    const long long own = (long long)(D->kb[S.rank] >> D->D) * per_layer;
    VT_CUDA(cudaMemcpyAsync(D->rho_full + own, S.rho[D->D], S.lv[D->D]->nel_local() * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
    o.pack(S.rho[D->D], 0, S.lv[D->D]->nel_local());
    for (int i = 0; i < o.nwait; ++i) {
      const int r = o.wpeer[i];
      const long long a = (long long)(D->kb[r] >> D->D) * per_layer;
      const long long b = (long long)(D->kb[r + 1] >> D->D) * per_layer;
      o.pull(r, 0, D->rho_full + a, b - a);
    }
    VT_TRY(peer_exchange(D, o, s));
  } else {
    auto& A = nccl();
    VT_CUDA(cudaMemcpyAsync(D->rho_full + (long long)(D->kb[D->sl[0].rank] >> D->D) * per_layer,
                            D->sl[0].rho[D->D], D->sl[0].lv[D->D]->nel_local() * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
    VT_NCCL(A.GroupStart());
    for (int r = 0; r < D->N; ++r) {
      const long long a = (long long)(D->kb[r] >> D->D) * per_layer;
      const long long b = (long long)(D->kb[r + 1] >> D->D) * per_layer;
      VT_NCCL(A.Broadcast(D->rho_full + a, D->rho_full + a, (size_t)(b - a), ncclDouble, r, D->comm, s));
    }
    VT_NCCL(A.GroupEnd());
  }
  VT_TRY(launch_scale(D->full, D->rho_full, p, kmin, E, D->scale_full, bad, s));
  int hb = 0;
  VT_CUDA(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  VT_CUDA(cudaStreamSynchronize(s));
  VT_TRY(peer_check(D));
  if (hb) return fail(VT_EDENSITY, "density outside [0, 1]");
  VT_TRY(vt_hier_refresh(D->tail, D->rho_full, D->scale_full, p, kmin, E, stream));
  D->refreshed = true;
  return VT_OK;
}

// v = K u on every local slab (u zero on fixed dofs, e.g. a solver vector);
// u's ghost planes are exchanged first (u is modified in its ghost planes).
vt_status vt_dist_apply(vt_dist* D, double* const* u, double* const* v, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  std::vector<double*> uu(u, u + D->nlocal);
  VT_TRY(halo_nodes(D, 0, uu, s));
  for (int i = 0; i < D->nlocal; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_hex8(S.lv[0], H8_APPLY, false, S.scale[0], u[i], nullptr, nullptr, v[i], 0.0,
                       nullptr, nullptr, s));
  }
  return VT_OK;
}

// x . y over all slabs of all ranks (rank-ordered sum); blocking
vt_status vt_dist_dot(vt_dist* D, const double* const* x, const double* const* y, double* out,
                      void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  for (int i = 0; i < D->nlocal; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    int n = 0;
    VT_TRY(launch_dot(G, x[i], y[i], G->partial + 4 * 4096, &n, s));
    VT_TRY(slab_sum(D, i, G->partial + 4 * 4096, n, 0, 4, nullptr, s));
  }
  return host_slot_sum(D, 4, s, out);
}

// z = V-cycle(f) through the slab hierarchy (f zero on fixed dofs)
vt_status vt_dist_vcycle(vt_dist* D, const double* const* f, double* const* z, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!D->refreshed) return fail(VT_ESETUP, "hierarchy was not refreshed before use");
  std::vector<const double*> ff(f, f + D->nlocal);
  VT_TRY(dist_vcycle(D, ff, nullptr, false, s));
  for (int i = 0; i < D->nlocal; ++i)
    VT_CUDA(cudaMemcpyAsync(z[i], D->sl[i].z, D->sl[i].lv[0]->vec_len() * sizeof(double),
                            cudaMemcpyDeviceToDevice, s));
  return VT_OK;
}

// Multigrid-preconditioned CG across the slabs, same recurrences and checks as
// vt_pcg [ref: solver.py:62-191].  f, x: level-0 slab vectors (x: warm start
// in, solution out).  Blocking; every rank must call it.
vt_status vt_dist_pcg(vt_dist* D, const double* const* f, double* const* x, int warm, double tol,
                      int maxit, vt_solve_report* rep, void* stream) {
  VT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  VT_CUDA(cudaSetDevice(D->device));
  cudaStream_t s = D->stream;
  if (!rep) return fail(VT_EINVAL, "null report");
  memset(rep, 0, sizeof(*rep));
  if (!D->refreshed) return fail(VT_ESETUP, "hierarchy was not refreshed before use");
  const int NL = D->nlocal;
  // ||f||                                          [ref: solver.py:81-95]
  for (int i = 0; i < NL; ++i) {
    vt_grid* G = D->sl[i].lv[0];
    int n = 0;
    VT_TRY(launch_dot(G, f[i], f[i], G->partial, &n, s));
    VT_TRY(slab_sum(D, i, G->partial, n, 0, 5, nullptr, s));
  }
  double ff = 0.0;
  VT_TRY(host_slot_sum(D, 5, s, &ff));
  const double fnorm = sqrt(ff);
  if (!isfinite(fnorm)) {
    rep->breakdown = 5;
    return fail(VT_EBREAKDOWN, "rhs contains non-finite entries");
  }
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    vt_grid* G = S.lv[0];
    const size_t vb = G->vec_len() * sizeof(double);
    if (warm)
      VT_TRY(launch_project(G, x[i], S.x, s));
    else
      VT_CUDA(cudaMemsetAsync(S.x, 0, vb, s));
    VT_CUDA(cudaMemcpyAsync(S.fv, f[i], vb, cudaMemcpyDeviceToDevice, s));
  }
  auto finish = [&]() -> vt_status {
    for (int i = 0; i < NL; ++i)
      VT_CUDA(cudaMemcpyAsync(x[i], D->sl[i].x, D->sl[i].lv[0]->vec_len() * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
    VT_CUDA(cudaStreamSynchronize(s));
    return peer_check(D);
  };
  if (fnorm == 0.0) {
    VT_TRY(finish());
    rep->converged = 1;
    return VT_OK;
  }
  auto true_residual = [&](double* rel) -> vt_status {
    std::vector<double*> xs(NL);
    for (int i = 0; i < NL; ++i) xs[i] = D->sl[i].x;
    VT_TRY(halo_nodes(D, 0, xs, s));
    for (int i = 0; i < NL; ++i) {
      DSlab& S = D->sl[i];
      vt_grid* G = S.lv[0];
      VT_TRY(launch_hex8(G, H8_RESID, true, S.scale[0], S.x, S.x, S.fv, S.rr, 0.0,
                         G->partial + 4096, nullptr, s));
      VT_TRY(slab_sum(D, i, G->partial + 4096, G->h8.grid, 0, 6, nullptr, s));
    }
    double rr = 0.0;
    VT_TRY(host_slot_sum(D, 6, s, &rr));
    *rel = sqrt(rr) / fnorm;
    return VT_OK;
  };
  double rel = 0.0;
  VT_TRY(true_residual(&rel));
  if (rel <= tol) {
    VT_TRY(finish());
    rep->converged = 1;
    rep->final_rel_residual = rel;
    return VT_OK;
  }
  // z = M r, p = z, rz = r.z                      [ref: solver.py:105-118]
  std::vector<const double*> r0(NL);
  for (int i = 0; i < NL; ++i) r0[i] = D->sl[i].rr;
  VT_TRY(dist_vcycle(D, r0, nullptr, true, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    vt_grid* G = S.lv[0];
    VT_TRY(slab_sum(D, i, G->partial + 3 * 4096, G->h8.grid, 0, 3, nullptr, s));
    VT_CUDA(cudaMemcpyAsync(S.p, S.z, G->vec_len() * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  double rz = 0.0;
  VT_TRY(host_slot_sum(D, 3, s, &rz));
  rep->precond_applications = 1;
  if (!isfinite(rz) || rz <= 0.0) {
    rep->breakdown = 1;
    rep->breakdown_value = rz;
    return fail(VT_EBREAKDOWN, "preconditioned product r'z is not positive at iteration 0; "
                               "preconditioner is not SPD");
  }
  PcgCtl c0;
  memset(&c0, 0, sizeof(c0));
  c0.rz = rz;
  c0.fnorm = fnorm;
  c0.tol = tol;
  c0.rel = rel;
  c0.precond_apps = 1;
  c0.skip_cand = 1;
  c0.skip_swap = 1;
  VT_CUDA(cudaMemcpyAsync(D->ctl, &c0, sizeof(c0), cudaMemcpyHostToDevice, s));
  if (!D->graph) {
    VT_CUDA(cudaStreamSynchronize(s));
    VT_TRY(dist_capture(D, s));
  }
  PcgCtl* ring = D->ctl_host;
  cudaEvent_t ev[2];
  VT_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  VT_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  auto launch_iter = [&](int i) -> vt_status {
    VT_CUDA(cudaGraphLaunch(D->graph, s));
    g_launches += D->nodes;
    VT_CUDA(cudaMemcpyAsync(&ring[i & 1], D->ctl, sizeof(PcgCtl), cudaMemcpyDeviceToHost, s));
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
    if (e != cudaSuccess) { st = cuda_fail(e, "dist pcg iteration"); break; }
    if ((st = peer_check(D)) != VT_OK) break;
    if (ring[i & 1].stop) break;
  }
  cudaStreamSynchronize(s);
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  if (st != VT_OK) return st;
  PcgCtl c;
  VT_CUDA(cudaMemcpy(&c, D->ctl, sizeof(c), cudaMemcpyDeviceToHost));
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
  if (!c.converged) VT_TRY(true_residual(&final_rel));  // [ref: solver.py:161-167]
  rep->final_rel_residual = final_rel;
  rep->converged = final_rel <= tol;
  return finish();
}

}  // extern "C"
