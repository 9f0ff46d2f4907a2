// The reference's default coarse scheme (Galerkin) on z-slabs
// [ref: multigrid.py:216-278; SURVEY 8(e)].
//
// Level 0 (the fine hex8 operator) and level 1 are slab-distributed; levels
// >= 2 run replicated on every rank:
//  * Level 1 is applied matrix-free, K1 x = Pi1 P^T (Pi0 K0 Pi0) P Pi1 x, with
//    the slab pieces of the single-GPU path: prolongation into the fine slab,
//    the TMA hex8 apply, restriction back (one halo-plane exchange before each
//    pass), then the level-1 epilogue with the level-1 diagonal.
//  * Its diagonal and the stored matrices of levels >= 2 depend on all fine
//    scales of a coarse element's children (64 fine elements for a level-2
//    element), which straddle slab boundaries; so every refresh gathers the
//    whole fine scale field (one element layer per rank and layer, cheap next
//    to a solve) into a replicated whole-grid Galerkin hierarchy `gtail` and
//    builds the level-1 diagonal, the level >= 2 matrices and the coarsest
//    factor there with the single-GPU kernels -- the same operations in the
//    same order, so the slab V-cycle equals the single-GPU one.
//  * Each slab restricts its level-1 residual into the level-2 planes whose
//    centre plane it owns (written into gtail's level-2 rhs, ranges
//    exchanged), the replicated tail V-cycle runs from level 2, and its
//    correction is prolongated straight into each level-1 slab.
#include <string.h>

#include "dist_internal.h"

namespace vt {

void dist_galerkin_free(vt_dist* D) {
  for (double* p : D->gfa) cudaFree(p);
  for (double* p : D->gfb) cudaFree(p);
  for (double* p : D->gc1) cudaFree(p);
  for (double* p : D->gd1) cudaFree(p);
  D->gfa.clear();
  D->gfb.clear();
  D->gc1.clear();
  D->gd1.clear();
  if (D->gtail) vt_hier_destroy(D->gtail);
  if (D->gfine) vt_grid_destroy(D->gfine);
  D->gtail = nullptr;
  D->gfine = nullptr;
}

static vt_status zalloc(double** p, size_t n) {
  VT_CUDA(cudaMalloc(p, n * sizeof(double)));
  VT_CUDA(cudaMemset(*p, 0, n * sizeof(double)));
  return VT_OK;
}

// every rank's element layers of the fine scale -> the replicated whole-grid
// scale (vt element layout; layer k of the grid is layer q = k + 1)
static vt_status gather_fine_scale(vt_dist* D, cudaStream_t s) {
  double* full = D->gtail->scale[0];
  const long long ep = D->gfine->g.eplane;
  for (int i = 0; i < D->nlocal; ++i) {  // own layers (every transport)
    const DSlab& S = D->sl[i];
    const Geom& g = S.lv[0]->g;
    VT_CUDA(cudaMemcpyAsync(full + (long long)(g.k0 + 1) * ep, S.scale[0] + ep,
                            (size_t)(g.k1 - g.k0) * ep * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  if (!D->remote()) return VT_OK;
  const int me = D->sl[0].rank;
  if (D->px) {  // in chunks of the staging area: every rank pulls every other rank's layers
    const long long chunk = (long long)D->px->stage_doubles;
    long long maxn = 0;
    for (int r = 0; r < D->N; ++r) maxn = std::max<long long>(maxn, (long long)(D->kb[r + 1] - D->kb[r]) * ep);
    for (long long off = 0; off < maxn; off += chunk) {
      PeerOps o = peer_all_but_self(D);
      const long long mine = (long long)(D->kb[me + 1] - D->kb[me]) * ep;
      if (off < mine)
        o.pack(full + (long long)(D->kb[me] + 1) * ep + off, 0, std::min(chunk, mine - off));
      for (int w = 0; w < o.nwait; ++w) {
        const int r = o.wpeer[w];
        const long long n = (long long)(D->kb[r + 1] - D->kb[r]) * ep;
        if (off < n) o.pull(r, 0, full + (long long)(D->kb[r] + 1) * ep + off, std::min(chunk, n - off));
      }
      VT_TRY(peer_exchange(D, o, s));
    }
    return VT_OK;
  }
  auto& A = nccl();
  VT_NCCL(A.GroupStart());
  for (int r = 0; r < D->N; ++r) {
    double* p = full + (long long)(D->kb[r] + 1) * ep;
    VT_NCCL(A.Broadcast(p, p, (size_t)(D->kb[r + 1] - D->kb[r]) * ep, ncclDouble, r, D->comm, s));
  }
  VT_NCCL(A.GroupEnd());
  return VT_OK;
}

vt_status dist_refresh_galerkin(vt_dist* D, double p, double kmin, double E, cudaStream_t s) {
  // level 0: damped inverse diagonal of the slab operator (as the homogenized path)
  for (DSlab& S : D->sl) VT_TRY(launch_wdiag(S.lv[0], S.scale[0], D->omega, S.wd[0], s));
  VT_TRY(gather_fine_scale(D, s));
  // level-1 diagonal, level >= 2 matrices, coarsest factor on the whole grid
  VT_TRY(hier_refresh_levels(D->gtail, p, kmin, E, s));
  // each slab's owned planes of the level-1 diagonal (same plane layout)
  for (int i = 0; i < D->nlocal; ++i) {
    const DSlab& S = D->sl[i];
    const Geom& g = S.lv[1]->g;
    VT_CUDA(cudaMemcpyAsync(D->gd1[i] + (long long)g.pA * g.nplane,
                            D->gtail->gdiag[1] + (long long)(g.pA + g.k0) * g.nplane,
                            (size_t)(g.pB - g.pA) * g.nplane * sizeof(double), cudaMemcpyDeviceToDevice, s));
  }
  VT_CUDA(cudaStreamSynchronize(s));
  return peer_check(D);
}

// level-1 operator on the slabs: mode 1 residual (out = f - K1 u), mode 2 damped Jacobi
static vt_status level1_op(vt_dist* D, int mode, const std::vector<double*>& u,
                           const std::vector<const double*>& f, const std::vector<double*>& out,
                           const int* stop, cudaStream_t s) {
  const int NL = (int)D->sl.size();
  std::vector<double*> uu(u), fa(NL), fb(NL);
  VT_TRY(halo_nodes(D, 1, uu, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_prolong_set(S.lv[1], S.lv[0], u[i], D->gfa[i], stop, s));
    fa[i] = D->gfa[i];
    fb[i] = D->gfb[i];
  }
  VT_TRY(halo_nodes(D, 0, fa, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_hex8(S.lv[0], H8_APPLY, false, S.scale[0], D->gfa[i], nullptr, nullptr, D->gfb[i], 0.0,
                       nullptr, stop, s));
  }
  VT_TRY(halo_nodes(D, 0, fb, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_restrict(S.lv[0], S.lv[1], D->gfb[i], D->gc1[i], stop, -1, -1, s));
    VT_TRY(launch_gal_vec_epilogue(S.lv[1], mode, D->gc1[i], u[i], f[i], D->gd1[i], D->omega, out[i],
                                   stop, s));
  }
  return VT_OK;
}

// z = V(1,1) cycle of the level-0 slab vectors f0 (Galerkin); the rz partials
// of the last fine smoother land in each slab's partial + 3*4096.  Capturable.
vt_status dist_vcycle_galerkin(vt_dist* D, const std::vector<const double*>& f0, const int* stop,
                               bool want_rz, cudaStream_t s) {
  const int NL = (int)D->sl.size();
  vt_hier* T = D->gtail;
  std::vector<double*> u0(NL), r0(NL), u1(NL), r1(NL), u1b(NL);
  std::vector<const double*> f1(NL);
  // level 0: u = w f, r = f - K u, restrict into the level-1 slabs
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_jacobi0w(S.lv[0], S.wd[0], f0[i], S.u[0], stop, s));
    u0[i] = S.u[0];
    r0[i] = S.r[0];
    u1[i] = S.u[1];
    u1b[i] = S.u2[1];
    r1[i] = S.r[1];
    f1[i] = S.f[1];
  }
  VT_TRY(halo_nodes(D, 0, u0, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_hex8(S.lv[0], H8_RESID, false, S.scale[0], S.u[0], S.u[0], f0[i], S.r[0], 0.0, nullptr,
                       stop, s));
  }
  VT_TRY(halo_nodes(D, 0, r0, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_restrict(S.lv[0], S.lv[1], S.r[0], S.f[1], stop, -1, -1, s));
  }
  // level 1: first sweep from zero, residual (matrix-free), restrict into the tail's level 2
  for (int i = 0; i < NL; ++i)
    VT_TRY(launch_gal_jacobi0(D->sl[i].lv[1], D->sl[i].f[1], D->gd1[i], D->omega, D->sl[i].u[1], stop, s));
  VT_TRY(level1_op(D, 1, u1, f1, r1, stop, s));
  VT_TRY(halo_nodes(D, 1, r1, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_restrict(S.lv[1], T->lv[2], S.r[1], T->f[2], stop, S.tkb, S.tke, s));
  }
  VT_TRY(gather_tail_f(D, T->lv[2], T->f[2], s));
  // replicated stored-matrix tail, levels >= 2
  const double* zt = nullptr;
  VT_TRY(hier_vcycle_launch(T, T->f[2], stop, nullptr, false, s, &zt, 2));
  // up: level 2 -> 1, smooth (matrix-free), level 1 -> 0, smooth (+ r.z)
  for (int i = 0; i < NL; ++i)
    VT_TRY(launch_prolong_add(T->lv[2], D->sl[i].lv[1], zt, D->sl[i].u[1], stop, s));
  VT_TRY(level1_op(D, 2, u1, f1, u1b, stop, s));
  VT_TRY(halo_nodes(D, 1, u1b, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_prolong_add(S.lv[1], S.lv[0], S.u2[1], S.u[0], stop, s));
  }
  VT_TRY(halo_nodes(D, 0, u0, s));
  for (int i = 0; i < NL; ++i) {
    DSlab& S = D->sl[i];
    VT_TRY(launch_hex8(S.lv[0], H8_SMOOTH, want_rz, S.scale[0], S.u[0], nullptr, f0[i], S.u2[0], D->omega,
                       S.lv[0]->partial + 3 * 4096, stop, s));
    S.z = S.u2[0];
  }
  return VT_OK;
}

}  // namespace vt

using namespace vt;

extern "C" {

// switch a slab set to the Galerkin scheme (before the first refresh)
vt_status vt_dist_set_scheme(vt_dist* D, int scheme) {
  if (!D) return fail(VT_EINVAL, "null slab set");
  if (scheme == D->scheme) return VT_OK;
  if (scheme != 1) return fail(VT_EINVAL, "a slab set can only be switched to the Galerkin scheme (1)");
  if (D->D != 1) return fail(VT_EINVAL, "the Galerkin slab scheme distributes levels 0 and 1 (dist_level 1)");
  if (D->L < 3) return fail(VT_EINVAL, "the Galerkin slab scheme needs at least 3 multigrid levels");
  VT_CUDA(cudaSetDevice(D->device));
  vt_status st = vt_grid_create(&D->gfine, D->nx, D->ny, D->nz, D->h, D->nu, D->node_mask.data(), 0, D->nz,
                                D->device);
  if (st != VT_OK) return st;
  st = vt_hier_create_ex(&D->gtail, D->gfine, D->L, D->omega, D->sweeps, 1);
  if (st != VT_OK) {
    dist_galerkin_free(D);
    return st;
  }
  // the replicated hierarchy only runs levels >= 2: drop its whole-grid
  // level-0 / level-1 work vectors (its level-0 scale and level-1 diagonal stay)
  vt_hier* T = D->gtail;
  for (int l = 0; l < 2; ++l) {
    double** v[] = {&T->u[l], &T->u2[l], &T->r[l], &T->rho[l], &T->wd[l]};
    for (double** q : v) {
      cudaFree(*q);
      *q = nullptr;
    }
  }
  cudaFree(T->f[1]); T->f[1] = nullptr;
  cudaFree(T->gfa); T->gfa = nullptr;
  cudaFree(T->gfb); T->gfb = nullptr;
  cudaFree(T->gc1); T->gc1 = nullptr;
  D->gfa.assign(D->nlocal, nullptr);
  D->gfb.assign(D->nlocal, nullptr);
  D->gc1.assign(D->nlocal, nullptr);
  D->gd1.assign(D->nlocal, nullptr);
  for (int i = 0; i < D->nlocal; ++i) {
    const DSlab& S = D->sl[i];
    if ((st = zalloc(&D->gfa[i], S.lv[0]->vec_len())) || (st = zalloc(&D->gfb[i], S.lv[0]->vec_len())) ||
        (st = zalloc(&D->gc1[i], S.lv[1]->vec_len())) || (st = zalloc(&D->gd1[i], S.lv[1]->vec_len()))) {
      dist_galerkin_free(D);
      return st;
    }
  }
  if (D->graph) {
    cudaGraphExecDestroy(D->graph);
    D->graph = nullptr;
  }
  D->scheme = 1;
  D->refreshed = false;
  VT_CUDA(cudaDeviceSynchronize());
  return VT_OK;
}

int vt_dist_scheme(const vt_dist* D) { return D ? D->scheme : -1; }

}  // extern "C"
