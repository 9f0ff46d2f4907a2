// Internals of the z-slab runtime shared by dist.cu (solve) and
// dist_design.cu (per-SIMP-iteration design kernels).
#pragma once
#include <nccl.h>

#include <string>
#include <vector>

#include "vt_internal.h"
#include "vt_pcg.cuh"

namespace vt {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl();

struct DSlab {
  int rank = 0;
  std::vector<vt_grid*> lv;                       // levels 0..D (slab geometry)
  std::vector<double*> u, u2, r, f, scale, rho;   // per level; f[0] unused
  std::vector<double*> wd;                        // omega / diag per dof (refresh)
  double *x = nullptr, *fv = nullptr, *rr = nullptr, *p = nullptr, *q = nullptr, *t = nullptr;
  const double* z = nullptr;                      // V-cycle output buffer (level 0)
  int tkb = 0, tke = 0;                           // tail-level coarse planes restricted here
};

constexpr int NSLOT = 16;

}  // namespace vt

struct vt_dist {
  int N = 1, rank0 = 0, nlocal = 1, L = 1, D = 0, device = 0, sweeps = 1;
  double omega = 0.4;
  int nx = 0, ny = 0, nz = 0;
  std::vector<int> kb;                 // level-0 slab boundaries (N + 1)
  std::vector<vt::DSlab> sl;           // slabs of this process
  vt_grid* full = nullptr;             // replicated full grid of level D
  vt_hier* tail = nullptr;             // levels D..L-1 on every rank
  double* rho_full = nullptr;          // level-D densities, plain, full grid
  double* scale_full = nullptr;        // level-D scale, vt element layout
  double* scal = nullptr;              // device [NSLOT][N] per-rank scalars
  double* host_scal = nullptr;         // pinned mirror
  vt::PcgCtl* ctl = nullptr;
  vt::PcgCtl* ctl_host = nullptr;      // pinned ring of 2
  cudaGraphExec_t graph = nullptr;
  unsigned long long nodes = 0;
  cudaStream_t stream = nullptr;
  ncclComm_t comm = nullptr;
  bool refreshed = false;
  // distributed sensitivity filter (dist_design.cu)
  int fR = -1;
  double* fw = nullptr;                 // (2R+1)^3 kernel
  std::vector<double*> fwsum, fprod;    // per slab: correlate(1), rho*dc with R ghost layers
  double* opart = nullptr;              // OC / change partials (per slab, 4096 x 4)
  std::vector<double*> gpad;            // per slab: rho with the element layer below (gravity)

  bool remote() const { return comm != nullptr; }
};

namespace vt {
#define VT_NCCL(call)                                                                        \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      return ::vt::fail(VT_ECUDA, std::string("NCCL error ") +                               \
                                      (nccl().GetErrorString ? nccl().GetErrorString(r_) : "") + \
                                      " at " #call);                                         \
  } while (0)

vt_status halo_nodes(vt_dist* D, int l, const std::vector<double*>& v, cudaStream_t s);
vt_status halo_elems(vt_dist* D, int l, const std::vector<double*>& e, cudaStream_t s);
vt_status gather_scal(vt_dist* D, int slot, cudaStream_t s);
vt_status slab_sum(vt_dist* D, int i, const double* partial, int n, int n50, int slot,
                   const PcgCtl* ctl, cudaStream_t s);
vt_status host_slot_sum(vt_dist* D, int slot, cudaStream_t s, double* out);
vt_status host_slot_values(vt_dist* D, int slot, cudaStream_t s, double* out);
}  // namespace vt
