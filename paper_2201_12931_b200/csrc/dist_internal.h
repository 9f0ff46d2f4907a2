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

// ------------------------------------------------------------------ peer transport (peer.cu)
constexpr int XP_MAXOPS = 16;
constexpr int PEER_MAX_R = 8;  // filter half-widths the peer staging area holds

// one exchange: pack own data into the staging area, pull peers' staged data
struct PeerOps {
  int npack = 0, npull = 0, nwait = 0;
  const double* psrc[XP_MAXOPS];
  long long poff[XP_MAXOPS], pn[XP_MAXOPS];  // staging offset / count (doubles)
  int qpeer[XP_MAXOPS];
  long long qoff[XP_MAXOPS], qn[XP_MAXOPS];
  double* qdst[XP_MAXOPS];
  int wpeer[XP_MAXOPS];                       // ranks synchronised with (symmetric)
  const int* skip = nullptr;                  // device word: nonzero = skip the whole exchange
                                              // (every rank reads the same value)
  void pack(const double* src, long long off, long long n) {
    psrc[npack] = src; poff[npack] = off; pn[npack] = n; ++npack;
  }
  void pull(int peer, long long off, double* dst, long long n) {
    qpeer[npull] = peer; qoff[npull] = off; qdst[npull] = dst; qn[npull] = n; ++npull;
  }
  void wait(int peer) { wpeer[nwait++] = peer; }
};

struct XArgs {
  int npack, npull, nwait;
  const double* psrc[XP_MAXOPS];
  long long poff[XP_MAXOPS], pn[XP_MAXOPS];
  const double* qsrc[XP_MAXOPS];
  double* qdst[XP_MAXOPS];
  long long qn[XP_MAXOPS];
  unsigned long long* wflag[XP_MAXOPS];
  double* stage;
  unsigned long long* self;   // own flags: [0] ready, [1] done
  unsigned long long* ctr;    // local: [0] epoch
  unsigned* cnt;              // local: [0] packers, [1] pullers
  int* err;                   // mapped host word
  const int* skip;            // see PeerOps::skip
  unsigned long long timeout_ns;
};

struct PeerXport {
  void* block = nullptr;              // IPC-shared: 256 B flags + staging
  void* local = nullptr;              // epoch + CTA counters (not shared)
  size_t stage_doubles = 0, half = 0; // staging area; halo exchanges use [0, half) down, [half, 2 half) up
  std::vector<void*> peer_block;      // every rank's block in this address space
  int* err_host = nullptr;
  int* err_dev = nullptr;
  unsigned long long timeout_ns = 0;
  bool opened = false;
};

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

  vt::PeerXport* px = nullptr;         // peer-memory transport (peer.cu), else NCCL when comm
  // Galerkin scheme on slabs (dist_galerkin.cu)
  int scheme = 0;                      // 0 homogenized, 1 galerkin (needs dist level 1)
  double h = 0.0, nu = 0.3;
  std::vector<uint8_t> node_mask;      // host copy of the fine fixed mask (whole grid)
  vt_grid* gfine = nullptr;            // the whole fine grid (replicated)
  vt_hier* gtail = nullptr;            // whole Galerkin hierarchy; its levels >= 2 are the tail
  std::vector<double*> gfa, gfb, gc1, gd1;  // per slab: level-0 / level-1 scratch, level-1 diagonal

  bool remote() const { return comm != nullptr || px != nullptr; }
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

// skip (peer transport only): device word read by the exchange kernel; nonzero
// on every rank = no exchange (the other transports always exchange)
vt_status halo_nodes(vt_dist* D, int l, const std::vector<double*>& v, cudaStream_t s,
                     const int* skip = nullptr);
vt_status halo_elems(vt_dist* D, int l, const std::vector<double*>& e, cudaStream_t s);
vt_status gather_scal(vt_dist* D, int slot, cudaStream_t s);
vt_status slab_sum(vt_dist* D, int i, const double* partial, int n, int n50, int slot,
                   const PcgCtl* ctl, cudaStream_t s);
vt_status host_slot_sum(vt_dist* D, int slot, cudaStream_t s, double* out);
vt_status host_slot_values(vt_dist* D, int slot, cudaStream_t s, double* out);
vt_status gather_tail_f(vt_dist* D, vt_grid* C, double* f, cudaStream_t s);
vt_status dist_vcycle_galerkin(vt_dist* D, const std::vector<const double*>& f0, const int* stop,
                               bool want_rz, cudaStream_t s);
vt_status dist_refresh_galerkin(vt_dist* D, double p, double kmin, double E, cudaStream_t s);
void dist_galerkin_free(vt_dist* D);
vt_status peer_init(vt_dist* D, size_t stage_doubles);
void peer_free(vt_dist* D);
vt_status peer_check(vt_dist* D);
vt_status peer_exchange(vt_dist* D, const PeerOps& ops, cudaStream_t s);
PeerOps peer_all_but_self(vt_dist* D);
// neighbour halo: send `down` (n doubles) to rank-1 and `up` to rank+1, receive
// rank-1's `up` into below and rank+1's `down` into above
vt_status peer_halo(vt_dist* D, const double* down, const double* up, double* below, double* above,
                    long long n, cudaStream_t s, const int* skip = nullptr);
}  // namespace vt
