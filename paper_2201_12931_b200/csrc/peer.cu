// Peer-memory transport of the z-slab decomposition: one slab per process,
// exchanges by direct loads from the neighbours' device memory (CUDA IPC;
// over NVLink / NVSwitch when the ranks sit on different GPUs of one box, or
// the same HBM when several ranks share one GPU, which is how the
// multi-process path is tested on a single B200).
//
// Every rank owns one IPC-shared block: a 256-byte flag header (monotonic
// `ready` / `done` epochs) followed by a staging area.  One exchange is ONE
// kernel (capturable into the PCG iteration graph, no host round trip):
//
//   1. pack: copy the rank's outgoing planes / scalars into its own staging
//      area (so any buffer, library- or torch-owned, can be exchanged);
//   2. the last CTA to finish packing publishes ready = e (release, system scope);
//   3. every CTA waits for ready >= e of the peers it pulls from, then pulls
//      their staged data straight into its ghost planes / slots;
//   4. the last CTA to finish pulling publishes done = e and waits for the
//      peers' done >= e, so no peer repacks its staging area while this rank
//      is still reading it (and vice versa).
//
// All ranks issue the same sequence of exchanges (the same precondition the
// NCCL transport has), so the epoch e -- a device-resident counter bumped by
// every exchange kernel -- names the same exchange on every rank.  A spin
// that waits more than VT_PEER_TIMEOUT_S seconds (default 60) gives up, sets
// an error word in mapped host memory and the host call fails with VT_ECUDA
// instead of hanging the device.
#include <stdlib.h>
#include <string.h>

#include "dist_internal.h"

namespace vt {

constexpr int XP_THREADS = 256;
constexpr size_t XP_HEADER = 256;  // bytes of flags before the staging area

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// wait until flag >= e on every listed peer; false on timeout
__device__ bool wait_flags(unsigned long long* const* fl, int nw, int which, unsigned long long e,
                           unsigned long long timeout_ns, int* err) {
  const unsigned long long t0 = globaltimer();
  for (int w = 0; w < nw; ++w) {
    const unsigned long long* f = fl[w] + which;
    unsigned spins = 0;
    while (ld_acquire_sys(f) < e) {
      if (*(volatile int*)err) return false;
      if ((++spins & 1023u) == 0 && globaltimer() - t0 > timeout_ns) {
        atomicExch(err, 1);
        __threadfence_system();
        return false;
      }
    }
  }
  return true;
}

__global__ void __launch_bounds__(XP_THREADS)
    xchg_kernel(XArgs a) {
  // a conditional exchange (same flag value on every rank): no epoch is used
  if (a.skip && *(volatile const int*)a.skip) return;
  __shared__ unsigned long long e;
  __shared__ int ok;
  if (threadIdx.x == 0) {
    e = *(volatile unsigned long long*)&a.ctr[0] + 1;
    ok = 1;
  }
  __syncthreads();
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nth = (long long)gridDim.x * blockDim.x;
  // 1. pack outgoing data into the own staging area
  for (int o = 0; o < a.npack; ++o) {
    const double* src = a.psrc[o];
    double* dst = a.stage + a.poff[o];
    for (long long i = tid; i < a.pn[o]; i += nth) dst[i] = src[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(&a.cnt[0], 1u);
    if (prev == gridDim.x - 1) {  // every CTA packed: publish
      a.cnt[0] = 0;
      st_release_sys(&a.self[0], e);
    }
    // 2. the peers this rank pulls from have packed
    if (!wait_flags(a.wflag, a.nwait, 0, e, a.timeout_ns, a.err)) ok = 0;
  }
  __syncthreads();
  // 3. pull the peers' staged data (bypassing L1: the same addresses are
  //    reused by every exchange)
  if (ok) {
    for (int o = 0; o < a.npull; ++o) {
      const double* src = a.qsrc[o];
      double* dst = a.qdst[o];
      for (long long i = tid; i < a.qn[o]; i += nth) dst[i] = __ldcg(src + i);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned prev = atomicAdd(&a.cnt[1], 1u);
    if (prev == gridDim.x - 1) {  // 4. every CTA pulled: release the peers, wait for theirs
      a.cnt[1] = 0;
      st_release_sys(&a.self[1], e);
      wait_flags(a.wflag, a.nwait, 1, e, a.timeout_ns, a.err);
      *(volatile unsigned long long*)&a.ctr[0] = e;
      __threadfence();
    }
  }
}

}  // namespace vt

using namespace vt;

namespace vt {

static double peer_timeout_s() {
  const char* t = getenv("VT_PEER_TIMEOUT_S");
  const double v = t ? atof(t) : 60.0;
  return v > 0 ? v : 60.0;
}

vt_status peer_init(vt_dist* D, size_t stage_doubles) {
  PeerXport* P = new PeerXport();
  D->px = P;
  P->stage_doubles = stage_doubles;
  P->half = stage_doubles / 2;
  const size_t bytes = XP_HEADER + stage_doubles * sizeof(double);
  VT_CUDA(cudaMalloc(&P->block, bytes));
  VT_CUDA(cudaMemset(P->block, 0, bytes));
  VT_CUDA(cudaMalloc(&P->local, 64));
  VT_CUDA(cudaMemset(P->local, 0, 64));
  VT_CUDA(cudaHostAlloc(&P->err_host, sizeof(int), cudaHostAllocMapped));
  *P->err_host = 0;
  VT_CUDA(cudaHostGetDevicePointer(&P->err_dev, P->err_host, 0));
  P->peer_block.assign(D->N, nullptr);
  P->timeout_ns = (unsigned long long)(peer_timeout_s() * 1e9);
  return VT_OK;
}

void peer_free(vt_dist* D) {
  PeerXport* P = D->px;
  if (!P) return;
  const int me = D->sl.empty() ? -1 : D->sl[0].rank;
  for (int r = 0; r < (int)P->peer_block.size(); ++r)
    if (P->peer_block[r] && r != me) cudaIpcCloseMemHandle(P->peer_block[r]);
  cudaFree(P->block);
  cudaFree(P->local);
  if (P->err_host) cudaFreeHost(P->err_host);
  delete P;
  D->px = nullptr;
}

static unsigned long long* flags_of(void* block) { return reinterpret_cast<unsigned long long*>(block); }
static double* stage_of(void* block) {
  return reinterpret_cast<double*>(reinterpret_cast<char*>(block) + XP_HEADER);
}

vt_status peer_check(vt_dist* D) {
  if (D->px && *(volatile int*)D->px->err_host)
    return fail(VT_ECUDA, "peer exchange timed out (a rank stopped exchanging or the ranks issued "
                          "different exchange sequences)");
  return VT_OK;
}

vt_status peer_exchange(vt_dist* D, const PeerOps& ops, cudaStream_t s) {
  PeerXport* P = D->px;
  if (!P || !P->opened) return fail(VT_ESETUP, "peer transport is not connected");
  if (ops.npack > XP_MAXOPS || ops.npull > XP_MAXOPS || ops.nwait > XP_MAXOPS)
    return fail(VT_EINVAL, "too many peer exchange operations");
  XArgs a = {};
  a.stage = stage_of(P->block);
  a.self = flags_of(P->block);
  a.ctr = reinterpret_cast<unsigned long long*>(P->local);
  a.cnt = reinterpret_cast<unsigned*>(reinterpret_cast<char*>(P->local) + 16);
  a.err = P->err_dev;
  a.timeout_ns = P->timeout_ns;
  a.skip = ops.skip;
  long long total = 0;
  a.npack = ops.npack;
  for (int i = 0; i < ops.npack; ++i) {
    if (ops.poff[i] < 0 || (size_t)(ops.poff[i] + ops.pn[i]) > P->stage_doubles)
      return fail(VT_EINVAL, "peer exchange exceeds the staging area");
    a.psrc[i] = ops.psrc[i];
    a.poff[i] = ops.poff[i];
    a.pn[i] = ops.pn[i];
    total = ops.pn[i] > total ? ops.pn[i] : total;
  }
  a.npull = ops.npull;
  for (int i = 0; i < ops.npull; ++i) {
    const int r = ops.qpeer[i];
    if (r < 0 || r >= D->N || !P->peer_block[r]) return fail(VT_EINVAL, "bad peer rank");
    if (ops.qoff[i] < 0 || (size_t)(ops.qoff[i] + ops.qn[i]) > P->stage_doubles)
      return fail(VT_EINVAL, "peer exchange exceeds the staging area");
    a.qsrc[i] = stage_of(P->peer_block[r]) + ops.qoff[i];
    a.qdst[i] = ops.qdst[i];
    a.qn[i] = ops.qn[i];
    total = ops.qn[i] > total ? ops.qn[i] : total;
  }
  a.nwait = ops.nwait;
  for (int i = 0; i < ops.nwait; ++i) {
    const int r = ops.wpeer[i];
    if (r < 0 || r >= D->N || !P->peer_block[r]) return fail(VT_EINVAL, "bad peer rank");
    a.wflag[i] = flags_of(P->peer_block[r]);
  }
  // every CTA must be resident at once (they spin on the peers): one per SM at most
  const int grid = fit_grid(total, 4LL * XP_THREADS, D->sl[0].lv[0]->nsm);
  xchg_kernel<<<grid, XP_THREADS, 0, s>>>(a);
  count_launch();
  VT_CUDA(cudaGetLastError());
  return VT_OK;
}

// all peers except this rank
PeerOps peer_all_but_self(vt_dist* D) {
  PeerOps o;
  const int me = D->sl[0].rank;
  for (int r = 0; r < D->N; ++r)
    if (r != me) o.wpeer[o.nwait++] = r;
  return o;
}

}  // namespace vt

extern "C" {

vt_status vt_dist_peer_handle(vt_dist* D, uint8_t* out, int nbytes) {
  if (!D || !D->px) return fail(VT_EINVAL, "not a peer-transport slab set");
  if (!out || nbytes < (int)sizeof(cudaIpcMemHandle_t)) return fail(VT_EINVAL, "handle buffer too small");
  cudaIpcMemHandle_t h;
  VT_CUDA(cudaIpcGetMemHandle(&h, D->px->block));
  memcpy(out, &h, sizeof(h));
  return VT_OK;
}

int vt_peer_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }

// handles: nranks consecutive handles in rank order (this rank's own entry is ignored)
vt_status vt_dist_peer_open(vt_dist* D, const uint8_t* handles, int nbytes) {
  if (!D || !D->px) return fail(VT_EINVAL, "not a peer-transport slab set");
  const int hb = (int)sizeof(cudaIpcMemHandle_t);
  if (!handles || nbytes < D->N * hb) return fail(VT_EINVAL, "handle array too small");
  VT_CUDA(cudaSetDevice(D->device));
  PeerXport* P = D->px;
  const int me = D->sl[0].rank;
  for (int r = 0; r < D->N; ++r) {
    if (r == me) {
      P->peer_block[r] = P->block;
      continue;
    }
    if (P->peer_block[r]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + (size_t)r * hb, hb);
    void* p = nullptr;
    VT_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    P->peer_block[r] = p;
  }
  P->opened = true;
  return VT_OK;
}

}  // extern "C"

namespace vt {

vt_status peer_halo(vt_dist* D, const double* down, const double* up, double* below, double* above,
                    long long n, cudaStream_t s, const int* skip) {
  PeerXport* P = D->px;
  if ((size_t)n > P->half) return fail(VT_EINVAL, "halo exceeds the peer staging area");
  const int r = D->sl[0].rank;
  PeerOps o;
  if (r > 0) {
    o.pack(down, 0, n);                          // my first planes -> rank-1
    o.pull(r - 1, (long long)P->half, below, n);  // rank-1's last planes
    o.wait(r - 1);
  }
  if (r < D->N - 1) {
    o.pack(up, (long long)P->half, n);           // my last planes -> rank+1
    o.pull(r + 1, 0, above, n);                  // rank+1's first planes
    o.wait(r + 1);
  }
  o.skip = skip;
  return peer_exchange(D, o, s);
}

}  // namespace vt
