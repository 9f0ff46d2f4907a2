// Microbenchmark (runs ON the GPU box): cost of one "phase" of the fused tail
// kernel -- cluster barrier alone, and barrier + one dependent L2 load/store
// round trip per thread -- for 16-CTA clusters of 512 threads.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/micro scripts/micro_phase.cu && /tmp/micro
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gt() {
  unsigned long long g;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
  return g;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) phases(double* buf, int n, unsigned long long* out, int iters) {
  cg::cluster_group cl = cg::this_cluster();
  const int t = blockIdx.x * blockDim.x + threadIdx.x, nt = gridDim.x * blockDim.x;
  cl.sync();
  const unsigned long long t0 = gt();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1) {
      // read a neighbour's value written in the previous phase, write own
      for (int i = t; i < n; i += nt) buf[(it & 1) * n + i] = __ldcg(buf + ((it + 1) & 1) * n + (i + 97) % n) + 1.0;
    } else if (MODE == 2) {
      // 24 independent loads per item (element-phase shape)
      for (int i = t; i < n; i += nt) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 24; ++k) s += __ldcg(buf + ((it + 1) & 1) * n + (i * 7 + k * 131) % n);
        buf[(it & 1) * n + i] = s;
      }
    }
    cl.sync();
  }
  const unsigned long long t1 = gt();
  if (t == 0) out[MODE] = (t1 - t0) / iters;
}

int main() {
  double* buf;
  unsigned long long* out;
  const int n = 8192;
  cudaMalloc(&buf, 2 * n * sizeof(double));
  cudaMemset(buf, 0, 2 * n * sizeof(double));
  cudaMallocManaged(&out, 8 * sizeof(unsigned long long));
  for (int cs : {8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaFuncSetAttribute(phases<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(phases<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(phases<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaLaunchKernelEx(&cfg, phases<0>, buf, n, out, 1000);
      cudaLaunchKernelEx(&cfg, phases<1>, buf, n, out, 1000);
      cudaLaunchKernelEx(&cfg, phases<2>, buf, n, out, 1000);
      cudaError_t e = cudaDeviceSynchronize();
      printf("cluster %d: barrier only %llu ns, + 1 ldcg/st per thread %llu ns, + 24 ldcg per item %llu ns (%s)\n",
             cs, out[0], out[1], out[2], cudaGetErrorString(e));
    }
  }
  return 0;
}
