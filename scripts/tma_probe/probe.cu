// Standalone probe: one 3D TMA load of a double tensor into smem (debug tool).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include "../../paper_2201_12931_b200/csrc/vt_device.cuh"
using namespace vt;
__global__ void k(const __grid_constant__ CUtensorMap m, int x, int y, int z, int bytes, double* out, int n) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_fence_init(); }
  __syncthreads();
  if (threadIdx.x == 0) { mbar_expect_tx(&bar, bytes); tma_load_3d(sm, &m, &bar, x, y, z); }
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = ((double*)sm)[i];
}
int main(int argc, char** argv) {
  int d0 = atoi(argv[1]), d1 = atoi(argv[2]), d2 = atoi(argv[3]), b0 = atoi(argv[4]), b1 = atoi(argv[5]);
  int x = atoi(argv[6]), y = atoi(argv[7]); int pitch = atoi(argv[8]); int dyn = argc > 9 ? atoi(argv[9]) : 0;
  size_t N = (size_t)pitch * d1 * d2;
  double* h = (double*)malloc(N * 8); for (size_t i = 0; i < N; ++i) h[i] = (double)i;
  double *g, *o; cudaMalloc(&g, N * 8); cudaMemcpy(g, h, N * 8, cudaMemcpyHostToDevice);
  int n = b0 * b1; cudaMalloc(&o, n * 8);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m; cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t st[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)pitch * 8 * d1};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, 1}, es[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d  ", (int)r);
  if (dyn) cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  int z = argc > 10 ? atoi(argv[10]) : 0;
  k<<<1, 128, dyn ? 140000 : n * 8 + 128>>>(m, x, y, z, n * 8, o, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("dims(%d,%d,%d) box(%d,%d) at(%d,%d) pitch %d dyn %d -> %s", d0, d1, d2, b0, b1, x, y, pitch, dyn, cudaGetErrorString(e));
  if (e == cudaSuccess) { double* ho = (double*)malloc(n * 8); cudaMemcpy(ho, o, n * 8, cudaMemcpyDeviceToHost);
    printf("  first %g %g .. row1 %g", ho[0], ho[1], ho[b0]); }
  printf("\n");
  return 0;
}
