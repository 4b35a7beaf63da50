// Minimal TMA 2D load test: variants via argv[1]:
//  0: map as __grid_constant__ param, entry point default
//  1: map as __grid_constant__ param, entry point by version 12000
//  2: map in global memory, entry point by version 12000
//  3: like 1 + 3.5 KB of extra kernel params
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../../paper_1511_02490_b200/csrc/stencil/kernels.cuh"
using namespace sk;
struct Big { long long w[441]; };
__global__ void k_param(const __grid_constant__ CUtensorMap map, float* out, int bw, int bh) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, bw * bh * 4); tma_load_2d(smem, &map, bar, -1, -1); }
  __syncthreads();
  mbar_wait_parity(bar, 0);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}
__global__ void k_big(const __grid_constant__ CUtensorMap map, float* out, int bw, int bh, const __grid_constant__ Big b) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, bw * bh * 4); tma_load_2d(smem, &map, bar, -1, -1); }
  __syncthreads();
  mbar_wait_parity(bar, 0);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i] + (float)b.w[i % 441];
}
__global__ void k_global(const CUtensorMap* map, float* out, int bw, int bh) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_barrier_init(); fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, bw * bh * 4); tma_load_2d(smem, map, bar, -1, -1); }
  __syncthreads();
  mbar_wait_parity(bar, 0);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int v = argc > 1 ? atoi(argv[1]) : 0;
  int W = 64, H = 32, bw = 36, bh = 10;
  float* in; float* out; cudaMalloc(&in, W * H * 4); cudaMalloc(&out, bw * bh * 4);
  float* h = (float*)malloc(W * H * 4); for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  cudaMemcpy(in, h, W * H * 4, cudaMemcpyHostToDevice);
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaError_t e;
  if (v == 0) e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  else e = cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
  printf("entry e=%d q=%d p=%p\n", (int)e, (int)q, p);
  CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H}; cuuint64_t str[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}; cuuint32_t es[2] = {1, 1};
  CUresult r = ((Enc)p)(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, in, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode r=%d\n", (int)r);
  cudaFuncSetAttribute(k_param, cudaFuncAttributeMaxDynamicSharedMemorySize, 9000);
  cudaFuncSetAttribute(k_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 9000);
  cudaFuncSetAttribute(k_global, cudaFuncAttributeMaxDynamicSharedMemorySize, 9000);
  if (v == 2) { CUtensorMap* dm; cudaMalloc(&dm, sizeof(CUtensorMap)); cudaMemcpy(dm, &m, sizeof m, cudaMemcpyHostToDevice); k_global<<<1, 128, 9000>>>(dm, out, bw, bh); }
  else if (v == 3) { Big b{}; k_big<<<1, 128, 9000>>>(m, out, bw, bh, b); }
  else k_param<<<1, 128, 9000>>>(m, out, bw, bh);
  e = cudaDeviceSynchronize();
  printf("variant %d: %s\n", v, cudaGetErrorString(e));
  float* ho = (float*)malloc(bw * bh * 4); cudaMemcpy(ho, out, bw * bh * 4, cudaMemcpyDeviceToHost);
  printf("out[0]=%g out[1]=%g out[37]=%g (want 0, 0, 0 then row1: out[37]=%g)\n", ho[0], ho[1], ho[37], 0.0);
  return 0;
}
