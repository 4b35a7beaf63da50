// argv: x0 y0 bw l2promo use_cccl direct_link
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda/ptx>
#include <cstdio>
#include <cstdlib>
#include "../../paper_1511_02490_b200/csrc/stencil/kernels.cuh"
using namespace sk;
__global__ void k(const __grid_constant__ CUtensorMap map, float* out, int bw, int bh, int x0, int y0, int cccl) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8192);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1); fence_barrier_init(); fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, bw * bh * 4);
    if (cccl) {
      int32_t c[2] = {x0, y0};
      cuda::ptx::cp_async_bulk_tensor(cuda::ptx::space_cluster, cuda::ptx::space_global, smem, &map, c, bar);
    } else {
      tma_load_2d(smem, &map, bar, x0, y0);
    }
  }
  __syncthreads();
  mbar_wait_parity(bar, 0);
  for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) out[i] = reinterpret_cast<float*>(smem)[i];
}
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main(int argc, char** argv) {
  int x0 = atoi(argv[1]), y0 = atoi(argv[2]), bw = atoi(argv[3]), promo = atoi(argv[4]), cccl = atoi(argv[5]), direct = atoi(argv[6]);
  int W = 64, H = 32, bh = 10;
  float* in; float* out; cudaMalloc(&in, W * H * 4); cudaMalloc(&out, bw * bh * 4);
  float* h = (float*)malloc(W * H * 4); for (int i = 0; i < W * H; ++i) h[i] = (float)i;
  cudaMemcpy(in, h, W * H * 4, cudaMemcpyHostToDevice);
  Enc fn;
  if (direct) fn = cuTensorMapEncodeTiled;
  else { void* p; cudaDriverEntryPointQueryResult q; cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q); fn = (Enc)p; }
  CUtensorMap m; cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)H}; cuuint64_t str[1] = {(cuuint64_t)W * 4};
  cuuint32_t box[2] = {(cuuint32_t)bw, (cuuint32_t)bh}; cuuint32_t es[2] = {1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, in, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 9000);
  k<<<1, 128, 9000>>>(m, out, bw, bh, x0, y0, cccl);
  cudaError_t e = cudaDeviceSynchronize();
  float* ho = (float*)malloc(bw * bh * 4); cudaMemcpy(ho, out, bw * bh * 4, cudaMemcpyDeviceToHost);
  printf("x0=%d y0=%d bw=%d promo=%d cccl=%d direct=%d encode=%d -> %s  out[0]=%g out[bw]=%g\n", x0, y0, bw, promo, cccl, direct, (int)r, cudaGetErrorString(e), ho[0], ho[bw]);
  return 0;
}
