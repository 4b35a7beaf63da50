// Exhaustive check of sk::div_const_rn<28> against IEEE division for all
// 2^32 fp32 bit patterns (NaN results compare as NaN); prints the mismatch
// count and exits non-zero on any.  Built and run by tests/test_div_const.py.
#include <cstdio>
#include <cstdint>
#include "ops.cuh"

__global__ void check(unsigned long long base, unsigned long long* bad, unsigned* first) {
  const unsigned long long i = base + blockIdx.x * static_cast<unsigned long long>(blockDim.x) + threadIdx.x;
  const float s = __uint_as_float(static_cast<uint32_t>(i));
  const float a = sk::div_const_rn<28>(s);
  const float b = __fdiv_rn(s, 28.0f);
  const bool same = __float_as_uint(a) == __float_as_uint(b) || (a != a && b != b);
  if (!same) {
    atomicAdd(bad, 1ull);
    atomicMin(first, static_cast<uint32_t>(i));
  }
}

int main() {
  unsigned long long* bad;
  unsigned* first;
  cudaMalloc(&bad, sizeof(*bad));
  cudaMalloc(&first, sizeof(*first));
  cudaMemset(bad, 0, sizeof(*bad));
  cudaMemset(first, 0xff, sizeof(*first));
  const unsigned long long chunk = 1ull << 30;
  for (unsigned long long base = 0; base < (1ull << 32); base += chunk) {
    check<<<static_cast<unsigned>(chunk / 256), 256>>>(base, bad, first);
  }
  unsigned long long h = 0;
  unsigned f = 0;
  cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
  cudaMemcpy(&f, first, sizeof(f), cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  std::printf("div_const_rn<28>: %llu mismatches of 4294967296 (first 0x%08x) %s\n", h, f,
              e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  return (h == 0 && e == cudaSuccess) ? 0 : 1;
}
