// sk_stencil_iterate_nccl with P thread-ranks on one GPU over the NCCL test
// double (tests/cpp/fake_nccl.cpp): the row-sharded result, gathered, must
// equal the single-GPU sk_stencil_iterate result bit for bit (which the
// parity tests pin to the CPU oracle).  Covers ragged shards (H not a
// multiple of P), asymmetric halos (boxmean 5,1,3,0), both border modes,
// the scalar and vector load paths, and shards exactly N + S rows tall.
// Built into paper_1511_02490_b200/lib/nccl_halo_test; run by
// tests/test_nccl_halo.py (-m gpu).  Prints "OK" and exits 0 on success.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "sk_stencil.h"

extern "C" void fake_nccl_make_comms(int nranks, void** comms);

static int fails = 0;

static bool run_case(const char* name, sk_stencil_desc d, int W, int H, int P, int iters, int wc, int wr) {
  const size_t es = d.dtype == SK_FLOAT64 ? 8 : 4;
  std::vector<unsigned char> host(size_t(W) * H * es);
  sk_fill_host(d.dtype, d.op == SK_OP_GOL ? 2 : 0, 5, host.data(), int64_t(W) * H);
  // single GPU
  void *a, *b;
  cudaMalloc(&a, host.size());
  cudaMalloc(&b, host.size());
  cudaMemcpy(a, host.data(), host.size(), cudaMemcpyHostToDevice);
  int32_t in_b = 0;
  if (sk_stencil_iterate(&d, a, b, W, H, W, iters, wc, wr, nullptr, &in_b) != SK_OK) {
    std::printf("FAIL %s: single-GPU iterate: %s\n", name, sk_last_error());
    return false;
  }
  std::vector<unsigned char> want(host.size());
  cudaMemcpy(want.data(), in_b ? b : a, host.size(), cudaMemcpyDeviceToHost);
  cudaFree(a);
  cudaFree(b);

  // P ranks, each a thread with its own stream and N + rows + S buffers
  std::vector<void*> comms(P);
  fake_nccl_make_comms(P, comms.data());
  std::vector<unsigned char> got(host.size());
  std::vector<int> rcs(P, 0);
  const int N = d.north, S = d.south;
  auto rank_fn = [&](int r) {
    const int r0 = int((long long)H * r / P), r1 = int((long long)H * (r + 1) / P);
    const int rows = r1 - r0;
    const size_t rb = size_t(W) * es, bytes = size_t(N + rows + S) * rb;
    void *xa, *xb;
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaMalloc(&xa, bytes);
    cudaMalloc(&xb, bytes);
    cudaMemset(xa, 0xab, bytes);  // stale halo garbage must never leak in
    cudaMemset(xb, 0xcd, bytes);
    cudaMemcpy(static_cast<char*>(xa) + N * rb, host.data() + size_t(r0) * rb, size_t(rows) * rb,
               cudaMemcpyHostToDevice);
    int32_t res_b = 0;
    rcs[r] = sk_stencil_iterate_nccl(&d, xa, xb, W, rows, W, iters, wc, wr, comms[r], r, P, st, &res_b);
    cudaStreamSynchronize(st);
    if (rcs[r] == SK_OK) {
      cudaMemcpy(got.data() + size_t(r0) * rb, static_cast<char*>(res_b ? xb : xa) + N * rb, size_t(rows) * rb,
                 cudaMemcpyDeviceToHost);
    } else {
      std::printf("  rank %d: %s\n", r, sk_last_error());
    }
    cudaFree(xa);
    cudaFree(xb);
    cudaStreamDestroy(st);
  };
  std::vector<std::thread> ts;
  for (int r = 0; r < P; ++r) ts.emplace_back(rank_fn, r);
  for (auto& t : ts) t.join();
  for (int r = 0; r < P; ++r) {
    if (rcs[r] != SK_OK) {
      std::printf("FAIL %s: rank %d returned %d\n", name, r, rcs[r]);
      return false;
    }
  }
  if (std::memcmp(got.data(), want.data(), got.size()) != 0) {
    size_t i = 0;
    while (got[i] == want[i]) ++i;
    std::printf("FAIL %s: first differing byte %zu (row %zu)\n", name, i, i / (size_t(W) * es));
    return false;
  }
  std::printf("ok   %s (P=%d, %dx%d, %d generations)\n", name, P, W, H, iters);
  return true;
}

static sk_stencil_desc desc(int op, int dtype, int n, int s, int e, int w, int border, int path) {
  sk_stencil_desc d;
  std::memset(&d, 0, sizeof d);
  d.op = op;
  d.dtype = dtype;
  d.north = n;
  d.south = s;
  d.east = e;
  d.west = w;
  d.border_mode = border;
  d.load_path = path;
  return d;
}

int main() {
  struct Case {
    const char* name;
    sk_stencil_desc d;
    int W, H, P, iters, wc, wr;
  } cases[] = {
      {"heat f32 nearest auto", desc(SK_OP_HEAT, SK_FLOAT32, 1, 1, 1, 1, SK_BORDER_NEAREST, SK_LOAD_AUTO), 520, 301, 2, 9, 32, 8},
      {"heat f32 nearest tma, 4 ranks", desc(SK_OP_HEAT, SK_FLOAT32, 1, 1, 1, 1, SK_BORDER_NEAREST, SK_LOAD_TMA), 520, 301, 4, 7, 16, 4},
      {"gol i32 pad, 3 ranks", desc(SK_OP_GOL, SK_INT32, 1, 1, 1, 1, SK_BORDER_PAD, SK_LOAD_AUTO), 264, 203, 3, 12, 32, 4},
      {"gol i32 pad vector, 8 ranks", desc(SK_OP_GOL, SK_INT32, 1, 1, 1, 1, SK_BORDER_PAD, SK_LOAD_VECTOR), 512, 512, 8, 10, 16, 8},
      {"boxmean 5,1,3,0 f32 nearest, 3 ranks", desc(SK_OP_BOXMEAN, SK_FLOAT32, 5, 1, 3, 0, SK_BORDER_NEAREST, SK_LOAD_AUTO), 300, 250, 3, 4, 24, 4},
      {"five_point f64 pad explicit, 2 ranks", desc(SK_OP_FIVE_POINT, SK_FLOAT64, 1, 1, 1, 1, SK_BORDER_PAD, SK_LOAD_EXPLICIT), 130, 97, 2, 5, 8, 8},
      {"heat f32 shards of N+S rows", desc(SK_OP_HEAT, SK_FLOAT32, 1, 1, 1, 1, SK_BORDER_NEAREST, SK_LOAD_AUTO), 256, 8, 4, 6, 32, 2},
      {"heat f32 one rank", desc(SK_OP_HEAT, SK_FLOAT32, 1, 1, 1, 1, SK_BORDER_NEAREST, SK_LOAD_AUTO), 256, 100, 1, 6, 32, 2},
  };
  for (auto& c : cases) fails += run_case(c.name, c.d, c.W, c.H, c.P, c.iters, c.wc, c.wr) ? 0 : 1;
  // contract: fused generations / strip and bit-plane paths are refused
  sk_stencil_desc f = desc(SK_OP_HEAT, SK_FLOAT32, 1, 1, 1, 1, SK_BORDER_NEAREST, SK_LOAD_AUTO);
  f.fused_iterations = 2;
  void* comm[1];
  fake_nccl_make_comms(1, comm);
  void* buf;
  cudaMalloc(&buf, 1 << 20);
  if (sk_stencil_iterate_nccl(&f, buf, buf, 64, 16, 64, 1, 32, 2, comm[0], 0, 1, nullptr, nullptr) != SK_ENOTSUP) {
    std::printf("FAIL fused_iterations accepted\n");
    ++fails;
  }
  f.fused_iterations = 0;
  if (sk_stencil_iterate_nccl(&f, buf, buf, 64, 1, 64, 1, 32, 2, comm[0], 0, 1, nullptr, nullptr) != SK_EINVAL) {
    std::printf("FAIL a 1-row shard of a 1,1 stencil accepted\n");
    ++fails;
  }
  cudaFree(buf);
  if (fails == 0) std::printf("OK\n");
  return fails == 0 ? 0 : 1;
}
