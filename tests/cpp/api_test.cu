// C++ API test (GPU): wgtb::Stencil<T> over the C-ABI and wgtb::CustomStencil
// with a user customising function, checked against direct host loops.
// Built by paper_1511_02490_b200/Makefile into lib/api_test; run by
// tests/test_cpp_api.py (-m gpu).  Prints "OK" and exits 0 on success.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "wgtb/stencil.hpp"
#include "wgtb/stencil_custom.cuh"

// user functor: max of the cross taps (N=2, S=1, E=1, W=3) minus the centre
struct AsymCross {
  template <class V>
  __device__ float operator()(const V& v) const {
    float m = v.at(-2, 0);
    m = fmaxf(m, v.at(-1, 0));
    m = fmaxf(m, v.at(1, 0));
    m = fmaxf(m, v.at(0, 1));
    m = fmaxf(m, v.at(0, -1));
    m = fmaxf(m, v.at(0, -2));
    m = fmaxf(m, v.at(0, -3));
    return m - v.at(0, 0);
  }
};

static float host_asym(const std::vector<float>& g, int W, int H, int r, int c, float pad, bool nearest) {
  auto at = [&](int rr, int cc) {
    if (rr >= 0 && rr < H && cc >= 0 && cc < W) return g[size_t(rr) * W + cc];
    if (!nearest) return pad;
    rr = rr < 0 ? 0 : (rr >= H ? H - 1 : rr);
    cc = cc < 0 ? 0 : (cc >= W ? W - 1 : cc);
    return g[size_t(rr) * W + cc];
  };
  float m = at(r - 2, c);
  for (auto [dr, dc] : {std::pair{-1, 0}, {1, 0}, {0, 1}, {0, -1}, {0, -2}, {0, -3}}) m = fmaxf(m, at(r + dr, c + dc));
  return m - at(r, c);
}

static int fails = 0;
#define CHECK(cond, ...)            \
  do {                              \
    if (!(cond)) {                  \
      std::printf(__VA_ARGS__);     \
      std::printf("\n");            \
      ++fails;                      \
    }                               \
  } while (0)

int main() {
  const int W = 301, H = 257;
  std::vector<float> g(size_t(W) * H);
  for (size_t i = 0; i < g.size(); ++i) g[i] = float((i * 2654435761u) % 1000) / 997.0f;
  float *d_in, *d_out;
  cudaMalloc(&d_in, g.size() * 4);
  cudaMalloc(&d_out, g.size() * 4);
  cudaMemcpy(d_in, g.data(), g.size() * 4, cudaMemcpyHostToDevice);
  std::vector<float> out(g.size());
  for (bool nearest : {false, true}) {
    for (auto path : {SK_LOAD_AUTO, SK_LOAD_EXPLICIT}) {
      for (int k : {0, 1, 8}) {
        wgtb::CustomStencil<float, AsymCross> st({2, 1, 1, 3},
                                                 nearest ? wgtb::Border::nearest() : wgtb::Border::padding(0.25),
                                                 k);
        st.load_path(path);
        for (auto [wc, wr] : {std::pair{32, 8}, {2, 2}, {16, 16}, {6, 10}}) {
          st(d_in, d_out, W, H, wc, wr);
          cudaMemcpy(out.data(), d_out, out.size() * 4, cudaMemcpyDeviceToHost);
          int bad = 0;
          for (int r = 0; r < H; ++r)
            for (int c = 0; c < W; ++c) bad += out[size_t(r) * W + c] != host_asym(g, W, H, r, c, 0.25f, nearest);
          CHECK(bad == 0, "custom functor mismatch: nearest=%d path=%d k=%d %dx%d bad=%d", nearest, path, k, wc, wr, bad);
        }
      }
    }
  }
  // refusal / oversize surface as the reference's exceptions
  try {
    wgtb::CustomStencil<float, AsymCross> st({2, 1, 1, 3});
    st(d_in, d_out, W, H, 64, 32);
    CHECK(false, "expected IllegalWorkgroupSize");
  } catch (const wgtb::IllegalWorkgroupSize&) {
  }
  // built-in op through the host API: GoL blinker, period 2
  {
    const int n = 64;
    std::vector<int32_t> b(n * n, 0), r(n * n);
    b[20 * n + 30] = b[20 * n + 31] = b[20 * n + 32] = 1;
    int32_t *a, *bb;
    cudaMalloc(&a, n * n * 4);
    cudaMalloc(&bb, n * n * 4);
    cudaMemcpy(a, b.data(), n * n * 4, cudaMemcpyHostToDevice);
    wgtb::Stencil<int32_t> gol(SK_OP_GOL, {1, 1, 1, 1}, wgtb::Border::padding(0));
    int32_t* res = gol.iterate(a, bb, n, n, 10, 32, 4);
    cudaMemcpy(r.data(), res, n * n * 4, cudaMemcpyDeviceToHost);
    CHECK(r == b, "gol blinker not periodic");
    gol.run_host(b.data(), r.data(), n, n, 1, 8, 8);
    CHECK(r[19 * n + 31] == 1 && r[20 * n + 31] == 1 && r[21 * n + 31] == 1 && r[20 * n + 30] == 0,
          "gol run_host one step wrong");
    CHECK(gol.probe(n, n, 64, 32) == SK_OVERSIZED, "probe should report oversized");
    // temporally blocked paths through the same API: bit-plane GoL (TB 8) and
    // streamed host jobs must reproduce the one-pass results
    wgtb::Stencil<int32_t> bits(SK_OP_GOL, {1, 1, 1, 1}, wgtb::Border::padding(0));
    bits.load_path(SK_LOAD_BITPLANE).fused_iterations(8);
    cudaMemcpy(a, b.data(), n * n * 4, cudaMemcpyHostToDevice);
    res = bits.iterate(a, bb, n, n, 10, 32, 8);
    cudaMemcpy(r.data(), res, n * n * 4, cudaMemcpyDeviceToHost);
    CHECK(r == b, "bit-plane gol blinker not periodic");
    std::vector<int32_t> r1(n * n), r2(n * n);
    const int64_t t1 = gol.submit_host(b.data(), r1.data(), n, n, 1, 8, 8);
    const int64_t t2 = gol.submit_host(b.data(), r2.data(), n, n, 2, 8, 8);
    wgtb::Stencil<int32_t>::wait_host(t1);
    wgtb::Stencil<int32_t>::wait_host(t2);
    CHECK(r1[19 * n + 31] == 1 && r1[20 * n + 30] == 0 && r2 == b, "streamed host jobs wrong");
  }
  // register-strip heat (TB 6) equals six one-pass generations
  {
    const int W = 300, H = 97;
    std::vector<float> h(W * H), o1(W * H), o2(W * H);
    for (int i = 0; i < W * H; ++i) h[i] = static_cast<float>((i * 2654435761u) % 1000) / 1000.0f;
    wgtb::Stencil<float> one(SK_OP_HEAT, {}, wgtb::Border::nearest());
    wgtb::Stencil<float> tb(SK_OP_HEAT, {}, wgtb::Border::nearest());
    tb.load_path(SK_LOAD_STRIPS).fused_iterations(6);
    one.run_host(h.data(), o1.data(), W, H, 13, 32, 8);
    tb.run_host(h.data(), o2.data(), W, H, 13, 32, 12);
    CHECK(o1 == o2, "strip heat differs from one-pass");
  }
  // vector work-items (SK_LOAD_VECTOR) through the host API equal the scalar TMA kernel
  {
    const int W = 264, H = 203;
    std::vector<float> h(W * H), o1(W * H), o2(W * H);
    for (int i = 0; i < W * H; ++i) h[i] = static_cast<float>((i * 2654435761u) % 1000) / 1000.0f;
    wgtb::Stencil<float> vec(SK_OP_BOXMEAN, {5, 1, 3, 0}, wgtb::Border::nearest());
    wgtb::Stencil<float> sca(SK_OP_BOXMEAN, {5, 1, 3, 0}, wgtb::Border::nearest());
    vec.load_path(SK_LOAD_VECTOR);
    sca.load_path(SK_LOAD_TMA);
    vec.run_host(h.data(), o1.data(), W, H, 3, 16, 8);
    sca.run_host(h.data(), o2.data(), W, H, 3, 32, 8);
    CHECK(o1 == o2, "vector box mean differs from the scalar kernel");
    int32_t km = 0;
    CHECK(vec.probe(W, H, 16, 8, &km) == SK_OK && km >= 512, "vector probe");
  }
  std::printf(fails ? "FAILED %d\n" : "OK\n", fails);
  return fails ? 1 : 0;
}
