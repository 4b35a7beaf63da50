// wgtb::Stencil<T> — the SkelCL stencil pattern as a C++
// host API over the C-ABI (include/sk_stencil.h).  Plain host C++: no nvcc
// needed for the built-in customising functions.  User-written functors use
// wgtb::CustomStencil<T, F> from stencil_custom.cuh (compiled with nvcc).
//
//   wgtb::Stencil<float> blur(SK_OP_GAUSSIAN, {5, 5, 5, 5}, wgtb::Border::nearest());
//   blur(d_in, d_out, W, H, /*wc=*/32, /*wr=*/8);               // one pass
//   blur.iterate(d_a, d_b, W, H, 100, 32, 8);                   // ping-pong
//   wgtb::Stencil<float> heat(SK_OP_HEAT, {}, wgtb::Border::nearest());
//   heat.load_path(SK_LOAD_STRIPS).fused_iterations(8).iterate(d_a, d_b, W, H, 100, 32, 12);
//
// Errors follow the reference's taxonomy (errors.hpp): IllegalWorkgroupSize
// for wc*wr above the maximum, RefusedParameter(w_c, w_r) for a refused
// launch, DeviceError for CUDA failures, InvalidArgument otherwise.
#pragma once

#include <cstdint>
#include <string>
#include <type_traits>
#include <vector>

#include "sk_stencil.h"
#include "wgtb/common.hpp"
#include "wgtb_c.h"

namespace wgtb {

// N/S/E/W border region (cells); north = smaller row index.
struct BorderRegion {
  int north = 1, south = 1, east = 1, west = 1;
};

// Out-of-matrix substitution: a pad value or the nearest in-matrix cell.
struct Border {
  int mode = SK_BORDER_PAD;
  double pad = 0.0;
  static Border padding(double value) { return {SK_BORDER_PAD, value}; }
  static Border nearest() { return {SK_BORDER_NEAREST, 0.0}; }
};

template <typename T>
constexpr int sk_dtype_for() {
  static_assert(std::is_same_v<T, int32_t> || std::is_same_v<T, float> || std::is_same_v<T, double>,
                "Stencil element type must be int32_t, float or double");
  return std::is_same_v<T, int32_t> ? SK_INT32 : std::is_same_v<T, float> ? SK_FLOAT32 : SK_FLOAT64;
}

// Throws the exception matching an sk_status.
inline void throw_status(int rc, int wc, int wr, const char* where) {
  if (rc == SK_OK) return;
  const std::string msg = std::string(where) + ": " + sk_last_error();
  switch (rc) {
    case SK_OVERSIZED: throw IllegalWorkgroupSize(msg);
    case SK_REFUSED: throw RefusedParameter(msg, wc, wr);
    case SK_ECUDA: throw DeviceError(msg);
    default: throw InvalidArgument(msg);
  }
}

template <typename T>
class Stencil {
 public:
  Stencil(sk_op op, BorderRegion region = {}, Border border = {}, int cells_per_thread = 0) {
    desc_.op = op;
    desc_.dtype = sk_dtype_for<T>();
    desc_.north = region.north;
    desc_.south = region.south;
    desc_.east = region.east;
    desc_.west = region.west;
    desc_.border_mode = border.mode;
    desc_.pad_value = border.pad;
    desc_.load_path = SK_LOAD_AUTO;
    desc_.cells_per_thread = cells_per_thread;
  }

  // Synthetic-kernel knobs (generate_kernels, synthgen.cpp:57-80).
  Stencil& synthetic(bool heavy, int instructions) {
    desc_.complexity = heavy ? 1 : 0;
    desc_.instructions = instructions;
    return *this;
  }
  Stencil& load_path(sk_load_path p) {
    desc_.load_path = p;
    return *this;
  }
  // Temporal blocking: TB generations per launch (per-cell fused 2/4,
  // bit-plane GoL 1..128, register-strip cross ops 1..32; sk_stencil.h).
  Stencil& fused_iterations(int tb) {
    desc_.fused_iterations = tb;
    return *this;
  }

  // One pass over a W x H device grid (row pitch in elements; 0 = W).
  void operator()(const T* d_in, T* d_out, int64_t W, int64_t H, int wc, int wr,
                  void* stream = nullptr, int64_t pitch = 0, int64_t rows_above = 0,
                  int64_t rows_below = 0) const {
    const int64_t p = pitch ? pitch : W;
    throw_status(sk_stencil_launch(&desc_, d_in, d_out, W, H, p, p, rows_above, rows_below, wc, wr,
                                   stream),
                 wc, wr, "Stencil");
  }

  // `iterations` passes ping-ponging a/b; returns the buffer with the result.
  T* iterate(T* d_a, T* d_b, int64_t W, int64_t H, int iterations, int wc, int wr,
             void* stream = nullptr) const {
    int32_t in_b = 0;
    throw_status(sk_stencil_iterate(&desc_, d_a, d_b, W, H, W, iterations, wc, wr, stream, &in_b), wc,
                 wr, "Stencil::iterate");
    return in_b ? d_b : d_a;
  }

  // Host arrays in, host array out (H2D, passes, D2H).
  void run_host(const T* h_in, T* h_out, int64_t W, int64_t H, int iterations, int wc, int wr) const {
    throw_status(sk_stencil_run_host(&desc_, h_in, h_out, W, H, iterations, wc, wr), wc, wr,
                 "Stencil::run_host");
  }

  // Streamed host jobs (pinned buffers): submit returns a ticket at once,
  // three jobs in flight per thread; wait blocks until h_out holds the result.
  int64_t submit_host(const T* h_in, T* h_out, int64_t W, int64_t H, int iterations, int wc,
                      int wr) const {
    int64_t ticket = -1;
    throw_status(sk_stencil_submit_host(&desc_, h_in, h_out, W, H, iterations, wc, wr, &ticket), wc,
                 wr, "Stencil::submit_host");
    return ticket;
  }
  static void wait_host(int64_t ticket) {
    throw_status(sk_stencil_wait_host(ticket), 0, 0, "Stencil::wait_host");
  }

  // Legality without launching: SK_OK, SK_OVERSIZED or SK_REFUSED.
  int probe(int64_t W, int64_t H, int wc, int wr, int32_t* kernel_max = nullptr) const {
    const int rc = sk_stencil_probe(&desc_, W, H, wc, wr, kernel_max, nullptr, nullptr);
    if (rc != SK_OK && rc != SK_OVERSIZED && rc != SK_REFUSED) throw_status(rc, wc, wr, "Stencil::probe");
    return rc;
  }

  std::vector<double> time(const T* d_in, T* d_out, int64_t W, int64_t H, int wc, int wr,
                           int samples = 30, int warmup = 3, bool flush_l2 = true) const {
    std::vector<double> ms(static_cast<std::size_t>(samples));
    throw_status(sk_stencil_time(&desc_, d_in, d_out, W, H, W, wc, wr, warmup, samples, flush_l2, ms.data()),
                 wc, wr, "Stencil::time");
    return ms;
  }

  const sk_stencil_desc& desc() const { return desc_; }

  // Online-tuned launches (wgtb_c.h, libwgtb): the trained model picks the
  // workgroup size per (grid, device) and re-picks when a launch is refused.
  //   auto tuned = heat.autotuned("results/b200/model.json", "he.json");
  //   tuned(d_in, d_out, W, H);   // tuned.wc(), tuned.wr(): the size that ran
  class Tuned {
   public:
    Tuned(const Stencil& s, std::string model_json, std::string kernel_json)
        : desc_(s.desc_), model_(std::move(model_json)), kernel_(std::move(kernel_json)) {}
    void operator()(const T* d_in, T* d_out, int64_t W, int64_t H, void* stream = nullptr, int64_t pitch = 0) {
      const int64_t p = pitch ? pitch : W;
      if (wgtb_launch_tuned(model_.c_str(), kernel_.c_str(), &desc_, d_in, d_out, W, H, p, p, stream, &wc_, &wr_,
                            &proposals_) != 0) {
        throw NoLegalParameter(std::string("Stencil::Tuned: ") + wgtb_last_error());
      }
    }
    // external refusal feedback for the W x H session
    void refuse(int64_t W, int64_t H, int wc, int wr) {
      if (wgtb_tuned_refuse(model_.c_str(), kernel_.c_str(), &desc_, W, H, wc, wr) != 0) {
        throw InvalidArgument(std::string("Stencil::Tuned::refuse: ") + wgtb_last_error());
      }
    }
    int wc() const { return wc_; }
    int wr() const { return wr_; }
    int proposals() const { return proposals_; }

   private:
    sk_stencil_desc desc_;
    std::string model_, kernel_;
    int32_t wc_ = 0, wr_ = 0, proposals_ = 0;
  };
  Tuned autotuned(std::string model_json, std::string kernel_json) const {
    return Tuned(*this, std::move(model_json), std::move(kernel_json));
  }

 private:
  sk_stencil_desc desc_{};
};

}  // namespace wgtb
