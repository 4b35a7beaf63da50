// wgtb::CustomStencil<T, F> — a stencil with a USER customising function
// (PAPER.md:91-96), compiled with nvcc in the caller's translation unit.
//
// F is a functor with  `template <class V> __device__ T operator()(const V& v) const`
// where v.at(dr, dc) is the cell dr rows south (negative = north) and dc
// columns east (negative = west) of the work-item's cell, within the declared
// border region.  Example:
//
//   struct Cross {  // max of the four neighbours minus the centre
//     template <class V> __device__ float operator()(const V& v) const {
//       return fmaxf(fmaxf(v.at(-1, 0), v.at(1, 0)), fmaxf(v.at(0, -1), v.at(0, 1))) - v.at(0, 0);
//     }
//   };
//   wgtb::CustomStencil<float, Cross> st({1, 1, 1, 1}, wgtb::Border::nearest());
//   st(d_in, d_out, W, H, 32, 8);
//
// The executor's kernel templates (TMA-pipelined and explicit-load, K = 1, 2,
// 4, 8 cells per work-item) are instantiated here for F; their driver
// handles go to libsk_stencil through sk_stencil_launch_custom, which owns
// geometry, TMA descriptors, legality and the launch.
#pragma once

#include <cuda_runtime.h>

#include "kernels.cuh"  // paper_1511_02490_b200/csrc/stencil (add to the include path)
#include "wgtb/stencil.hpp"

namespace wgtb {

namespace detail {

// Adapts a user functor to the executor's op interface.
template <class F>
struct UserOp {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const sk::OpParams<T>&) const {
    return F{}(v);
  }
};

template <class F, typename T, int K>
void table_entry(sk_kernel_table& t, int i) {
  cudaFunction_t tma = nullptr, expl = nullptr;
  if (cudaGetFuncBySymbol(&tma, reinterpret_cast<const void*>(&sk::k_stencil_tma<UserOp<F>, T, K, 1024>)) !=
          cudaSuccess ||
      cudaGetFuncBySymbol(&expl, reinterpret_cast<const void*>(&sk::k_stencil_explicit<UserOp<F>, T, K, 1024>)) !=
          cudaSuccess) {
    throw DeviceError("cudaGetFuncBySymbol failed for a custom stencil kernel");
  }
  t.tma[i] = reinterpret_cast<const void*>(tma);
  t.explicit_load[i] = reinterpret_cast<const void*>(expl);
}

}  // namespace detail

template <typename T, class F>
class CustomStencil {
 public:
  explicit CustomStencil(BorderRegion region, Border border = {}, int cells_per_thread = 0) {
    desc_.op = SK_OP_BOXMEAN;  // ignored by sk_stencil_launch_custom
    desc_.dtype = sk_dtype_for<T>();
    desc_.north = region.north;
    desc_.south = region.south;
    desc_.east = region.east;
    desc_.west = region.west;
    desc_.border_mode = border.mode;
    desc_.pad_value = border.pad;
    desc_.cells_per_thread = cells_per_thread;
    detail::table_entry<F, T, 1>(table_, 0);
    detail::table_entry<F, T, 2>(table_, 1);
    detail::table_entry<F, T, 4>(table_, 2);
    detail::table_entry<F, T, 8>(table_, 3);
  }

  void operator()(const T* d_in, T* d_out, int64_t W, int64_t H, int wc, int wr,
                  cudaStream_t stream = nullptr, int64_t pitch = 0) const {
    const int64_t p = pitch ? pitch : W;
    throw_status(sk_stencil_launch_custom(&desc_, &table_, d_in, d_out, W, H, p, p, 0, 0, wc, wr, stream),
                 wc, wr, "CustomStencil");
  }

  CustomStencil& load_path(sk_load_path p) {
    desc_.load_path = p;
    return *this;
  }

 private:
  sk_stencil_desc desc_{};
  sk_kernel_table table_{};
};

}  // namespace wgtb
