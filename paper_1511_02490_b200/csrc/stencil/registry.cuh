// Kernel registry: (op, dtype, K) -> {TMA kernel, explicit kernel}.  The
// template instantiations live in one translation unit per element type
// (kernels_i32.cu, kernels_f32.cu, kernels_f64.cu) so they build in parallel.
#pragma once

#include "sk_stencil.h"

namespace sk {

using KernelPtr = const void*;

struct KernelPair {
  KernelPtr tma;
  KernelPtr explicit_;
};

// Vector-work-item one-pass kernels (SK_LOAD_VECTOR, vector.cuh):
// k_stencil_tma<Op, T, K, 1024, false, 16 / sizeof(T)>; nullptr when the op
// (with this descriptor's border) has no vector form.
KernelPtr vector_i32(const sk_stencil_desc& d, int K);
KernelPtr vector_f32(const sk_stencil_desc& d, int K);
KernelPtr vector_f64(const sk_stencil_desc& d, int K);

// K in {1, 2, 4, 8}: cells per work-item.
KernelPair kernels_i32(const sk_stencil_desc& d, int K);
KernelPair kernels_f32(const sk_stencil_desc& d, int K);
KernelPair kernels_f64(const sk_stencil_desc& d, int K);

// Temporal-blocking kernels (TMA only): TB in {2, 4}; nullptr when the op has
// no fused instantiation.
KernelPtr fused_i32(const sk_stencil_desc& d, int K, int TB);
KernelPtr fused_f32(const sk_stencil_desc& d, int K, int TB);
KernelPtr fused_f64(const sk_stencil_desc& d, int K, int TB);

// Bit-sliced temporally blocked Game of Life (gol_bits.cuh): T grid <->
// packed bit grid conversion per element type, and the register-strip
// generation kernel k_gol_strips<R> (R rows per lane in {8, 16, 32}).
KernelPtr gol_pack_i32();
KernelPtr gol_pack_f32();
KernelPtr gol_pack_f64();
KernelPtr gol_unpack_i32();
KernelPtr gol_unpack_f32();
KernelPtr gol_unpack_f64();
KernelPtr gol_strips(int R);

// Register-strip temporal blocking of the 5-point cross ops (cross_strips.cuh):
// k_cross_strips<Op, T, R>, R rows per lane in {4, 8, 16}; nullptr for other ops.
KernelPtr cross_strips_i32(const sk_stencil_desc& d, int R);
KernelPtr cross_strips_f32(const sk_stencil_desc& d, int R);
KernelPtr cross_strips_f64(const sk_stencil_desc& d, int R);

// Peer-memory halo exchange fused into the boundary-strip pass (halo.cuh):
// k_halo_strips<Op, T> per op, and the row put k_halo_put<T>.
KernelPtr halo_strips_i32(const sk_stencil_desc& d);
KernelPtr halo_strips_f32(const sk_stencil_desc& d);
KernelPtr halo_strips_f64(const sk_stencil_desc& d);
KernelPtr halo_put_i32();
KernelPtr halo_put_f32();
KernelPtr halo_put_f64();
KernelPtr halo_wait();

// k_stencil_tma<Op, T, K, 1024, PEER = true>: the one-pass kernel with the
// peer exchange fused into its boundary tile-rows; nullptr for other ops.
KernelPtr peer_tma_i32(const sk_stencil_desc& d, int K);
KernelPtr peer_tma_f32(const sk_stencil_desc& d, int K);
KernelPtr peer_tma_f64(const sk_stencil_desc& d, int K);

}  // namespace sk
