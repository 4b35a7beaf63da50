// Instantiates every (op, K) kernel pair for one element type SK_T and
// defines the registry function SK_REGISTRY_FN (see registry.cuh).
#include "kernels.cuh"
#include "fused.cuh"
#include "gol_bits.cuh"
#include "cross_strips.cuh"
#include "halo.cuh"
#include "registry.cuh"

namespace sk {
namespace {

template <class Op, typename T, int K>
KernelPair pair_for() {
  return {reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, K, 1024>),
          reinterpret_cast<KernelPtr>(&k_stencil_explicit<Op, T, K, 1024>)};
}

template <class Op, typename T, int MAXT = 1024>
KernelPtr vector_for_k(int K) {
  constexpr int V = 16 / sizeof(T);
  switch (K) {
    case 1: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 1, MAXT, false, V>);
    case 2: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 2, MAXT, false, V>);
    case 4: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 4, MAXT, false, V>);
    case 8: return reinterpret_cast<KernelPtr>(&k_stencil_tma_r80<Op, T, 8, V>);
    default: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 16, 512, false, V>);  // 128 registers
  }
}

template <class Op, typename T>
KernelPtr peer_for_k(int K) {
  switch (K) {
    case 1: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 1, 1024, true>);
    case 2: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 2, 1024, true>);
    case 4: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 4, 1024, true>);
    default: return reinterpret_cast<KernelPtr>(&k_stencil_tma<Op, T, 8, 1024, true>);
  }
}

template <class Op, typename T>
KernelPair pair_for_k(int K) {
  switch (K) {
    case 1: return pair_for<Op, T, 1>();
    case 2: return pair_for<Op, T, 2>();
    case 4: return pair_for<Op, T, 4>();
    default: return pair_for<Op, T, 8>();
  }
}

template <class Op, typename T, int K>
KernelPtr fused_for_tb(int TB) {
  return TB == 2 ? reinterpret_cast<KernelPtr>(&k_stencil_tma_fused<Op, T, K, 2, 1024>)
                 : reinterpret_cast<KernelPtr>(&k_stencil_tma_fused<Op, T, K, 4, 1024>);
}

template <class Op, typename T>
KernelPtr fused_for(int K, int TB) {
  switch (K) {
    case 1: return fused_for_tb<Op, T, 1>(TB);
    case 2: return fused_for_tb<Op, T, 2>(TB);
    case 4: return fused_for_tb<Op, T, 4>(TB);
    default: return fused_for_tb<Op, T, 8>(TB);
  }
}

template <class Op, typename T>
KernelPtr cross_for(int R) {
  switch (R) {
    case 4: return reinterpret_cast<KernelPtr>(&k_cross_strips<Op, T, 4>);
    case 8: return reinterpret_cast<KernelPtr>(&k_cross_strips<Op, T, 8>);
    case 16: return reinterpret_cast<KernelPtr>(&k_cross_strips<Op, T, 16>);
    default: return nullptr;
  }
}

}  // namespace

KernelPtr SK_CROSS_FN(const sk_stencil_desc& d, int R) {
  switch (d.op) {
    case SK_OP_FIVE_POINT: return cross_for<FivePoint, SK_T>(R);
    case SK_OP_HEAT: return cross_for<Heat, SK_T>(R);
    default: return nullptr;
  }
}

KernelPtr SK_HALO_FN(const sk_stencil_desc& d) {
  using T = SK_T;
  switch (d.op) {
    case SK_OP_FIVE_POINT: return reinterpret_cast<KernelPtr>(&k_halo_strips<FivePoint, T>);
    case SK_OP_HEAT: return reinterpret_cast<KernelPtr>(&k_halo_strips<Heat, T>);
    case SK_OP_GOL: return reinterpret_cast<KernelPtr>(&k_halo_strips<Gol, T>);
    case SK_OP_BOXMEAN: return reinterpret_cast<KernelPtr>(&k_halo_strips<BoxMean, T>);
    case SK_OP_GAUSSIAN: return reinterpret_cast<KernelPtr>(&k_halo_strips<Gaussian, T>);
    case SK_OP_SOBEL: return reinterpret_cast<KernelPtr>(&k_halo_strips<Sobel, T>);
    case SK_OP_NMS: return reinterpret_cast<KernelPtr>(&k_halo_strips<Nms, T>);
    case SK_OP_THRESHOLD: return reinterpret_cast<KernelPtr>(&k_halo_strips<Threshold, T>);
    case SK_OP_SYNTHETIC: return reinterpret_cast<KernelPtr>(&k_halo_strips<Synthetic, T>);
  }
  return nullptr;
}

// One-pass TMA kernel with the peer exchange fused in (iterated ops only).
KernelPtr SK_PEER_FN(const sk_stencil_desc& d, int K) {
  using T = SK_T;
  switch (d.op) {
    case SK_OP_FIVE_POINT: return peer_for_k<FivePoint, T>(K);
    case SK_OP_HEAT: return peer_for_k<Heat, T>(K);
    case SK_OP_GOL: return peer_for_k<Gol, T>(K);
    case SK_OP_BOXMEAN:
      if (d.north == 5 && d.south == 1 && d.east == 3 && d.west == 0) {
        return peer_for_k<BoxMeanFixed<5, 1, 3, 0>, T>(K);
      }
      return peer_for_k<BoxMean, T>(K);
    default: return nullptr;
  }
}

// Vector work-items: only for the border region the op's vector form has.
KernelPtr SK_VECTOR_FN(const sk_stencil_desc& d, int K) {
  using T = SK_T;
  const bool unit = d.north == 1 && d.south == 1 && d.east == 1 && d.west == 1;
  switch (d.op) {
    case SK_OP_FIVE_POINT: return unit ? vector_for_k<FivePoint, T>(K) : nullptr;
    case SK_OP_HEAT: return unit ? vector_for_k<Heat, T>(K) : nullptr;
    case SK_OP_GOL: return unit ? vector_for_k<Gol, T>(K) : nullptr;
    case SK_OP_SOBEL: return unit ? vector_for_k<Sobel, T>(K) : nullptr;
    case SK_OP_NMS: return unit ? vector_for_k<Nms, T>(K) : nullptr;
    case SK_OP_BOXMEAN:
      if (d.north == 5 && d.south == 1 && d.east == 3 && d.west == 0) {
        return vector_for_k<BoxMeanFixed<5, 1, 3, 0>, T>(K);
      }
      return nullptr;
    default: return nullptr;
  }
}

KernelPtr SK_HALO_PUT_FN() { return reinterpret_cast<KernelPtr>(&k_halo_put<SK_T>); }

KernelPtr SK_PACK_FN() { return reinterpret_cast<KernelPtr>(&k_gol_pack<SK_T>); }
KernelPtr SK_UNPACK_FN() { return reinterpret_cast<KernelPtr>(&k_gol_unpack<SK_T>); }

#ifdef SK_STRIPS_HOME
KernelPtr halo_wait() { return reinterpret_cast<KernelPtr>(&k_halo_wait<0>); }

KernelPtr gol_strips(int R) {
  switch (R) {
    case 8: return reinterpret_cast<KernelPtr>(&k_gol_strips<8>);
    case 16: return reinterpret_cast<KernelPtr>(&k_gol_strips<16>);
    case 32: return reinterpret_cast<KernelPtr>(&k_gol_strips<32>);
    default: return nullptr;
  }
}
#endif

KernelPtr SK_FUSED_FN(const sk_stencil_desc& d, int K, int TB) {
  using T = SK_T;
  if (TB != 2 && TB != 4) return nullptr;
  switch (d.op) {
    case SK_OP_FIVE_POINT: return fused_for<FivePoint, T>(K, TB);
    case SK_OP_HEAT: return fused_for<Heat, T>(K, TB);
    case SK_OP_GOL: return fused_for<Gol, T>(K, TB);
    case SK_OP_BOXMEAN: return fused_for<BoxMean, T>(K, TB);
    default: return nullptr;
  }
}

KernelPair SK_REGISTRY_FN(const sk_stencil_desc& d, int K) {
  using T = SK_T;
  switch (d.op) {
    case SK_OP_FIVE_POINT: return pair_for_k<FivePoint, T>(K);
    case SK_OP_HEAT: return pair_for_k<Heat, T>(K);
    case SK_OP_GOL: return pair_for_k<Gol, T>(K);
    case SK_OP_BOXMEAN:
      if (d.north == 5 && d.south == 1 && d.east == 3 && d.west == 0) {
        return pair_for_k<BoxMeanFixed<5, 1, 3, 0>, T>(K);
      }
      return pair_for_k<BoxMean, T>(K);
    case SK_OP_GAUSSIAN:
      if (d.north == 5) return pair_for_k<GaussianFixed<5>, T>(K);
      return pair_for_k<Gaussian, T>(K);
    case SK_OP_SOBEL: return pair_for_k<Sobel, T>(K);
    case SK_OP_NMS: return pair_for_k<Nms, T>(K);
    case SK_OP_THRESHOLD: return pair_for_k<Threshold, T>(K);
    case SK_OP_SYNTHETIC: return pair_for_k<Synthetic, T>(K);
  }
  return {nullptr, nullptr};
}

}  // namespace sk
