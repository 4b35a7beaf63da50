// Kernel instantiations for double.
#include <cstdint>
#define SK_T double
#define SK_REGISTRY_FN kernels_f64
#define SK_FUSED_FN fused_f64
#define SK_CROSS_FN cross_strips_f64
#define SK_VECTOR_FN vector_f64
#define SK_PEER_FN peer_tma_f64
#define SK_HALO_FN halo_strips_f64
#define SK_HALO_PUT_FN halo_put_f64
#define SK_PACK_FN gol_pack_f64
#define SK_UNPACK_FN gol_unpack_f64
#include "kernels_inst.cuh"
