// Kernel instantiations for int32_t.
#include <cstdint>
#define SK_T int32_t
#define SK_REGISTRY_FN kernels_i32
#define SK_FUSED_FN fused_i32
#define SK_CROSS_FN cross_strips_i32
#define SK_VECTOR_FN vector_i32
#define SK_PEER_FN peer_tma_i32
#define SK_HALO_FN halo_strips_i32
#define SK_HALO_PUT_FN halo_put_i32
#define SK_PACK_FN gol_pack_i32
#define SK_UNPACK_FN gol_unpack_i32
#define SK_STRIPS_HOME 1
#include "kernels_inst.cuh"
