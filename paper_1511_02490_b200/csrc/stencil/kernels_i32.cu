// Kernel instantiations for int32_t.
#include <cstdint>
#define SK_T int32_t
#define SK_REGISTRY_FN kernels_i32
#define SK_FUSED_FN fused_i32
#define SK_BITS_FN gol_bits_i32
#include "kernels_inst.cuh"
