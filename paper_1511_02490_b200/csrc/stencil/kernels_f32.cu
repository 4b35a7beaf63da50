// Kernel instantiations for float.
#include <cstdint>
#define SK_T float
#define SK_REGISTRY_FN kernels_f32
#define SK_FUSED_FN fused_f32
#define SK_BITS_FN gol_bits_f32
#include "kernels_inst.cuh"
