// Kernel instantiations for double.
#include <cstdint>
#define SK_T double
#define SK_REGISTRY_FN kernels_f64
#define SK_FUSED_FN fused_f64
#define SK_BITS_FN gol_bits_f64
#include "kernels_inst.cuh"
