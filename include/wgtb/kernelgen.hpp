// Executable synthetic kernels: template substitution
// that turns a KernelDescriptor - border region N/S/E/W and the per-category
// instruction counts the reference draws as fixture splits
// (src/synthgen.cpp:16-38, 89-94) - into a CUDA customising function for
// wgtb::CustomStencil, plus the same computation in C for the CPU check.
// The paper's synthetic benchmarks are generated the same way (PAPER.md:
// 206-222).  Counts map to code as:
//   load        taps v.at(dr, dc) spread over the border region (the four arm
//               extremes first, then seeded positions), each added to acc;
//   float_arith further dependent fp32 mul / add steps on acc (taps count
//               as one float op each);
//   int_arith   an FNV-style integer mixing chain, folded in at the end;
//   branch      data-dependent two-way updates of acc;
//   vector, store, call, other   no extra code (the executor's own store is
//               the kernel's store).
// Every float operation is an explicitly rounded __fadd_rn / __fmul_rn on the
// GPU and a plain float operation in C compiled with -ffp-contract=off, so
// the two are bit-identical.
#pragma once

#include <string>

#include "wgtb/scenario.hpp"

namespace wgtb {

struct GeneratedKernel {
  std::string cuda;      // translation unit: functor + extern "C" sk_gen_table()
  std::string c_ref;     // C99: extern "C"-compatible gen_grid() reference
  std::string functor;   // functor type name
};

// fp32 kernels; deterministic in the descriptor (positions seeded by the name).
GeneratedKernel generate_kernel(const KernelDescriptor& k);

}  // namespace wgtb
