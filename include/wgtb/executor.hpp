// The hot-path seam on real hardware: the B200 replacement for the
// reference's simulated execution oracle (simoracle.hpp:15-58).  Same
// operations, same contracts, real numbers:
//
//   kernel_max_wgsize  cudaFuncAttributes.maxThreadsPerBlock of the kernel
//                      the executor would launch (simoracle.cpp:62-70)
//   is_refused         the executor's zero-work legality probe: tile above
//                      the opt-in shared memory / no resident block /
//                      launch-config error (simoracle.cpp:72-80)
//   scenario_context   W_max(s) and the refused set (simoracle.cpp:82-88)
//   run                `samples` cudaEvent-timed passes of the real kernel
//                      (simoracle.cpp:122-141); throws IllegalWorkgroupSize /
//                      RefusedParameter like the simulator
//   collect            the exhaustive wc x wr sweep (simoracle.cpp:143-161),
//                      with the paper's gold-standard output check
//                       on every measured size
#pragma once

#include <cstdint>
#include <functional>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "sk_stencil.h"
#include "wgtb/autotune.hpp"
#include "wgtb/io.hpp"
#include "wgtb/scenario.hpp"
#include "wgtb/space.hpp"

namespace wgtb {

struct SweepConfig {
  int samples = 30;          // runtimes per test case (simoracle.hpp:18)
  int warmup = 3;            // untimed launches before the samples
  bool flush_l2 = true;      // overwrite 2 x L2 before every sample
  int max_wgsize_cap = 0;    // optional cap on the effective maximum (0 = none)
  bool validate = true;      // every size's output must equal the gold standard (else rejected)
  std::uint64_t seed = 1;    // input grid seed (reference Rng stream)
  int border_mode = SK_BORDER_NEAREST;
  double pad_value = 0.0;
  int cells_per_thread = 0;  // executor K (0 = auto)
};

// Executable stencil for a scenario's kernel + dataset descriptors.
sk_stencil_desc stencil_desc_for(const KernelDescriptor& k, ElementType type,
                                 const SweepConfig& cfg = {});

int kernel_max_wgsize(const DeviceDescriptor& device, const KernelDescriptor& kernel,
                      ElementType type = ElementType::FLOAT32);
bool is_refused(const DeviceDescriptor& device, const KernelDescriptor& kernel, WorkgroupSize w,
                int out_elem_bytes = 4);
ConstraintContext scenario_context(const Scenario& s, const SweepConfig& cfg,
                                   std::set<WorkgroupSize> refused = {});

std::vector<double> run(const Scenario& s, WorkgroupSize w, const SweepConfig& cfg);

struct CollectResult {
  SampleTable table;
  RefusedRecord refused;
  ContextRecord contexts;
  // sizes whose output differed from the gold standard (an explicit-load
  // pass): rejected before timing, also listed as refused; must be empty
  std::map<std::string, std::set<WorkgroupSize>> rejected;
  std::map<std::string, std::size_t> gold_mismatches;  // per scenario, must be 0
};

using ProgressFn = std::function<void(const Scenario&, std::size_t done, std::size_t total)>;
CollectResult collect(const std::vector<Scenario>& scenarios, const SweepConfig& cfg,
                      const ProgressFn& progress = {});

// Live legality probe for online tuning (Algorithm 1/2 against the device).
ProbeFn live_probe(const Scenario& s, const SweepConfig& cfg = {});

}  // namespace wgtb
