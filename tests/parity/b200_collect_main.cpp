// The reference's own sweep harness (wgtune::collect, simoracle.cpp:143-161)
// driving the real B200 executor through the reference-side binding
// integration/b200_backend.cpp.  Linked by
// oracle/build_ref.sh against the reference library with run /
// kernel_max_wgsize / is_refused of simoracle.o weakened, so the binding's
// definitions replace the simulator's while collect and scenario_context stay
// the reference's code.  Checks the collect contract of
// tests/test_simoracle.cpp:183-250 on real measurements; prints "OK".
#include <cstdio>
#include <set>

#include "sk_stencil.h"
#include "wgtune/simoracle.hpp"
#include "wgtune/space.hpp"

using namespace wgtune;

int main() {
  sk_device_props p{};
  if (sk_device_features(0, &p) != SK_OK) {
    std::printf("FAIL sk_device_features: %s\n", sk_last_error());
    return 1;
  }
  DeviceDescriptor dev;
  dev.id = "B200-collect";
  dev.device_type = DeviceType::GPU;
  dev.vendor_class = VendorClass::NVIDIA_GPU;
  dev.compute_units = p.compute_units;
  dev.frequency_mhz = p.frequency_mhz;
  dev.local_mem_kb = p.local_mem_kb;
  dev.global_cache_kb = p.global_cache_kb;
  dev.global_mem_mb = p.global_mem_mb;
  dev.device_max_wgsize = p.device_max_wgsize;
  dev.simd_width = p.simd_width;
  KernelDescriptor k;
  k.name = "he";
  k.north = k.south = k.east = k.west = 1;
  k.instr_counts = {28, 10, 16, 38, 8, 0, 5, 8};
  k.total_instructions = 113;
  k.complexity = true;
  DatasetDescriptor ds{512, 512, ElementType::FLOAT32, ElementType::FLOAT32};
  const Scenario s = make_scenario(dev, k, ds);

  OracleConfig cfg;
  cfg.min_samples = 10;
  cfg.max_wgsize_cap = 96;
  const CollectResult r = collect({s}, cfg);  // the reference's collect

  const ConstraintContext& ctx = r.contexts.at(s.id);
  const auto space = enumerate_space(ctx.effective_max());
  const auto& refused = r.refused.at(s.id);
  int fails = 0;
  std::size_t sampled = 0;
  for (const auto& w : space) {
    const bool has = r.table.has(s.id, w);
    if (has == (refused.count(w) > 0)) {
      std::printf("FAIL %s: sampled=%d refused=%d\n", w.str().c_str(), int(has), int(refused.count(w)));
      ++fails;
    }
    if (has) {
      ++sampled;
      const auto& rt = r.table.runtimes(s.id, w);
      if (rt.size() != 10) {
        std::printf("FAIL %s: %zu samples\n", w.str().c_str(), rt.size());
        ++fails;
      }
      for (double t : rt) fails += !(t > 0.0);
    }
  }
  if (r.table.scenario_rows(s.id).size() != sampled) ++fails;
  // argmin of the measured means is the oracle size
  const WorkgroupSize omega = oracle(s.id, r.table);
  for (const auto& [w, rt] : r.table.scenario_rows(s.id)) {
    if (r.table.mean_runtime(s.id, w) < r.table.mean_runtime(s.id, omega)) {
      std::printf("FAIL oracle %s is beaten by %s\n", omega.str().c_str(), w.str().c_str());
      ++fails;
    }
  }
  // kernel_max is the real one (cudaFuncAttributes), not the simulated rule
  int32_t km = 0;
  sk_stencil_desc d{};
  d.op = SK_OP_HEAT;
  d.dtype = SK_FLOAT32;
  d.north = d.south = d.east = d.west = 1;
  d.border_mode = SK_BORDER_NEAREST;
  sk_kernel_max_wgsize(&d, &km);
  if (ctx.kernel_max() != km) {
    std::printf("FAIL kernel_max %d != device %d\n", ctx.kernel_max(), km);
    ++fails;
  }
  std::printf("collect: %zu legal sizes sampled, %zu refused, oracle %s (%.4f ms)\n", sampled, refused.size(),
              omega.str().c_str(), r.table.mean_runtime(s.id, omega));
  if (fails == 0) std::printf("OK\n");
  return fails == 0 ? 0 : 1;
}
