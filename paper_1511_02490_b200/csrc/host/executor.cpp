// Real-hardware execution seam (see executor.hpp).  Device buffers and
// timing go through the C-ABI of libsk_stencil (sk_stencil_time /
// sk_stencil_probe) plus plain cudaMalloc/cudaMemcpy for the scenario grids.
#include "wgtb/executor.hpp"

#include <cuda_runtime.h>

#include <cstdio>
#include <memory>
#include <mutex>

namespace wgtb {

namespace {

int sk_dtype_of(ElementType t) {
  switch (t) {
    case ElementType::INT32: return SK_INT32;
    case ElementType::FLOAT32: return SK_FLOAT32;
    case ElementType::FLOAT64: return SK_FLOAT64;
  }
  return SK_FLOAT32;
}

ElementType element_of_bytes(int bytes) { return bytes == 8 ? ElementType::FLOAT64 : ElementType::FLOAT32; }

[[noreturn]] void device_fail(const std::string& what) {
  throw DeviceError(what + ": " + sk_last_error());
}

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw DeviceError(std::string(what) + ": " + cudaGetErrorString(e));
}

// Device grids of one scenario: input (reference-Rng synthetic data) and output.
struct Grids {
  void* in = nullptr;
  void* out = nullptr;
  std::size_t bytes = 0;
  Grids(const Scenario& s, const SweepConfig& cfg) {
    const auto& ds = s.dataset;
    if (ds.in_type != ds.out_type) throw InvalidArgument("executor needs in_type == out_type: " + s.id);
    const std::size_t n = static_cast<std::size_t>(ds.element_count());
    bytes = n * static_cast<std::size_t>(element_size_bytes(ds.in_type));
    std::unique_ptr<unsigned char[]> host(new unsigned char[bytes]);
    // gol: live/dead cells; other int kernels: 0..255 "pixels"; float: 2u-1
    const int kind = ds.in_type == ElementType::INT32 ? (s.kernel.name == "gol" ? 2 : 3) : 0;
    if (sk_fill_host(sk_dtype_of(ds.in_type), kind, cfg.seed, host.get(), static_cast<int64_t>(n)) != SK_OK) {
      device_fail("sk_fill_host");
    }
    check_cuda(cudaMalloc(&in, bytes), "cudaMalloc(in)");
    check_cuda(cudaMalloc(&out, bytes), "cudaMalloc(out)");
    check_cuda(cudaMemcpy(in, host.get(), bytes, cudaMemcpyHostToDevice), "cudaMemcpy(in)");
  }
  ~Grids() {
    cudaFree(in);
    cudaFree(out);
  }
  Grids(const Grids&) = delete;
  Grids& operator=(const Grids&) = delete;
};

int effective_max(const Scenario& s, const SweepConfig& cfg) {
  int m = std::min(s.device.device_max_wgsize,
                   kernel_max_wgsize(s.device, s.kernel, s.dataset.out_type));
  if (cfg.max_wgsize_cap > 0) m = std::min(m, cfg.max_wgsize_cap);
  return m;
}

std::vector<double> timed_samples(const sk_stencil_desc& d, const Scenario& s, const Grids& g,
                                  WorkgroupSize w, const SweepConfig& cfg) {
  std::vector<double> ms(static_cast<std::size_t>(std::max(cfg.samples, 1)));
  const int rc = sk_stencil_time(&d, g.in, g.out, s.dataset.width, s.dataset.height, s.dataset.width,
                                 w.cols(), w.rows(), cfg.warmup, cfg.samples, cfg.flush_l2 ? 1 : 0,
                                 ms.data());
  if (rc == SK_REFUSED) throw RefusedParameter("size " + w.str() + " refused for " + s.id, w.cols(), w.rows());
  if (rc == SK_OVERSIZED) throw IllegalWorkgroupSize("size " + w.str() + " exceeds the maximum for " + s.id);
  if (rc != SK_OK) device_fail("sk_stencil_time(" + s.id + ", " + w.str() + ")");
  ms.resize(static_cast<std::size_t>(cfg.samples));
  for (double& t : ms) t = std::max(t, 1e-6);  // event resolution floor; runtimes must be > 0
  return ms;
}

}  // namespace

sk_stencil_desc stencil_desc_for(const KernelDescriptor& k, ElementType type, const SweepConfig& cfg) {
  sk_stencil_desc d{};
  const std::string& n = k.name;
  if (n.starts_with("synthetic-")) d.op = SK_OP_SYNTHETIC;
  else if (n == "gaussian") d.op = SK_OP_GAUSSIAN;
  else if (n == "gol") d.op = SK_OP_GOL;
  else if (n == "he" || n == "heat") d.op = SK_OP_HEAT;
  else if (n == "nms") d.op = SK_OP_NMS;
  else if (n == "sobel") d.op = SK_OP_SOBEL;
  else if (n == "threshold") d.op = SK_OP_THRESHOLD;
  else if (n == "five_point") d.op = SK_OP_FIVE_POINT;
  else if (n == "boxmean" || n.starts_with("boxmean-")) d.op = SK_OP_BOXMEAN;
  else throw InvalidArgument("no executable functor for kernel '" + n + "'");
  d.dtype = sk_dtype_of(type);
  d.north = k.north;
  d.south = k.south;
  d.east = k.east;
  d.west = k.west;
  // gol's dead boundary is pad 0; the other kernels use the sweep's mode
  d.border_mode = d.op == SK_OP_GOL ? SK_BORDER_PAD : cfg.border_mode;
  d.pad_value = d.op == SK_OP_GOL ? 0.0 : cfg.pad_value;
  d.complexity = k.complexity ? 1 : 0;
  d.instructions = k.total_instructions;
  d.load_path = SK_LOAD_AUTO;
  d.cells_per_thread = cfg.cells_per_thread;
  return d;
}

int kernel_max_wgsize(const DeviceDescriptor& device, const KernelDescriptor& kernel, ElementType type) {
  const sk_stencil_desc d = stencil_desc_for(kernel, type);
  int32_t km = 0;
  if (sk_kernel_max_wgsize(&d, &km) != SK_OK) device_fail("sk_kernel_max_wgsize");
  return std::min(km, device.device_max_wgsize);
}

bool is_refused(const DeviceDescriptor& device, const KernelDescriptor& kernel, WorkgroupSize w,
                int out_elem_bytes) {
  (void)device;  // the current CUDA device is the one probed
  const sk_stencil_desc d = stencil_desc_for(kernel, element_of_bytes(out_elem_bytes));
  const int rc = sk_stencil_probe(&d, 4096, 4096, w.cols(), w.rows(), nullptr, nullptr, nullptr);
  if (rc == SK_OK || rc == SK_OVERSIZED) return false;
  if (rc == SK_REFUSED) return true;
  device_fail("sk_stencil_probe");
}

ConstraintContext scenario_context(const Scenario& s, const SweepConfig& cfg,
                                   std::set<WorkgroupSize> refused) {
  int device_max = s.device.device_max_wgsize;
  if (cfg.max_wgsize_cap > 0) device_max = std::min(device_max, cfg.max_wgsize_cap);
  return ConstraintContext(device_max, kernel_max_wgsize(s.device, s.kernel, s.dataset.out_type),
                           std::move(refused));
}

std::vector<double> run(const Scenario& s, WorkgroupSize w, const SweepConfig& cfg) {
  const int eff = effective_max(s, cfg);
  if (w.area() > eff) {
    throw IllegalWorkgroupSize("size " + w.str() + " exceeds the effective maximum " + std::to_string(eff) +
                               " for " + s.id);
  }
  const sk_stencil_desc d = stencil_desc_for(s.kernel, s.dataset.out_type, cfg);
  Grids g(s, cfg);
  return timed_samples(d, s, g, w, cfg);
}

// The gold standard of a scenario: one pass through the explicit-load
// kernel (one column per work-item, K = 1, 32x8 block) - an independent code
// path from the TMA / vector kernels whose sizes are being timed.
void gold_output(const sk_stencil_desc& d, const Scenario& s, const Grids& g, void* gold) {
  sk_stencil_desc e = d;
  e.load_path = SK_LOAD_EXPLICIT;
  e.cells_per_thread = 1;
  const int rc = sk_stencil_launch(&e, g.in, gold, s.dataset.width, s.dataset.height, s.dataset.width,
                                   s.dataset.width, 0, 0, 32, 8, nullptr);
  if (rc != SK_OK) device_fail("gold-standard pass (" + s.id + ")");
  check_cuda(cudaDeviceSynchronize(), "gold-standard pass");
}

CollectResult collect(const std::vector<Scenario>& scenarios, const SweepConfig& cfg,
                      const ProgressFn& progress) {
  if (scenarios.empty()) throw InvalidArgument("collect requires at least one scenario");
  CollectResult res;
  for (const Scenario& s : scenarios) {
    const sk_stencil_desc d = stencil_desc_for(s.kernel, s.dataset.out_type, cfg);
    Grids g(s, cfg);
    const auto space = enumerate_space(effective_max(s, cfg));
    std::set<WorkgroupSize>& refused = res.refused[s.id];
    std::set<WorkgroupSize>& rejected = res.rejected[s.id];
    void* gold = nullptr;
    if (cfg.validate) {
      check_cuda(cudaMalloc(&gold, g.bytes), "cudaMalloc(gold)");
      gold_output(d, s, g, gold);
    }
    std::size_t done = 0;
    for (const WorkgroupSize& w : space) {
      const int rc = sk_stencil_probe(&d, s.dataset.width, s.dataset.height, w.cols(), w.rows(), nullptr,
                                      nullptr, nullptr);
      if (rc == SK_REFUSED) {
        refused.insert(w);
      } else if (rc != SK_OK) {
        device_fail("sk_stencil_probe(" + s.id + ", " + w.str() + ")");
      } else {
        // validate before timing: a size whose output differs from the gold
        // standard is rejected (recorded, never timed)
        bool ok = true;
        if (cfg.validate) {
          const int lrc = sk_stencil_launch(&d, g.in, g.out, s.dataset.width, s.dataset.height,
                                            s.dataset.width, s.dataset.width, 0, 0, w.cols(), w.rows(), nullptr);
          if (lrc == SK_REFUSED) {
            refused.insert(w);
            if (progress) progress(s, ++done, space.size());
            continue;
          }
          if (lrc != SK_OK) device_fail("validation pass (" + s.id + ", " + w.str() + ")");
          int32_t equal = 0;
          if (sk_buffers_equal(gold, g.out, static_cast<int64_t>(g.bytes), &equal) != SK_OK) {
            device_fail("sk_buffers_equal");
          }
          ok = equal != 0;
        }
        if (!ok) {
          rejected.insert(w);
          refused.insert(w);  // unusable: the evaluation treats it like a refusal
          std::fprintf(stderr, "GOLD MISMATCH %s %s (rejected, not timed)\n", s.id.c_str(), w.str().c_str());
        } else {
          try {
            res.table.add_row(s.id, w, timed_samples(d, s, g, w, cfg));
          } catch (const RefusedParameter&) {
            refused.insert(w);  // launch-time refusal (non-sticky)
          }
        }
      }
      if (progress) progress(s, ++done, space.size());
    }
    cudaFree(gold);
    res.gold_mismatches[s.id] = rejected.size();
    res.contexts.emplace(s.id, scenario_context(s, cfg, refused));
  }
  return res;
}

ProbeFn live_probe(const Scenario& s, const SweepConfig& cfg) {
  const sk_stencil_desc d = stencil_desc_for(s.kernel, s.dataset.out_type, cfg);
  const int W = s.dataset.width, H = s.dataset.height;
  return [d, W, H](WorkgroupSize w) {
    const int rc = sk_stencil_probe(&d, W, H, w.cols(), w.rows(), nullptr, nullptr, nullptr);
    if (rc == SK_OK) return ProbeResult::Legal;
    if (rc == SK_OVERSIZED) return ProbeResult::Oversized;
    if (rc == SK_REFUSED) return ProbeResult::Refused;
    throw DeviceError(std::string("sk_stencil_probe: ") + sk_last_error());
  };
}

}  // namespace wgtb
