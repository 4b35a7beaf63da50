// The reference-side binding: proj/src/b200_backend.cpp,
// linked instead of the simulated parts of simoracle.cpp.  Every signature
// is the reference's (include/wgtune/simoracle.hpp:26, :34-35, :45); every
// body goes through the C-ABI of libsk_stencil (include/sk_stencil.h).  The
// reference's own collect() and scenario_context() (simoracle.cpp:82-88,
// 143-161) then sweep the real B200 executor.  Built and run against the
// reference sources by oracle/build_ref.sh + tests/test_integration_backend.py.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "sk_stencil.h"
#include "wgtune/errors.hpp"
#include "wgtune/simoracle.hpp"

namespace wgtune {

static sk_stencil_desc desc_for(const KernelDescriptor& k, ElementType type) {
  sk_stencil_desc d{};
  const std::string& n = k.name;
  d.op = n.rfind("synthetic-", 0) == 0 ? SK_OP_SYNTHETIC
         : n == "gaussian"             ? SK_OP_GAUSSIAN
         : n == "gol"                  ? SK_OP_GOL
         : n == "he"                   ? SK_OP_HEAT
         : n == "nms"                  ? SK_OP_NMS
         : n == "sobel"                ? SK_OP_SOBEL
                                       : SK_OP_THRESHOLD;
  d.dtype = type == ElementType::INT32 ? SK_INT32 : type == ElementType::FLOAT64 ? SK_FLOAT64 : SK_FLOAT32;
  d.north = k.north;
  d.south = k.south;
  d.east = k.east;
  d.west = k.west;
  d.border_mode = d.op == SK_OP_GOL ? SK_BORDER_PAD : SK_BORDER_NEAREST;
  d.complexity = k.complexity ? 1 : 0;
  d.instructions = k.total_instructions;
  return d;
}

// simoracle.hpp:26 - the kernel's real maximum (cudaFuncAttributes)
int kernel_max_wgsize(const DeviceDescriptor& device, const KernelDescriptor& kernel) {
  const sk_stencil_desc d = desc_for(kernel, ElementType::FLOAT32);
  int32_t km = 0;
  if (sk_kernel_max_wgsize(&d, &km) != SK_OK) throw InvalidArgument(sk_last_error());
  return std::min<int>(km, device.device_max_wgsize);
}

// simoracle.hpp:34-35 - refused = the device cannot run the tile
bool is_refused(const DeviceDescriptor&, const KernelDescriptor& kernel, WorkgroupSize w, int out_elem_bytes) {
  const sk_stencil_desc d =
      desc_for(kernel, out_elem_bytes == 8 ? ElementType::FLOAT64 : ElementType::FLOAT32);
  return sk_stencil_probe(&d, 4096, 4096, w.cols(), w.rows(), nullptr, nullptr, nullptr) == SK_REFUSED;
}

// simoracle.hpp:45 - min_samples cudaEvent-timed passes on the B200
std::vector<double> run(const Scenario& s, WorkgroupSize w, const OracleConfig& cfg) {
  const sk_stencil_desc d = desc_for(s.kernel, s.dataset.in_type);
  const size_t n = size_t(s.dataset.width) * size_t(s.dataset.height);
  const size_t bytes = n * size_t(element_size_bytes(s.dataset.in_type));
  std::vector<char> h(bytes);
  sk_fill_host(d.dtype, d.op == SK_OP_GOL ? 2 : 0, cfg.seed, h.data(), int64_t(n));
  void *in = nullptr, *out = nullptr;
  if (cudaMalloc(&in, bytes) != cudaSuccess || cudaMalloc(&out, bytes) != cudaSuccess) {
    cudaFree(in);
    throw InvalidArgument("cudaMalloc failed");
  }
  cudaMemcpy(in, h.data(), bytes, cudaMemcpyHostToDevice);
  std::vector<double> ms(size_t(std::max(cfg.min_samples, 1)));
  const int rc = sk_stencil_time(&d, in, out, s.dataset.width, s.dataset.height, s.dataset.width, w.cols(),
                                 w.rows(), 3, cfg.min_samples, 1, ms.data());
  cudaFree(in);
  cudaFree(out);
  if (rc == SK_OVERSIZED) throw IllegalWorkgroupSize(sk_last_error());
  if (rc == SK_REFUSED) throw RefusedParameter(sk_last_error(), w.cols(), w.rows());
  if (rc != SK_OK) throw InvalidArgument(sk_last_error());
  for (double& t : ms) t = std::max(t, 1e-6);  // runtimes must be > 0 (space.cpp)
  return ms;
}

}  // namespace wgtune
