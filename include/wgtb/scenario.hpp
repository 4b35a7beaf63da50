// Scenarios (device x kernel x dataset), their feature vectors and the
// synthetic benchmark generator.  Interface parity with the reference's
// scenario.hpp:12-84, features.hpp:11-43 and synthgen.hpp:10-33.
//
// B200 change (north-star subsystem 3): DeviceDescriptor is read from
// cudaDeviceProp (device_from_cuda), not from a fixture table; kernel and
// dataset descriptors are unchanged, and each kernel descriptor also selects
// an executable sm_100a functor (executor.hpp).
#pragma once

#include <array>
#include <map>
#include <span>
#include <string>
#include <string_view>
#include <vector>

#include "wgtb/common.hpp"

namespace wgtb {

enum class DeviceType { CPU, GPU };
enum class VendorClass { INTEL_CPU, AMD_GPU, NVIDIA_GPU, OTHER };
enum class ElementType { INT32, FLOAT32, FLOAT64 };
enum class InstrCategory { Load, Store, IntArith, FloatArith, Branch, Vector, Call, Other };
inline constexpr int kInstrCategoryCount = 8;
using InstrCounts = std::array<int, kInstrCategoryCount>;

std::string_view to_string(DeviceType);
std::string_view to_string(VendorClass);
std::string_view to_string(ElementType);
std::string_view to_string(InstrCategory);
DeviceType device_type_from_string(std::string_view);
VendorClass vendor_class_from_string(std::string_view);
ElementType element_type_from_string(std::string_view);
InstrCategory instr_category_from_string(std::string_view);
int element_size_bytes(ElementType);

struct DeviceDescriptor {
  std::string id;
  DeviceType device_type = DeviceType::CPU;
  VendorClass vendor_class = VendorClass::OTHER;
  int compute_units = 1;
  int frequency_mhz = 1;
  int local_mem_kb = 1;
  int global_cache_kb = 0;
  int global_mem_mb = 1;
  int device_max_wgsize = 64;
  int simd_width = 8;
  void validate() const;
};

struct KernelDescriptor {
  std::string name;
  int north = 0, south = 0, east = 0, west = 0;
  InstrCounts instr_counts{};
  int total_instructions = 1;
  bool complexity = false;
  void validate() const;
};

struct DatasetDescriptor {
  int width = 1, height = 1;
  ElementType in_type = ElementType::FLOAT32;
  ElementType out_type = ElementType::FLOAT32;
  long long element_count() const { return static_cast<long long>(width) * height; }
  void validate() const;
};

struct Scenario {
  DeviceDescriptor device;
  KernelDescriptor kernel;
  DatasetDescriptor dataset;
  std::string id;  // "<device.id>/<kernel.name>/<W>x<H>/<IN>-<OUT>"
};

std::string scenario_id(const DeviceDescriptor&, const KernelDescriptor&,
                        const DatasetDescriptor&);
Scenario make_scenario(const DeviceDescriptor&, const KernelDescriptor&,
                       const DatasetDescriptor&);

// ------------------------------------------------------------- features
inline constexpr int kFeatureCount = 29;
inline constexpr std::string_view kFeatureSchemaVersion = "fv1";
const std::array<std::string_view, kFeatureCount>& feature_names();

class FeatureVector {
 public:
  FeatureVector() = default;
  explicit FeatureVector(const std::array<double, kFeatureCount>& v) : v_(v) {}
  std::span<const double, kFeatureCount> values() const { return v_; }
  double operator[](int i) const { return v_[static_cast<std::size_t>(i)]; }
  double at_name(std::string_view name) const;
  bool operator==(const FeatureVector&) const = default;

 private:
  std::array<double, kFeatureCount> v_{};
};

FeatureVector extract(const Scenario& s);
std::array<double, kInstrCategoryCount> densities(const InstrCounts& counts, int total);
std::map<InstrCategory, double> densities(const std::map<InstrCategory, int>& counts, int total);

// ------------------------------------------------------------- synthgen
std::vector<KernelDescriptor> generate_kernels(int n, std::uint64_t seed);
std::vector<KernelDescriptor> reference_kernels(int gaussian_border = 5);
std::vector<DatasetDescriptor> generate_datasets();
std::vector<DeviceDescriptor> reference_devices();        // the paper's Table 1 rig
std::vector<Scenario> standard_scenarios(std::uint64_t seed);

// The device this process runs on, from cudaDeviceProp (via the C-ABI's
// sk_device_features).  Throws DeviceError without a CUDA device.
DeviceDescriptor device_from_cuda(int device = 0);

}  // namespace wgtb
