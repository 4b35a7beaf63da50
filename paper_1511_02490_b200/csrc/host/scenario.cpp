// Descriptors, scenario ids, the fv1 feature schema and the synthetic
// benchmark generator.  Semantics follow the reference's scenario.cpp:55-141,
// features.cpp:10-93 and synthgen.cpp:16-160 (RNG draw order included, so
// generated kernels are identical); device descriptors additionally come
// from cudaDeviceProp (device_from_cuda).
#include <numeric>

#include "sk_stencil.h"
#include "wgtb/scenario.hpp"

namespace wgtb {

namespace {

template <typename E, std::size_t N>
E enum_from(std::string_view s, const std::array<std::string_view, N>& names, const char* what) {
  for (std::size_t i = 0; i < N; ++i) {
    if (names[i] == s) return static_cast<E>(i);
  }
  throw ParseError(std::string("unknown ") + what + " '" + std::string(s) + "'");
}

constexpr std::array<std::string_view, 2> kDeviceTypes = {"CPU", "GPU"};
constexpr std::array<std::string_view, 4> kVendors = {"INTEL_CPU", "AMD_GPU", "NVIDIA_GPU",
                                                      "OTHER"};
constexpr std::array<std::string_view, 3> kElements = {"INT32", "FLOAT32", "FLOAT64"};
constexpr std::array<std::string_view, kInstrCategoryCount> kCategories = {
    "load", "store", "int_arith", "float_arith", "branch", "vector", "call", "other"};

bool bad_name(const std::string& s) { return s.empty() || s.find_first_of("/,\n") != s.npos; }

}  // namespace

std::string_view to_string(DeviceType v) { return kDeviceTypes[static_cast<int>(v)]; }
std::string_view to_string(VendorClass v) { return kVendors[static_cast<int>(v)]; }
std::string_view to_string(ElementType v) { return kElements[static_cast<int>(v)]; }
std::string_view to_string(InstrCategory v) { return kCategories[static_cast<int>(v)]; }
DeviceType device_type_from_string(std::string_view s) {
  return enum_from<DeviceType>(s, kDeviceTypes, "device type");
}
VendorClass vendor_class_from_string(std::string_view s) {
  return enum_from<VendorClass>(s, kVendors, "vendor class");
}
ElementType element_type_from_string(std::string_view s) {
  return enum_from<ElementType>(s, kElements, "element type");
}
InstrCategory instr_category_from_string(std::string_view s) {
  return enum_from<InstrCategory>(s, kCategories, "instruction category");
}

int element_size_bytes(ElementType t) { return t == ElementType::FLOAT64 ? 8 : 4; }

// ---------------------------------------------------------- validation
void DeviceDescriptor::validate() const {
  if (bad_name(id)) throw InvalidDescriptor("device id must be non-empty without '/', ',': '" + id + "'");
  if (compute_units < 1 || frequency_mhz < 1 || local_mem_kb < 1 || global_mem_mb < 1 ||
      global_cache_kb < 0) {
    throw InvalidDescriptor("device '" + id + "' has a non-positive hardware field");
  }
  const int m = device_max_wgsize;
  if (m < 64 || (m & (m - 1)) != 0) {
    throw InvalidDescriptor("device '" + id + "' max workgroup size must be a power of two >= 64");
  }
  if (simd_width != 8 && simd_width != 16 && simd_width != 32 && simd_width != 64) {
    throw InvalidDescriptor("device '" + id + "' simd width must be 8, 16, 32 or 64");
  }
  if (vendor_class == VendorClass::INTEL_CPU && device_type != DeviceType::CPU) {
    throw InvalidDescriptor("device '" + id + "': INTEL_CPU vendor class requires a CPU device");
  }
}

void KernelDescriptor::validate() const {
  if (bad_name(name)) throw InvalidDescriptor("kernel name must be non-empty without '/', ','");
  for (int b : {north, south, east, west}) {
    if (b < 0 || b > 64) throw InvalidDescriptor("kernel '" + name + "' border outside [0, 64]");
  }
  if (total_instructions < 1) throw InvalidDescriptor("kernel '" + name + "' needs instructions >= 1");
  long long sum = 0;
  for (int c : instr_counts) {
    if (c < 0) throw InvalidDescriptor("kernel '" + name + "' has a negative instruction count");
    sum += c;
  }
  if (sum != total_instructions) {
    throw InvalidDescriptor("kernel '" + name + "' instruction counts sum to " +
                            std::to_string(sum) + ", not " + std::to_string(total_instructions));
  }
}

void DatasetDescriptor::validate() const {
  if (width < 1 || height < 1) {
    throw InvalidDescriptor("dataset dimensions must be >= 1, got " + std::to_string(width) + "x" +
                            std::to_string(height));
  }
}

std::string scenario_id(const DeviceDescriptor& d, const KernelDescriptor& k,
                        const DatasetDescriptor& ds) {
  std::string id;
  id.append(d.id).append("/").append(k.name).append("/");
  id.append(std::to_string(ds.width)).append("x").append(std::to_string(ds.height)).append("/");
  id.append(to_string(ds.in_type)).append("-").append(to_string(ds.out_type));
  return id;
}

Scenario make_scenario(const DeviceDescriptor& d, const KernelDescriptor& k,
                       const DatasetDescriptor& ds) {
  d.validate();
  k.validate();
  ds.validate();
  return Scenario{d, k, ds, scenario_id(d, k, ds)};
}

// ------------------------------------------------------------ features
const std::array<std::string_view, kFeatureCount>& feature_names() {
  static const std::array<std::string_view, kFeatureCount> names = {
      "compute_units", "frequency_mhz", "local_mem_kb", "global_cache_kb", "global_mem_mb",
      "device_max_wgsize", "simd_width", "is_cpu", "is_gpu", "vendor_class",
      "border_north", "border_south", "border_east", "border_west", "total_instructions",
      "density_load", "density_store", "density_int_arith", "density_float_arith",
      "density_branch", "density_vector", "density_call", "density_other", "complexity",
      "width", "height", "in_type_size", "out_type_size", "element_count"};
  return names;
}

double FeatureVector::at_name(std::string_view name) const {
  const auto& names = feature_names();
  for (std::size_t i = 0; i < names.size(); ++i) {
    if (names[i] == name) return v_[i];
  }
  throw InvalidArgument("unknown feature '" + std::string(name) + "'");
}

std::array<double, kInstrCategoryCount> densities(const InstrCounts& counts, int total) {
  if (total <= 0) throw InvalidArgument("instruction total must be positive");
  const int sum = std::accumulate(counts.begin(), counts.end(), 0);
  if (sum != total) {
    throw InconsistentCounts("instruction counts sum to " + std::to_string(sum) + ", expected " +
                             std::to_string(total));
  }
  std::array<double, kInstrCategoryCount> out{};
  for (int i = 0; i < kInstrCategoryCount; ++i) {
    out[static_cast<std::size_t>(i)] = static_cast<double>(counts[static_cast<std::size_t>(i)]) / total;
  }
  return out;
}

std::map<InstrCategory, double> densities(const std::map<InstrCategory, int>& counts, int total) {
  InstrCounts flat{};
  for (const auto& [cat, n] : counts) flat[static_cast<std::size_t>(cat)] = n;
  const auto d = densities(flat, total);
  std::map<InstrCategory, double> out;
  for (int i = 0; i < kInstrCategoryCount; ++i) out[static_cast<InstrCategory>(i)] = d[static_cast<std::size_t>(i)];
  return out;
}

FeatureVector extract(const Scenario& s) {
  std::array<double, kFeatureCount> f{};
  std::size_t n = 0;
  auto put = [&](double v) { f[n++] = v; };
  const DeviceDescriptor& d = s.device;
  put(d.compute_units);
  put(d.frequency_mhz);
  put(d.local_mem_kb);
  put(d.global_cache_kb);
  put(d.global_mem_mb);
  put(d.device_max_wgsize);
  put(d.simd_width);
  put(d.device_type == DeviceType::CPU);
  put(d.device_type == DeviceType::GPU);
  put(static_cast<int>(d.vendor_class));
  const KernelDescriptor& k = s.kernel;
  put(k.north);
  put(k.south);
  put(k.east);
  put(k.west);
  put(k.total_instructions);
  for (double x : densities(k.instr_counts, k.total_instructions)) put(x);
  put(k.complexity);
  const DatasetDescriptor& ds = s.dataset;
  put(ds.width);
  put(ds.height);
  put(element_size_bytes(ds.in_type));
  put(element_size_bytes(ds.out_type));
  put(static_cast<double>(ds.element_count()));
  return FeatureVector(f);
}

// ------------------------------------------------------------ synthgen
namespace {

// Per-category weights of the synthetic instruction split (lightweight vs
// compute-intensive templates, §3.3); data of synthgen.cpp:18-21.
constexpr std::array<double, kInstrCategoryCount> kLightSplit = {0.30, 0.15, 0.15, 0.10,
                                                                 0.10, 0.05, 0.05, 0.10};
constexpr std::array<double, kInstrCategoryCount> kHeavySplit = {0.25, 0.08, 0.12, 0.30,
                                                                 0.08, 0.07, 0.04, 0.06};

InstrCounts categorical_split(Rng& rng, int total, const std::array<double, kInstrCategoryCount>& w) {
  std::array<double, kInstrCategoryCount> cdf{};
  double acc = 0.0;
  for (std::size_t i = 0; i < w.size(); ++i) cdf[i] = (acc += w[i]);
  InstrCounts counts{};
  for (int draw = 0; draw < total; ++draw) {
    const double u = rng.uniform01() * acc;
    std::size_t c = 0;
    while (c + 1 < cdf.size() && u >= cdf[c]) ++c;
    ++counts[c];
  }
  return counts;
}

KernelDescriptor fixed_kernel(const char* name, int n, int s, int e, int w, InstrCounts counts,
                              bool heavy) {
  KernelDescriptor k;
  k.name = name;
  k.north = n;
  k.south = s;
  k.east = e;
  k.west = w;
  k.instr_counts = counts;
  k.total_instructions = std::accumulate(counts.begin(), counts.end(), 0);
  k.complexity = heavy;
  k.validate();
  return k;
}

}  // namespace

std::vector<KernelDescriptor> generate_kernels(int n, std::uint64_t seed) {
  if (n < 1) throw InvalidArgument("kernel count must be >= 1, got " + std::to_string(n));
  Rng rng(fnv1a64_mix(fnv1a64("synthgen"), seed));
  std::vector<KernelDescriptor> out;
  out.reserve(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    KernelDescriptor k;
    k.name = "synthetic-" + std::to_string(seed) + "-" + std::to_string(i);
    // draw order: complexity, N, S, E, W, total, split (Table 2 ranges)
    k.complexity = rng.coin();
    k.north = static_cast<int>(rng.range(1, 30));
    k.south = static_cast<int>(rng.range(1, 30));
    k.east = static_cast<int>(rng.range(1, 30));
    k.west = static_cast<int>(rng.range(1, 30));
    k.total_instructions = static_cast<int>(k.complexity ? rng.range(592, 706) : rng.range(67, 137));
    k.instr_counts = categorical_split(rng, k.total_instructions,
                                       k.complexity ? kHeavySplit : kLightSplit);
    k.validate();
    out.push_back(std::move(k));
  }
  return out;
}

std::vector<KernelDescriptor> reference_kernels(int g) {
  if (g < 1 || g > 10) throw InvalidArgument("gaussian border must be in [1, 10]");
  // PAPER.md Table 2 borders and totals; per-category splits are the
  // reference's fixture (synthgen.cpp:89-94).
  return {fixed_kernel("gaussian", g, g, g, g, {20, 8, 12, 24, 6, 0, 4, 8}, false),
          fixed_kernel("gol", 1, 1, 1, 1, {52, 20, 48, 0, 40, 0, 10, 20}, false),
          fixed_kernel("he", 1, 1, 1, 1, {28, 10, 16, 38, 8, 0, 5, 8}, true),
          fixed_kernel("nms", 1, 1, 1, 1, {60, 18, 38, 52, 32, 0, 8, 16}, false),
          fixed_kernel("sobel", 1, 1, 1, 1, {64, 20, 40, 74, 18, 0, 10, 20}, false),
          fixed_kernel("threshold", 0, 0, 0, 0, {12, 6, 10, 4, 8, 0, 2, 4}, false)};
}

std::vector<DatasetDescriptor> generate_datasets() {
  std::vector<DatasetDescriptor> out;
  for (int side : {512, 1024, 2048, 4096}) {
    for (ElementType t : {ElementType::INT32, ElementType::FLOAT32, ElementType::FLOAT64}) {
      out.push_back(DatasetDescriptor{side, side, t, t});
    }
  }
  return out;
}

std::vector<DeviceDescriptor> reference_devices() {
  // PAPER.md Table 1 (:404-414); max wgsize / simd width as in the
  // reference fixture (synthgen.cpp:131-138).
  struct Row {
    const char* id;
    DeviceType t;
    VendorClass v;
    int cu, mhz, lmem, cache, mem, maxwg, simd;
  };
  static const Row rows[] = {
      {"i5-2430M", DeviceType::CPU, VendorClass::INTEL_CPU, 4, 2400, 32, 256, 7937, 512, 8},
      {"i5-4570", DeviceType::CPU, VendorClass::INTEL_CPU, 4, 3200, 32, 256, 7901, 512, 8},
      {"i7-3820", DeviceType::CPU, VendorClass::INTEL_CPU, 8, 1200, 32, 256, 7944, 512, 16},
      {"tahiti-7970", DeviceType::GPU, VendorClass::AMD_GPU, 32, 1000, 32, 16, 2959, 256, 64},
      {"gtx-590", DeviceType::GPU, VendorClass::NVIDIA_GPU, 1, 1215, 48, 256, 1536, 512, 32},
      {"gtx-690", DeviceType::GPU, VendorClass::NVIDIA_GPU, 8, 1019, 48, 128, 2048, 512, 32},
      {"gtx-titan", DeviceType::GPU, VendorClass::NVIDIA_GPU, 14, 980, 48, 224, 6144, 1024, 32},
  };
  std::vector<DeviceDescriptor> out;
  for (const Row& r : rows) {
    DeviceDescriptor d{r.id, r.t, r.v, r.cu, r.mhz, r.lmem, r.cache, r.mem, r.maxwg, r.simd};
    d.validate();
    out.push_back(d);
  }
  return out;
}

std::vector<Scenario> standard_scenarios(std::uint64_t seed) {
  const auto devices = reference_devices();
  const auto datasets = generate_datasets();
  const auto synthetic = generate_kernels(40, seed);
  const auto real = reference_kernels();
  std::vector<Scenario> out;
  for (std::size_t i = 0; i < 40; ++i) {
    out.push_back(make_scenario(devices[i % 7], synthetic[i], datasets[(i * 5 + 3) % 12]));
  }
  for (std::size_t j = 0; j < 10; ++j) {
    out.push_back(make_scenario(devices[(j * 3 + 1) % 7], real[j % 6], datasets[(j * 7 + 2) % 12]));
  }
  return out;
}

DeviceDescriptor device_from_cuda(int device) {
  sk_device_props p{};
  if (sk_device_features(device, &p) != SK_OK) {
    throw DeviceError(std::string("cannot read CUDA device properties: ") + sk_last_error());
  }
  DeviceDescriptor d;
  d.id = p.name;
  d.device_type = DeviceType::GPU;
  d.vendor_class = VendorClass::NVIDIA_GPU;
  d.compute_units = p.compute_units;
  d.frequency_mhz = p.frequency_mhz;
  d.local_mem_kb = p.local_mem_kb;
  d.global_cache_kb = p.global_cache_kb;
  d.global_mem_mb = p.global_mem_mb;
  d.device_max_wgsize = p.device_max_wgsize;
  d.simd_width = p.simd_width;
  d.validate();
  return d;
}

}  // namespace wgtb
