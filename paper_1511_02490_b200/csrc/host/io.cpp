// CSV / JSON persistence; formats and error behaviour follow the reference's
// datastore.cpp:18-400 so files interchange in both directions.
#include "wgtb/io.hpp"

#include <algorithm>
#include <charconv>
#include <cstdio>
#include <sstream>

namespace wgtb {

namespace fs = std::filesystem;
using nlohmann::json;

namespace {

constexpr std::string_view kSamplesHeader = "scenario_id,w_c,w_r,runtime_ms";
constexpr std::string_view kRefusedHeader = "scenario_id,w_c,w_r";
constexpr std::string_view kContextsHeader = "scenario_id,device_max,kernel_max";

// Iterates the data lines of a CSV with the given header:
// fn(fields, line_no).  CR is stripped; blank lines are skipped.
template <typename Fn>
void for_each_record(const std::string& text, std::string_view header, Fn&& fn) {
  std::istringstream in(text);
  std::string line;
  std::size_t line_no = 0;
  bool header_seen = false;
  while (std::getline(in, line)) {
    ++line_no;
    if (!line.empty() && line.back() == '\r') line.pop_back();
    if (!header_seen) {
      if (line != header) throw ParseError("expected header '" + std::string(header) + "'", line_no);
      header_seen = true;
      continue;
    }
    if (line.empty()) continue;
    std::vector<std::string_view> fields;
    std::string_view rest(line);
    for (;;) {
      auto comma = rest.find(',');
      fields.push_back(rest.substr(0, comma));
      if (comma == std::string_view::npos) break;
      rest.remove_prefix(comma + 1);
    }
    fn(fields, line_no);
  }
  if (!header_seen) throw ParseError("missing header '" + std::string(header) + "'", 1);
}

int int_field(std::string_view s, std::size_t line, const char* what) {
  int v = 0;
  auto [end, ec] = std::from_chars(s.data(), s.data() + s.size(), v);
  if (ec != std::errc{} || end != s.data() + s.size()) {
    throw ParseError(std::string("bad ") + what + " '" + std::string(s) + "'", line);
  }
  return v;
}

WorkgroupSize size_fields(std::string_view c, std::string_view r, std::size_t line) {
  int wc = int_field(c, line, "w_c");
  int wr = int_field(r, line, "w_r");
  if (wc < 1 || wr < 1) throw ParseError("workgroup size dimensions must be >= 1", line);
  return {wc, wr};
}

// One observation line of a samples CSV -> fn(id, w, ms, line).
template <typename Fn>
void parse_samples(const std::string& text, Fn&& fn) {
  for_each_record(text, kSamplesHeader, [&](const auto& f, std::size_t line) {
    if (f.size() != 4) throw ParseError("expected 4 fields, got " + std::to_string(f.size()), line);
    if (f[0].empty()) throw ParseError("empty scenario id", line);
    WorkgroupSize w = size_fields(f[1], f[2], line);
    double ms = 0.0;
    auto [end, ec] = std::from_chars(f[3].data(), f[3].data() + f[3].size(), ms);
    if (ec != std::errc{} || end != f[3].data() + f[3].size()) {
      throw ParseError("bad runtime '" + std::string(f[3]) + "'", line);
    }
    if (!(ms > 0.0)) throw ParseError("runtime must be positive, got '" + std::string(f[3]) + "'", line);
    fn(std::string(f[0]), w, ms, line);
  });
}

json parse_json(const fs::path& p) {
  try {
    return json::parse(read_text(p));
  } catch (const json::parse_error& e) {
    throw ParseError("bad JSON in " + p.string() + ": " + e.what());
  }
}

template <typename T, typename FromJson>
std::vector<T> load_dir(const fs::path& dir, FromJson&& from_json) {
  if (!fs::is_directory(dir)) throw IoError("missing descriptor directory " + dir.string());
  std::vector<fs::path> files;
  for (const auto& e : fs::directory_iterator(dir)) {
    if (e.path().extension() == ".json") files.push_back(e.path());
  }
  std::sort(files.begin(), files.end());
  std::vector<T> out;
  for (const auto& f : files) {
    try {
      out.push_back(from_json(parse_json(f)));
    } catch (const json::exception& e) {
      throw ParseError("bad descriptor " + f.string() + ": " + e.what());
    }
  }
  return out;
}

}  // namespace

std::string read_text(const fs::path& path) {
  std::error_code ec;
  const auto size = fs::file_size(path, ec);
  std::FILE* f = ec ? nullptr : std::fopen(path.c_str(), "rb");
  if (!f) throw IoError(path.string() + ": cannot be opened for reading");
  std::string text(size, '\0');
  const std::size_t got = size ? std::fread(text.data(), 1, size, f) : 0;
  std::fclose(f);
  if (got != size) throw IoError(path.string() + ": short read");
  return text;
}

void write_text(const fs::path& path, const std::string& text) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw IoError(path.string() + ": cannot be opened for writing");
  const std::size_t put = std::fwrite(text.data(), 1, text.size(), f);
  const bool closed = std::fclose(f) == 0;
  if (put != text.size() || !closed) throw IoError(path.string() + ": write failed");
}

// ---------------------------------------------------------------- samples
// "<id>,<w_c>,<w_r>" - the leading columns of every samples / refused line
static std::string case_key(const std::string& id, WorkgroupSize w) {
  std::string k = id;
  k += ',';
  k += std::to_string(w.cols());
  k += ',';
  k += std::to_string(w.rows());
  return k;
}

std::string samples_to_csv(const SampleTable& table) {
  std::string out(kSamplesHeader);
  out.push_back('\n');
  for (const auto& [id, sizes] : table.rows()) {
    for (const auto& [w, runs] : sizes) {
      const std::string key = case_key(id, w);
      for (double t : runs) (out += key) += ',' + format_double(t) + '\n';
    }
  }
  return out;
}

// Lines of one test case must be contiguous (datastore.cpp:21-25): a case
// that was already started and then left may not start again.
SampleTable samples_from_csv(const std::string& text) {
  SampleTable table;
  std::string cur_id;
  WorkgroupSize cur_w;
  bool started = false;
  parse_samples(text, [&](std::string id, WorkgroupSize w, double ms, std::size_t line) {
    const bool same = started && w == cur_w && id == cur_id;
    if (!same) {
      if (table.has(id, w)) {
        throw DuplicateTestCase("test case " + id + " " + w.str() + " reappears on line " + std::to_string(line) +
                                " after other cases");
      }
      cur_id = id;
      cur_w = w;
      started = true;
    }
    table.add_runtime(id, w, ms);
  });
  return table;
}

void save_samples(const SampleTable& t, const fs::path& p) { write_text(p, samples_to_csv(t)); }
SampleTable load_samples(const fs::path& p) { return samples_from_csv(read_text(p)); }

// ---------------------------------------------------------------- refused
std::string refused_to_csv(const RefusedRecord& refused) {
  std::string out(kRefusedHeader);
  out.push_back('\n');
  for (const auto& [id, sizes] : refused) {
    for (const WorkgroupSize& w : sizes) (out += case_key(id, w)) += '\n';
  }
  return out;
}

RefusedRecord refused_from_csv(const std::string& text) {
  RefusedRecord rec;
  for_each_record(text, kRefusedHeader, [&](const auto& f, std::size_t line) {
    if (f.size() != 3 || f[0].empty()) throw ParseError("expected 'scenario_id,w_c,w_r'", line);
    rec[std::string(f[0])].insert(size_fields(f[1], f[2], line));
  });
  return rec;
}

void save_refused(const RefusedRecord& r, const fs::path& p) { write_text(p, refused_to_csv(r)); }
RefusedRecord load_refused(const fs::path& p) { return refused_from_csv(read_text(p)); }

// --------------------------------------------------------------- contexts
std::string contexts_to_csv(const ContextRecord& contexts) {
  std::string out(kContextsHeader);
  out += '\n';
  for (const auto& [id, ctx] : contexts) {
    out += id + ',' + std::to_string(ctx.device_max()) + ',' + std::to_string(ctx.kernel_max()) + '\n';
  }
  return out;
}

ContextRecord contexts_from_csv(const std::string& text, const RefusedRecord& refused) {
  ContextRecord rec;
  for_each_record(text, kContextsHeader, [&](const auto& f, std::size_t line) {
    if (f.size() != 3 || f[0].empty()) throw ParseError("expected 'scenario_id,device_max,kernel_max'", line);
    std::string id(f[0]);
    std::set<WorkgroupSize> ref;
    if (auto it = refused.find(id); it != refused.end()) ref = it->second;
    rec.emplace(id, ConstraintContext(int_field(f[1], line, "device_max"),
                                      int_field(f[2], line, "kernel_max"), std::move(ref)));
  });
  return rec;
}

void save_contexts(const ContextRecord& c, const fs::path& p) { write_text(p, contexts_to_csv(c)); }
ContextRecord load_contexts(const fs::path& p, const RefusedRecord& refused) {
  return contexts_from_csv(read_text(p), refused);
}

// ------------------------------------------------------------ descriptors
// The integer fields of each descriptor as (JSON key, member) tables: one
// loop writes them, one reads them back.  nlohmann::json objects are ordered
// by key, so the dumped text is the reference's byte for byte.
namespace {

constexpr std::pair<const char*, int DeviceDescriptor::*> kDeviceInts[] = {
    {"compute_units", &DeviceDescriptor::compute_units},     {"frequency_mhz", &DeviceDescriptor::frequency_mhz},
    {"local_mem_kb", &DeviceDescriptor::local_mem_kb},       {"global_cache_kb", &DeviceDescriptor::global_cache_kb},
    {"global_mem_mb", &DeviceDescriptor::global_mem_mb},     {"device_max_wgsize", &DeviceDescriptor::device_max_wgsize},
    {"simd_width", &DeviceDescriptor::simd_width},
};
constexpr std::pair<const char*, int KernelDescriptor::*> kKernelInts[] = {
    {"north", &KernelDescriptor::north}, {"south", &KernelDescriptor::south},
    {"east", &KernelDescriptor::east},   {"west", &KernelDescriptor::west},
    {"total_instructions", &KernelDescriptor::total_instructions},
};
constexpr std::pair<const char*, int DatasetDescriptor::*> kDatasetInts[] = {
    {"width", &DatasetDescriptor::width}, {"height", &DatasetDescriptor::height}};

template <typename D, std::size_t N>
void put_ints(json& j, const D& d, const std::pair<const char*, int D::*> (&fields)[N]) {
  for (const auto& [key, member] : fields) j[key] = d.*member;
}

template <typename D, std::size_t N>
void get_ints(const json& j, D& d, const std::pair<const char*, int D::*> (&fields)[N]) {
  for (const auto& [key, member] : fields) d.*member = j.at(key).template get<int>();
}

std::string category_key(int i) { return std::string(to_string(static_cast<InstrCategory>(i))); }

std::string dataset_stem(const DatasetDescriptor& d) {
  std::string stem = std::to_string(d.width);
  stem += 'x';
  stem += std::to_string(d.height);
  stem += '-';
  stem += to_string(d.in_type);
  stem += '-';
  stem += to_string(d.out_type);
  return stem;
}

}  // namespace

json device_to_json(const DeviceDescriptor& d) {
  json j = json::object();
  j["id"] = d.id;
  j["device_type"] = to_string(d.device_type);
  j["vendor_class"] = to_string(d.vendor_class);
  put_ints(j, d, kDeviceInts);
  return j;
}

static std::string text_of(const json& j, const char* key) { return j.at(key).get<std::string>(); }

DeviceDescriptor device_from_json(const json& j) {
  DeviceDescriptor d;
  d.id = text_of(j, "id");
  d.device_type = device_type_from_string(text_of(j, "device_type"));
  d.vendor_class = vendor_class_from_string(text_of(j, "vendor_class"));
  get_ints(j, d, kDeviceInts);
  d.validate();
  return d;
}

json kernel_to_json(const KernelDescriptor& k) {
  json j = json::object();
  j["name"] = k.name;
  j["complexity"] = k.complexity;
  put_ints(j, k, kKernelInts);
  json& counts = j["instr_counts"] = json::object();
  for (int i = 0; i < kInstrCategoryCount; ++i) counts[category_key(i)] = k.instr_counts[static_cast<std::size_t>(i)];
  return j;
}

KernelDescriptor kernel_from_json(const json& j) {
  KernelDescriptor k;
  k.name = text_of(j, "name");
  k.complexity = j.at("complexity").get<bool>();
  get_ints(j, k, kKernelInts);
  const json& counts = j.at("instr_counts");
  for (int i = 0; i < kInstrCategoryCount; ++i) {
    k.instr_counts[static_cast<std::size_t>(i)] = counts.at(category_key(i)).get<int>();
  }
  k.validate();
  return k;
}

json dataset_to_json(const DatasetDescriptor& d) {
  json j = json::object();
  put_ints(j, d, kDatasetInts);
  j["in_type"] = to_string(d.in_type);
  j["out_type"] = to_string(d.out_type);
  return j;
}

DatasetDescriptor dataset_from_json(const json& j) {
  DatasetDescriptor d;
  get_ints(j, d, kDatasetInts);
  d.in_type = element_type_from_string(text_of(j, "in_type"));
  d.out_type = element_type_from_string(text_of(j, "out_type"));
  d.validate();
  return d;
}

void save_descriptors(const DescriptorSet& set, const fs::path& dir) {
  auto put = [&](const char* sub, const std::string& stem, const json& j) {
    fs::create_directories(dir / sub);
    write_text(dir / sub / (stem + ".json"), j.dump(2) + "\n");
  };
  for (const auto& d : set.devices) {
    d.validate();
    put("devices", d.id, device_to_json(d));
  }
  for (const auto& k : set.kernels) {
    k.validate();
    put("kernels", k.name, kernel_to_json(k));
  }
  for (const auto& d : set.datasets) {
    d.validate();
    put("datasets", dataset_stem(d), dataset_to_json(d));
  }
  for (const char* sub : {"devices", "kernels", "datasets"}) fs::create_directories(dir / sub);
}

DescriptorSet load_descriptors(const fs::path& dir) {
  DescriptorSet s;
  s.devices = load_dir<DeviceDescriptor>(dir / "devices", device_from_json);
  s.kernels = load_dir<KernelDescriptor>(dir / "kernels", kernel_from_json);
  s.datasets = load_dir<DatasetDescriptor>(dir / "datasets", dataset_from_json);
  return s;
}

// Every (device, kernel, dataset) combination, in scenario-id order.
std::vector<Scenario> cross_scenarios(const DescriptorSet& set) {
  std::vector<Scenario> all;
  all.reserve(set.devices.size() * set.kernels.size() * set.datasets.size());
  for (std::size_t n = 0; n < all.capacity(); ++n) {
    const std::size_t ds = n % set.datasets.size(), rest = n / set.datasets.size();
    all.push_back(make_scenario(set.devices[rest / set.kernels.size()], set.kernels[rest % set.kernels.size()],
                                set.datasets[ds]));
  }
  std::ranges::sort(all, {}, &Scenario::id);
  return all;
}

SampleTable import_external(const fs::path& csv_path, const fs::path& descriptor_dir) {
  std::set<std::string> known;
  for (const auto& s : cross_scenarios(load_descriptors(descriptor_dir))) known.insert(s.id);
  SampleTable table;
  parse_samples(read_text(csv_path), [&](std::string id, WorkgroupSize w, double ms, std::size_t line) {
    if (!known.contains(id)) {
      throw UnknownScenario("scenario '" + id + "' matches no registered descriptor combination (line " +
                            std::to_string(line) + ")");
    }
    table.add_runtime(id, w, ms);
  });
  return table;
}

}  // namespace wgtb
