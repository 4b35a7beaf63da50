// CSV / JSON persistence; formats and error behaviour follow the reference's
// datastore.cpp:18-400 so files interchange in both directions.
#include "wgtb/io.hpp"

#include <algorithm>
#include <charconv>
#include <fstream>
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
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open " + path.string());
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void write_text(const fs::path& path, const std::string& text) {
  std::ofstream out(path, std::ios::binary | std::ios::trunc);
  if (!out) throw IoError("cannot write " + path.string());
  out << text;
  if (!out) throw IoError("write failed for " + path.string());
}

// ---------------------------------------------------------------- samples
std::string samples_to_csv(const SampleTable& table) {
  std::string out(kSamplesHeader);
  out += '\n';
  for (const auto& [id, sizes] : table.rows()) {
    for (const auto& [w, runs] : sizes) {
      const std::string key = id + ',' + std::to_string(w.cols()) + ',' + std::to_string(w.rows()) + ',';
      for (double t : runs) out.append(key).append(format_double(t)).append("\n");
    }
  }
  return out;
}

SampleTable samples_from_csv(const std::string& text) {
  SampleTable table;
  std::set<std::pair<std::string, WorkgroupSize>> closed;
  std::pair<std::string, WorkgroupSize> open_key;
  bool have_open = false;
  parse_samples(text, [&](std::string id, WorkgroupSize w, double ms, std::size_t line) {
    auto key = std::make_pair(std::move(id), w);
    if (!have_open || key != open_key) {
      // a group may not reappear once another group has started
      if (closed.contains(key)) {
        throw DuplicateTestCase("duplicate test case " + key.first + " " + w.str() + " (line " +
                                std::to_string(line) + ")");
      }
      if (have_open) closed.insert(open_key);
      open_key = key;
      have_open = true;
    }
    table.add_runtime(key.first, w, ms);
  });
  return table;
}

void save_samples(const SampleTable& t, const fs::path& p) { write_text(p, samples_to_csv(t)); }
SampleTable load_samples(const fs::path& p) { return samples_from_csv(read_text(p)); }

// ---------------------------------------------------------------- refused
std::string refused_to_csv(const RefusedRecord& refused) {
  std::string out(kRefusedHeader);
  out += '\n';
  for (const auto& [id, sizes] : refused) {
    for (const WorkgroupSize& w : sizes) {
      out += id + ',' + std::to_string(w.cols()) + ',' + std::to_string(w.rows()) + '\n';
    }
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
json device_to_json(const DeviceDescriptor& d) {
  return json{{"id", d.id},
              {"device_type", to_string(d.device_type)},
              {"vendor_class", to_string(d.vendor_class)},
              {"compute_units", d.compute_units},
              {"frequency_mhz", d.frequency_mhz},
              {"local_mem_kb", d.local_mem_kb},
              {"global_cache_kb", d.global_cache_kb},
              {"global_mem_mb", d.global_mem_mb},
              {"device_max_wgsize", d.device_max_wgsize},
              {"simd_width", d.simd_width}};
}

DeviceDescriptor device_from_json(const json& j) {
  DeviceDescriptor d;
  d.id = j.at("id").get<std::string>();
  d.device_type = device_type_from_string(j.at("device_type").get<std::string>());
  d.vendor_class = vendor_class_from_string(j.at("vendor_class").get<std::string>());
  j.at("compute_units").get_to(d.compute_units);
  j.at("frequency_mhz").get_to(d.frequency_mhz);
  j.at("local_mem_kb").get_to(d.local_mem_kb);
  j.at("global_cache_kb").get_to(d.global_cache_kb);
  j.at("global_mem_mb").get_to(d.global_mem_mb);
  j.at("device_max_wgsize").get_to(d.device_max_wgsize);
  j.at("simd_width").get_to(d.simd_width);
  d.validate();
  return d;
}

json kernel_to_json(const KernelDescriptor& k) {
  json counts = json::object();
  for (int i = 0; i < kInstrCategoryCount; ++i) {
    counts[std::string(to_string(static_cast<InstrCategory>(i)))] = k.instr_counts[static_cast<std::size_t>(i)];
  }
  return json{{"name", k.name},   {"north", k.north}, {"south", k.south},
              {"east", k.east},   {"west", k.west},   {"instr_counts", counts},
              {"total_instructions", k.total_instructions}, {"complexity", k.complexity}};
}

KernelDescriptor kernel_from_json(const json& j) {
  KernelDescriptor k;
  k.name = j.at("name").get<std::string>();
  j.at("north").get_to(k.north);
  j.at("south").get_to(k.south);
  j.at("east").get_to(k.east);
  j.at("west").get_to(k.west);
  for (int i = 0; i < kInstrCategoryCount; ++i) {
    k.instr_counts[static_cast<std::size_t>(i)] =
        j.at("instr_counts").at(std::string(to_string(static_cast<InstrCategory>(i)))).get<int>();
  }
  j.at("total_instructions").get_to(k.total_instructions);
  j.at("complexity").get_to(k.complexity);
  k.validate();
  return k;
}

json dataset_to_json(const DatasetDescriptor& d) {
  return json{{"width", d.width}, {"height", d.height}, {"in_type", to_string(d.in_type)},
              {"out_type", to_string(d.out_type)}};
}

DatasetDescriptor dataset_from_json(const json& j) {
  DatasetDescriptor d;
  j.at("width").get_to(d.width);
  j.at("height").get_to(d.height);
  d.in_type = element_type_from_string(j.at("in_type").get<std::string>());
  d.out_type = element_type_from_string(j.at("out_type").get<std::string>());
  d.validate();
  return d;
}

void save_descriptors(const DescriptorSet& set, const fs::path& dir) {
  for (const char* sub : {"devices", "kernels", "datasets"}) fs::create_directories(dir / sub);
  for (const auto& d : set.devices) {
    d.validate();
    write_text(dir / "devices" / (d.id + ".json"), device_to_json(d).dump(2) + "\n");
  }
  for (const auto& k : set.kernels) {
    k.validate();
    write_text(dir / "kernels" / (k.name + ".json"), kernel_to_json(k).dump(2) + "\n");
  }
  for (const auto& d : set.datasets) {
    d.validate();
    const std::string stem = std::to_string(d.width) + "x" + std::to_string(d.height) + "-" +
                             std::string(to_string(d.in_type)) + "-" + std::string(to_string(d.out_type));
    write_text(dir / "datasets" / (stem + ".json"), dataset_to_json(d).dump(2) + "\n");
  }
}

DescriptorSet load_descriptors(const fs::path& dir) {
  DescriptorSet s;
  s.devices = load_dir<DeviceDescriptor>(dir / "devices", device_from_json);
  s.kernels = load_dir<KernelDescriptor>(dir / "kernels", kernel_from_json);
  s.datasets = load_dir<DatasetDescriptor>(dir / "datasets", dataset_from_json);
  return s;
}

std::vector<Scenario> cross_scenarios(const DescriptorSet& set) {
  std::vector<Scenario> out;
  for (const auto& d : set.devices) {
    for (const auto& k : set.kernels) {
      for (const auto& ds : set.datasets) out.push_back(make_scenario(d, k, ds));
    }
  }
  std::sort(out.begin(), out.end(), [](const Scenario& a, const Scenario& b) { return a.id < b.id; });
  return out;
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
