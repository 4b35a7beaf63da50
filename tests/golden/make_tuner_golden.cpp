// Generates tests/golden/tuner/ from the REFERENCE library (oracle/_ref):
// the standard 50-scenario fixture (seed 17) as descriptor JSON, a simulated
// sweep (sigma 0.05, 5 samples, max workgroup size capped at 64 to keep the
// fixture small) as samples / refused / contexts CSV, and the reference's own
// evaluate() metrics for every technique under the synthetic->real split and
// 10-fold cross-validation (time_ms zeroed: it is wall-clock).
// Build + run: bash tests/golden/make_tuner_golden.sh
#include <filesystem>
#include <fstream>
#include <iostream>

#include "wgtune/bench.hpp"
#include "wgtune/datastore.hpp"
#include "wgtune/simoracle.hpp"
#include "wgtune/synthgen.hpp"

using namespace wgtune;
namespace fs = std::filesystem;

int main(int argc, char** argv) {
  const fs::path out = argc > 1 ? argv[1] : "tests/golden/tuner";
  fs::create_directories(out);
  auto scenarios = standard_scenarios(17);
  DescriptorSet set;
  std::set<std::string> seen_dev, seen_k, seen_ds;
  for (const auto& s : scenarios) {
    if (seen_dev.insert(s.device.id).second) set.devices.push_back(s.device);
    if (seen_k.insert(s.kernel.name).second) set.kernels.push_back(s.kernel);
    std::string dk = std::to_string(s.dataset.width) + std::string(to_string(s.dataset.in_type));
    if (seen_ds.insert(dk).second) set.datasets.push_back(s.dataset);
  }
  save_descriptors(set, out / "descriptors");
  OracleConfig cfg;
  cfg.seed = 17;
  cfg.noise_sigma = 0.05;
  cfg.min_samples = 5;
  cfg.max_wgsize_cap = 64;
  CollectResult col = collect(scenarios, cfg);
  save_samples(col.table, out / "samples.csv");
  save_refused(col.refused, out / "refused.csv");
  {
    std::ofstream f(out / "contexts.csv");
    f << "scenario_id,device_max,kernel_max\n";
    for (const auto& [id, c] : col.contexts) f << id << ',' << c.device_max() << ',' << c.kernel_max() << '\n';
  }
  EvalData data;
  data.table = col.table;
  for (const auto& s : scenarios) {
    data.scenarios.emplace(s.id, s);
    data.contexts.emplace(s.id, col.contexts.at(s.id));
  }
  // ids in EvalData map order, as the reference CLI's cmd_evaluate builds
  // them (tools/wgtune.cpp:129-134)
  std::vector<std::string> ids;
  std::vector<Scenario> ordered;
  for (const auto& [id, s] : data.scenarios) {
    ids.push_back(id);
    ordered.push_back(s);
  }
  std::vector<std::pair<std::string, std::vector<Partition>>> plans = {
      {"synthreal", {partition_synthetic_real(ordered)}}, {"kfold", partition_kfold(ids, 10, 0)}};
  for (const auto& [pname, parts] : plans) {
    std::vector<MetricsRow> rows;
    for (const auto& tech : technique_ids()) {
      for (const auto& [train, test] : parts) {
        auto t = make_technique(tech);
        for (auto& r : rows_of(evaluate(*t, train, test, data, 0))) {
          r.time_ms = 0.0;
          rows.push_back(r);
        }
      }
    }
    write_metrics_csv(rows, out / ("expected_metrics_" + pname + ".csv"));
    std::cout << pname << ": " << rows.size() << " rows\n" << format_report(summarize(rows));
  }
  std::cout << "scenarios " << scenarios.size() << ", test cases " << col.table.row_count() << "\n";
  return 0;
}
