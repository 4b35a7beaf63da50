// The reference's own evaluate() (bench.cpp:354-411) on B200 sweep data
// ("strongest end-to-end oracle"): EvalData is built from the
// RECORDED contexts (device max, real kernel max, refusals) as bench.hpp:37-41
// allows, instead of the simulator's assemble_eval_data.  Prints the
// reference's metrics CSV; tests/test_reference_evaluate.py compares it with
// `wgtb evaluate` on the same files.  TEST INFRASTRUCTURE (oracle/_ref).
//   ref_evaluate DESC_DIR SAMPLES REFUSED CONTEXTS TECHNIQUE PARTITION [FOLDS] [SEED]
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "wgtune/bench.hpp"
#include "wgtune/datastore.hpp"

using namespace wgtune;

int main(int argc, char** argv) {
  if (argc < 7) {
    std::cerr << "usage: ref_evaluate DESC SAMPLES REFUSED CONTEXTS TECHNIQUE PARTITION [FOLDS] [SEED]\n";
    return 2;
  }
  const std::string tech_id = argv[5], part = argv[6];
  const int folds = argc > 7 ? std::stoi(argv[7]) : 10;
  const std::uint64_t seed = argc > 8 ? std::stoull(argv[8]) : 0;
  const auto all = cross_scenarios(load_descriptors(argv[1]));
  SampleTable table = load_samples(argv[2]);
  const RefusedRecord refused = load_refused(argv[3]);
  std::ifstream cf(argv[4]);
  std::string line;
  std::getline(cf, line);  // scenario_id,device_max,kernel_max
  std::map<std::string, std::pair<int, int>> maxima;
  while (std::getline(cf, line)) {
    if (line.empty()) continue;
    std::stringstream ss(line);
    std::string id, dm, km;
    std::getline(ss, id, ',');
    std::getline(ss, dm, ',');
    std::getline(ss, km, ',');
    maxima[id] = {std::stoi(dm), std::stoi(km)};
  }
  EvalData data;
  std::vector<Scenario> scen;
  for (const auto& s : all) {
    if (!table.has_scenario(s.id) || !maxima.count(s.id)) continue;
    std::set<WorkgroupSize> r;
    if (auto it = refused.find(s.id); it != refused.end()) r = it->second;
    data.contexts.emplace(s.id, ConstraintContext(maxima[s.id].first, maxima[s.id].second, r));
    data.scenarios.emplace(s.id, s);
    scen.push_back(s);
  }
  data.table = std::move(table);
  std::vector<std::string> ids;
  for (const auto& [id, _] : data.scenarios) ids.push_back(id);
  std::vector<Partition> parts;
  if (part == "kfold") parts = partition_kfold(ids, folds, seed);
  else if (part == "synthreal") parts = {partition_synthetic_real(scen)};
  else if (part == "loo-kernel") parts = partition_leave_one_out(scen, LeaveOneOutDimension::Kernel);
  else if (part == "loo-dataset") parts = partition_leave_one_out(scen, LeaveOneOutDimension::Dataset);
  else {
    std::cerr << "unknown partition " << part << "\n";
    return 2;
  }
  std::vector<std::string> techs = tech_id == "all" ? technique_ids() : std::vector<std::string>{tech_id};
  std::vector<MetricsRow> rows;
  for (const auto& t : techs) {
    for (const auto& [train, test] : parts) {
      auto tech = make_technique(t);
      for (const auto& rec : evaluate(*tech, train, test, data, seed)) rows.push_back(rec.row);
    }
  }
  std::cout << metrics_to_csv(rows);
  return 0;
}
