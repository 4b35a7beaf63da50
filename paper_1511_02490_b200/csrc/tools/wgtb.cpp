// wgtb — command-line driver of the B200 autotuner (mirrors the reference's
// tools/wgtune.cpp:87-408 subcommands, without CLI11):
//
//   wgtb generate  --out DIR [--kernels N] [--seed S] [--reference] [--gaussian-border G]
//                  [--device cuda|fixture] [--datasets standard|SIDExSIDE,...]
//   wgtb collect   --scenarios DIR --out samples.csv [--refused F] [--contexts F]
//                  [--samples 30] [--warmup 3] [--no-flush] [--no-validate] [--cap M]
//                  [--border nearest|pad] [--k K] [--store all|mean] [--resume] [filters]
//   wgtb evaluate  --scenarios DIR --samples F --refused F --contexts F
//                  --technique T|all --partition kfold|synthreal|loo-kernel|loo-dataset|loo-device
//                  [--folds 10] [--seed S] [--metrics out.csv] [--pin-baseline WxH] [--expert]
//   wgtb train     --scenarios DIR --samples F --refused F --contexts F --technique T --out model.json
//   wgtb predict   --model model.json --kernel-json F --dataset WxH-IN-OUT [--device cuda|fixture:ID|json:PATH]
//                  [--refused F --contexts F]   (prints "wc wr")
//   wgtb features  [--device 0]                 (cudaDeviceProp -> DeviceDescriptor JSON)
//
// Exit codes: 0 success, 1 internal error, 2 usage / input error.
#include <chrono>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "wgtb/evaluation.hpp"
#include "wgtb/executor.hpp"
#include "wgtb/kernelgen.hpp"
#include "wgtb/io.hpp"
#include "wgtb/learn.hpp"

namespace fs = std::filesystem;
using namespace wgtb;

namespace {

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Args {
  std::map<std::string, std::vector<std::string>> opts;
  std::set<std::string> flags;

  Args(int argc, char** argv, int first, const std::set<std::string>& boolean) {
    for (int i = first; i < argc; ++i) {
      std::string a = argv[i];
      if (a.rfind("--", 0) != 0) throw UsageError("unexpected argument '" + a + "'");
      if (boolean.contains(a)) {
        flags.insert(a);
      } else {
        if (i + 1 >= argc) throw UsageError("missing value for " + a);
        opts[a].push_back(argv[++i]);
      }
    }
  }
  bool has(const std::string& k) const { return opts.contains(k) || flags.contains(k); }
  std::string get(const std::string& k, const std::string& def = "") const {
    auto it = opts.find(k);
    return it == opts.end() ? def : it->second.back();
  }
  std::string need(const std::string& k) const {
    if (!opts.contains(k)) throw UsageError("missing required option " + k);
    return get(k);
  }
  std::vector<std::string> all(const std::string& k) const {
    auto it = opts.find(k);
    return it == opts.end() ? std::vector<std::string>{} : it->second;
  }
  long long num(const std::string& k, long long def) const {
    return has(k) ? std::stoll(get(k)) : def;
  }
};

std::string dataset_key(const Scenario& s) {
  return std::to_string(s.dataset.width) + "x" + std::to_string(s.dataset.height) + "-" +
         std::string(to_string(s.dataset.in_type)) + "-" + std::string(to_string(s.dataset.out_type));
}

std::vector<Scenario> filtered(const DescriptorSet& set, const Args& a) {
  auto match = [](const std::vector<std::string>& want, const std::string& v) {
    return want.empty() || std::find(want.begin(), want.end(), v) != want.end();
  };
  std::vector<Scenario> out;
  for (auto& s : cross_scenarios(set)) {
    if (match(a.all("--device"), s.device.id) && match(a.all("--kernel"), s.kernel.name) &&
        match(a.all("--dataset"), dataset_key(s))) {
      out.push_back(std::move(s));
    }
  }
  const long long limit = a.num("--limit", 0);
  if (limit > 0 && static_cast<long long>(out.size()) > limit) out.resize(static_cast<std::size_t>(limit));
  return out;
}

EvalData load_eval(const Args& a) {
  auto scenarios = filtered(load_descriptors(a.need("--scenarios")), a);
  // --samples / --refused / --contexts may repeat: the files are layered in
  // order, a later file replacing whole scenarios of the earlier ones (e.g.
  // the round-1 study + the 30-observation re-sweep of the real kernels)
  a.need("--samples");
  a.need("--contexts");
  SampleTable table;
  for (const auto& f : a.all("--samples")) {
    SampleTable layer = load_samples(f);
    for (const auto& id : layer.scenario_ids()) {
      table.erase_scenario(id);
      for (const auto& [w, runs] : layer.scenario_rows(id)) table.add_row(id, w, runs);
    }
  }
  // the i-th --refused file belongs to the i-th --contexts file
  const auto ctx_files = a.all("--contexts"), ref_files = a.all("--refused");
  if (!ref_files.empty() && ref_files.size() != ctx_files.size()) {
    throw UsageError("give one --refused per --contexts (or none)");
  }
  ContextRecord contexts;
  for (std::size_t i = 0; i < ctx_files.size(); ++i) {
    const RefusedRecord refused = ref_files.empty() ? RefusedRecord{} : load_refused(ref_files[i]);
    for (auto& [id, ctx] : load_contexts(ctx_files[i], refused)) {
      contexts.erase(id);
      contexts.emplace(id, std::move(ctx));
    }
  }
  std::vector<Scenario> with_data;
  for (auto& s : scenarios) {
    if (table.has_scenario(s.id) && contexts.contains(s.id)) with_data.push_back(std::move(s));
  }
  if (with_data.empty()) throw InvalidArgument("no scenario has both samples and a recorded context");
  return assemble_eval_data(with_data, std::move(table), contexts);
}

int cmd_generate(const Args& a) {
  DescriptorSet set;
  const std::string dev = a.get("--device", "cuda");
  if (dev == "cuda") set.devices = {device_from_cuda(0)};
  else if (dev == "fixture") set.devices = reference_devices();
  else throw UsageError("--device must be cuda or fixture");
  const int n = static_cast<int>(a.num("--kernels", 40));
  if (n > 0) set.kernels = generate_kernels(n, static_cast<std::uint64_t>(a.num("--seed", 17)));
  if (a.has("--reference")) {
    auto real = reference_kernels(static_cast<int>(a.num("--gaussian-border", 5)));
    set.kernels.insert(set.kernels.end(), real.begin(), real.end());
  }
  set.datasets = generate_datasets();
  save_descriptors(set, a.need("--out"));
  std::cout << "wrote " << set.devices.size() << " devices, " << set.kernels.size() << " kernels, "
            << set.datasets.size() << " datasets under " << a.get("--out") << "\n";
  return 0;
}

int cmd_collect(const Args& a) {
  auto scenarios = filtered(load_descriptors(a.need("--scenarios")), a);
  if (scenarios.empty()) throw InvalidArgument("no scenarios match the filters");
  SweepConfig cfg;
  cfg.samples = static_cast<int>(a.num("--samples", 30));
  cfg.warmup = static_cast<int>(a.num("--warmup", 3));
  cfg.flush_l2 = !a.has("--no-flush");
  cfg.validate = !a.has("--no-validate");
  cfg.max_wgsize_cap = static_cast<int>(a.num("--cap", 0));
  cfg.cells_per_thread = static_cast<int>(a.num("--k", 0));
  cfg.border_mode = a.get("--border", "nearest") == "pad" ? SK_BORDER_PAD : SK_BORDER_NEAREST;
  const fs::path out = a.need("--out");
  const fs::path refused_path = a.get("--refused", out.string() + ".refused.csv");
  const fs::path ctx_path = a.get("--contexts", out.string() + ".contexts.csv");

  // Resume: scenarios already complete in the output files are skipped and
  // their rows kept (append-style harness).
  SampleTable table;
  RefusedRecord refused;
  ContextRecord contexts;
  if (a.has("--resume") && fs::exists(out) && fs::exists(ctx_path)) {
    table = load_samples(out);
    if (fs::exists(refused_path)) refused = load_refused(refused_path);
    contexts = load_contexts(ctx_path, refused);
  }
  std::size_t mismatches = 0;
  for (const Scenario& s : scenarios) {
    if (contexts.contains(s.id)) continue;
    const auto t0 = std::chrono::steady_clock::now();
    CollectResult r = collect({s}, cfg, [&](const Scenario& sc, std::size_t done, std::size_t total) {
      if (done == total) {
        const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        std::cerr << "  " << sc.id << ": " << total << " sizes in " << secs << " s\n";
      }
    });
    // --store mean: one observation per test case, the sample mean (the
    // evaluation only ever uses means; keeps full sweeps small on disk)
    const bool mean_only = a.get("--store", "all") == "mean";
    for (const auto& [w, runs] : r.table.scenario_rows(s.id)) {
      if (mean_only) table.add_row(s.id, w, {r.table.mean_runtime(s.id, w)});
      else table.add_row(s.id, w, runs);
    }
    refused[s.id] = r.refused[s.id];
    contexts.emplace(s.id, r.contexts.at(s.id));
    mismatches += r.gold_mismatches[s.id];
    save_samples(table, out);  // checkpoint after every scenario
    save_refused(refused, refused_path);
    save_contexts(contexts, ctx_path);
  }
  std::size_t nref = 0;
  for (const auto& [_, sz] : refused) nref += sz.size();
  std::cout << "collected " << table.row_count() << " test cases over " << contexts.size() << " scenarios ("
            << nref << " refused sizes, " << mismatches << " gold-standard mismatches)\n";
  return mismatches == 0 ? 0 : 1;
}

std::vector<Partition> partitions(const Args& a, const EvalData& d) {
  std::vector<Scenario> scen;
  std::vector<std::string> ids;
  for (const auto& [id, s] : d.scenarios) {
    scen.push_back(s);
    ids.push_back(id);
  }
  const std::string p = a.get("--partition", "kfold");
  if (p == "kfold") return partition_kfold(ids, static_cast<int>(a.num("--folds", 10)), a.num("--seed", 0));
  if (p == "synthreal") return {partition_synthetic_real(scen)};
  if (p == "loo-device") return partition_leave_one_out(scen, LeaveOneOutDimension::Device);
  if (p == "loo-kernel") return partition_leave_one_out(scen, LeaveOneOutDimension::Kernel);
  if (p == "loo-dataset") return partition_leave_one_out(scen, LeaveOneOutDimension::Dataset);
  throw UsageError("unknown partition '" + p + "'");
}

int cmd_evaluate(const Args& a) {
  const EvalData d = load_eval(a);
  const auto parts = partitions(a, d);
  std::vector<std::string> techniques = {a.need("--technique")};
  if (techniques[0] == "all") techniques = technique_ids();
  EvalOptions opt;
  if (a.has("--pin-baseline")) opt.pinned_baseline = WorkgroupSize::parse(a.get("--pin-baseline"));
  std::vector<EvalRecord> records;
  for (const auto& t : techniques) {
    for (const auto& [train, test] : parts) {
      auto tech = make_technique(t);
      auto recs = evaluate(*tech, train, test, d, static_cast<std::uint64_t>(a.num("--seed", 0)), opt);
      records.insert(records.end(), recs.begin(), recs.end());
    }
  }
  const auto rows = rows_of(records);
  std::cout << format_report(summarize(rows));
  if (a.has("--expert")) {
    std::cout << "\nvs human expert w(32x4):\n" << format_report(human_expert_summary(records, d));
  }
  if (a.has("--metrics")) write_metrics_csv(rows, a.get("--metrics"));
  return 0;
}

int cmd_train(const Args& a) {
  const EvalData d = load_eval(a);
  std::vector<std::string> ids;
  for (const auto& [id, _] : d.scenarios) ids.push_back(id);
  const std::string t = a.need("--technique");
  const std::uint64_t seed = static_cast<std::uint64_t>(a.num("--seed", 0));
  nlohmann::json bundle;
  bundle["technique"] = t;
  bundle["schema"] = kFeatureSchemaVersion;
  std::set<WorkgroupSize> refused_union;
  for (const auto& [id, c] : d.contexts) refused_union.insert(c.refused().begin(), c.refused().end());
  nlohmann::json prior = nlohmann::json::array();
  for (auto w : refused_union) prior.push_back({w.cols(), w.rows()});
  bundle["prior_refused"] = prior;
  if (t == "runtime-reg" || t == "speedup-reg") {
    const RegressionMode mode = t == "runtime-reg" ? RegressionMode::Runtime : RegressionMode::Speedup;
    std::vector<ConstraintContext> cs;
    int widest = 0;
    for (const auto& [id, c] : d.contexts) {
      cs.push_back(c);
      widest = std::max(widest, c.effective_max());
    }
    WorkgroupSize base = baseline_param(ids, d.table, safe_set(cs, enumerate_space(widest)));
    RegressionDataset ds;
    ds.mode = mode;
    for (const auto& id : ids) {
      const FeatureVector f = extract(d.scenarios.at(id));
      for (const auto& [w, _] : d.table.scenario_rows(id)) {
        ds.rows.push_back({f, w, mode == RegressionMode::Runtime ? d.table.mean_runtime(id, w)
                                                                 : speedup(id, w, base, d.table)});
      }
    }
    bundle["regressor"] = train_regressor(ds, seed)->to_json();
    bundle["baseline"] = {base.cols(), base.rows()};
  } else {
    const auto dash = t.find('-');
    if (dash == std::string::npos) throw UsageError("unknown technique '" + t + "'");
    static const std::map<std::string, ClassifierAlgo> algos = {
        {"zeror", ClassifierAlgo::ZeroR}, {"nb", ClassifierAlgo::NaiveBayes},
        {"tree", ClassifierAlgo::DecisionTree}, {"forest", ClassifierAlgo::RandomForest}};
    auto it = algos.find(t.substr(0, dash));
    if (it == algos.end()) throw UsageError("unknown technique '" + t + "'");
    LabelledDataset ds;
    for (const auto& id : ids) {
      ds.features.push_back(extract(d.scenarios.at(id)));
      ds.labels.push_back(oracle(id, d.table));
    }
    bundle["classifier"] = train_classifier(it->second, ds, seed)->to_json();
    bundle["fallback"] = t.substr(dash + 1);
  }
  write_text(a.need("--out"), bundle.dump() + "\n");
  std::cout << "trained " << t << " on " << ids.size() << " scenarios -> " << a.get("--out") << "\n";
  return 0;
}

int cmd_predict(const Args& a) {
  const nlohmann::json bundle = nlohmann::json::parse(read_text(a.need("--model")));
  DeviceDescriptor dev = a.get("--device", "cuda") == "cuda" ? device_from_cuda(0) : DeviceDescriptor{};
  if (a.get("--device", "cuda").starts_with("json:")) {
    dev = device_from_json(nlohmann::json::parse(read_text(a.get("--device").substr(5))));
  }
  if (a.get("--device", "cuda").starts_with("fixture:")) {
    const std::string id = a.get("--device").substr(8);
    for (const auto& d : reference_devices()) {
      if (d.id == id) dev = d;
    }
  }
  const KernelDescriptor k = kernel_from_json(nlohmann::json::parse(read_text(a.need("--kernel-json"))));
  DatasetDescriptor ds;
  {
    const std::string spec = a.need("--dataset");  // WxH-IN-OUT
    const auto x = spec.find('x'), d1 = spec.find('-'), d2 = spec.rfind('-');
    if (x == std::string::npos || d1 == std::string::npos || d1 == d2) throw UsageError("--dataset WxH-IN-OUT");
    ds.width = std::stoi(spec.substr(0, x));
    ds.height = std::stoi(spec.substr(x + 1, d1 - x - 1));
    ds.in_type = element_type_from_string(spec.substr(d1 + 1, d2 - d1 - 1));
    ds.out_type = element_type_from_string(spec.substr(d2 + 1));
  }
  const Scenario s = make_scenario(dev, k, ds);
  const FeatureVector f = extract(s);
  std::set<WorkgroupSize> prior;
  for (const auto& w : bundle.value("prior_refused", nlohmann::json::array())) prior.insert({w[0].get<int>(), w[1].get<int>()});
  const bool on_device = a.get("--device", "cuda") == "cuda";
  const int kmax = on_device ? kernel_max_wgsize(s.device, s.kernel, s.dataset.out_type) : s.device.device_max_wgsize;
  std::set<WorkgroupSize> known;
  for (auto w : prior) {
    if (w.area() <= std::min(kmax, s.device.device_max_wgsize)) known.insert(w);
  }
  const ConstraintContext ctx(s.device.device_max_wgsize, kmax, known);
  const ProbeFn probe = on_device ? live_probe(s) : ProbeFn([&](WorkgroupSize w) {
    return w.area() <= ctx.effective_max() ? ProbeResult::Legal : ProbeResult::Oversized;
  });
  // --shortlist N: the model's N best-ranked accepted sizes, one per line
  // (the first is the plain prediction)
  const int n = static_cast<int>(a.num("--shortlist", 0));
  if (a.has("--shortlist") && n < 1) throw UsageError("--shortlist needs N >= 1");
  std::vector<WorkgroupSize> ws;
  if (bundle.contains("regressor")) {
    auto model = regressor_from_json(bundle["regressor"]);
    const FitnessMode fm = model->mode() == RegressionMode::Runtime ? FitnessMode::RuntimeReciprocal : FitnessMode::Speedup;
    ws = n > 0 ? shortlist_regress(*model, f, ctx, fm, probe, n)
               : std::vector<WorkgroupSize>{tune_regress(*model, f, ctx, fm, probe).w};
  } else {
    auto model = classifier_from_json(bundle["classifier"]);
    const std::string fb = bundle.value("fallback", "nn");
    FallbackStrategy st = fb == "random" ? FallbackStrategy::random(fnv1a64(s.id, 0)) : FallbackStrategy::nearest_neighbour();
    ws = n > 0 ? shortlist_classify(*model, f, ctx, st, probe, n)
               : std::vector<WorkgroupSize>{tune_classify(*model, f, ctx, st, probe).w};
  }
  for (const auto& w : ws) std::cout << w.cols() << " " << w.rows() << "\n";
  return 0;
}

int cmd_features(const Args& a) {
  std::cout << device_to_json(device_from_cuda(static_cast<int>(a.num("--device", 0)))).dump(2) << "\n";
  return 0;
}

// Executable synthetic kernel for a descriptor (§8f rank 3): writes
// <out>/<name>.cu (the CUDA functor + sk_gen_table) and <out>/<name>_ref.c.
int cmd_gen_kernel(const Args& a) {
  const KernelDescriptor k = kernel_from_json(nlohmann::json::parse(read_text(a.need("--kernel-json"))));
  const GeneratedKernel g = generate_kernel(k);
  const fs::path out = a.need("--out");
  fs::create_directories(out);
  write_text(out / (k.name + ".cu"), g.cuda);
  write_text(out / (k.name + "_ref.c"), g.c_ref);
  std::cout << "generated " << g.functor << " -> " << (out / (k.name + ".cu")).string() << "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: wgtb generate|collect|evaluate|train|predict|features|gen-kernel [options]\n";
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    const std::set<std::string> boolean = {"--reference", "--no-flush", "--no-validate", "--resume", "--expert"};
    Args a(argc, argv, 2, boolean);
    if (cmd == "generate") return cmd_generate(a);
    if (cmd == "collect") return cmd_collect(a);
    if (cmd == "evaluate") return cmd_evaluate(a);
    if (cmd == "train") return cmd_train(a);
    if (cmd == "predict") return cmd_predict(a);
    if (cmd == "features") return cmd_features(a);
    if (cmd == "gen-kernel") return cmd_gen_kernel(a);
    throw UsageError("unknown subcommand '" + cmd + "'");
  } catch (const UsageError& e) {
    std::cerr << "wgtb: " << e.what() << "\n";
    return 2;
  } catch (const ParseError& e) {
    std::cerr << "wgtb: " << e.what() << "\n";
    return 2;
  } catch (const InvalidArgument& e) {
    std::cerr << "wgtb: " << e.what() << "\n";
    return 2;
  } catch (const InvalidPartition& e) {
    std::cerr << "wgtb: " << e.what() << "\n";
    return 2;
  } catch (const IoError& e) {
    std::cerr << "wgtb: " << e.what() << "\n";
    return 2;
  } catch (const std::exception& e) {
    std::cerr << "wgtb: internal error: " << e.what() << "\n";
    return 1;
  }
}
