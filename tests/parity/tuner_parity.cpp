// Tuner-side parity harness: the B200 framework's host C++ autotuner (wgtb)
// against the compiled reference library (wgtune, oracle/_ref) on identical
// inputs.  TEST INFRASTRUCTURE: built by oracle/build_ref.sh, run by
// tests/test_tuner_parity.py.  Prints one "PASS <check>" / "FAIL <check>:
// <detail>" line per check and exits non-zero on any failure.
//
// Inputs come from the reference's own fixture and simulator (the standard
// 50-scenario set, seed 17, simoracle::collect with sigma 0.05) so both
// sides see exactly the tables the reference's tests and CLI produce.
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <string>
#include <vector>

// reference (namespace wgtune)
#include "wgtune/bench.hpp"
#include "wgtune/datastore.hpp"
#include "wgtune/errors.hpp"
#include "wgtune/features.hpp"
#include "wgtune/learn.hpp"
#include "wgtune/rng.hpp"
#include "wgtune/simoracle.hpp"
#include "wgtune/space.hpp"
#include "wgtune/synthgen.hpp"
#include "wgtune/tuner.hpp"
// framework (namespace wgtb)
#include "wgtb/autotune.hpp"
#include "wgtb/evaluation.hpp"
#include "wgtb/io.hpp"
#include "wgtb/learn.hpp"
#include "wgtb/scenario.hpp"
#include "wgtb/space.hpp"

namespace R = wgtune;
namespace B = wgtb;

static int g_fail = 0;
static int g_pass = 0;

static void check(const std::string& name, bool ok, const std::string& detail = "") {
  if (ok) {
    ++g_pass;
    std::printf("PASS %s\n", name.c_str());
  } else {
    ++g_fail;
    std::printf("FAIL %s: %s\n", name.c_str(), detail.c_str());
  }
}

static bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

// ------------------------------------------------------------ converters
static B::WorkgroupSize cv(R::WorkgroupSize w) { return {w.cols(), w.rows()}; }
static R::WorkgroupSize cv(B::WorkgroupSize w) { return {w.cols(), w.rows()}; }

static B::DeviceDescriptor cv(const R::DeviceDescriptor& d) {
  return B::DeviceDescriptor{d.id, static_cast<B::DeviceType>(d.device_type),
                             static_cast<B::VendorClass>(d.vendor_class), d.compute_units,
                             d.frequency_mhz, d.local_mem_kb, d.global_cache_kb, d.global_mem_mb,
                             d.device_max_wgsize, d.simd_width};
}
static B::KernelDescriptor cv(const R::KernelDescriptor& k) {
  B::KernelDescriptor o;
  o.name = k.name;
  o.north = k.north;
  o.south = k.south;
  o.east = k.east;
  o.west = k.west;
  for (int i = 0; i < 8; ++i) o.instr_counts[i] = k.instr_counts[i];
  o.total_instructions = k.total_instructions;
  o.complexity = k.complexity;
  return o;
}
static B::DatasetDescriptor cv(const R::DatasetDescriptor& d) {
  return B::DatasetDescriptor{d.width, d.height, static_cast<B::ElementType>(d.in_type),
                              static_cast<B::ElementType>(d.out_type)};
}
static B::Scenario cv(const R::Scenario& s) {
  return B::make_scenario(cv(s.device), cv(s.kernel), cv(s.dataset));
}
static std::set<B::WorkgroupSize> cv(const std::set<R::WorkgroupSize>& s) {
  std::set<B::WorkgroupSize> o;
  for (auto w : s) o.insert(cv(w));
  return o;
}
static B::ConstraintContext cv(const R::ConstraintContext& c) {
  return B::ConstraintContext(c.device_max(), c.kernel_max(), cv(c.refused()));
}
static B::FeatureVector cv(const R::FeatureVector& f) {
  std::array<double, B::kFeatureCount> v{};
  for (int i = 0; i < B::kFeatureCount; ++i) v[i] = f[i];
  return B::FeatureVector(v);
}

static bool same_kernel(const R::KernelDescriptor& a, const B::KernelDescriptor& b) {
  if (a.name != b.name || a.north != b.north || a.south != b.south || a.east != b.east ||
      a.west != b.west || a.total_instructions != b.total_instructions || a.complexity != b.complexity)
    return false;
  for (int i = 0; i < 8; ++i) {
    if (a.instr_counts[i] != b.instr_counts[i]) return false;
  }
  return true;
}

int main() {
  // -------------------------------------------------------------- rng
  {
    bool ok = true;
    for (std::uint64_t seed : {0ull, 1ull, 17ull, 0xdeadbeefull}) {
      R::Rng r(seed);
      B::Rng b(seed);
      for (int i = 0; i < 2000 && ok; ++i) {
        switch (i % 6) {
          case 0: ok = r.next() == b.next(); break;
          case 1: ok = r.bounded(1 + i) == b.bounded(1 + i); break;
          case 2: ok = r.range(-5, 1000) == b.range(-5, 1000); break;
          case 3: ok = same_bits(r.uniform01(), b.uniform01()); break;
          case 4: ok = same_bits(r.normal(), b.normal()); break;
          default: ok = r.coin() == b.coin(); break;
        }
      }
      std::vector<int> v1(97), v2(97);
      for (int i = 0; i < 97; ++i) v1[i] = v2[i] = i;
      r.shuffle(v1);
      b.shuffle(v2);
      ok = ok && v1 == v2;
      ok = ok && R::fnv1a64("kfold") == B::fnv1a64("kfold") &&
           R::fnv1a64_mix(R::fnv1a64("x"), seed) == B::fnv1a64_mix(B::fnv1a64("x"), seed);
    }
    check("rng.streams_fnv_shuffle", ok);
  }
  // ---------------------------------------------------- enumerate_space
  {
    bool ok = true;
    for (int m : {4, 5, 8, 16, 64, 100, 256, 512, 1000, 1024, 4096}) {
      auto a = R::enumerate_space(m);
      auto b = B::enumerate_space(m);
      ok = ok && a.size() == b.size();
      for (std::size_t i = 0; ok && i < a.size(); ++i) ok = cv(a[i]) == b[i];
    }
    bool both_throw = false;
    try { B::enumerate_space(3); } catch (const B::EmptySpace&) { both_throw = true; }
    check("space.enumerate_space", ok && both_throw && B::enumerate_space(1024).size() == 1466);
  }
  // ---------------------------------------------------------- synthgen
  {
    bool ok = true;
    for (std::uint64_t seed : {0ull, 1ull, 17ull, 42ull, 12345ull}) {
      auto a = R::generate_kernels(60, seed);
      auto b = B::generate_kernels(60, seed);
      for (std::size_t i = 0; i < a.size(); ++i) ok = ok && same_kernel(a[i], b[i]);
    }
    for (int g = 1; g <= 10; ++g) {
      auto a = R::reference_kernels(g);
      auto b = B::reference_kernels(g);
      for (std::size_t i = 0; i < a.size(); ++i) ok = ok && same_kernel(a[i], b[i]);
    }
    auto da = R::generate_datasets();
    auto db = B::generate_datasets();
    ok = ok && da.size() == db.size();
    for (std::size_t i = 0; i < da.size(); ++i) {
      ok = ok && da[i].width == db[i].width && static_cast<int>(da[i].in_type) == static_cast<int>(db[i].in_type);
    }
    auto va = R::reference_devices();
    auto vb = B::reference_devices();
    for (std::size_t i = 0; i < va.size(); ++i) {
      ok = ok && va[i].id == vb[i].id && va[i].compute_units == vb[i].compute_units &&
           va[i].device_max_wgsize == vb[i].device_max_wgsize && va[i].simd_width == vb[i].simd_width;
    }
    check("synthgen.kernels_datasets_devices", ok);
  }
  // ---------------------------------------------- scenarios + features
  auto rs = R::standard_scenarios(17);
  std::vector<B::Scenario> bs;
  for (const auto& s : rs) bs.push_back(cv(s));
  {
    auto bstd = B::standard_scenarios(17);
    bool ok = rs.size() == bstd.size();
    for (std::size_t i = 0; ok && i < rs.size(); ++i) ok = rs[i].id == bstd[i].id && rs[i].id == bs[i].id;
    check("scenario.standard_ids", ok);
    bool fok = true;
    for (std::size_t i = 0; i < rs.size(); ++i) {
      auto fa = R::extract(rs[i]);
      auto fb = B::extract(bs[i]);
      for (int j = 0; j < B::kFeatureCount; ++j) fok = fok && same_bits(fa[j], fb[j]);
    }
    for (int j = 0; j < B::kFeatureCount; ++j) fok = fok && R::feature_names()[j] == B::feature_names()[j];
    check("features.extract_fv1", fok);
  }
  // ------------------------------------------- simulated corpus -> CSV
  R::OracleConfig ocfg;
  ocfg.seed = 17;
  ocfg.noise_sigma = 0.05;
  ocfg.min_samples = 30;
  const R::CollectResult col = R::collect(rs, ocfg);
  const std::string csv = R::samples_to_csv(col.table);
  const B::SampleTable btab = B::samples_from_csv(csv);
  check("datastore.samples_csv_roundtrip", B::samples_to_csv(btab) == csv && btab.row_count() == col.table.row_count());
  {
    std::ostringstream ref_refused;
    B::RefusedRecord brr;
    for (const auto& [id, sz] : col.refused) brr[id] = cv(sz);
    const std::string mine = B::refused_to_csv(brr);
    const B::RefusedRecord back = B::refused_from_csv(mine);
    const std::filesystem::path tmp = std::filesystem::temp_directory_path() / "wgtb_parity_refused.csv";
    R::save_refused(col.refused, tmp);
    const std::string theirs = B::read_text(tmp);
    std::filesystem::remove(tmp);
    std::size_t nonempty = 0;
    for (const auto& [id, sz] : brr) nonempty += !sz.empty();
    check("datastore.refused_csv_roundtrip",
          mine == theirs && back.size() == nonempty && B::refused_to_csv(back) == mine,
          "csv bytes differ from the reference's save_refused");
    // descriptor JSON: identical dumps
    bool jok = true;
    for (const auto& s : rs) {
      jok = jok && R::device_to_json(s.device).dump(2) == B::device_to_json(cv(s.device)).dump(2) &&
            R::kernel_to_json(s.kernel).dump(2) == B::kernel_to_json(cv(s.kernel)).dump(2) &&
            R::dataset_to_json(s.dataset).dump(2) == B::dataset_to_json(cv(s.dataset)).dump(2);
    }
    check("datastore.descriptor_json", jok);
    // parse-error behaviour on malformed CSV
    int both = 0;
    for (const char* bad : {"scenario_id,w_c,w_r,runtime_ms\na,1,1,-1\n", "nope\n",
                            "scenario_id,w_c,w_r,runtime_ms\na,1,x,1\n",
                            "scenario_id,w_c,w_r,runtime_ms\na,2,2,1\nb,2,2,1\na,2,2,3\n"}) {
      bool r_threw = false, b_threw = false;
      try { R::samples_from_csv(bad); } catch (const R::Error&) { r_threw = true; }
      try { B::samples_from_csv(bad); } catch (const B::Error&) { b_threw = true; }
      both += r_threw && b_threw;
    }
    check("datastore.csv_error_behaviour", both == 4);
  }
  // --------------------------------------------------- space arithmetic
  std::vector<std::string> ids;
  for (const auto& s : rs) ids.push_back(s.id);
  {
    bool ok = true;
    for (const auto& id : ids) {
      auto oa = R::oracle(id, col.table);
      auto ob = B::oracle(id, btab);
      ok = ok && cv(oa) == ob;
      for (const auto& [w, _] : col.table.scenario_rows(id)) {
        ok = ok && same_bits(R::performance(id, w, col.table), B::performance(id, cv(w), btab));
        ok = ok && same_bits(R::speedup(id, w, oa, col.table), B::speedup(id, cv(w), ob, btab));
      }
    }
    check("space.oracle_performance_speedup", ok);
    std::vector<R::ConstraintContext> rc;
    std::vector<B::ConstraintContext> bc;
    for (const auto& id : ids) {
      rc.push_back(col.contexts.at(id));
      bc.push_back(cv(col.contexts.at(id)));
    }
    auto sa = R::safe_set(rc, R::enumerate_space(1024));
    auto sb = B::safe_set(bc, B::enumerate_space(1024));
    std::vector<std::string> train(ids.begin(), ids.begin() + 40);
    auto ra = R::baseline_ranking(train, col.table, sa);
    auto rb = B::baseline_ranking(train, btab, sb);
    bool rok = ra.size() == rb.size() && cv(sa) == sb;
    for (std::size_t i = 0; rok && i < ra.size(); ++i) rok = cv(ra[i]) == rb[i];
    check("space.safe_set_baseline_ranking", rok, "safe " + std::to_string(sa.size()) + "/" + std::to_string(sb.size()));
  }
  // ---------------------------------------------------------- learning
  std::vector<std::string> train(ids.begin(), ids.begin() + 40);
  {
    R::LabelledDataset la;
    B::LabelledDataset lb;
    for (std::size_t i = 0; i < 40; ++i) {
      la.features.push_back(R::extract(rs[i]));
      la.labels.push_back(R::oracle(rs[i].id, col.table));
      lb.features.push_back(B::extract(bs[i]));
      lb.labels.push_back(B::oracle(bs[i].id, btab));
    }
    for (auto algo : {0, 1, 2, 3}) {
      for (std::uint64_t seed : {0ull, 7ull}) {
        auto ma = R::train_classifier(static_cast<R::ClassifierAlgo>(algo), la, seed);
        auto mb = B::train_classifier(static_cast<B::ClassifierAlgo>(algo), lb, seed);
        bool ok = ma->to_json().dump() == mb->to_json().dump();
        for (std::size_t i = 0; ok && i < rs.size(); ++i) {
          ok = cv(ma->predict(R::extract(rs[i]))) == mb->predict(B::extract(bs[i]));
        }
        // JSON round trip of our model preserves predictions
        auto mc = B::classifier_from_json(mb->to_json());
        for (std::size_t i = 0; ok && i < bs.size(); ++i) ok = mc->predict(B::extract(bs[i])) == mb->predict(B::extract(bs[i]));
        check("learn.classifier_" + std::string(B::to_string(static_cast<B::ClassifierAlgo>(algo))) + "_seed" +
                  std::to_string(seed),
              ok);
      }
    }
    // regressors (runtime and speedup targets), 40 training scenarios
    std::vector<R::ConstraintContext> train_ctx;
    for (const auto& id : train) train_ctx.push_back(col.contexts.at(id));
    auto base = R::baseline_param(train, col.table, R::safe_set(train_ctx, R::enumerate_space(1024)));
    for (int mode : {0, 1}) {
      R::RegressionDataset ra;
      B::RegressionDataset rb;
      ra.mode = static_cast<R::RegressionMode>(mode);
      rb.mode = static_cast<B::RegressionMode>(mode);
      for (std::size_t i = 0; i < 40; ++i) {
        for (const auto& [w, _] : col.table.scenario_rows(rs[i].id)) {
          double t = mode == 0 ? col.table.mean_runtime(rs[i].id, w) : R::speedup(rs[i].id, w, base, col.table);
          ra.rows.push_back({R::extract(rs[i]), w, t});
          rb.rows.push_back({B::extract(bs[i]), cv(w), t});
        }
      }
      auto ma = R::train_regressor(ra, 3);
      auto mb = B::train_regressor(rb, 3);
      bool ok = ma->to_json().dump() == mb->to_json().dump();
      for (std::size_t i = 40; ok && i < rs.size(); ++i) {
        for (const auto& w : R::enumerate_space(256)) {
          ok = ok && same_bits(ma->predict(R::extract(rs[i]), w), mb->predict(B::extract(bs[i]), cv(w)));
        }
      }
      check(std::string("learn.forest_regressor_") + (mode == 0 ? "runtime" : "speedup"), ok,
            "rows " + std::to_string(ra.rows.size()));
    }
  }
  // ------------------------------------------------------------ tuners
  {
    // Fixed classifier predictions through the fallbacks, with probes
    // replaying the simulated corpus.
    bool ok = true;
    R::LabelledDataset la;
    B::LabelledDataset lb;
    for (std::size_t i = 0; i < 40; ++i) {
      la.features.push_back(R::extract(rs[i]));
      la.labels.push_back(R::WorkgroupSize(2 + 2 * (i % 40), 2 + 2 * (i % 9)));  // many illegal labels
      lb.features.push_back(B::extract(bs[i]));
      lb.labels.push_back(cv(la.labels.back()));
    }
    auto ma = R::train_classifier(R::ClassifierAlgo::DecisionTree, la, 1);
    auto mb = B::train_classifier(B::ClassifierAlgo::DecisionTree, lb, 1);
    std::set<R::WorkgroupSize> safe = R::safe_set({col.contexts.at(ids[0]), col.contexts.at(ids[3])}, R::enumerate_space(512));
    auto rank_a = R::baseline_ranking({ids[0], ids[3]}, col.table, safe);
    std::vector<B::WorkgroupSize> rank_b;
    for (auto w : rank_a) rank_b.push_back(cv(w));
    int fallbacks = 0;
    for (std::size_t i = 0; i < rs.size(); ++i) {
      const auto& id = rs[i].id;
      const auto& rctx = col.contexts.at(id);
      const B::ConstraintContext bctx = cv(rctx);
      R::ProbeFn rp = [&](R::WorkgroupSize w) {
        if (w.area() > rctx.effective_max()) return R::ProbeResult::Oversized;
        if (rctx.refused().count(w) || !col.table.has(id, w)) return R::ProbeResult::Refused;
        return R::ProbeResult::Legal;
      };
      B::ProbeFn bp = [&](B::WorkgroupSize w) {
        return static_cast<B::ProbeResult>(static_cast<int>(rp(cv(w))));
      };
      // empty prior-refused context so fallbacks discover refusals by probing
      R::ConstraintContext rctx0(rctx.device_max(), rctx.kernel_max());
      B::ConstraintContext bctx0(bctx.device_max(), bctx.kernel_max());
      for (int fb = 0; fb < 3; ++fb) {
        R::FallbackStrategy sa = fb == 0 ? R::FallbackStrategy::baseline(rank_a)
                                 : fb == 1 ? R::FallbackStrategy::random(R::fnv1a64(id, 5))
                                           : R::FallbackStrategy::nearest_neighbour();
        B::FallbackStrategy sb = fb == 0 ? B::FallbackStrategy::baseline(rank_b)
                                 : fb == 1 ? B::FallbackStrategy::random(B::fnv1a64(id, 5))
                                           : B::FallbackStrategy::nearest_neighbour();
        std::string ea, eb;
        R::ClassifyOutcome oa;
        B::ClassifyOutcome ob;
        try { oa = R::tune_classify(*ma, R::extract(rs[i]), rctx0, sa, rp); } catch (const R::Error&) { ea = "threw"; }
        try { ob = B::tune_classify(*mb, B::extract(bs[i]), bctx0, sb, bp); } catch (const B::Error&) { eb = "threw"; }
        ok = ok && ea == eb;
        if (ea.empty() && eb.empty()) {
          ok = ok && cv(oa.w) == ob.w && oa.fallback_iterations == ob.fallback_iterations &&
               cv(oa.initial) == ob.initial && static_cast<int>(oa.initial_probe) == static_cast<int>(ob.initial_probe);
          fallbacks += oa.fallback_iterations > 0;
        }
      }
    }
    check("tuner.tune_classify_all_fallbacks", ok && fallbacks > 10, "fallback episodes " + std::to_string(fallbacks));
  }
  // ------------------------------------------------- full evaluations
  {
    R::EvalData rd;
    rd.table = col.table;
    B::EvalData bd;
    bd.table = btab;
    for (std::size_t i = 0; i < rs.size(); ++i) {
      rd.scenarios.emplace(rs[i].id, rs[i]);
      rd.contexts.emplace(rs[i].id, col.contexts.at(rs[i].id));
      bd.scenarios.emplace(bs[i].id, bs[i]);
      bd.contexts.emplace(bs[i].id, cv(col.contexts.at(rs[i].id)));
    }
    auto pa = R::partition_synthetic_real(rs);
    auto pb = B::partition_synthetic_real(bs);
    auto ka = R::partition_kfold(ids, 10, 3);
    auto kb = B::partition_kfold(ids, 10, 3);
    bool pok = pa == pb && ka == kb;
    for (int dim = 0; dim < 3; ++dim) {
      pok = pok && R::partition_leave_one_out(rs, static_cast<R::LeaveOneOutDimension>(dim)) ==
                       B::partition_leave_one_out(bs, static_cast<B::LeaveOneOutDimension>(dim));
    }
    check("bench.partitions", pok);
    std::vector<std::pair<std::string, std::vector<std::pair<std::vector<std::string>, std::vector<std::string>>>>> plans = {
        {"synthreal", {pa}}, {"kfold", {ka.begin(), ka.begin() + 3}}};
    for (const auto& tech : R::technique_ids()) {
      for (const auto& [pname, parts] : plans) {
        bool ok = true;
        std::string detail;
        std::vector<R::EvalRecord> all_a;
        std::vector<B::EvalRecord> all_b;
        for (const auto& [tr, te] : parts) {
          auto ta = R::make_technique(tech);
          auto tb = B::make_technique(tech);
          auto ra = R::evaluate(*ta, tr, te, rd, 11);
          auto rb = B::evaluate(*tb, tr, te, bd, 11);
          ok = ok && ra.size() == rb.size();
          for (std::size_t i = 0; ok && i < ra.size(); ++i) {
            const auto& x = ra[i].row;
            const auto& y = rb[i].row;
            ok = x.technique == y.technique && x.scenario_id == y.scenario_id && x.accuracy == y.accuracy &&
                 x.validity == y.validity && x.refused == y.refused && same_bits(x.performance, y.performance) &&
                 same_bits(x.speedup, y.speedup) && x.fallback_iterations == y.fallback_iterations &&
                 cv(ra[i].chosen) == rb[i].chosen && cv(ra[i].baseline) == rb[i].baseline;
            if (!ok) detail = x.scenario_id + " chose " + ra[i].chosen.str() + " vs " + rb[i].chosen.str();
          }
          all_a.insert(all_a.end(), ra.begin(), ra.end());
          all_b.insert(all_b.end(), rb.begin(), rb.end());
        }
        if (ok) {
          auto sa = R::summarize(R::rows_of(all_a));
          auto sb = B::summarize(B::rows_of(all_b));
          ok = sa.size() == sb.size() && same_bits(sa[0].mean_performance_pct, sb[0].mean_performance_pct) &&
               same_bits(sa[0].median_speedup, sb[0].median_speedup) && same_bits(sa[0].mean_speedup, sb[0].mean_speedup);
          if (!ok) detail = "summary differs";
        }
        check("bench.evaluate_" + tech + "_" + pname, ok, detail);
      }
    }
  }
  std::printf("parity: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
