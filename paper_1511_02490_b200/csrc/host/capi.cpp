// extern "C" entry points of libwgtb (include/wgtb_c.h).
#include <cuda_runtime.h>

#include <chrono>
#include <map>
#include <memory>
#include <mutex>

#include "wgtb/autotune.hpp"
#include "wgtb/io.hpp"
#include "wgtb/learn.hpp"
#include "wgtb/scenario.hpp"
#include "wgtb_c.h"

namespace {

thread_local std::string g_error;

struct Bundle {
  std::unique_ptr<wgtb::Classifier> classifier;
  std::unique_ptr<wgtb::Regressor> regressor;
  std::string fallback = "nn";
  std::set<wgtb::WorkgroupSize> prior_refused;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Bundle>> g_bundles;  // parsed once per path

std::shared_ptr<Bundle> load_bundle(const std::string& path) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_bundles.find(path);
  if (it != g_bundles.end()) return it->second;
  const auto j = nlohmann::json::parse(wgtb::read_text(path));
  auto b = std::make_shared<Bundle>();
  if (j.contains("regressor")) b->regressor = wgtb::regressor_from_json(j.at("regressor"));
  else b->classifier = wgtb::classifier_from_json(j.at("classifier"));
  b->fallback = j.value("fallback", std::string("nn"));
  for (const auto& w : j.value("prior_refused", nlohmann::json::array())) {
    b->prior_refused.insert({w.at(0).get<int>(), w.at(1).get<int>()});
  }
  g_bundles[path] = b;
  return b;
}

wgtb::ElementType element_of(int dtype) {
  return dtype == SK_INT32 ? wgtb::ElementType::INT32
                           : dtype == SK_FLOAT64 ? wgtb::ElementType::FLOAT64 : wgtb::ElementType::FLOAT32;
}

}  // namespace

extern "C" {

const char* wgtb_last_error(void) { return g_error.c_str(); }

int wgtb_predict(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                 int64_t width, int64_t height, int32_t* wc, int32_t* wr, int32_t* probes,
                 double* elapsed_ms) {
  g_error.clear();
  try {
    if (!model_json || !kernel_json || !desc || !wc || !wr) throw wgtb::InvalidArgument("null argument");
    auto bundle = load_bundle(model_json);
    const wgtb::KernelDescriptor k = wgtb::kernel_from_json(nlohmann::json::parse(wgtb::read_text(kernel_json)));
    wgtb::DatasetDescriptor ds{static_cast<int>(width), static_cast<int>(height), element_of(desc->dtype),
                               element_of(desc->dtype)};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) throw wgtb::DeviceError("cudaGetDevice failed");
    const wgtb::Scenario s = wgtb::make_scenario(wgtb::device_from_cuda(dev), k, ds);
    const wgtb::FeatureVector f = wgtb::extract(s);
    int32_t kmax = 0;
    if (sk_kernel_max_wgsize(desc, &kmax) != SK_OK) throw wgtb::DeviceError(sk_last_error());
    std::set<wgtb::WorkgroupSize> known;
    const int eff = std::min<int>(kmax, s.device.device_max_wgsize);
    for (auto w : bundle->prior_refused) {
      if (w.area() <= eff) known.insert(w);
    }
    const wgtb::ConstraintContext ctx(s.device.device_max_wgsize, kmax, known);
    int n_probes = 0;
    const wgtb::ProbeFn probe = [&](wgtb::WorkgroupSize w) {
      ++n_probes;
      const int rc = sk_stencil_probe(desc, width, height, w.cols(), w.rows(), nullptr, nullptr, nullptr);
      if (rc == SK_OK) return wgtb::ProbeResult::Legal;
      if (rc == SK_OVERSIZED) return wgtb::ProbeResult::Oversized;
      if (rc == SK_REFUSED) return wgtb::ProbeResult::Refused;
      throw wgtb::DeviceError(sk_last_error());
    };
    const auto t0 = std::chrono::steady_clock::now();
    wgtb::WorkgroupSize w;
    if (bundle->regressor) {
      const auto fm = bundle->regressor->mode() == wgtb::RegressionMode::Runtime ? wgtb::FitnessMode::RuntimeReciprocal
                                                                                 : wgtb::FitnessMode::Speedup;
      w = wgtb::tune_regress(*bundle->regressor, f, ctx, fm, probe).w;
    } else {
      const auto strategy = bundle->fallback == "random" ? wgtb::FallbackStrategy::random(wgtb::fnv1a64(s.id, 0))
                                                         : wgtb::FallbackStrategy::nearest_neighbour();
      w = wgtb::tune_classify(*bundle->classifier, f, ctx, strategy, probe).w;
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    *wc = w.cols();
    *wr = w.rows();
    if (probes) *probes = n_probes;
    if (elapsed_ms) *elapsed_ms = ms;
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

}  // extern "C"
