// extern "C" entry points of libwgtb (include/wgtb_c.h).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

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

namespace {

// The session's known-refused sizes under the effective maximum, plus the
// bundle's prior refusals.
wgtb::ConstraintContext session_context(const Bundle& b, int dev_max, int kmax,
                                        const std::set<wgtb::WorkgroupSize>& refused) {
  std::set<wgtb::WorkgroupSize> known;
  const int eff = std::min(kmax, dev_max);
  for (const auto& w : b.prior_refused) {
    if (w.area() <= eff) known.insert(w);
  }
  for (const auto& w : refused) {
    if (w.area() <= eff) known.insert(w);
  }
  return wgtb::ConstraintContext(dev_max, kmax, known);
}

// Algorithm 1 or 2 (whichever the bundle holds) against `probe`.
wgtb::WorkgroupSize choose(const Bundle& b, const wgtb::Scenario& s, const wgtb::FeatureVector& f,
                           const wgtb::ConstraintContext& ctx, const wgtb::ProbeFn& probe) {
  if (b.regressor) {
    const auto fm = b.regressor->mode() == wgtb::RegressionMode::Runtime ? wgtb::FitnessMode::RuntimeReciprocal
                                                                         : wgtb::FitnessMode::Speedup;
    return wgtb::tune_regress(*b.regressor, f, ctx, fm, probe).w;
  }
  const auto strategy = b.fallback == "random" ? wgtb::FallbackStrategy::random(wgtb::fnv1a64(s.id, 0))
                                               : wgtb::FallbackStrategy::nearest_neighbour();
  return wgtb::tune_classify(*b.classifier, f, ctx, strategy, probe).w;
}

// One tuning context on the current device: the inputs of the prediction
// and what this session has learnt about legality.
struct Scene {
  std::shared_ptr<Bundle> bundle;
  wgtb::Scenario scenario;
  wgtb::FeatureVector features;
  int kmax = 0;
};

Scene make_scene(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc, int64_t width,
                 int64_t height) {
  if (!model_json || !kernel_json || !desc) throw wgtb::InvalidArgument("null argument");
  Scene sc;
  sc.bundle = load_bundle(model_json);
  const wgtb::KernelDescriptor k = wgtb::kernel_from_json(nlohmann::json::parse(wgtb::read_text(kernel_json)));
  wgtb::DatasetDescriptor ds{static_cast<int>(width), static_cast<int>(height), element_of(desc->dtype),
                             element_of(desc->dtype)};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) throw wgtb::DeviceError("cudaGetDevice failed");
  sc.scenario = wgtb::make_scenario(wgtb::device_from_cuda(dev), k, ds);
  sc.features = wgtb::extract(sc.scenario);
  if (sk_kernel_max_wgsize(desc, &sc.kmax) != SK_OK) throw wgtb::DeviceError(sk_last_error());
  return sc;
}

// Online tuning sessions (the in-process form of serve.cpp's Session),
// keyed by (model, kernel, descriptor, W, H, device).
struct Session {
  Scene scene;
  std::set<wgtb::WorkgroupSize> refused;  // learnt from launches / callers
  wgtb::WorkgroupSize w;
  bool proposed = false;
  int proposals = 0;
};
std::mutex g_sess_mu;
std::map<std::string, Session> g_sessions;

std::string format_double_key(double v) {
  char buf[32];
  std::snprintf(buf, sizeof buf, "%a", v);
  return buf;
}

std::string session_key(const char* model_json, const char* kernel_json, const sk_stencil_desc* d, int64_t width,
                        int64_t height) {
  int dev = 0;
  cudaGetDevice(&dev);
  // field by field (the struct has padding bytes a caller need not zero)
  std::string key = std::string(model_json) + '\n' + kernel_json + '\n';
  for (int v : {d->op, d->dtype, d->north, d->south, d->east, d->west, d->border_mode, d->complexity,
                d->instructions, d->load_path, d->cells_per_thread, d->fused_iterations}) {
    key += std::to_string(v) + ',';
  }
  key += format_double_key(d->pad_value);
  key += '\n' + std::to_string(width) + 'x' + std::to_string(height) + '@' + std::to_string(dev);
  return key;
}

Session& session_for(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc, int64_t width,
                     int64_t height) {
  const std::string key = session_key(model_json, kernel_json, desc, width, height);
  auto it = g_sessions.find(key);
  if (it == g_sessions.end()) {
    Session s;
    s.scene = make_scene(model_json, kernel_json, desc, width, height);
    it = g_sessions.emplace(key, std::move(s)).first;
  }
  return it->second;
}

// A new proposal: the live device probe, except that sizes this session has
// seen refused stay refused (serve.cpp:59-61, 150-157).
void propose(Session& s, const sk_stencil_desc* desc, int64_t width, int64_t height) {
  const Bundle& b = *s.scene.bundle;
  const int dev_max = s.scene.scenario.device.device_max_wgsize;
  const auto ctx = session_context(b, dev_max, s.scene.kmax, s.refused);
  const wgtb::ProbeFn probe = [&](wgtb::WorkgroupSize w) {
    if (s.refused.count(w)) return wgtb::ProbeResult::Refused;
    const int rc = sk_stencil_probe(desc, width, height, w.cols(), w.rows(), nullptr, nullptr, nullptr);
    if (rc == SK_OK) return wgtb::ProbeResult::Legal;
    if (rc == SK_OVERSIZED) return wgtb::ProbeResult::Oversized;
    if (rc == SK_REFUSED) return wgtb::ProbeResult::Refused;
    throw wgtb::DeviceError(sk_last_error());
  };
  s.w = choose(b, s.scene.scenario, s.scene.features, ctx, probe);
  s.proposed = true;
  ++s.proposals;
}

// Live legality of one size for the scene's stencil.
wgtb::ProbeResult device_probe(const sk_stencil_desc* desc, int64_t width, int64_t height, wgtb::WorkgroupSize w) {
  const int rc = sk_stencil_probe(desc, width, height, w.cols(), w.rows(), nullptr, nullptr, nullptr);
  if (rc == SK_OK) return wgtb::ProbeResult::Legal;
  if (rc == SK_OVERSIZED) return wgtb::ProbeResult::Oversized;
  if (rc == SK_REFUSED) return wgtb::ProbeResult::Refused;
  throw wgtb::DeviceError(sk_last_error());
}

// The model's shortlist for a scene (autotune.hpp: shortlist_*), with live
// device probes; *probes counts them.
std::vector<wgtb::WorkgroupSize> shortlist(const Scene& sc, const sk_stencil_desc* desc, int64_t width,
                                           int64_t height, int n, int* probes) {
  const Bundle& b = *sc.bundle;
  const auto ctx = session_context(b, sc.scenario.device.device_max_wgsize, sc.kmax, {});
  const wgtb::ProbeFn probe = [&](wgtb::WorkgroupSize w) {
    ++*probes;
    return device_probe(desc, width, height, w);
  };
  if (b.regressor) {
    const auto fm = b.regressor->mode() == wgtb::RegressionMode::Runtime ? wgtb::FitnessMode::RuntimeReciprocal
                                                                         : wgtb::FitnessMode::Speedup;
    return wgtb::shortlist_regress(*b.regressor, sc.features, ctx, fm, probe, n);
  }
  const auto strategy = b.fallback == "random" ? wgtb::FallbackStrategy::random(wgtb::fnv1a64(sc.scenario.id, 0))
                                               : wgtb::FallbackStrategy::nearest_neighbour();
  return wgtb::shortlist_classify(*b.classifier, sc.features, ctx, strategy, probe, n);
}

}  // namespace

extern "C" {

const char* wgtb_last_error(void) { return g_error.c_str(); }

int wgtb_shortlist(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc, int64_t width,
                   int64_t height, int32_t max_n, int32_t* wcs, int32_t* wrs, int32_t* n_out) {
  g_error.clear();
  try {
    if (!wcs || !wrs || !n_out || max_n < 1) throw wgtb::InvalidArgument("null argument or max_n < 1");
    const Scene sc = make_scene(model_json, kernel_json, desc, width, height);
    int probes = 0;
    const auto list = shortlist(sc, desc, width, height, max_n, &probes);
    for (std::size_t i = 0; i < list.size(); ++i) {
      wcs[i] = list[i].cols();
      wrs[i] = list[i].rows();
    }
    *n_out = static_cast<int32_t>(list.size());
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

int wgtb_tune_measured(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                       const void* d_in, void* d_out, int64_t width, int64_t height, int64_t pitch,
                       int32_t max_n, int32_t samples, int32_t* wc, int32_t* wr, int32_t* timed, double* best_ms,
                       double* elapsed_ms) {
  g_error.clear();
  try {
    if (!wc || !wr || max_n < 1 || samples < 1) throw wgtb::InvalidArgument("null argument, max_n or samples < 1");
    const auto t0 = std::chrono::steady_clock::now();
    const Scene sc = make_scene(model_json, kernel_json, desc, width, height);
    int probes = 0;
    const auto list = shortlist(sc, desc, width, height, max_n, &probes);
    if (list.empty()) throw wgtb::NoLegalParameter("the shortlist holds no legal size");
    std::vector<double> ms(static_cast<std::size_t>(samples));
    double best = 0.0;
    wgtb::WorkgroupSize pick = list.front();
    for (const auto& w : list) {
      const int rc = sk_stencil_time(desc, d_in, d_out, width, height, pitch, w.cols(), w.rows(), 1, samples, 1,
                                     ms.data());
      if (rc != SK_OK) throw wgtb::DeviceError(sk_last_error());
      std::vector<double> s = ms;
      std::nth_element(s.begin(), s.begin() + s.size() / 2, s.end());
      const double med = s[s.size() / 2];
      if (&w == &list.front() || med < best) {
        best = med;
        pick = w;
      }
    }
    *wc = pick.cols();
    *wr = pick.rows();
    if (timed) *timed = static_cast<int32_t>(list.size());
    if (best_ms) *best_ms = best;
    if (elapsed_ms) {
      *elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    }
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

int wgtb_predict(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                 int64_t width, int64_t height, int32_t* wc, int32_t* wr, int32_t* probes,
                 double* elapsed_ms) {
  g_error.clear();
  try {
    if (!wc || !wr) throw wgtb::InvalidArgument("null argument");
    const Scene sc = make_scene(model_json, kernel_json, desc, width, height);
    const auto ctx = session_context(*sc.bundle, sc.scenario.device.device_max_wgsize, sc.kmax, {});
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
    const wgtb::WorkgroupSize w = choose(*sc.bundle, sc.scenario, sc.features, ctx, probe);
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

int wgtb_launch_tuned(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                      const void* d_in, void* d_out, int64_t width, int64_t height, int64_t pitch_in,
                      int64_t pitch_out, void* stream, int32_t* wc_used, int32_t* wr_used,
                      int32_t* proposals) {
  g_error.clear();
  try {
    std::lock_guard<std::mutex> lk(g_sess_mu);
    Session& s = session_for(model_json, kernel_json, desc, width, height);
    for (int attempt = 0; attempt < 64; ++attempt) {
      if (!s.proposed) propose(s, desc, width, height);
      const int rc = sk_stencil_launch(desc, d_in, d_out, width, height, pitch_in, pitch_out, 0, 0, s.w.cols(),
                                       s.w.rows(), stream);
      if (rc == SK_OK) {
        if (wc_used) *wc_used = s.w.cols();
        if (wr_used) *wr_used = s.w.rows();
        if (proposals) *proposals = s.proposals;
        return 0;
      }
      if (rc != SK_REFUSED && rc != SK_OVERSIZED) throw wgtb::DeviceError(sk_last_error());
      // refusal feedback: never propose this size again in this session
      s.refused.insert(s.w);
      s.proposed = false;
    }
    throw wgtb::NoLegalParameter("64 proposals in a row were refused at launch");
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

int wgtb_tuned_refuse(const char* model_json, const char* kernel_json, const sk_stencil_desc* desc,
                      int64_t width, int64_t height, int32_t wc, int32_t wr) {
  g_error.clear();
  try {
    std::lock_guard<std::mutex> lk(g_sess_mu);
    Session& s = session_for(model_json, kernel_json, desc, width, height);
    const wgtb::WorkgroupSize w(wc, wr);
    s.refused.insert(w);
    if (s.proposed && s.w == w) s.proposed = false;
    return 0;
  } catch (const std::exception& e) {
    g_error = e.what();
    return -1;
  }
}

void wgtb_tuned_reset(void) {
  std::lock_guard<std::mutex> lk(g_sess_mu);
  g_sessions.clear();
}

}  // extern "C"
