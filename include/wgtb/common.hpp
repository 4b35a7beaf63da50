// wgtb — host-side autotuner for the B200 stencil executor.
//
// Common vocabulary: the exception taxonomy (mirrors the reference's
// errors.hpp:9-63 so callers can catch the same conditions), the
// deterministic hashing / random streams (rng.hpp:13-72: FNV-1a-64 and
// mt19937_64 with hand-rolled transforms, needed bit-for-bit so synthetic
// kernels, bootstraps and folds equal the reference's), and the tuned
// parameter itself, the workgroup size (space.hpp:15-33).
#pragma once

#include <cmath>
#include <compare>
#include <cstdint>
#include <random>
#include <stdexcept>
#include <string>
#include <string_view>
#include <utility>
#include <vector>

namespace wgtb {

// ----------------------------------------------------------------- errors
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define WGTB_DECLARE_ERROR(Name) \
  struct Name : Error {          \
    using Error::Error;          \
  }
WGTB_DECLARE_ERROR(InvalidArgument);
WGTB_DECLARE_ERROR(EmptySpace);
WGTB_DECLARE_ERROR(UnknownScenario);
WGTB_DECLARE_ERROR(UnknownTestCase);
WGTB_DECLARE_ERROR(NoSafeParameter);
WGTB_DECLARE_ERROR(InvalidDescriptor);
WGTB_DECLARE_ERROR(InconsistentCounts);
WGTB_DECLARE_ERROR(IllegalWorkgroupSize);
WGTB_DECLARE_ERROR(DuplicateTestCase);
WGTB_DECLARE_ERROR(EmptyTrainingSet);
WGTB_DECLARE_ERROR(SchemaError);
WGTB_DECLARE_ERROR(NoLegalParameter);
WGTB_DECLARE_ERROR(InvalidPartition);
WGTB_DECLARE_ERROR(IncompleteSpace);
WGTB_DECLARE_ERROR(InvalidPrediction);
WGTB_DECLARE_ERROR(IoError);
WGTB_DECLARE_ERROR(DeviceError);  // a CUDA failure that is not a refusal
#undef WGTB_DECLARE_ERROR

// Text input that could not be parsed; line is 1-based (0 = unknown).
struct ParseError : Error {
  explicit ParseError(const std::string& msg, std::size_t line = 0)
      : Error(line == 0 ? msg : msg + " (line " + std::to_string(line) + ")"), line_(line) {}
  std::size_t line() const { return line_; }

 private:
  std::size_t line_;
};

// A legal-sized workgroup the device refused to launch.
struct RefusedParameter : Error {
  RefusedParameter(const std::string& msg, int w_c, int w_r) : Error(msg), w_c_(w_c), w_r_(w_r) {}
  int w_c() const { return w_c_; }
  int w_r() const { return w_r_; }

 private:
  int w_c_, w_r_;
};

// ------------------------------------------------------------- hashing / rng
inline constexpr std::uint64_t kFnvOffset = 0xcbf29ce484222325ULL;
inline constexpr std::uint64_t kFnvPrime = 0x100000001b3ULL;

inline std::uint64_t fnv1a64(std::string_view bytes, std::uint64_t h = kFnvOffset) {
  for (unsigned char b : bytes) h = (h ^ b) * kFnvPrime;
  return h;
}

// Folds the 8 little-endian bytes of v into h.
inline std::uint64_t fnv1a64_mix(std::uint64_t h, std::uint64_t v) {
  for (int shift = 0; shift < 64; shift += 8) h = (h ^ ((v >> shift) & 0xffu)) * kFnvPrime;
  return h;
}

// Deterministic stream over the standard-specified mt19937_64 engine.
class Rng {
 public:
  explicit Rng(std::uint64_t seed) : eng_(seed) {}
  std::uint64_t next() { return eng_(); }
  std::uint64_t bounded(std::uint64_t n) { return eng_() % n; }  // [0, n)
  std::int64_t range(std::int64_t lo, std::int64_t hi) {          // [lo, hi]
    return lo + static_cast<std::int64_t>(bounded(static_cast<std::uint64_t>(hi - lo + 1)));
  }
  double uniform01() { return static_cast<double>(eng_() >> 11) * 0x1.0p-53; }
  bool coin() { return (eng_() & 1u) == 1u; }
  double normal() {  // Box-Muller, one value per call
    double a = uniform01();
    double b = uniform01();
    if (a <= 0.0) a = 0x1.0p-53;
    return std::sqrt(-2.0 * std::log(a)) * std::cos(6.283185307179586 * b);
  }
  template <typename T>
  void shuffle(std::vector<T>& v) {  // Fisher-Yates from the back
    for (std::size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[bounded(i)]);
  }

 private:
  std::mt19937_64 eng_;
};

// ---------------------------------------------------------- workgroup size
// (w_c columns, w_r rows); ordered lexicographically by (w_c, w_r), the
// tie-break order of every argmin/argmax in the tuner.
class WorkgroupSize {
 public:
  WorkgroupSize() = default;
  WorkgroupSize(int cols, int rows);
  int cols() const { return c_; }
  int rows() const { return r_; }
  long long area() const { return static_cast<long long>(c_) * r_; }
  std::string str() const;                           // "<w_c>x<w_r>"
  static WorkgroupSize parse(std::string_view text);  // inverse of str()
  friend auto operator<=>(const WorkgroupSize&, const WorkgroupSize&) = default;

 private:
  int c_ = 1;
  int r_ = 1;
};

// Shortest round-trip decimal text of a double (std::to_chars).
std::string format_double(double v);

}  // namespace wgtb
