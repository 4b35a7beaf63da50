// Customising functions of the B200 stencil executor (device side).
//
// Each op is a functor `T operator()(const View&) const` where View::at(dr, dc)
// returns the staged tile value dr rows south (negative = north) and dc
// columns east (negative = west) of the work-item's cell.  The formulas are
// the ones fixed in DESIGN.md §3; the CPU oracle (oracle/stencil_oracle.c)
// restates them independently.  This file is compiled with -fmad=false so
// every float expression rounds exactly as written (the oracle is built with
// -ffp-contract=off), which makes fp32/fp64 outputs bit-identical to the CPU.
//
// Reference kernel set: PAPER.md Table 2 (:465-488), synthgen.cpp:82-96.
#pragma once

#include <cstdint>
#include <type_traits>

namespace sk {

// Gaussian weight type: int32 stencils use exact int64 binomial products.
template <typename T>
using WeightT = std::conditional_t<std::is_same_v<T, int32_t>, long long, T>;

// Parameters shared by all ops (runtime borders, synthetic knobs, gaussian
// weights).  Passed by value as a kernel parameter (constant bank).
template <typename T>
struct OpParams {
  int north, south, east, west;
  int complexity;
  int alu_iters;                 // synthetic: dependent ALU iterations per cell
  int gauss_radius;              // gaussian: g
  WeightT<T> gauss_w[21 * 21];   // gaussian: row-major (2g+1)^2 weights
};

// Integer accumulator for int32 stencils: wraps modulo 2^64 so overflow is
// defined and identical on CPU and GPU.
template <typename T> struct Acc { using type = T; };
template <> struct Acc<int32_t> { using type = long long; };

template <typename T>
__device__ __forceinline__ T from_acc(typename Acc<T>::type a) { return static_cast<T>(a); }

__device__ __forceinline__ long long wrap_add(long long a, long long b) {
  return static_cast<long long>(static_cast<unsigned long long>(a) +
                                static_cast<unsigned long long>(b));
}
__device__ __forceinline__ long long wrap_mul(long long a, long long b) {
  return static_cast<long long>(static_cast<unsigned long long>(a) *
                                static_cast<unsigned long long>(b));
}

template <typename T> __device__ __forceinline__ T tmax(T a, T b) { return a > b ? a : b; }

// ---------------------------------------------------------------- five_point
// float/double: ((((n + s) + e) + w) + c) * 0.2      int: (n+s+e+w+c) / 5
struct FivePoint {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    if constexpr (std::is_same_v<T, int32_t>) {
      long long s = (long long)v.at(-1, 0) + v.at(1, 0) + v.at(0, 1) + v.at(0, -1) + v.at(0, 0);
      return static_cast<int32_t>(s / 5);
    } else {
      T s = v.at(-1, 0) + v.at(1, 0);
      s = s + v.at(0, 1);
      s = s + v.at(0, -1);
      s = s + v.at(0, 0);
      return s * T(0.2);
    }
  }
};

// ---------------------------------------------------------------------- heat
// float/double: c + 0.2 * ((((n + s) + e) + w) - 4c)   int: c + (lap - 4c) / 5
struct Heat {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    T c = v.at(0, 0);
    if constexpr (std::is_same_v<T, int32_t>) {
      long long lap = (long long)v.at(-1, 0) + v.at(1, 0) + v.at(0, 1) + v.at(0, -1) - 4LL * c;
      return static_cast<int32_t>(c + lap / 5);
    } else {
      T lap = v.at(-1, 0) + v.at(1, 0);
      lap = lap + v.at(0, 1);
      lap = lap + v.at(0, -1);
      lap = lap - T(4) * c;
      return c + T(0.2) * lap;
    }
  }
};

// Ops may also provide a column form evaluating a work-item's K vertically
// adjacent cells at once (kColumn = true): `column<T, K>(centre, pitch, p, res)`
// with centre = the first cell.  It must equal K calls of apply() exactly.
template <class Op, class = void>
struct has_column : std::false_type {};
template <class Op>
struct has_column<Op, std::void_t<decltype(Op::kColumn)>> : std::bool_constant<Op::kColumn> {};

// ----------------------------------------------------------------------- gol
// Conway B3/S23 on the 3x3 Moore neighbourhood; a cell is alive iff != 0.
// Column form: the alive count of row i over columns c-1..c+1 is shared by
// the three cells i-1, i, i+1 of the work-item's column (same integer count).
struct Gol {
  static constexpr bool kColumn = true;

  template <typename T, int K>
  __device__ __forceinline__ void column(const T* centre, int pitch, const OpParams<T>&,
                                         T (&res)[K]) const {
    int mid[K + 2];
    int row[K + 2];
#pragma unroll
    for (int i = 0; i < K + 2; ++i) {
      const T* r = centre + (i - 1) * pitch;
      const int l = r[-1] != T(0), m = r[0] != T(0), rr = r[1] != T(0);
      mid[i] = m;
      row[i] = l + m + rr;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const int n = row[k] + row[k + 1] + row[k + 2] - mid[k + 1];
      res[k] = (n == 3 || (mid[k + 1] && n == 2)) ? T(1) : T(0);
    }
  }

  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    int n = (v.at(-1, -1) != T(0)) + (v.at(-1, 0) != T(0)) + (v.at(-1, 1) != T(0)) +
            (v.at(0, -1) != T(0)) + (v.at(0, 1) != T(0)) +
            (v.at(1, -1) != T(0)) + (v.at(1, 0) != T(0)) + (v.at(1, 1) != T(0));
    bool alive = v.at(0, 0) != T(0);
    return (n == 3 || (alive && n == 2)) ? T(1) : T(0);
  }
};

// ------------------------------------------------------------------- boxmean
// Sum of the whole border region, rows north..south outer, columns west..east
// inner, then float: sum / count, int: sum / count (truncating).
struct BoxMean {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>& p) const {
    using A = typename Acc<T>::type;
    A s = A(0);
    for (int dr = -p.north; dr <= p.south; ++dr) {
      for (int dc = -p.west; dc <= p.east; ++dc) {
        if constexpr (std::is_same_v<T, int32_t>) s = wrap_add(s, v.at(dr, dc));
        else s = s + v.at(dr, dc);
      }
    }
    int count = (p.north + p.south + 1) * (p.east + p.west + 1);
    if constexpr (std::is_same_v<T, int32_t>) return static_cast<int32_t>(s / count);
    else return s / T(count);
  }
};

// Asymmetric (5,1,3,0) box mean with compile-time extents: the BASELINE
// config-4 kernel.  Same arithmetic and summation order as BoxMean.
template <int N, int S, int E, int W>
struct BoxMeanFixed {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    using A = typename Acc<T>::type;
    A s = A(0);
#pragma unroll
    for (int dr = -N; dr <= S; ++dr) {
#pragma unroll
      for (int dc = -W; dc <= E; ++dc) {
        if constexpr (std::is_same_v<T, int32_t>) s = wrap_add(s, v.at(dr, dc));
        else s = s + v.at(dr, dc);
      }
    }
    constexpr int count = (N + S + 1) * (E + W + 1);
    if constexpr (std::is_same_v<T, int32_t>) return static_cast<int32_t>(s / count);
    else return s / T(count);
  }
};

// ------------------------------------------------------------------ gaussian
// Binomial blur: w(i,j) = C(2g,g+i) C(2g,g+j) / 2^(4g), row-major sum of
// w * v (mul then add, no FMA).  int32: integer weights C*C, wrap-around
// int64 sum, arithmetic shift right by 4g.
struct Gaussian {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>& p) const {
    const int g = p.gauss_radius;
    const int d = 2 * g + 1;
    using A = typename Acc<T>::type;
    A s = A(0);
    for (int i = -g; i <= g; ++i) {
      for (int j = -g; j <= g; ++j) {
        WeightT<T> w = p.gauss_w[(i + g) * d + (j + g)];
        if constexpr (std::is_same_v<T, int32_t>) {
          s = wrap_add(s, wrap_mul(w, (long long)v.at(i, j)));
        } else {
          s = s + w * v.at(i, j);
        }
      }
    }
    if constexpr (std::is_same_v<T, int32_t>) return static_cast<int32_t>(s >> (4 * g));
    else return s;
  }
};

// --------------------------------------------------------------------- sobel
// gx = (ne + 2e + se) - (nw + 2w + sw); gy = (sw + 2s + se) - (nw + 2n + ne)
// float: sqrt(gx*gx + gy*gy)      int: |gx| + |gy|
struct Sobel {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    if constexpr (std::is_same_v<T, int32_t>) {
      long long gx = ((long long)v.at(-1, 1) + 2LL * v.at(0, 1) + v.at(1, 1)) -
                     ((long long)v.at(-1, -1) + 2LL * v.at(0, -1) + v.at(1, -1));
      long long gy = ((long long)v.at(1, -1) + 2LL * v.at(1, 0) + v.at(1, 1)) -
                     ((long long)v.at(-1, -1) + 2LL * v.at(-1, 0) + v.at(-1, 1));
      long long m = (gx < 0 ? -gx : gx) + (gy < 0 ? -gy : gy);
      return static_cast<int32_t>(m);
    } else {
      T ex = v.at(-1, 1) + T(2) * v.at(0, 1);
      ex = ex + v.at(1, 1);
      T wx = v.at(-1, -1) + T(2) * v.at(0, -1);
      wx = wx + v.at(1, -1);
      T gx = ex - wx;
      T sy = v.at(1, -1) + T(2) * v.at(1, 0);
      sy = sy + v.at(1, 1);
      T ny = v.at(-1, -1) + T(2) * v.at(-1, 0);
      ny = ny + v.at(-1, 1);
      T gy = sy - ny;
      T m2 = gx * gx;
      m2 = m2 + gy * gy;
      return sqrt(m2);
    }
  }
};

// ----------------------------------------------------------------------- nms
// Non-maximum suppression: keep the centre if it is >= every 3x3 neighbour.
struct Nms {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    T m = v.at(-1, -1);
    m = tmax(m, v.at(-1, 0));
    m = tmax(m, v.at(-1, 1));
    m = tmax(m, v.at(0, -1));
    m = tmax(m, v.at(0, 1));
    m = tmax(m, v.at(1, -1));
    m = tmax(m, v.at(1, 0));
    m = tmax(m, v.at(1, 1));
    T c = v.at(0, 0);
    return c >= m ? c : T(0);
  }
};

// ----------------------------------------------------------------- threshold
struct Threshold {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    return v.at(0, 0) > T(0.5) ? T(1) : T(0);
  }
};

// ----------------------------------------------------------------- synthetic
// Cross-shaped access of the full border extents (the column dr = -N..S, then
// the row dc = -W..-1 and 1..E), mean over the taps, then `alu_iters`
// dependent ALU steps: float x = x * 0.999 + 0.001 (mul then add); int
// 32-bit LCG x = x * 1664525 + 1013904223 (mod 2^32).
struct Synthetic {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>& p) const {
    using A = typename Acc<T>::type;
    A s = A(0);
    for (int dr = -p.north; dr <= p.south; ++dr) {
      if constexpr (std::is_same_v<T, int32_t>) s = wrap_add(s, v.at(dr, 0));
      else s = s + v.at(dr, 0);
    }
    for (int dc = -p.west; dc <= -1; ++dc) {
      if constexpr (std::is_same_v<T, int32_t>) s = wrap_add(s, v.at(0, dc));
      else s = s + v.at(0, dc);
    }
    for (int dc = 1; dc <= p.east; ++dc) {
      if constexpr (std::is_same_v<T, int32_t>) s = wrap_add(s, v.at(0, dc));
      else s = s + v.at(0, dc);
    }
    int taps = p.north + p.south + 1 + p.east + p.west;
    if constexpr (std::is_same_v<T, int32_t>) {
      uint32_t x = static_cast<uint32_t>(static_cast<int32_t>(s / taps));
      for (int k = 0; k < p.alu_iters; ++k) x = x * 1664525u + 1013904223u;
      return static_cast<int32_t>(x);
    } else {
      T x = s / T(taps);
      for (int k = 0; k < p.alu_iters; ++k) {
        x = x * T(0.999);
        x = x + T(0.001);
      }
      return x;
    }
  }
};

}  // namespace sk
