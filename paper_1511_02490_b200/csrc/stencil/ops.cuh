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
  WeightT<T> gauss_b[21];        // gaussian: 1-D binomial weights b_j, j = -g..g
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

  // alive(v) = v != 0 as 0/1: one unsigned min for int32 (any non-zero bit
  // pattern, negatives included, maps to 1); floats drop the sign bit first
  // so -0.0 stays dead and NaN stays alive, exactly like `v != 0`.
  template <typename T>
  __device__ __forceinline__ static unsigned alive(T v) {
    if constexpr (std::is_same_v<T, int32_t>) {
      return min(static_cast<unsigned>(v), 1u);
    } else if constexpr (std::is_same_v<T, float>) {
      return min(__float_as_uint(v) & 0x7fffffffu, 1u);
    } else {
      const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
      return b != 0ull;
    }
  }

  // Per row i: x = l + m + r (3-sum) and y = l + r (2-sum, the centre row's
  // neighbours); the 8-neighbour count of cell k is x[k] + y[k+1] + x[k+2].
  // B3/S23: alive next iff n8 == 3 or (alive and n8 == 2), i.e. (n8 | alive) == 3.
  template <typename T, int K>
  __device__ __forceinline__ void column(const T* centre, int pitch, const OpParams<T>&,
                                         T (&res)[K]) const {
    unsigned mid[K + 2], x[K + 2], y[K + 2];
#pragma unroll
    for (int i = 0; i < K + 2; ++i) {
      const T* r = centre + (i - 1) * pitch;
      const unsigned l = alive(r[-1]), m = alive(r[0]), rr = alive(r[1]);
      mid[i] = m;
      y[i] = l + rr;
      x[i] = y[i] + m;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const unsigned n8 = x[k] + y[k + 1] + x[k + 2];
      res[k] = ((n8 | mid[k + 1]) == 3u) ? T(1) : T(0);
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
// Sum of row sums: each row of the region is summed west to east, then the
// row sums north to south; divided by the cell count (int: truncating).
// The column form shares every row sum between the K cells of a work-item.
template <typename T>
__device__ __forceinline__ typename Acc<T>::type acc_add(typename Acc<T>::type a, T b) {
  if constexpr (std::is_same_v<T, int32_t>) return wrap_add(a, b);
  else return a + b;
}
template <typename T>
__device__ __forceinline__ typename Acc<T>::type acc_add2(typename Acc<T>::type a,
                                                          typename Acc<T>::type b) {
  if constexpr (std::is_same_v<T, int32_t>) return wrap_add(a, b);
  else return a + b;
}
template <typename T>
__device__ __forceinline__ T acc_div(typename Acc<T>::type s, int count) {
  if constexpr (std::is_same_v<T, int32_t>) return static_cast<int32_t>(s / count);
  else return s / T(count);
}

// fp32 s / D, correctly rounded, for a compile-time divisor: q0 = s * RN(1/D),
// the exact remainder r = s - q0 D (one FMA), q = q0 + r * RN(1/D).  Away
// from zero, subnormals, overflow and non-finite s this equals the IEEE
// quotient for D = 28 - verified for all 2^32 inputs on the GPU
// (tests/test_div_const.py) - and costs 3 FP instructions instead of the
// ~11 of a general division (MUFU.RCP, 4 FFMA, FCHK and its slow-path
// branch).  The rare out-of-range inputs take the IEEE division.
template <int D>
__device__ __forceinline__ float div_const_fast(float s) {
  constexpr float y = 1.0f / static_cast<float>(D);
  const float q0 = __fmul_rn(s, y);
  const float r = __fmaf_rn(-q0, static_cast<float>(D), s);
  return __fmaf_rn(r, y, q0);
}
__device__ __forceinline__ bool div_const_in_range(float s) {
  const float a = fabsf(s);
  return a >= 0x1p-100f && a <= 0x1p+120f;  // false for 0, subnormals, inf, NaN
}
template <int D>
__device__ __forceinline__ float div_const_rn(float s) {
  return div_const_in_range(s) ? div_const_fast<D>(s) : __fdiv_rn(s, static_cast<float>(D));
}

// Division by a compile-time cell count: the exact fp32 sequence above for
// the divisors it is verified for, the IEEE division otherwise.
template <typename T, int D>
__device__ __forceinline__ T acc_div_const(typename Acc<T>::type s) {
  if constexpr (std::is_same_v<T, float> && D == 28) return div_const_rn<D>(s);
  else return acc_div<T>(s, D);
}

struct BoxMean {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>& p) const {
    using A = typename Acc<T>::type;
    A s = A(0);
    for (int dr = -p.north; dr <= p.south; ++dr) {
      A row = A(v.at(dr, -p.west));
      for (int dc = -p.west + 1; dc <= p.east; ++dc) row = acc_add<T>(row, v.at(dr, dc));
      s = dr == -p.north ? row : acc_add2<T>(s, row);
    }
    return acc_div<T>(s, (p.north + p.south + 1) * (p.east + p.west + 1));
  }
};

// Compile-time extents (the BASELINE config-4 (5,1,3,0) kernel).
template <int N, int S, int E, int W>
struct BoxMeanFixed {
  static constexpr bool kColumn = true;
  static constexpr int kCount = (N + S + 1) * (E + W + 1);

  template <typename T>
  __device__ __forceinline__ typename Acc<T>::type row_sum(const T* r) const {
    using A = typename Acc<T>::type;
    A row = A(r[-W]);
#pragma unroll
    for (int dc = -W + 1; dc <= E; ++dc) row = acc_add<T>(row, r[dc]);
    return row;
  }

  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>&) const {
    using A = typename Acc<T>::type;
    A s = A(0);
#pragma unroll
    for (int dr = -N; dr <= S; ++dr) {
      A row = A(v.at(dr, -W));
#pragma unroll
      for (int dc = -W + 1; dc <= E; ++dc) row = acc_add<T>(row, v.at(dr, dc));
      s = dr == -N ? row : acc_add2<T>(s, row);
    }
    return acc_div_const<T, kCount>(s);
  }

  template <typename T, int K>
  __device__ __forceinline__ void column(const T* centre, int pitch, const OpParams<T>&,
                                         T (&res)[K]) const {
    using A = typename Acc<T>::type;
    A rows[K + N + S];
#pragma unroll
    for (int i = 0; i < K + N + S; ++i) rows[i] = row_sum<T>(centre + (i - N) * pitch);
    A sums[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      A s = rows[k];
#pragma unroll
      for (int j = 1; j <= N + S; ++j) s = acc_add2<T>(s, rows[k + j]);
      sums[k] = s;
    }
    if constexpr (std::is_same_v<T, float> && kCount == 28) {
      // one branch per work-item: the K quotients take the 3-instruction
      // exact sequence unless one of them is out of its range
      bool fast = true;
#pragma unroll
      for (int k = 0; k < K; ++k) fast = fast && div_const_in_range(sums[k]);
      if (fast) {
#pragma unroll
        for (int k = 0; k < K; ++k) res[k] = div_const_fast<kCount>(sums[k]);
      } else {
#pragma unroll
        for (int k = 0; k < K; ++k) res[k] = __fdiv_rn(sums[k], static_cast<float>(kCount));
      }
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) res[k] = acc_div_const<T, kCount>(sums[k]);
    }
  }
};

// ------------------------------------------------------------------ gaussian
// Separable binomial blur: b_j = C(2g, g+j) / 2^(2g) (exact in fp32/fp64).
// Row pass r_i = b_{-g} v(i,-g) + ... + b_g v(i,g) west to east (mul, then
// add), then s = b_{-g} r_{-g} + ... + b_g r_g north to south.  int32: integer
// b_j = C(2g, g+j), wrap-around int64 sums, arithmetic shift right by 4g.
template <typename T>
__device__ __forceinline__ typename Acc<T>::type gauss_term(WeightT<T> w, typename Acc<T>::type x) {
  if constexpr (std::is_same_v<T, int32_t>) return wrap_mul(w, x);
  else return w * x;
}

template <typename T>
__device__ __forceinline__ T gauss_result(typename Acc<T>::type s, int g) {
  if constexpr (std::is_same_v<T, int32_t>) return static_cast<int32_t>(s >> (4 * g));
  else return s;
}

struct Gaussian {
  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>& p) const {
    using A = typename Acc<T>::type;
    const int g = p.gauss_radius;
    A s = A(0);
    for (int i = -g; i <= g; ++i) {
      A row = gauss_term<T>(p.gauss_b[0], A(v.at(i, -g)));
      for (int j = -g + 1; j <= g; ++j) row = acc_add2<T>(row, gauss_term<T>(p.gauss_b[j + g], A(v.at(i, j))));
      const A t = gauss_term<T>(p.gauss_b[i + g], row);
      s = i == -g ? t : acc_add2<T>(s, t);
    }
    return gauss_result<T>(s, g);
  }
};

// Fixed radius (the reference kernel's default g = 5) with a column form:
// the K + 2G row passes are shared by the K cells of a work-item.
template <int G>
struct GaussianFixed {
  static constexpr bool kColumn = true;

  template <typename T, class V>
  __device__ __forceinline__ T apply(const V& v, const OpParams<T>& p) const {
    return Gaussian{}.template apply<T>(v, p);
  }

  template <typename T, int K>
  __device__ __forceinline__ void column(const T* centre, int pitch, const OpParams<T>& p,
                                         T (&res)[K]) const {
    using A = typename Acc<T>::type;
    A rows[K + 2 * G];
#pragma unroll
    for (int i = 0; i < K + 2 * G; ++i) {
      const T* r = centre + (i - G) * pitch;
      A row = gauss_term<T>(p.gauss_b[0], A(r[-G]));
#pragma unroll
      for (int j = -G + 1; j <= G; ++j) row = acc_add2<T>(row, gauss_term<T>(p.gauss_b[j + G], A(r[j])));
      rows[i] = row;
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      A s = gauss_term<T>(p.gauss_b[0], rows[k]);
#pragma unroll
      for (int i = 1; i <= 2 * G; ++i) s = acc_add2<T>(s, gauss_term<T>(p.gauss_b[i], rows[k + i]));
      res[k] = gauss_result<T>(s, G);
    }
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
