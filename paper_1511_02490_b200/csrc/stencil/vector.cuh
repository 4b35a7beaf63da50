// Vector work-items for the one-pass TMA kernel (SK_LOAD_VECTOR).
//
// A work-item owns V = 16 B / sizeof(T) adjacent columns x K rows (the
// scalar path owns 1 column x K rows), so a (wc x wr) workgroup's tile is
// (V*wc) x (K*wr) cells.  Its first cell sits 16-B aligned in the staged
// tile, so every row of its window is read with one 128-bit shared load for
// the V centre cells plus the narrowest aligned loads covering the W / E
// border columns, and every output row leaves as one 128-bit global store.
// The window is streamed row by row through registers: each input row is
// loaded once and serves as north, centre and south row of the outputs that
// need it.
//
// Per op the arithmetic is the scalar path's (the generic form calls the
// op's own apply() on a register view; the Gol and BoxMeanFixed forms share
// partial sums exactly as their column() forms do), so results are
// bit-identical to the scalar kernels and to the CPU oracle.
#pragma once

#include "ops.cuh"

namespace sk {

template <typename T, int V>
struct alignas(16) Vec {
  T v[V];
};

template <typename T, int N>
struct alignas(8) Half {
  T v[N];
};

// w[0 .. L+V+R) = row[-L .. V+R), with row 16-B aligned: one 128-bit load
// for the V centre cells; a side of one cell is a scalar load, a side of
// two 4-byte cells a 64-bit load, wider sides whole 128-bit vectors.
template <typename T, int V, int L, int R>
__device__ __forceinline__ void load_window(const T* row, T (&w)[L + V + R]) {
  const Vec<T, V> c = *reinterpret_cast<const Vec<T, V>*>(row);
#pragma unroll
  for (int j = 0; j < V; ++j) w[L + j] = c.v[j];
  if constexpr (L == 1) {
    w[0] = row[-1];
  } else if constexpr (L == 2 && sizeof(T) == 4) {
    const Half<T, 2> h = *reinterpret_cast<const Half<T, 2>*>(row - 2);
    w[0] = h.v[0];
    w[1] = h.v[1];
  } else if constexpr (L > 1) {
    constexpr int NV = (L + V - 1) / V;
#pragma unroll
    for (int n = 0; n < NV; ++n) {
      const Vec<T, V> h = *reinterpret_cast<const Vec<T, V>*>(row - (NV - n) * V);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const int q = n * V + j;  // column -NV*V + q
        if (q >= NV * V - L) w[q - (NV * V - L)] = h.v[j];
      }
    }
  }
  if constexpr (R == 1) {
    w[L + V] = row[V];
  } else if constexpr (R == 2 && sizeof(T) == 4) {
    const Half<T, 2> h = *reinterpret_cast<const Half<T, 2>*>(row + V);
    w[L + V] = h.v[0];
    w[L + V + 1] = h.v[1];
  } else if constexpr (R > 1) {
    constexpr int NV = (R + V - 1) / V;
#pragma unroll
    for (int n = 0; n < NV; ++n) {
      const Vec<T, V> h = *reinterpret_cast<const Vec<T, V>*>(row + (n + 1) * V);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        if (n * V + j < R) w[L + V + n * V + j] = h.v[j];
      }
    }
  }
}

// Packed fp32 pairs: sm_100's FADD2 / FMUL2 / FFMA2 issue two IEEE
// round-to-nearest operations per instruction, each lane rounded exactly as
// its scalar FADD / FMUL / FFMA (no flush-to-zero), so pairing two columns of
// a work-item halves the instructions of a chain without changing a bit.
struct F2 {
  float x, y;
};

#define SK_F2_OP2(name, ptx)                                                                  \
  __device__ __forceinline__ F2 name(F2 a, F2 b) {                                            \
    F2 r;                                                                                     \
    asm("{\n .reg .b64 a, b, r;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n " ptx        \
        " r, a, b;\n mov.b64 {%0, %1}, r;\n}"                                                 \
        : "=f"(r.x), "=f"(r.y)                                                                \
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));                                            \
    return r;                                                                                 \
  }
SK_F2_OP2(add2, "add.rn.f32x2")
SK_F2_OP2(mul2, "mul.rn.f32x2")
#undef SK_F2_OP2

__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 r;
  asm("{\n .reg .b64 a, b, c, r;\n mov.b64 a, {%2, %3};\n mov.b64 b, {%4, %5};\n"
      " mov.b64 c, {%6, %7};\n fma.rn.f32x2 r, a, b, c;\n mov.b64 {%0, %1}, r;\n}"
      : "=f"(r.x), "=f"(r.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return r;
}

// div_const_fast<D> (ops.cuh) on a pair: q0 = s RN(1/D); r = q0 (-D) + s
// (the same exact remainder as -q0 D + s); q = r RN(1/D) + q0.
template <int D>
__device__ __forceinline__ F2 div_const_fast2(F2 s) {
  constexpr float y = 1.0f / static_cast<float>(D);
  const F2 q0 = mul2(s, F2{y, y});
  const F2 r = fma2(q0, F2{-static_cast<float>(D), -static_cast<float>(D)}, s);
  return fma2(r, F2{y, y}, q0);
}

// Register view over a rolling window of 3 rows (north, centre, south) for
// the generic 3x3 form: at(dr, dc) of output column j.
template <typename T, int RW>
struct Win3 {
  const T (&n)[RW];
  const T (&c)[RW];
  const T (&s)[RW];
  int j;  // compile-time after unrolling
  __device__ __forceinline__ T at(int dr, int dc) const {
    return dr < 0 ? n[j + 1 + dc] : (dr > 0 ? s[j + 1 + dc] : c[j + 1 + dc]);
  }
};

// Generic 3x3 vector form: apply() per cell on a register window.
template <class Op, typename T, int K, int V, class Emit>
__device__ __forceinline__ void vblock3(const Op& op, const T* first, int pitch, const OpParams<T>& p,
                                        Emit&& emit) {
  constexpr int RW = V + 2;
  T a[RW], b[RW], c[RW];
  load_window<T, V, 1, 1>(first - pitch, a);
  load_window<T, V, 1, 1>(first, b);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    load_window<T, V, 1, 1>(first + (k + 1) * pitch, c);
    T out[V];
#pragma unroll
    for (int j = 0; j < V; ++j) out[j] = op.template apply<T>(Win3<T, RW>{a, b, c, j}, p);
    emit(k, out);
#pragma unroll
    for (int j = 0; j < RW; ++j) {
      a[j] = b[j];
      b[j] = c[j];
    }
  }
}

// Game of Life: per input row, alive flags of the V + 2 columns, then per
// column the 3-sum x and the 2-sum y (the scalar column form's partial
// counts); cell (k, j) = B3/S23 of x[k-1] + y[k] + x[k+1] at column j.
template <typename T, int K, int V, class Emit>
__device__ __forceinline__ void vblock_gol(const T* first, int pitch, Emit&& emit) {
  unsigned x0[V], x1[V], y1[V], m1[V];
  auto row_counts = [&](const T* row, unsigned (&x)[V], unsigned (&y)[V], unsigned (&m)[V]) {
    T w[V + 2];
    load_window<T, V, 1, 1>(row, w);
    unsigned al[V + 2];
#pragma unroll
    for (int j = 0; j < V + 2; ++j) al[j] = Gol::alive(w[j]);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      m[j] = al[j + 1];
      y[j] = al[j] + al[j + 2];
      x[j] = y[j] + m[j];
    }
  };
  unsigned yd[V], md[V];
  row_counts(first - pitch, x0, yd, md);
  row_counts(first, x1, y1, m1);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    unsigned x2[V], y2[V], m2[V];
    row_counts(first + (k + 1) * pitch, x2, y2, m2);
    T out[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const unsigned n8 = x0[j] + y1[j] + x2[j];
      out[j] = ((n8 | m1[j]) == 3u) ? T(1) : T(0);
    }
    emit(k, out);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      x0[j] = x1[j];
      x1[j] = x2[j];
      y1[j] = y2[j];
      m1[j] = m2[j];
    }
  }
}

// Box mean with compile-time extents: per input row the V row sums (west to
// east), kept for the NR = N + S + 1 rows of the window; cell (k, j) = the
// row sums of rows k-N .. k+S added north to south, divided by the count.
// fp32 with count 28: the exact 3-instruction division (div_const_fast) per
// output row unless a sum of that row is outside its verified range.  (An
// optimistic form - no branch per row, the work-item re-run on a flag - was
// measured slower at K = 8: the re-run doubles the kernel's code.)
template <int N, int S, int E, int W, typename T, int K, int V, class Emit>
__device__ __forceinline__ void vblock_boxmean(const T* first, int pitch, Emit&& emit) {
  using A = typename Acc<T>::type;
  constexpr int NR = N + S + 1;
  constexpr int kCount = (N + S + 1) * (E + W + 1);
  constexpr bool kFastDiv = std::is_same_v<T, float> && kCount == 28;
  A rs[NR][V];
  auto row_sums = [&](const T* row, A (&out)[V]) {
    T w[W + V + E];
    load_window<T, V, W, E>(row, w);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      A s = A(w[j]);
#pragma unroll
      for (int d = 1; d <= W + E; ++d) s = acc_add<T>(s, w[j + d]);
      out[j] = s;
    }
  };
#pragma unroll
  for (int i = 0; i < NR - 1; ++i) row_sums(first + (i - N) * pitch, rs[i]);
#pragma unroll
  for (int k = 0; k < K; ++k) {
    row_sums(first + (k + S) * pitch, rs[NR - 1]);
    A sum[V];
    if constexpr (std::is_same_v<T, float> && V % 2 == 0) {
      // two columns per packed add, north to south as the scalar chain
#pragma unroll
      for (int j = 0; j < V; j += 2) {
        F2 s{rs[0][j], rs[0][j + 1]};
#pragma unroll
        for (int i = 1; i < NR; ++i) s = add2(s, F2{rs[i][j], rs[i][j + 1]});
        sum[j] = s.x;
        sum[j + 1] = s.y;
      }
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) {
        A s = rs[0][j];
#pragma unroll
        for (int i = 1; i < NR; ++i) s = acc_add2<T>(s, rs[i][j]);
        sum[j] = s;
      }
    }
    T out[V];
    if constexpr (kFastDiv) {
      bool fast = true;
#pragma unroll
      for (int j = 0; j < V; ++j) fast = fast && div_const_in_range(sum[j]);
      if (!fast) {  // rare: a sum outside the exact sequence's range
#pragma unroll
        for (int j = 0; j < V; ++j) out[j] = __fdiv_rn(sum[j], static_cast<float>(kCount));
      } else if constexpr (V % 2 == 0) {
#pragma unroll
        for (int j = 0; j < V; j += 2) {
          const F2 q = div_const_fast2<kCount>(F2{sum[j], sum[j + 1]});
          out[j] = q.x;
          out[j + 1] = q.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < V; ++j) out[j] = div_const_fast<kCount>(sum[j]);
      }
    } else {
#pragma unroll
      for (int j = 0; j < V; ++j) out[j] = acc_div_const<T, kCount>(sum[j]);
    }
    emit(k, out);
#pragma unroll
    for (int i = 0; i < NR - 1; ++i) {
#pragma unroll
      for (int j = 0; j < V; ++j) rs[i][j] = rs[i + 1][j];
    }
  }
}

// Dispatch to an op's vector form.  Only ops with a compile-time border
// region have one; the host takes the vector kernel only when the
// descriptor's border equals it (registry: vector_for).
template <class Op> struct VectorForm : std::false_type {};
template <> struct VectorForm<FivePoint> : std::true_type {};
template <> struct VectorForm<Heat> : std::true_type {};
template <> struct VectorForm<Sobel> : std::true_type {};
template <> struct VectorForm<Nms> : std::true_type {};
template <> struct VectorForm<Gol> : std::true_type {};
template <int N, int S, int E, int W> struct VectorForm<BoxMeanFixed<N, S, E, W>> : std::true_type {};

template <class Op> struct BoxExtents;
template <int N, int S, int E, int W>
struct BoxExtents<BoxMeanFixed<N, S, E, W>> {
  static constexpr int n = N, s = S, e = E, w = W;
};

template <class Op, typename T, int K, int V, class Emit>
__device__ __forceinline__ void vector_tile(const T* first, int pitch, const OpParams<T>& p, Emit&& emit) {
  static_assert(VectorForm<Op>::value, "op has no vector form");
  if constexpr (std::is_same_v<Op, Gol>) {
    vblock_gol<T, K, V>(first, pitch, emit);
  } else if constexpr (std::is_same_v<Op, FivePoint> || std::is_same_v<Op, Heat> ||
                       std::is_same_v<Op, Sobel> || std::is_same_v<Op, Nms>) {
    vblock3<Op, T, K, V>(Op{}, first, pitch, p, emit);
  } else {
    using B = BoxExtents<Op>;
    vblock_boxmean<B::n, B::s, B::e, B::w, T, K, V>(first, pitch, emit);
  }
}

}  // namespace sk
