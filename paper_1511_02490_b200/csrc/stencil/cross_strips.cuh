// K1x  k_cross_strips — temporally blocked 5-point cross stencils (heat,
// five_point; N = S = E = W = 1) with the tile held in registers.
//
// The per-cell fused kernel (fused.cuh) recomputes every intermediate
// generation through shared memory: each cell update is 5 LDS + 1 STS + a
// block barrier per generation, and the loaded tile must fit the TMA ring.
// That caps heat f32 16384^2 at ~0.97 Tcells/s (TB = 4).  Here a block owns a
// tile of 32 lanes x 4 columns = 128 columns by nwarps x R rows; lane l of
// warp w holds columns 4l .. 4l+3 of rows wR .. wR+R-1 in registers, so a
// generation is, per row and lane:
//   west / east neighbours of the lane's outer columns: 2 warp shuffles;
//   north / south: the rows above / below in registers, except the warp's
//   first / last row, which come from the warps above / below through a
//   2 x nwarps x 2 x 32 x 16-B exchange area in shared memory (one barrier
//   per generation, double-buffered by generation parity, as k_gol_strips);
//   the op's own apply() on a 5-value view, so the arithmetic is the
//   executor's, bit for bit (-fmad=false).
// Garbage enters at the tile's outer lanes / rows and moves one cell per
// generation, so after TB generations columns [TB, 128 - TB) and rows
// [TB, nwarps R - TB) are exact: the tile stores 4 (32 - 2 ceil(TB/4))
// columns x (nwarps R - 2 TB) rows.
//
// Border semantics (DESIGN.md §2/§4.2) without a fix-up pass: a cross
// stencil only reads its 4 edge neighbours, and the substitute of an
// out-of-window neighbour is the pad value or - the nearest cell of a cross
// neighbour being the centre itself - the centre.  In edge tiles each
// in-window cell therefore takes its substitute directly when its
// neighbour lies outside the readable window [lo, hi] x [0, W); cells outside
// the window compute values nobody reads.  That is exactly what the one-pass
// executor reads at every generation, so the result is bit-identical.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

#include "ops.cuh"

namespace sk {

struct CrossGeom {
  long long pitch_in, pitch_out;  // elements
  int W, H;                       // output region
  int lo, hi;                     // readable input rows [lo, hi] (row 0 = output row 0)
  int tb;                         // generations this launch
  int hl;                         // halo lanes per side: ceil(tb / 4)
  int oc, th;                     // output columns / rows per tile
  int tiles_x, tiles_y;
  int mode;                       // sk_border_mode
  int vec;                        // 16-B aligned rows: vector loads / stores
};

// Four consecutive elements as 16-B accesses (two for double).
template <typename T>
struct alignas(4 * sizeof(T)) Quad {
  T x[4];
};

template <typename T>
__device__ __forceinline__ T from_bits(uint32_t u) {
  if constexpr (std::is_same_v<T, float>) return __uint_as_float(u);
  else return static_cast<T>(static_cast<int32_t>(u));
}
__device__ __forceinline__ uint32_t to_bits(float v) { return __float_as_uint(v); }
__device__ __forceinline__ uint32_t to_bits(int32_t v) { return static_cast<uint32_t>(v); }

template <typename T>
__device__ __forceinline__ Quad<T> ld_quad(const T* p, int gc, int W, bool vec) {
  Quad<T> q;
  if (vec && gc + 3 < W) {
    if constexpr (sizeof(T) == 4) {
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
      q.x[0] = from_bits<T>(u.x);
      q.x[1] = from_bits<T>(u.y);
      q.x[2] = from_bits<T>(u.z);
      q.x[3] = from_bits<T>(u.w);
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(p));
      const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
      q.x[0] = a.x; q.x[1] = a.y; q.x[2] = b.x; q.x[3] = b.y;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) q.x[j] = (gc + j >= 0 && gc + j < W) ? __ldg(p + j) : T(0);
  }
  return q;
}

template <typename T>
__device__ __forceinline__ void st_quad(T* p, const T (&v)[4], int gc, int W, bool vec) {
  if (vec && gc + 3 < W) {
    if constexpr (sizeof(T) == 4) {
      const uint4 u = make_uint4(to_bits(v[0]), to_bits(v[1]), to_bits(v[2]), to_bits(v[3]));
      __stcs(reinterpret_cast<uint4*>(p), u);
    } else {
      __stcs(reinterpret_cast<double2*>(p), make_double2(v[0], v[1]));
      __stcs(reinterpret_cast<double2*>(p) + 1, make_double2(v[2], v[3]));
    }
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (gc + j < W) p[j] = v[j];
    }
  }
}

// The 5-value view an op's apply() reads (at(dr, dc), dr = rows south).
template <typename T>
struct Cross5 {
  T n, s, e, w, c;
  __device__ __forceinline__ T at(int dr, int dc) const {
    return dr < 0 ? n : (dr > 0 ? s : (dc > 0 ? e : (dc < 0 ? w : c)));
  }
};

template <typename T>
__device__ __forceinline__ T shfl_up1(T v) {
  if constexpr (sizeof(T) == 8) {
    return __longlong_as_double(__shfl_up_sync(0xffffffffu, __double_as_longlong(v), 1));
  } else {
    return __shfl_up_sync(0xffffffffu, v, 1);
  }
}
template <typename T>
__device__ __forceinline__ T shfl_down1(T v) {
  if constexpr (sizeof(T) == 8) {
    return __longlong_as_double(__shfl_down_sync(0xffffffffu, __double_as_longlong(v), 1));
  } else {
    return __shfl_down_sync(0xffffffffu, v, 1);
  }
}

// One generation of the warp's R x 4 register strip.  EDGE: the tile touches
// the window edge, so in-window cells substitute out-of-window neighbours.
template <bool EDGE, class Op, typename T, int R>
__device__ __forceinline__ void cross_generation(T (&v)[R][4], const T (&above)[4], const T (&below)[4],
                                                 const Op& op, const OpParams<T>& p, int r0, int gc,
                                                 const CrossGeom& g, T pad) {
  T prev[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) prev[j] = above[j];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    T cur[4], sth[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      cur[j] = v[i][j];
      sth[j] = i + 1 < R ? v[i + 1][j] : below[j];
    }
    const T wl = shfl_up1(cur[3]);
    const T er = shfl_down1(cur[0]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      T n = prev[j], s = sth[j];
      T w = j == 0 ? wl : cur[j - 1];
      T e = j == 3 ? er : cur[j + 1];
      if constexpr (EDGE) {
        const T sub = g.mode == 0 ? pad : cur[j];
        const int gr = r0 + i;
        n = gr == g.lo ? sub : n;
        s = gr == g.hi ? sub : s;
        w = gc + j == 0 ? sub : w;
        e = gc + j == g.W - 1 ? sub : e;
      }
      v[i][j] = op.template apply<T>(Cross5<T>{n, s, e, w, cur[j]}, p);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) prev[j] = cur[j];
  }
}

template <bool EDGE, class Op, typename T, int R>
__device__ __forceinline__ void cross_generations(T (&v)[R][4], Quad<T>* xchg, int lane, int warp,
                                                  int nwarps, const OpParams<T>& p, int r0, int gc,
                                                  const CrossGeom& g, T pad) {
  const Op op;
  for (int gen = 1; gen <= g.tb; ++gen) {
    Quad<T>* slot = xchg + (gen & 1) * nwarps * 64;
    Quad<T> top, bot;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      top.x[j] = v[0][j];
      bot.x[j] = v[R - 1][j];
    }
    slot[warp * 64 + lane] = top;
    slot[warp * 64 + 32 + lane] = bot;
    __syncthreads();
    // the tile's first / last rows read their own rows: halo garbage
    const Quad<T> a = warp > 0 ? slot[(warp - 1) * 64 + 32 + lane] : top;
    const Quad<T> b = warp < nwarps - 1 ? slot[(warp + 1) * 64 + lane] : bot;
    cross_generation<EDGE, Op, T, R>(v, a.x, b.x, op, p, r0, gc, g, pad);
  }
}

// Register budget per thread bounds the block (the per-kernel maximum
// workgroup size): R x 4 state values plus the rolling rows.
// R = 8 asks for two resident 384-thread blocks per SM (<= 80 registers):
// with one, the SM idles on every block's tile load (ncu: long_scoreboard).
template <int R>
struct CrossBounds {
  static constexpr int kThreads = R <= 4 ? 1024 : 384;
  static constexpr int kMinBlocks = R == 8 ? 2 : 1;
};

template <class Op, typename T, int R>
__global__ void __launch_bounds__(CrossBounds<R>::kThreads, CrossBounds<R>::kMinBlocks)
    k_cross_strips(const T* __restrict__ in, T* __restrict__ out, const CrossGeom g, const T pad,
                   const __grid_constant__ OpParams<T> p) {
  // programmatic dependent launch (launch.cu: launch_pdl_checked): no global
  // access before the previous launch has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) unsigned char sm_raw[];
  Quad<T>* xchg = reinterpret_cast<Quad<T>*>(sm_raw);  // [2 parities][nwarps][top, bottom][32]
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int tile_rows = nwarps * R;

  const int ty = blockIdx.x / g.tiles_x;
  const int tx = blockIdx.x - ty * g.tiles_x;
  const int row_base = ty * g.th - g.tb;      // global row of tile row 0
  const int col_base = tx * g.oc - 4 * g.hl;  // global column of lane 0's first cell
  const int gc = col_base + 4 * lane;
  const int r0 = row_base + warp * R;
  const bool vec = g.vec != 0;
  const bool edge = col_base < 0 || col_base + 128 > g.W || row_base < g.lo ||
                    row_base + tile_rows - 1 > g.hi;

  T v[R][4];
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int gr = r0 + i;
    if (gr >= g.lo && gr <= g.hi && gc + 3 >= 0 && gc < g.W) {
      const Quad<T> q = ld_quad(in + static_cast<long long>(gr) * g.pitch_in + gc, gc, g.W, vec);
#pragma unroll
      for (int j = 0; j < 4; ++j) v[i][j] = q.x[j];
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) v[i][j] = T(0);
    }
  }

  if (edge) {
    cross_generations<true, Op, T, R>(v, xchg, lane, warp, nwarps, p, r0, gc, g, pad);
  } else {
    cross_generations<false, Op, T, R>(v, xchg, lane, warp, nwarps, p, r0, gc, g, pad);
  }

  if (lane < g.hl || lane >= 32 - g.hl || gc >= g.W) return;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int t = warp * R + i;
    const int gr = r0 + i;
    if (t >= g.tb && t < g.tb + g.th && gr < g.H) {
      st_quad(out + static_cast<long long>(gr) * g.pitch_out + gc, v[i], gc, g.W, vec);
    }
  }
}

}  // namespace sk
