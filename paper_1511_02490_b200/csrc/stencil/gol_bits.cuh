// Game of Life on the bit-plane path (SK_LOAD_BITPLANE): bit-sliced and
// temporally blocked, bit-identical to one-pass-per-generation execution.
//
// The customising function (B3/S23 on the 3x3 Moore
// neighbourhood, a cell is alive iff != 0) depends on its neighbourhood only
// through alive/dead, so the grid can be held as one bit per cell: a packed
// grid of uint32 words, bit b of word j = column 32 j + b.  One 32-bit logic
// op then evaluates 32 cells.  A run is three kinds of launch:
//
//   k_gol_pack     T grid -> packed grid: a warp reads 32 consecutive cells
//                  per 128-B request and __ballot_sync(v != 0) makes a word
//                  (the one HBM read of the T grid);
//   k_gol_strips   TB generations of the packed grid per launch, in
//                  registers (below); the packed grids are W*H/8 bytes and
//                  stay in L2 between launches;
//   k_gol_unpack   packed grid -> T grid, one int4/float4 store per 4 cells
//                  (the one HBM write of the T grid).
//
// Border semantics are the executor's (DESIGN.md §2/§4.2): after the load
// and after every intermediate generation, the cells of an edge tile outside
// the readable window are re-substituted - pad value, or the nearest
// in-window cell of that generation - exactly what the one-pass executor
// would read at the next launch (tests/test_gol_bits.py).
//
// Neighbour count, bit-sliced.  Per row, with W/C/E the row shifted
// west/centre/east (carried across word boundaries), the horizontal 3-sum
// W+C+E is the 2-bit number (x1 x0) = (maj(W,C,E), W^C^E) and the 2-sum W+E
// is (y1 y0) = (W&E, W^E).  The 8-neighbour count of a centre row b between
// rows a and c is n8 = x(a) + y(b) + x(c):
//     l0 = a0^b0^c0, l1 = maj(a0,b0,c0), h0 = a1^b1^c1, h1 = maj(a1,b1,c1)
//     n8 = l0 + 2 (l1 + h0) + 4 h1
// B3/S23 is next = (n8 == 3) | (alive & n8 == 2) = ((n8 | alive) == 3), i.e.
//     next = (l0 | alive) & (l1 ^ h0) & ~h1
// (l1 & h0 set means n8 >= 4, and then l1 ^ h0 is 0).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace sk {

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (c & (a | b));
}

template <typename T>
struct Vec4;
template <> struct Vec4<int32_t> { using type = int4; };
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };

// ===========================================================================
// K1s  k_gol_strips<R> — register strips over packed bit grids.
//
// Packed grid: row-major uint32 words, row pitch pw words, bit b of word j =
// column 32 j + b.  k_gol_pack / k_gol_unpack convert a T grid to / from it
// (one HBM pass each); k_gol_strips advances TB generations of a packed grid
// (32x smaller than the T grid, so it lives in L2 across launches).
//
// A block owns a tile of 32 - 2 hw words x (nwarps R - 2 TB) rows.  Lane l of
// warp w holds word l of the tile for R consecutive rows (w R .. w R + R - 1)
// in registers.  Per generation: west/east words come from lanes l -+ 1
// (__shfl_up/down), the row above / below the warp's strip from the warps
// above / below through a 2 x nwarps x 32-word exchange area in shared memory
// (one barrier per generation, double-buffered by generation parity), and
// the R rows are updated in place over a rolling window of row sums.  The
// tile's outer lanes / rows are the halo: garbage (missing neighbours) enters
// there and moves one cell per generation, so after TB <= 32 hw generations
// lanes [hw, 32 - hw) and rows [TB, nwarps R - TB) are exact.
// ===========================================================================
struct StripGeom {
  long long pw_in, pw_out;   // packed row pitches (words)
  int W, H;                  // grid
  int lo, hi;                // readable rows [lo, hi] of the packed input
  int nwords;                // ceil(W / 32)
  int tb, hw, ow, th;        // generations, halo lanes, output words / rows per tile
  int tiles_x, tiles_y;
  int mode;                  // sk_border_mode
  uint32_t padword;          // 0 or ~0
};

// Explicit 3-input logic ops (one LOP3 each; immediates for a = 0xF0,
// b = 0xCC, c = 0xAA) so the ALU op count is exactly what is written.
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return d;
}

// Row sums of one row word c with its west/east neighbours l, r:
// x = W + C + E as (x1 x0), y = W + E as (y1 y0).  The two shifts are
// multiplies (IMAD / IMAD.HI on the FMA pipe) because the ALU pipe, which
// runs every LOP3, is the kernel's bound: west = c << 1 | l >> 31 =
// c * 2 + hi(l * 2), east = c >> 1 | r << 31 = r * 2^31 + hi(c * 2^31).
__device__ __forceinline__ void row_sums(uint32_t l, uint32_t c, uint32_t r, uint32_t& x0,
                                         uint32_t& x1, uint32_t& y0, uint32_t& y1) {
  uint32_t w, e;
  asm("{\n\t.reg .u32 t;\n\t"
      "mul.hi.u32 t, %2, 2;\n\t"
      "mad.lo.u32 %0, %3, 2, t;\n\t"
      "mul.hi.u32 t, %3, 0x80000000;\n\t"
      "mad.lo.u32 %1, %4, 0x80000000, t;\n\t}"
      : "=r"(w), "=r"(e)
      : "r"(l), "r"(c), "r"(r));
  x0 = lop3<0x96>(w, c, e);  // w ^ c ^ e
  x1 = lop3<0xE8>(w, c, e);  // maj(w, c, e)
  y0 = lop3<0x3C>(w, e, 0);  // w ^ e
  y1 = lop3<0xC0>(w, e, 0);  // w & e
}

// next state of centre row b (alive, 2-sum y) between rows with 3-sums xa, xc
__device__ __forceinline__ uint32_t next_state(uint32_t xa0, uint32_t xa1, uint32_t y0, uint32_t y1,
                                               uint32_t xc0, uint32_t xc1, uint32_t alive) {
  const uint32_t l0 = lop3<0x96>(xa0, y0, xc0);
  const uint32_t l1 = lop3<0xE8>(xa0, y0, xc0);
  const uint32_t h0 = lop3<0x96>(xa1, y1, xc1);
  const uint32_t h1 = lop3<0xE8>(xa1, y1, xc1);
  const uint32_t t = lop3<0x14>(l1, h0, h1);  // (l1 ^ h0) & ~h1
  return lop3<0xA8>(l0, alive, t);            // (l0 | alive) & t
}

template <int R>
__device__ __forceinline__ void strips_substitute(uint32_t (&w)[R], const StripGeom& g, int lane,
                                                  int warp, int row_base, int word_base,
                                                  int tile_rows, uint32_t* edge_rows) {
  const int gw = word_base + lane;
  if (word_base < 0 || 32 * (word_base + 32) > g.W) {
    const int gw_e = (g.W & 31) ? g.nwords - 1 : g.nwords;  // first word with bits >= W
    const bool west = gw < 0, east = gw >= gw_e;
    const int nvalid = g.W - 32 * gw;
    const uint32_t m = nvalid <= 0 ? 0u : (nvalid >= 32 ? ~0u : ((1u << nvalid) - 1u));
    const int j0 = min(31, max(0, -word_base));                // lane of column 0
    const int jl = min(31, max(0, g.nwords - 1 - word_base));  // lane of column W-1
    const int bl = (g.W - 1) & 31;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      uint32_t v = w[i];
      const uint32_t v0 = __shfl_sync(0xffffffffu, v, j0);
      const uint32_t vl = __shfl_sync(0xffffffffu, v, jl);
      const uint32_t wf = g.mode == 0 ? g.padword : 0u - (v0 & 1u);
      const uint32_t ef = g.mode == 0 ? g.padword : 0u - ((vl >> bl) & 1u);
      v = west ? wf : v;
      v = east ? ((v & m) | (ef & ~m)) : v;
      w[i] = v;
    }
  }
  const int i_lo = g.lo - row_base, i_hi = g.hi - row_base;  // tile rows of the window edges
  if (i_lo > 0 || i_hi < tile_rows - 1) {
    const int r0 = warp * R;
    if (g.mode != 0) {  // nearest: publish rows i_lo / i_hi of this generation
      __syncthreads();  // the previous readers of edge_rows are done
#pragma unroll
      for (int i = 0; i < R; ++i) {
        if (r0 + i == i_lo) edge_rows[lane] = w[i];
        if (r0 + i == i_hi) edge_rows[32 + lane] = w[i];
      }
      __syncthreads();
    }
    const uint32_t vlo = g.mode == 0 ? g.padword : (i_lo > 0 ? edge_rows[lane] : 0u);
    const uint32_t vhi = g.mode == 0 ? g.padword : (i_hi < tile_rows - 1 ? edge_rows[32 + lane] : 0u);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      w[i] = r0 + i < i_lo ? vlo : (r0 + i > i_hi ? vhi : w[i]);
    }
  }
}

// Register budget per thread bounds the block: R words of state plus the
// rolling window (the per-kernel maximum workgroup size).
template <int R>
__global__ void __launch_bounds__(R <= 8 ? 768 : (R <= 16 ? 512 : 256))
    k_gol_strips(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, const StripGeom g) {
  // programmatic dependent launch (launch.cu: launch_pdl_checked): no global
  // access before the previous launch has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) uint32_t sm_x[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  uint32_t* xchg = sm_x;                       // [2 parities][nwarps][2 (top, bottom)][32]
  uint32_t* edge_rows = sm_x + 2 * nwarps * 64;  // [2][32]
  const int tile_rows = nwarps * R;

  const int ty = blockIdx.x / g.tiles_x;
  const int tx = blockIdx.x - ty * g.tiles_x;
  const int row_base = ty * g.th - g.tb;       // global row of tile row 0
  const int word_base = tx * g.ow - g.hw;      // global word of lane 0
  const int gw = word_base + lane;
  const int r0 = row_base + warp * R;          // global row of this warp's first row
  const bool edge = word_base < 0 || 32 * (word_base + 32) > g.W || row_base < g.lo ||
                    row_base + tile_rows - 1 > g.hi;

  uint32_t w[R];
  const bool col_ok = gw >= 0 && gw < g.nwords;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int gr = r0 + i;
    w[i] = (col_ok && gr >= g.lo && gr <= g.hi) ? in[static_cast<long long>(gr) * g.pw_in + gw] : 0u;
  }
  if (edge) strips_substitute<R>(w, g, lane, warp, row_base, word_base, tile_rows, edge_rows);

  for (int gen = 1; gen <= g.tb; ++gen) {
    uint32_t* slot = xchg + (gen & 1) * nwarps * 64;
    slot[warp * 64 + lane] = w[0];
    slot[warp * 64 + 32 + lane] = w[R - 1];
    __syncthreads();
    const uint32_t above = warp > 0 ? slot[(warp - 1) * 64 + 32 + lane] : 0u;
    const uint32_t below = warp < nwarps - 1 ? slot[(warp + 1) * 64 + lane] : 0u;

    uint32_t pa0, pa1, ca0, ca1, cy0, cy1, t0, t1;  // rolling window: row i-1 (x), row i (x, y)
    {
      const uint32_t l = __shfl_up_sync(0xffffffffu, above, 1), r = __shfl_down_sync(0xffffffffu, above, 1);
      row_sums(l, above, r, pa0, pa1, t0, t1);
    }
    {
      const uint32_t c = w[0];
      const uint32_t l = __shfl_up_sync(0xffffffffu, c, 1), r = __shfl_down_sync(0xffffffffu, c, 1);
      row_sums(l, c, r, ca0, ca1, cy0, cy1);
    }
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const uint32_t c = i + 1 < R ? w[i + 1] : below;
      const uint32_t l = __shfl_up_sync(0xffffffffu, c, 1), r = __shfl_down_sync(0xffffffffu, c, 1);
      uint32_t na0, na1, ny0, ny1;
      row_sums(l, c, r, na0, na1, ny0, ny1);
      w[i] = next_state(pa0, pa1, cy0, cy1, na0, na1, w[i]);
      pa0 = ca0; pa1 = ca1;
      ca0 = na0; ca1 = na1; cy0 = ny0; cy1 = ny1;
    }
    if (edge && gen < g.tb) strips_substitute<R>(w, g, lane, warp, row_base, word_base, tile_rows, edge_rows);
  }

  // ---- store the tile's output rows / lanes
  if (lane < g.hw || lane >= 32 - g.hw || gw >= g.nwords) return;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    const int t = warp * R + i;
    const int gr = r0 + i;
    if (t >= g.tb && t < g.tb + g.th && gr < g.H) out[static_cast<long long>(gr) * g.pw_out + gw] = w[i];
  }
}

// T grid rows [row0, row0 + rows) -> packed rows [0, rows): one ballot per
// 32 cells; a warp packs 32 consecutive words of a row (128-B loads, 8 in
// flight) and stores them as one 128-B row segment.
template <typename T>
__global__ void __launch_bounds__(256)
    k_gol_pack(const T* __restrict__ in, long long pitch_in, int row0, int rows, int W,
               uint32_t* __restrict__ out, long long pw) {
  const int lane = threadIdx.x & 31;
  const int nwords = (W + 31) / 32;
  const int segs = (nwords + 31) / 32;  // 32-word segments per row
  const long long nwarp_total = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long item = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       item < static_cast<long long>(rows) * segs; item += nwarp_total) {
    const int r = static_cast<int>(item / segs);
    const int sg = static_cast<int>(item - static_cast<long long>(r) * segs);
    const T* grow = in + static_cast<long long>(row0 + r) * pitch_in + 32 * 32 * sg + lane;
    const bool full = 32 * 32 * (sg + 1) <= W;
    uint32_t mine = 0u;
#pragma unroll
    for (int u0 = 0; u0 < 32; u0 += 8) {
      T v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int col = 32 * 32 * sg + 32 * (u0 + u) + lane;
        v[u] = (full || col < W) ? grow[32 * (u0 + u)] : T(0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t b = __ballot_sync(0xffffffffu, v[u] != T(0));
        mine = lane == u0 + u ? b : mine;
      }
    }
    const int wd = 32 * sg + lane;
    if (wd < nwords) out[static_cast<long long>(r) * pw + wd] = mine;
  }
}

// packed rows [0, rows) -> T rows: lane = 4 cells (one int4/float4 store),
// 8 lanes per word, a warp writes 4 words = 128 cells per store instruction.
template <typename T>
__global__ void __launch_bounds__(256)
    k_gol_unpack(const uint32_t* __restrict__ in, long long pw, int rows, int W,
                 T* __restrict__ out, long long pitch_out, int vec_store) {
  using V = typename Vec4<T>::type;
  const int lane = threadIdx.x & 31;
  const int nwords = (W + 31) / 32;
  const int groups = (nwords + 3) / 4;  // 4-word groups per row
  const int nib = (lane & 7) * 4;
  const long long nwarp_total = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long item = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       item < static_cast<long long>(rows) * groups; item += nwarp_total) {
    const int r = static_cast<int>(item / groups);
    const int gq = static_cast<int>(item - static_cast<long long>(r) * groups);
    const int wd = 4 * gq + (lane >> 3);
    if (wd >= nwords) continue;
    const uint32_t bits = in[static_cast<long long>(r) * pw + wd] >> nib;
    const int col = 32 * wd + nib;
    T* o = out + static_cast<long long>(r) * pitch_out + col;
    if (vec_store && col + 3 < W) {
      V v;
      v.x = T(bits & 1u);
      v.y = T((bits >> 1) & 1u);
      v.z = T((bits >> 2) & 1u);
      v.w = T((bits >> 3) & 1u);
      *reinterpret_cast<V*>(o) = v;
    } else {
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (col + b < W) o[b] = T((bits >> b) & 1u);
      }
    }
  }
}

}  // namespace sk
