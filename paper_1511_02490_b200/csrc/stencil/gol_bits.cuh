// K1g  k_gol_bits — Game of Life, bit-sliced and temporally blocked:
// TB generations per launch, one HBM read and one HBM write per cell.
//
// The customising function (B3/S23 on the 3x3 Moore
// neighbourhood, a cell is alive iff != 0) depends on its neighbourhood only
// through alive/dead, so a tile can be held as one bit per cell: word j of
// a buffer row holds the 32 cells of columns 32*gw .. 32*gw+31 (bit b =
// column 32*gw + b).  One 32-bit logic op then evaluates 32 cells.
//
//   load      each warp reads 32 consecutive cells of a row (one coalesced
//             128-B request) and __ballot_sync(v != 0) turns them into a word;
//   TB gens   ping-pong between two shared-memory bit planes; a thread
//             evaluates KS rows x 32 cells per item with a bit-sliced adder
//             (below); the tile shrinks its valid margin by one row/column
//             per generation, so it is loaded with TB halo rows and
//             ceil(TB/32) halo words on each side;
//   store     each lane expands 4 bits of a word into an int4/float4 store.
//
// Border semantics are the executor's (DESIGN.md §2/§4.2): after the load
// and after every intermediate generation, the cells of an edge tile outside
// the readable window are re-substituted - pad value, or the nearest
// in-window cell of that generation - exactly what the one-pass executor
// would read at the next launch, so the result is bit-identical to TB
// single passes (tests/test_stencil_parity.py::test_gol_bits_*).
//
// Neighbour count, bit-sliced.  Per buffer row r, with W/C/E the row shifted
// west/centre/east (funnel shifts across word boundaries), the horizontal
// 3-sum is the 2-bit number (s1 s0) = (maj(W,C,E), W^C^E).  The 9-cell sum
// (centre included) of rows a, b, c is then
//     l0 = a0^b0^c0, l1 = maj(a0,b0,c0), h0 = a1^b1^c1, h1 = maj(a1,b1,c1)
//     m0 = l1^h0,    m1 = l1&h0,        total = l0 + 2 m0 + 4 (m1 + h1)
// and the next state is total == 3 | (alive & total == 4):
//     next = (l0 & m0 & ~m1 & ~h1) | (alive & ~l0 & ~m0 & (m1 ^ h1)).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace sk {

struct BitGeom {
  long long pitch_in, pitch_out;  // elements
  int W, H;                       // computed region
  int lo, hi;                     // readable rows [lo, hi] (halo rows of a shard)
  int nwords;                     // ceil(W / 32)
  int tw, th;                     // output words / rows per tile
  int tb, hw;                     // generations this launch; halo words per side
  int bw, bh;                     // buffer words / rows: tw + 2 hw, th + 2 tb
  int bp;                         // buffer row pitch in words (bw + 2 zero columns)
  int plane;                      // words per bit plane (bp * (bh + slack))
  int tiles_x, tiles_y;
  int mode;                       // sk_border_mode
  uint32_t padword;               // 0 or ~0 (pad value alive?)
  int vec_store;                  // out base 16-B aligned and pitch_out % 4 == 0
};

constexpr int kBitsKS = 4;        // rows per work item in a generation
constexpr int kBitsLoadU = 8;     // words in flight per warp while loading

__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) {
  return (a & b) | (c & (a | b));
}

// One generation over buffer rows [ra, rb) and words [ja, jb): src -> dst.
// Row r's word j lives at plane[r * bp + 1 + j]; columns 0 and bp-1 are zero.
__device__ __forceinline__ void bits_generation(const uint32_t* __restrict__ src,
                                                uint32_t* __restrict__ dst, const BitGeom& g,
                                                int ra, int rb, int ja, int jb, int tid,
                                                int nthreads) {
  const int nj = jb - ja;
  const int items = ((rb - ra + kBitsKS - 1) / kBitsKS) * nj;
  if (tid >= items) return;
  // item = strip * nj + j, advanced incrementally (no division per item)
  int s = tid / nj;
  int j = tid - s * nj;
  const int ds = nthreads / nj;
  const int dj = nthreads - ds * nj;
  for (int item = tid; item < items; item += nthreads) {
    const int r0 = ra + s * kBitsKS;
    const uint32_t* p = src + (r0 - 1) * g.bp + 1 + ja + j;
    uint32_t x0[kBitsKS + 2], x1[kBitsKS + 2], alive[kBitsKS + 2];
#pragma unroll
    for (int q = 0; q < kBitsKS + 2; ++q) {
      const uint32_t l = p[q * g.bp - 1], c = p[q * g.bp], r = p[q * g.bp + 1];
      const uint32_t w = __funnelshift_l(l, c, 1);  // west neighbour of every bit
      const uint32_t e = __funnelshift_r(c, r, 1);  // east neighbour
      x0[q] = w ^ c ^ e;
      x1[q] = maj3(w, c, e);
      alive[q] = c;
    }
    uint32_t* o = dst + r0 * g.bp + 1 + ja + j;
#pragma unroll
    for (int k = 0; k < kBitsKS; ++k) {
      const uint32_t l0 = x0[k] ^ x0[k + 1] ^ x0[k + 2];
      const uint32_t l1 = maj3(x0[k], x0[k + 1], x0[k + 2]);
      const uint32_t h0 = x1[k] ^ x1[k + 1] ^ x1[k + 2];
      const uint32_t h1 = maj3(x1[k], x1[k + 1], x1[k + 2]);
      const uint32_t m0 = l1 ^ h0, m1 = l1 & h0;
      o[k * g.bp] = (l0 & m0 & ~(m1 | h1)) | (alive[k + 1] & ~(l0 | m0) & (m1 ^ h1));
    }
    j += dj;
    s += ds;
    if (j >= nj) {
      j -= nj;
      ++s;
    }
  }
}

// Border substitution of an edge tile's plane (per bit):
// (a) in-window rows: words west of column 0 take column 0 (nearest) or the
//     pad; bits at or east of column W take column W-1 or the pad;
// (b) rows outside [lo, hi] copy row lo / hi (nearest) or are all pad.
// Only out-of-range bits are written and only in-range bits are read.
static __device__ __forceinline__ void bits_substitute(uint32_t* plane, const BitGeom& g, int row_base, int word_base,
                                int tid, int nthreads) {
  const int i_lo = max(0, g.lo - row_base);
  const int i_hi = min(g.bh - 1, g.hi - row_base);
  const int jw = min(g.bw, max(0, -word_base));                        // words west of col 0
  const int gw_e = (g.W & 31) ? g.nwords - 1 : g.nwords;               // first word with bits >= W
  const int je = min(g.bw, max(0, gw_e - word_base));                  // words [je, bw) need east fix
  const int nfix = jw + (g.bw - je);
  if (nfix > 0 && i_hi >= i_lo) {
    const int j0 = -word_base;                   // word of column 0
    const int jl = g.nwords - 1 - word_base;     // word of column W-1
    const int bl = (g.W - 1) & 31;
    const int total = (i_hi - i_lo + 1) * nfix;
    for (int idx = tid; idx < total; idx += nthreads) {
      const int i = i_lo + idx / nfix;
      const int f = idx % nfix;
      const int j = f < jw ? f : je + (f - jw);
      uint32_t* row = plane + i * g.bp + 1;
      const int gw = word_base + j;
      if (gw < 0) {
        row[j] = g.mode == 0 ? g.padword : (0u - (row[j0] & 1u));
      } else {
        const int nvalid = g.W - 32 * gw;  // < 32 here
        const uint32_t m = nvalid <= 0 ? 0u : ((1u << nvalid) - 1u);
        const uint32_t fill = g.mode == 0 ? g.padword : (0u - ((row[jl] >> bl) & 1u));
        row[j] = (row[j] & m) | (fill & ~m);
      }
    }
    __syncthreads();
  }
  const int above = i_lo;                 // rows [0, i_lo) are north of the window
  const int below = g.bh - 1 - i_hi;      // rows (i_hi, bh) are south of it
  if (above > 0 || below > 0) {
    const int total = (above + below) * g.bw;
    for (int idx = tid; idx < total; idx += nthreads) {
      const int k = idx / g.bw;
      const int j = idx - k * g.bw;
      const int i = k < above ? k : i_hi + 1 + (k - above);
      const int from = k < above ? i_lo : i_hi;
      plane[i * g.bp + 1 + j] = g.mode == 0 ? g.padword : plane[from * g.bp + 1 + j];
    }
    __syncthreads();
  }
}

template <typename T>
struct Vec4;
template <> struct Vec4<int32_t> { using type = int4; };
template <> struct Vec4<float> { using type = float4; };
template <> struct Vec4<double> { using type = double4; };

template <typename T>
__global__ void __launch_bounds__(1024)
    k_gol_bits(const T* __restrict__ in, T* __restrict__ out, const BitGeom g) {
  extern __shared__ __align__(16) uint32_t sm_bits[];
  uint32_t* A = sm_bits;
  uint32_t* B = sm_bits + g.plane;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nthreads = blockDim.x * blockDim.y;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nwarps = nthreads >> 5;  // whole warps: the host rounds wc*wr up to 32

  const int ty = blockIdx.x / g.tiles_x;
  const int tx = blockIdx.x - ty * g.tiles_x;
  const int row_base = ty * g.th - g.tb;   // global row of buffer row 0
  const int word_base = tx * g.tw - g.hw;  // global word of buffer word 0
  const bool edge = word_base < 0 || 32 * (word_base + g.bw) > g.W || row_base < g.lo ||
                    row_base + g.bh - 1 > g.hi;

  // zero both planes' guard columns and slack rows (never written below)
  const int rows_alloc = g.plane / g.bp;
  for (int r = tid; r < 2 * rows_alloc; r += nthreads) {
    uint32_t* row = sm_bits + r * g.bp;  // the planes are contiguous
    row[0] = 0u;
    row[g.bp - 1] = 0u;
  }
  for (int i = tid; i < (rows_alloc - g.bh) * g.bp; i += nthreads) {
    A[g.bh * g.bp + i] = 0u;
    B[g.bh * g.bp + i] = 0u;
  }

  // ---- load: one ballot per 32 cells, kBitsLoadU requests in flight per warp
  const int loadable_lo = max(0, g.lo - row_base), loadable_hi = min(g.bh - 1, g.hi - row_base);
  for (int i = warp; i < g.bh; i += nwarps) {
    uint32_t* prow = A + i * g.bp + 1;
    if (i < loadable_lo || i > loadable_hi) {  // outside the window: substituted below
      for (int j = lane; j < g.bw; j += 32) prow[j] = 0u;
      continue;
    }
    const T* grow = in + static_cast<long long>(row_base + i) * g.pitch_in;
    for (int j0 = 0; j0 < g.bw; j0 += kBitsLoadU) {
      T v[kBitsLoadU];
#pragma unroll
      for (int u = 0; u < kBitsLoadU; ++u) {
        const int col = 32 * (word_base + j0 + u) + lane;
        v[u] = (j0 + u < g.bw && col >= 0 && col < g.W) ? grow[col] : T(0);
      }
      uint32_t mine = 0u;  // lane u keeps word j0 + u
#pragma unroll
      for (int u = 0; u < kBitsLoadU; ++u) {
        const uint32_t bits = __ballot_sync(0xffffffffu, v[u] != T(0));
        if (lane == u) mine = bits;
      }
      if (lane < kBitsLoadU && j0 + lane < g.bw) prow[j0 + lane] = mine;
    }
  }
  __syncthreads();
  if (edge) bits_substitute(A, g, row_base, word_base, tid, nthreads);

  // ---- TB - 1 intermediate generations over the shrinking valid region
  uint32_t* src = A;
  uint32_t* dst = B;
  for (int gen = 1; gen < g.tb; ++gen) {
    bits_generation(src, dst, g, gen, g.bh - gen, 0, g.bw, tid, nthreads);
    __syncthreads();
    if (edge) bits_substitute(dst, g, row_base, word_base, tid, nthreads);
    uint32_t* t = src;
    src = dst;
    dst = t;
  }
  // ---- last generation: the output words only
  bits_generation(src, dst, g, g.tb, g.tb + g.th, g.hw, g.hw + g.tw, tid, nthreads);
  __syncthreads();

  // ---- store: lane = 4 cells of a word (8 lanes per word, 4 words per warp op)
  using V = typename Vec4<T>::type;
  const int r_end = min(g.th, g.H - ty * g.th);
  const int sub = lane >> 3;       // word within the warp's group of 4
  const int nib = (lane & 7) * 4;  // first bit of this lane
  const bool vec_ok = g.vec_store != 0;
  for (int i = warp; i < r_end; i += nwarps) {
    const uint32_t* prow = dst + (g.tb + i) * g.bp + 1 + g.hw;
    T* orow = out + static_cast<long long>(ty * g.th + i) * g.pitch_out;
    for (int j = sub; j < g.tw; j += 4) {
      const int gw = tx * g.tw + j;
      if (gw >= g.nwords) break;
      const uint32_t w = prow[j] >> nib;
      const int col = 32 * gw + nib;
      if (vec_ok && col + 3 < g.W) {
        V v;
        v.x = T(w & 1u);
        v.y = T((w >> 1) & 1u);
        v.z = T((w >> 2) & 1u);
        v.w = T((w >> 3) & 1u);
        *reinterpret_cast<V*>(orow + col) = v;
      } else {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if (col + b < g.W) orow[col + b] = T((w >> b) & 1u);
        }
      }
    }
  }
}

}  // namespace sk
