// K1t  k_stencil_tma_fused — temporal blocking: TB generations of an
// iterated stencil per launch.
//
// The producer streams the output tile plus a TB-deep border region
// (TB*N rows north, TB*S south, TB*W west, TB*E east) through the same TMA
// ring as K1a.  Generation g = 1 .. TB-1 is computed in shared memory over the
// tile grown by (TB-g) border regions into one of two scratch buffers; the
// final generation is computed into registers and stored.  HBM traffic per
// generation drops ~TB x at the price of recomputing the shrinking halo.
//
// Border semantics stay exact: after every intermediate generation, cells of
// an edge tile that lie outside the readable window are replaced by the pad
// value or by the nearest in-window cell OF THAT GENERATION - what the
// one-pass executor would read at the next launch.  (The clamp target lies
// inside the same region by the argument of DESIGN.md §4.2.)
#pragma once

#include "kernels.cuh"

namespace sk {

// K cells of one column: the op's column form or K single evaluations.
template <class Op, typename T, int K>
__device__ __forceinline__ void eval_column(const Op& op, const T* centre, int pitch,
                                            const OpParams<T>& p, T (&res)[K]) {
  if constexpr (has_column<Op>::value) {
    op.template column<T, K>(centre, pitch, p, res);
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) res[j] = op.template apply<T>(TileView<T>{centre + j * pitch, pitch}, p);
  }
}

// Out-of-window fix-up of one generation region held in `buf` (pitch bp):
// region cell (i, j) is global (gr0 + i, gc0 + j).
template <typename T>
__device__ __forceinline__ void fixup_region(T* buf, int bp, int rows, int cols, int gr0, int gc0,
                                             const Geom& g, T pad, int tid, int nthreads) {
  const int row_lo = -g.above, row_hi = g.H - 1 + g.below;
  for (int i = tid; i < rows * cols; i += nthreads) {
    const int r = i / cols;
    const int c = i - r * cols;
    const int gr = gr0 + r, gc = gc0 + c;
    if (gr >= row_lo && gr <= row_hi && gc >= 0 && gc < g.W) continue;
    T v;
    if (g.mode == 0) {
      v = pad;
    } else {
      const int cr = clampi(gr, row_lo, row_hi) - gr0;
      const int cc = clampi(gc, 0, g.W - 1) - gc0;
      v = buf[cr * bp + cc];
    }
    buf[r * bp + c] = v;
  }
}

template <class Op, typename T, int K, int TB, int MAXT>
__global__ void __launch_bounds__(MAXT)
    k_stencil_tma_fused(const __grid_constant__ CUtensorMap map, T* __restrict__ out, const Geom g,
                        const T pad, const __grid_constant__ OpParams<T> p) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* scratch0 = reinterpret_cast<T*>(smem + g.stages * g.stage_bytes);
  T* scratch1 = scratch0 + g.scratch_elems;
  uint64_t* full = reinterpret_cast<uint64_t*>(scratch1 + g.scratch_elems);
  uint64_t* empty = full + g.stages;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nthreads = blockDim.x * blockDim.y;
  const int nwarps = (nthreads + 31) >> 5;
  const int ntiles = g.tiles_x * g.tiles_y;
  const int lag = g.lag > 0 ? g.lag : g.stages >= 3 ? 2 : 1;
  const int lane = tid & 31;
  const int warp_lanes = min(32, nthreads - (tid & ~31));
  const unsigned warp_mask = warp_lanes == 32 ? 0xffffffffu : ((1u << warp_lanes) - 1u);
  const bool fix0 = !(g.mode == 0 && g.pad_is_zero);

  if (tid == 0) {
    prefetch_tensormap(&map);
    for (int s = 0; s < g.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
    for (int s = 0; s < g.stages; ++s) {
      int t = blockIdx.x + s * gridDim.x;
      if (t < ntiles) tma_issue_tile<T>(&map, reinterpret_cast<T*>(smem + s * g.stage_bytes), &full[s], g, t);
    }
  }
  __syncthreads();

  const int step_y = gridDim.x / g.tiles_x;
  const int step_x = gridDim.x - step_y * g.tiles_x;
  int ty = blockIdx.x / g.tiles_x;
  int tx = blockIdx.x - ty * g.tiles_x;
  int s = 0;
  uint32_t phase = 0;
  int ps = 0;
  uint32_t pphase = 0;
  const Op op;
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    if (tid == 0 && it >= lag) {
      int tn = t + (g.stages - lag) * gridDim.x;
      if (tn < ntiles) {
        mbar_wait_parity(&empty[ps], pphase);
        tma_issue_tile<T>(&map, reinterpret_cast<T*>(smem + ps * g.stage_bytes), &full[ps], g, tn);
      }
      if (++ps == g.stages) {
        ps = 0;
        pphase ^= 1u;
      }
    }
    const int r0 = ty * g.tile_rows;
    const int c0 = tx * g.wc;
    const bool edge = tile_is_edge(g, tx, ty);
    T* tile = reinterpret_cast<T*>(smem + s * g.stage_bytes) + tile_offset(g, c0);

    mbar_wait_parity(&full[s], phase);
    if (fix0 && edge) {
      __syncthreads();
      fixup_tile(tile, g, r0, c0, pad, tid, nthreads);
      fence_proxy_async_smem();
      __syncthreads();
    }

    // intermediate generations 1 .. TB-1 in shared memory
    const T* src = tile;
    int spitch = g.tile_w;
    T* dst = scratch0;
#pragma unroll
    for (int gen = 1; gen < TB; ++gen) {
      const int m = TB - gen;  // remaining margin in border regions
      const int rows = g.tile_rows + m * (g.bN + g.bS);
      const int cols = g.wc + m * (g.bW + g.bE);
      const int segs = cols * ((rows + K - 1) / K);
      for (int idx = tid; idx < segs; idx += nthreads) {
        const int i0 = (idx / cols) * K;
        const int j = idx - (i0 / K) * cols;
        T res[K];
        eval_column<Op, T, K>(op, src + (i0 + g.bN) * spitch + j + g.bW, spitch, p, res);
#pragma unroll
        for (int k = 0; k < K; ++k) dst[(i0 + k) * g.sp + j] = res[k];
      }
      __syncthreads();
      if (gen == 1) {  // the loaded tile is no longer read: release the stage
        __syncwarp(warp_mask);
        if (lane == 0) mbar_arrive(&empty[s]);
      }
      if (edge) {
        fixup_region(dst, g.sp, rows, cols, r0 - m * g.bN, c0 - m * g.bW, g, pad, tid, nthreads);
        __syncthreads();
      }
      src = dst;
      spitch = g.sp;
      dst = dst == scratch0 ? scratch1 : scratch0;
    }

    // final generation -> registers -> HBM
    T res[K];
    eval_column<Op, T, K>(op, src + (threadIdx.y * K + g.bN) * spitch + threadIdx.x + g.bW, spitch, p, res);
    store_tile<T, K>(out, g, r0, c0, edge, res);
    __syncthreads();  // scratch buffers are rewritten by the next tile

    tx += step_x;
    ty += step_y;
    if (tx >= g.tiles_x) {
      tx -= g.tiles_x;
      ++ty;
    }
    if (++s == g.stages) {
      s = 0;
      phase ^= 1u;
    }
  }
}

}  // namespace sk
