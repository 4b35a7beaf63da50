// B200 stencil executor kernels (sm_100a).
//
// K1a  k_stencil_tma      persistent, TMA-pipelined: one elected thread
//                         streams (tile + border region) boxes into an
//                         S-stage shared-memory ring with
//                         cp.async.bulk.tensor.2d + mbarrier complete_tx;
//                         out-of-bounds box elements arrive zero-filled, which
//                         is exactly SK_BORDER_PAD with pad 0; other modes
//                         patch the out-of-range cells of edge tiles in shared
//                         memory (clamp or pad) before compute.
// K1b  k_stencil_explicit one tile per block, coalesced loads of the tile with
//                         the border substitution applied at load time.
//
// Both keep the SkelCL execution model: a (wc x wr)
// workgroup of work-items, one per output cell, computing from a tile of
// (wc + E + W) x (wr + N + S) elements staged in shared memory.  The block
// shape is a launch parameter, not a template parameter.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "ops.cuh"
#include "vector.cuh"

namespace sk {

// Peer-memory halo exchange fused into the one-pass kernel (PEER
// instantiations only; zero otherwise).  The first and last tile-rows are
// processed first: their TMA loads wait for the neighbours' arrival flags,
// their first `north_rows` / last `south_rows` output rows are also stored
// into the neighbours' halo rows, and the last of them publishes
// `signal_value`.
struct PeerTile {
  const long long* flag_n;   // this rank's arrival flags (null: no neighbour)
  const long long* flag_s;
  long long wait_value;
  void* peer_n;              // neighbours' dst buffers (base = their halo row 0)
  void* peer_s;
  long long north_off, south_off;  // elements
  int north_rows, south_rows;
  long long* pflag_n;        // neighbours' flags this rank publishes to
  long long* pflag_s;
  unsigned* done;            // boundary-tile ticket counter
  long long signal_value;
  int boundary_tiles;
};

// Launch geometry, computed on the host (launch.cu) for one (desc, W, H, wc, wr).
struct Geom {
  int W, H;                 // computed region (columns, rows)
  long long pitch_in;       // elements
  long long pitch_out;      // elements
  int above, below;         // readable input rows beyond [0, H) (row-shard halos)
  int N, S, E, Wb;          // border region (Wb = west)
  int wc, wr;               // workgroup (block) shape, threads
  int K;                    // cells per work-item (consecutive rows of one column)
  int V;                    // columns per work-item (1, or 16 B / sizeof(T) on SK_LOAD_VECTOR)
  int tile_cols;            // output columns per tile = wc * V
  int tile_rows;            // output rows per tile = wr * K
  int ex_lo, ex_hi;         // tiles with ex_lo <= tx <= ex_hi and
  int ey_lo, ey_hi;         //   ey_lo <= ty <= ey_hi need no border work
  int lw;                   // logical tile width  = wc + E + Wb
  int tile_w;               // smem row pitch = TMA box width (16-B multiple)
  int vec;                  // elements per 16 B (TMA: box x start must be 16-B aligned)
  int tile_h;               // tile rows = tile_rows + N + S
  int tiles_x, tiles_y;
  int mode;                 // sk_border_mode
  int pad_is_zero;          // PAD mode with an all-zero pad value
  int stage_bytes;          // bytes per pipeline stage (128-aligned)
  int stages;               // TMA ring depth
  int box_h, nchunks;       // TMA box height and boxes per tile
  // temporal blocking (fused.cuh): TB generations per launch.  When TB > 1
  // the N/S/E/Wb above are the TB-scaled halo of the loaded box and
  // bN/bS/bE/bW the stencil's own border region.
  int TB;
  int bN, bS, bE, bW;
  int sp;                   // row pitch of the two scratch generation buffers
  int scratch_elems;        // elements per scratch buffer (incl. K slack rows)
  PeerTile peer;            // fused peer exchange (PEER kernels only)
  int lag;                  // ring refill lag (0: 2 for >= 3 stages, else 1)
};

// ------------------------------------------------------------------ PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "SK_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra SK_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ----------------------------------------------------------------- tile view
template <typename T>
struct TileView {
  const T* centre;  // the work-item's own cell in the staged tile
  int pitch;
  __device__ __forceinline__ T at(int dr, int dc) const { return centre[dr * pitch + dc]; }
};

template <typename T>
__device__ __forceinline__ T pad_value(const T pad) { return pad; }

__device__ __forceinline__ int clampi(int v, int lo, int hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

// Column offset of the tile's first logical cell inside its 16-B aligned
// TMA box: the box starts at align_down(c0 - W, vec) (the TMA unit faults on
// an unaligned innermost start coordinate).
__device__ __forceinline__ int tile_offset(const Geom& g, int c0) {
  return (c0 - g.Wb) & (g.vec - 1);
}

// True when a tile reaches outside the readable input or the matrix (needs
// border substitution and bounds-checked stores); bounds precomputed on the host.
__device__ __forceinline__ bool tile_is_edge(const Geom& g, int tx, int ty) {
  return tx < g.ex_lo || tx > g.ex_hi || ty < g.ey_lo || ty > g.ey_hi;
}

// Patch the out-of-range cells of an edge tile in shared memory: pad value,
// or a copy of the nearest in-range cell (which always lies inside the same
// tile).  Only out-of-range cells are written and only
// in-range cells are read, so one pass is race-free.
template <typename T>
__device__ __forceinline__ void fixup_tile(T* tile, const Geom& g, int r0, int c0, T pad,
                                           int tid, int nthreads) {
  // `tile` points at the first logical column (box start + tile_offset).
  // The in-range cells form one rectangle [tr_lo, tr_hi] x [tc_lo, tc_hi] of
  // the tile; only the cells around it are visited: the west / east strips
  // of the in-range rows, then the out-of-range rows in full.
  const int row_lo = -g.above, row_hi = g.H - 1 + g.below;
  const int gr0 = r0 - g.N, gc0 = c0 - g.Wb;  // global coords of tile cell (0, 0)
  const int tr_lo = max(0, row_lo - gr0), tr_hi = min(g.tile_h - 1, row_hi - gr0);
  const int tc_lo = max(0, -gc0), tc_hi = min(g.lw - 1, g.W - 1 - gc0);
  const int in_rows = max(0, tr_hi - tr_lo + 1);
  const int west = tc_lo, side = west + (g.lw - 1 - tc_hi);
  const int n_side = in_rows * side;
  const int n_rows = (g.tile_h - in_rows) * g.lw;
  auto patch = [&](int tr, int tc) {
    T v = pad;
    if (g.mode != 0) {
      const int cr = clampi(tr, tr_lo, tr_hi);
      const int cc = clampi(tc, tc_lo, tc_hi);
      v = tile[cr * g.tile_w + cc];
    }
    tile[tr * g.tile_w + tc] = v;
  };
  for (int i = tid; i < n_side; i += nthreads) {
    const int q = i / side;
    const int k = i - q * side;
    patch(tr_lo + q, k < west ? k : tc_hi + 1 + (k - west));
  }
  for (int i = tid; i < n_rows; i += nthreads) {
    const int q = i / g.lw;
    const int tc = i - q * g.lw;
    patch(q < tr_lo ? q : in_rows + q, tc);
  }
}

// ------------------------------------------------------- compute + store
// Work-item (threadIdx.x, threadIdx.y) owns column c0 + threadIdx.x, rows
// r0 + threadIdx.y*K ... + K-1 of the tile.  The K evaluations are unrolled
// so the compiler shares the overlapping shared-memory loads between them.
template <class Op, typename T, int K>
__device__ __forceinline__ void compute_tile(const T* tile, const Geom& g,
                                             const OpParams<T>& p, T (&res)[K]) {
  const Op op;
  const T* base = tile + (threadIdx.y * K + g.N) * g.tile_w + threadIdx.x + g.Wb;
  if constexpr (has_column<Op>::value) {
    op.template column<T, K>(base, g.tile_w, p, res);
  } else {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      TileView<T> view{base + j * g.tile_w, g.tile_w};
      res[j] = op.template apply<T>(view, p);
    }
  }
}

// Fused peer exchange: boundary tile-rows first (row order 0, last, 1, 2, ...).
__device__ __forceinline__ int peer_tile_row(const Geom& g, int ty) {
  if (g.tiles_y < 2) return ty;
  return ty == 0 ? 0 : (ty == 1 ? g.tiles_y - 1 : ty - 1);
}

__device__ __forceinline__ bool peer_boundary_row(const Geom& g, int tyr) {
  return tyr == 0 || tyr == g.tiles_y - 1;
}

__device__ __forceinline__ long long ld_acquire_sys_s64(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Producer side: a boundary tile's box includes halo rows, so its TMA load
// waits for the neighbour's flag; the acquire is then ordered before the
// async-proxy (TMA) reads of those rows.
__device__ __forceinline__ void peer_wait_rows(const Geom& g, int tyr) {
  bool waited = false;
  if (tyr == 0 && g.peer.flag_n) {
    while (ld_acquire_sys_s64(g.peer.flag_n) < g.peer.wait_value) __nanosleep(32);
    waited = true;
  }
  if (tyr == g.tiles_y - 1 && g.peer.flag_s) {
    while (ld_acquire_sys_s64(g.peer.flag_s) < g.peer.wait_value) __nanosleep(32);
    waited = true;
  }
  if (waited) asm volatile("fence.proxy.async.global;" ::: "memory");
}

// Consumer side, after a boundary tile's stores: the threads that stored
// into a neighbour's halo make those stores visible system-wide, then the
// last boundary tile of the grid publishes the generation to the neighbours.
// Nothing to publish (no neighbours): no fence, no barrier.
__device__ __forceinline__ void peer_tile_done(const Geom& g, int tid, bool stored_peer) {
  if (!g.peer.pflag_n && !g.peer.pflag_s) return;
  if (stored_peer) __threadfence_system();
  __syncthreads();
  if (tid == 0 && atomicAdd(g.peer.done, 1u) == static_cast<unsigned>(g.peer.boundary_tiles) - 1u) {
    __threadfence_system();
    if (g.peer.pflag_n) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(g.peer.pflag_n), "l"(g.peer.signal_value) : "memory");
    if (g.peer.pflag_s) asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(g.peer.pflag_s), "l"(g.peer.signal_value) : "memory");
    atomicExch(g.peer.done, 0u);
  }
}

// Returns whether this thread stored into a neighbour's halo.
template <typename T, int K>
__device__ __forceinline__ bool store_peer_rows(const Geom& g, int r0, int c0, const T (&res)[K]) {
  const int c = c0 + threadIdx.x;
  const int r = r0 + threadIdx.y * K;
  if (c >= g.W) return false;
  T* pn = static_cast<T*>(g.peer.peer_n);
  T* ps = static_cast<T*>(g.peer.peer_s);
  bool stored = false;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int rr = r + j;
    if (rr >= g.H) break;
    if (pn && rr < g.peer.north_rows) {
      pn[g.peer.north_off + static_cast<long long>(rr) * g.pitch_out + c] = res[j];
      stored = true;
    }
    if (ps && rr >= g.H - g.peer.south_rows) {
      ps[g.peer.south_off + static_cast<long long>(rr - (g.H - g.peer.south_rows)) * g.pitch_out + c] = res[j];
      stored = true;
    }
  }
  return stored;
}

template <typename T, int K>
__device__ __forceinline__ void store_tile(T* __restrict__ out, const Geom& g, int r0, int c0,
                                           bool edge, const T (&res)[K]) {
  const int c = c0 + threadIdx.x;
  const int r = r0 + threadIdx.y * K;
  T* dst = out + static_cast<long long>(r) * g.pitch_out + c;
  if (!edge) {
#pragma unroll
    for (int j = 0; j < K; ++j) dst[j * g.pitch_out] = res[j];
  } else if (c < g.W) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (r + j < g.H) dst[j * g.pitch_out] = res[j];
    }
  }
}

// --------------------------------------------------------------------- K1a
template <typename T, bool PEER = false>
__device__ __forceinline__ void tma_issue_tile(const CUtensorMap* map, T* stage, uint64_t* bar,
                                               const Geom& g, int t) {
  int ty = t / g.tiles_x;
  int tx = t - ty * g.tiles_x;
  if constexpr (PEER) {
    ty = peer_tile_row(g, ty);
    peer_wait_rows(g, ty);
  }
  int x = tx * g.tile_cols - g.Wb;
  x -= x & (g.vec - 1);                      // 16-B aligned innermost start
  int y = ty * g.tile_rows - g.N + g.above;  // tensor rows start `above` rows before row 0
  mbar_arrive_expect_tx(bar, static_cast<uint32_t>(g.nchunks * g.box_h * g.tile_w * sizeof(T)));
  for (int k = 0; k < g.nchunks; ++k) {
    tma_load_2d(stage + k * g.box_h * g.tile_w, map, bar, x, y + k * g.box_h);
  }
}

// V > 1: vector work-items (vector.cuh), V columns x K rows each.
template <typename T, int K, int V>
__device__ __forceinline__ void store_row_vec(T* __restrict__ out, const Geom& g, int r, int c, bool edge,
                                              const T (&v)[V]) {
  T* dst = out + static_cast<long long>(r) * g.pitch_out + c;
  if (!edge) {
    Vec<T, V> x;
#pragma unroll
    for (int j = 0; j < V; ++j) x.v[j] = v[j];
    *reinterpret_cast<Vec<T, V>*>(dst) = x;
  } else if (r < g.H) {
#pragma unroll
    for (int j = 0; j < V; ++j) {
      if (c + j < g.W) dst[j] = v[j];
    }
  }
}

// The persistent TMA pass, shared by the kernels below (they differ only in
// their register bound).
template <class Op, typename T, int K, bool PEER, int V>
__device__ __forceinline__ void tma_pass(const CUtensorMap& map, T* __restrict__ out, const Geom& g,
                                         const T pad, const OpParams<T>& p) {
  // Shared memory: [stages x stage_bytes tiles][full[stages]][empty[stages]].
  // full[s]  : 1 arrival (producer's expect_tx) + the TMA transaction bytes.
  // empty[s] : one arrival per warp once it has read the tile in stage s.
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + g.stages * g.stage_bytes);
  uint64_t* empty = full + g.stages;
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nthreads = blockDim.x * blockDim.y;
  const int nwarps = (nthreads + 31) >> 5;
  const int ntiles = g.tiles_x * g.tiles_y;
  const bool fix_edges = !(g.mode == 0 && g.pad_is_zero);
  // Refill lag: the stage read `lag` iterations ago is refilled, so the
  // producer rarely waits for slow warps (lag 1 for shallow rings).
  const int lag = g.lag > 0 ? g.lag : g.stages >= 3 ? 2 : 1;
  const int lane = tid & 31;
  const int warp_lanes = min(32, nthreads - (tid & ~31));
  const unsigned warp_mask = warp_lanes == 32 ? 0xffffffffu : ((1u << warp_lanes) - 1u);

  if (tid == 0) {
    prefetch_tensormap(&map);
    for (int s = 0; s < g.stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps);
    }
    fence_barrier_init();
    fence_proxy_async_smem();
    // Programmatic dependent launch (launch.cu: launch_tma): everything above
    // touches only shared memory and the tensor map, so it overlaps the tail
    // of the previous generation's kernel; no global read or write happens
    // before that kernel has completed and its stores are visible.  Then let
    // the next generation's CTAs be scheduled onto SMs as ours retire.
    // (Without a programmatic dependency both instructions are no-ops.)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int s = 0; s < g.stages; ++s) {
      int t = blockIdx.x + s * gridDim.x;
      if (t < ntiles) {
        tma_issue_tile<T, PEER>(&map, reinterpret_cast<T*>(smem + s * g.stage_bytes), &full[s], g, t);
      }
    }
  }
  __syncthreads();

  // Tile coordinates advance by gridDim.x tiles per iteration; kept
  // incrementally (no per-tile integer division on the hot path).
  const int step_y = gridDim.x / g.tiles_x;
  const int step_x = gridDim.x - step_y * g.tiles_x;
  int ty = blockIdx.x / g.tiles_x;
  int tx = blockIdx.x - ty * g.tiles_x;
  int s = 0;
  uint32_t phase = 0;
  int ps = 0;  // producer (thread 0): stage / phase of iteration it - lag
  uint32_t pphase = 0;
  int it = 0;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    if (tid == 0 && it >= lag) {
      // refill the stage read at iteration it-lag with tile (it-lag)+stages
      int tn = t + (g.stages - lag) * gridDim.x;
      if (tn < ntiles) {
        mbar_wait_parity(&empty[ps], pphase);
        tma_issue_tile<T, PEER>(&map, reinterpret_cast<T*>(smem + ps * g.stage_bytes), &full[ps], g,
                          tn);
      }
      if (++ps == g.stages) {
        ps = 0;
        pphase ^= 1u;
      }
    }
    const int tyr = PEER ? peer_tile_row(g, ty) : ty;  // boundary tile-rows first (PEER)
    const int r0 = tyr * g.tile_rows;
    const int c0 = tx * g.tile_cols;
    const bool edge = tile_is_edge(g, tx, tyr);
    T* tile = reinterpret_cast<T*>(smem + s * g.stage_bytes) + tile_offset(g, c0);

    mbar_wait_parity(&full[s], phase);
    if (fix_edges && edge) {
      __syncthreads();  // every warp is at this tile (uniform condition)
      fixup_tile(tile, g, r0, c0, pad, tid, nthreads);
      fence_proxy_async_smem();  // generic writes before the next async refill
      __syncthreads();
    }
    if constexpr (V > 1) {
      // stream the work-item's rows; each output row leaves as one vector
      const T* first = tile + (threadIdx.y * K + g.N) * g.tile_w + threadIdx.x * V + g.Wb;
      const int r = r0 + threadIdx.y * K;
      const int c = c0 + threadIdx.x * V;
      if (!edge) {
        // interior tile: one address per work-item, no bounds test per row
        T* dst = out + static_cast<long long>(r) * g.pitch_out + c;
        vector_tile<Op, T, K, V>(first, g.tile_w, p, [&](int k, const T (&v)[V]) {
          Vec<T, V> x;
#pragma unroll
          for (int j = 0; j < V; ++j) x.v[j] = v[j];
          *reinterpret_cast<Vec<T, V>*>(dst + static_cast<long long>(k) * g.pitch_out) = x;
        });
      } else {
        vector_tile<Op, T, K, V>(first, g.tile_w, p, [&](int k, const T (&v)[V]) {
          store_row_vec<T, K, V>(out, g, r + k, c, true, v);
        });
      }
    } else {
      T res[K];
      compute_tile<Op, T, K>(tile, g, p, res);
      store_tile<T, K>(out, g, r0, c0, edge, res);
      if constexpr (PEER) {
        if (peer_boundary_row(g, tyr)) {
          const bool stored = store_peer_rows<T, K>(g, r0, c0, res);
          peer_tile_done(g, tid, stored);
        }
      }
    }
    // Release the stage only after the stores: they consume every value the
    // warp loaded from it, so no shared-memory read of this tile can still be
    // in flight when the producer's TMA refill overwrites the stage.  (An
    // arrive issued right after the loads raced the refill: ~17% of runs on
    // heat 2048^2 at 2x32, K=2, 2-stage ring - scripts/stress_race.py.)
    __syncwarp(warp_mask);
    if (lane == 0) mbar_arrive(&empty[s]);

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

template <class Op, typename T, int K, int MAXT, bool PEER = false, int V = 1>
__global__ void __launch_bounds__(MAXT)
    k_stencil_tma(const __grid_constant__ CUtensorMap map, T* __restrict__ out, const Geom g,
                  const T pad, const __grid_constant__ OpParams<T> p) {
  tma_pass<Op, T, K, PEER, V>(map, out, g, pad, p);
}

// Vector work-items with K = 8 rows: AUTO gives them blocks of wr <= 8 rows
// and wc <= 63 columns (one TMA box), so at most 504 threads.  1024 threads'
// 64 registers spill them; 512 threads' bound lets ptxas take 96-115 and
// costs resident blocks.  80 registers: no spills, and five 128-thread
// blocks still fit an SM (launchable up to 768 threads).
template <class Op, typename T, int K, int V>
__global__ void __maxnreg__(80)
    k_stencil_tma_r80(const __grid_constant__ CUtensorMap map, T* __restrict__ out, const Geom g,
                      const T pad, const __grid_constant__ OpParams<T> p) {
  tma_pass<Op, T, K, false, V>(map, out, g, pad, p);
}

// --------------------------------------------------------------------- K1b
template <class Op, typename T, int K, int MAXT>
__global__ void __launch_bounds__(MAXT)
    k_stencil_explicit(const T* __restrict__ in, T* __restrict__ out, const Geom g, const T pad,
                       const __grid_constant__ OpParams<T> p) {
  extern __shared__ __align__(128) unsigned char smem[];
  T* tile = reinterpret_cast<T*>(smem);
  const int tid = threadIdx.y * blockDim.x + threadIdx.x;
  const int nthreads = blockDim.x * blockDim.y;
  const int by = blockIdx.x / g.tiles_x;  // 1-D grid of tiles (no 65535 limit)
  const int bx = blockIdx.x - by * g.tiles_x;
  const int r0 = by * g.tile_rows;
  const int c0 = bx * g.tile_cols;
  const int row_lo = -g.above, row_hi = g.H - 1 + g.below;
  const int total = g.tile_h * g.lw;
  const bool edge = tile_is_edge(g, bx, by);

  if (!edge) {
    for (int i = tid; i < total; i += nthreads) {
      int tr = i / g.lw;
      int tc = i - tr * g.lw;
      tile[tr * g.tile_w + tc] =
          in[static_cast<long long>(r0 - g.N + tr) * g.pitch_in + (c0 - g.Wb + tc)];
    }
  } else {
    for (int i = tid; i < total; i += nthreads) {
      int tr = i / g.lw;
      int tc = i - tr * g.lw;
      int gr = r0 - g.N + tr;
      int gc = c0 - g.Wb + tc;
      T v;
      if (gr >= row_lo && gr <= row_hi && gc >= 0 && gc < g.W) {
        v = in[static_cast<long long>(gr) * g.pitch_in + gc];
      } else if (g.mode == 0) {
        v = pad;
      } else {
        v = in[static_cast<long long>(clampi(gr, row_lo, row_hi)) * g.pitch_in +
               clampi(gc, 0, g.W - 1)];
      }
      tile[tr * g.tile_w + tc] = v;
    }
  }
  __syncthreads();
  T res[K];
  compute_tile<Op, T, K>(tile, g, p, res);
  store_tile<T, K>(out, g, r0, c0, edge, res);
}

}  // namespace sk
