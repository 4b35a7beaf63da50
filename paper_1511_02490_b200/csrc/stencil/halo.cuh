// K3p  Peer-memory halo exchange fused into the boundary-strip pass of a
// row-sharded iterated stencil (SURVEY.md §8e "fused variant").
//
// The NCCL schedule (distributed.py: iterate_sharded_overlapped) computes the
// boundary strips, then ncclSend/ncclRecv's the new boundary rows, while the
// interior runs.  Here the strip pass itself delivers the rows: every cell of
// the rows a neighbour needs is stored twice, into the local dst buffer and -
// through a peer (NVLink / NVSwitch) mapping of the neighbour's dst buffer -
// straight into its halo rows.  The last block to finish then publishes the
// generation number into the neighbour's arrival flag (release, system
// scope), and every block of the next generation's strip pass acquires its
// own flags before it reads a halo row.  No host round trip, no NCCL.
//
// One flag per direction is enough: rank p's strip pass of
// generation g+1 waits for the halos of generation g; the neighbour publishes
// them only after its own strip pass of generation g - the last reader of the
// buffer p is about to overwrite (ping-pong: dst of g+1 is src of g-1) - has
// completed.  Interior rows never read halo rows.
//
// Semantics are the executor's: the readable window of the
// shard is rows [-above, h - 1 + below] and columns [0, W); beyond it a
// neighbour reads the pad value or the nearest in-window cell.  Every op's
// apply() runs on that view, so the strips are bit-identical to the
// one-pass kernels.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "ops.cuh"

namespace sk {

struct HaloGeom {
  long long pitch;       // elements, src / dst / peer buffers alike
  int W, h;              // shard width, owned rows
  int above, below;      // readable halo rows in src (0 at the global edges)
  int m;                 // strip depth = max(N, S)
  int north_rows;        // rows of the top strip mirrored to the north peer (S of the stencil)
  int south_rows;        // rows of the bottom strip mirrored to the south peer (N)
  long long north_off;   // element offset of the north peer's south-halo row 0 in its dst
  long long south_off;   // element offset of the south peer's north-halo row 0 in its dst
  int mode;              // sk_border_mode
  long long wait_value;  // flags[0] / flags[1] must reach this before halos are read
  long long signal_value;
};

// Global-memory view with the executor's border substitution.
template <typename T>
struct WindowView {
  const T* base;  // shard row 0
  long long pitch;
  int r, c, lo, hi, W, mode;
  T pad;
  __device__ __forceinline__ T at(int dr, int dc) const {
    int rr = r + dr, cc = c + dc;
    if (rr < lo || rr > hi || cc < 0 || cc >= W) {
      if (mode == 0) return pad;
      rr = rr < lo ? lo : (rr > hi ? hi : rr);
      cc = cc < 0 ? 0 : (cc >= W ? W - 1 : cc);
    }
    return base[static_cast<long long>(rr) * pitch + cc];
  }
};

__device__ __forceinline__ long long ld_acquire_sys(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(long long* p, long long v) {
  asm volatile("st.release.sys.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Block-wide acquire of this rank's arrival flags (flags[0]: north halo from
// p-1, flags[1]: south halo from p+1); a null flag pointer skips a side.
__device__ __forceinline__ void halo_acquire(const long long* flag_n, const long long* flag_s,
                                             long long value) {
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    if (flag_n) {
      while (ld_acquire_sys(flag_n) < value) __nanosleep(64);
    }
    if (flag_s) {
      while (ld_acquire_sys(flag_s) < value) __nanosleep(64);
    }
  }
  __syncthreads();
}

// The last block of the grid publishes `value` to the peers' flags after every
// block's stores (local and remote) are visible system-wide.
__device__ __forceinline__ void halo_release(unsigned* done, long long* peer_flag_n,
                                             long long* peer_flag_s, long long value) {
  __threadfence_system();  // this thread's local and peer stores, system-wide
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    const unsigned nblocks = gridDim.x * gridDim.y;
    if (atomicAdd(done, 1u) == nblocks - 1) {
      __threadfence_system();
      if (peer_flag_n) st_release_sys(peer_flag_n, value);
      if (peer_flag_s) st_release_sys(peer_flag_s, value);
      atomicExch(done, 0u);  // ready for the next generation (stream-ordered)
    }
  }
}

// Boundary strips of one generation: blockIdx.y = 0 computes owned rows
// [0, m), blockIdx.y = 1 rows [h - m, h); one work-item per cell.  Rows
// [0, north_rows) are also stored to peer_n + north_off, rows
// [h - south_rows, h) to peer_s + south_off.
template <class Op, typename T>
__global__ void __launch_bounds__(256)
    k_halo_strips(const T* __restrict__ src, T* __restrict__ dst, T* peer_n, T* peer_s,
                  const long long* flag_n, const long long* flag_s, long long* peer_flag_n,
                  long long* peer_flag_s, unsigned* done, const HaloGeom g, const T pad,
                  const __grid_constant__ OpParams<T> p) {
  halo_acquire(flag_n, flag_s, g.wait_value);
  const int bottom = blockIdx.y;
  const long long cells = static_cast<long long>(g.m) * g.W;
  const Op op;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < cells;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int rr = static_cast<int>(i / g.W);
    const int c = static_cast<int>(i - static_cast<long long>(rr) * g.W);
    const int r = bottom ? g.h - g.m + rr : rr;
    if (bottom && r < g.m) continue;  // h < 2m: the top strip already owns the row
    const WindowView<T> v{src, g.pitch, r, c, -g.above, g.h - 1 + g.below, g.W, g.mode, pad};
    const T out = op.template apply<T>(v, p);
    dst[static_cast<long long>(r) * g.pitch + c] = out;
    if (peer_n && r < g.north_rows) peer_n[g.north_off + static_cast<long long>(r) * g.pitch + c] = out;
    if (peer_s && r >= g.h - g.south_rows) {
      peer_s[g.south_off + static_cast<long long>(r - (g.h - g.south_rows)) * g.pitch + c] = out;
    }
  }
  halo_release(done, peer_flag_n, peer_flag_s, g.signal_value);
}

// Initial (or re-synchronising) halo put: copy rows [0, north_rows) of `src`
// to the north peer and rows [h - south_rows, h) to the south peer, then
// publish `signal_value` (after waiting for `wait_value`: the peers must be
// done reading the halos about to be overwritten).
template <typename T>
__global__ void __launch_bounds__(256)
    k_halo_put(const T* __restrict__ src, T* peer_n, T* peer_s, const long long* flag_n,
               const long long* flag_s, long long* peer_flag_n, long long* peer_flag_s,
               unsigned* done, const HaloGeom g) {
  halo_acquire(flag_n, flag_s, g.wait_value);
  const long long nn = peer_n ? static_cast<long long>(g.north_rows) * g.W : 0;
  const long long ns = peer_s ? static_cast<long long>(g.south_rows) * g.W : 0;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < nn + ns;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    if (i < nn) {
      const int r = static_cast<int>(i / g.W);
      const int c = static_cast<int>(i - static_cast<long long>(r) * g.W);
      peer_n[g.north_off + static_cast<long long>(r) * g.pitch + c] = src[static_cast<long long>(r) * g.pitch + c];
    } else {
      const long long j = i - nn;
      const int r = static_cast<int>(j / g.W);
      const int c = static_cast<int>(j - static_cast<long long>(r) * g.W);
      peer_s[g.south_off + static_cast<long long>(r) * g.pitch + c] =
          src[static_cast<long long>(g.h - g.south_rows + r) * g.pitch + c];
    }
  }
  halo_release(done, peer_flag_n, peer_flag_s, g.signal_value);
}

// Stream-ordered acquire of this rank's arrival flags (the temporally
// blocked schedule waits here before its strip pass, whose kernel is the
// register-strip one).
// (A template so the header can be included by every translation unit.)
template <int Unused = 0>
__global__ void __launch_bounds__(32) k_halo_wait(const long long* flag_n, const long long* flag_s,
                                                  long long value) {
  halo_acquire(flag_n, flag_s, value);
}

}  // namespace sk
