/*
 * sk_stencil.h — C-ABI of the B200 SkelCL-style 2D stencil executor.
 *
 * This is the drop-in boundary that replaces the reference's simulated
 * execution seam (wgtune "simoracle", /root/reference/proj/include/wgtune/
 * simoracle.hpp) with real sm_100a kernels.  Plain pointers and sizes only:
 * no torch, no C++ types.  Every entry point names the reference interface it
 * replaces.
 *
 * Grid semantics (Fig. 1 at :122-128): a row-major H x W
 * matrix (row pitch >= W elements).  Each output cell is the customising
 * function applied to the rectangular border region around the input cell:
 * `north` rows above (row - 1 ... row - north), `south` rows below,
 * `east` columns to the right (col + 1 ...), `west` columns to the left.
 * Cells of the region outside the matrix take the pad value (SK_BORDER_PAD)
 * or the value of the nearest in-matrix cell (SK_BORDER_NEAREST, i.e.
 * clamp(row), clamp(col)).  The workgroup (CUDA block) is wc columns by wr
 * rows of work-items, one work-item per output cell; each block stages its
 * tile plus the perimeter border region in shared memory (PAPER.md:102-111,
 * tile shape (wc+E+W) x (wr+N+S) as in simoracle.cpp:21-28).
 */
#ifndef SK_STENCIL_H
#define SK_STENCIL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes.  SK_OVERSIZED / SK_REFUSED mirror the reference's
 * ProbeResult{Legal, Refused, Oversized} (tuner.hpp:16) and the exceptions
 * IllegalWorkgroupSize (errors.hpp:27) / RefusedParameter (errors.hpp:52-63)
 * thrown by simoracle::run (simoracle.cpp:122-131).  A refusal is a real,
 * non-sticky launch-configuration failure on the device (shared-memory tile
 * above the opt-in limit, no resident block possible, launch-config error);
 * a sticky CUDA fault is SK_ECUDA and aborts sweeps. */
typedef enum {
  SK_OK = 0,
  SK_OVERSIZED = 1, /* wc*wr above min(device max, per-kernel max)        */
  SK_REFUSED = 2,   /* legal size the device refuses to launch            */
  SK_EINVAL = 3,    /* bad argument (null pointer, bad enum, bad dims)    */
  SK_ECUDA = 4,     /* CUDA runtime error; see sk_last_error()            */
  SK_ENOTSUP = 5    /* combination not supported (e.g. in/out dtype mix)  */
} sk_status;

/* Element types, in the order of the reference's ElementType
 * (scenario.hpp:14: INT32, FLOAT32, FLOAT64). */
typedef enum { SK_INT32 = 0, SK_FLOAT32 = 1, SK_FLOAT64 = 2 } sk_dtype;

/* Border substitution. */
typedef enum { SK_BORDER_PAD = 0, SK_BORDER_NEAREST = 1 } sk_border_mode;

/* Customising functions.  The formulas are defined once in DESIGN.md §3 and
 * restated independently by the CPU oracle (oracle/stencil_oracle.c).
 * The real-world kernel set follows the reference's reference_kernels()
 * (synthgen.cpp:82-96 / PAPER.md Table 2): gaussian, gol, he, nms, sobel,
 * threshold; the synthetic family follows generate_kernels()
 * (synthgen.cpp:57-80).  FIVE_POINT and BOXMEAN are the BASELINE.json
 * config-1 and config-4 kernels. */
typedef enum {
  SK_OP_FIVE_POINT = 0, /* mean of centre + 4 neighbours, border (1,1,1,1)  */
  SK_OP_HEAT = 1,       /* "he": u + 0.2*(n+s+e+w-4u), border (1,1,1,1)     */
  SK_OP_GOL = 2,        /* "gol": Conway B3/S23, 3x3 Moore, border 1        */
  SK_OP_BOXMEAN = 3,    /* mean of the whole N/S/E/W region (any borders)   */
  SK_OP_GAUSSIAN = 4,   /* "gaussian": binomial blur, border g in [1,10]    */
  SK_OP_SOBEL = 5,      /* "sobel": gradient magnitude, border 1            */
  SK_OP_NMS = 6,        /* "nms": keep local 3x3 maxima, border 1           */
  SK_OP_THRESHOLD = 7,  /* "threshold": c > 0.5 ? 1 : 0, border 0           */
  SK_OP_SYNTHETIC = 8,  /* "synthetic-*": cross-shaped region mean + ALU loop */
  SK_OP_COUNT = 9
} sk_op;

/* Load strategy for the shared-memory tile. */
typedef enum {
  SK_LOAD_AUTO = 0,     /* TMA when the tile/tensor constraints allow       */
  SK_LOAD_TMA = 1,      /* force the TMA-pipelined persistent kernel        */
  SK_LOAD_EXPLICIT = 2, /* force explicit coalesced loads (one tile/block)  */
  SK_LOAD_BITPLANE = 3, /* gol only: bit-sliced tile (one bit per cell in
                           shared memory, 32 cells per logic op), any number
                           of fused generations; AUTO takes it for gol when
                           fused_iterations >= 2, except K in {1,2,4} with
                           TB in {2,4} (per-cell fused kernel).  Work-item = 32 cells of a
                           row x K rows; tile = wc words x wr*K rows.       */
  SK_LOAD_STRIPS = 4,   /* five_point / heat with N=S=E=W=1 only: register
                           strips, any TB in [1, 32] generations per launch;
                           AUTO takes it for those ops when TB > 4.  Work-
                           item = 4 cells of a row x K rows (K in {4, 8, 16},
                           0 = 8, float64 4); the block's tile is 128 columns x
                           (wc*wr/32)*K rows, of which 4(32 - 2 ceil(TB/4))
                           x ((wc*wr/32)*K - 2 TB) are stored.              */
  SK_LOAD_VECTOR = 5    /* one pass, TMA-staged tile, vector work-items:
                           V = 16 B / sizeof(T) adjacent cells of a row x K
                           rows (128-bit shared loads, one 128-bit global
                           store per row); tile = V*wc x wr*K cells.  For
                           five_point / heat / gol / sobel / nms with
                           N=S=E=W=1 and boxmean with (5,1,3,0); one pass
                           per launch (fused_iterations <= 1); needs 16-B
                           aligned buffers and pitches; a tile wider than a
                           TMA box (256 elements) is refused.               */
} sk_load_path;

/* Stencil descriptor: the kernel half of a reference KernelDescriptor
 * (scenario.hpp:46-56: name -> op, north/south/east/west, complexity,
 * total_instructions) plus the element type (DatasetDescriptor in/out type,
 * scenario.hpp:58-66; in == out) and the border mode / pad value that the
 * SkelCL user chooses. */
typedef struct {
  int32_t op;          /* sk_op                                             */
  int32_t dtype;       /* sk_dtype, input and output                        */
  int32_t north, south, east, west; /* border region, each in [0, 64]       */
  int32_t border_mode; /* sk_border_mode                                    */
  double pad_value;    /* cast to the element type                          */
  int32_t complexity;  /* synthetic only: 0 light (synthetic-a), 1 heavy (b) */
  int32_t instructions;/* synthetic only: static instruction total          */
  int32_t load_path;   /* sk_load_path                                      */
  int32_t cells_per_thread; /* K cells per work-item (rows of one column):
                          0 = auto, or 1, 2, 4, 8.  The workgroup (block) is
                          still wc x wr work-items; its tile covers
                          wc x (wr*K) cells.                                 */
  int32_t fused_iterations; /* temporal blocking: TB generations per launch
                          (0/1 = one pass per launch; 2 or 4 fuse TB passes in
                          shared memory).  sk_stencil_launch
                          then advances TB generations; sk_stencil_iterate
                          splits `iterations` into fused launches + single
                          passes.  Supported for five_point, heat, gol and
                          boxmean on the TMA path.  gol on the bit-plane
                          path (SK_LOAD_BITPLANE, or AUTO with TB >= 2)
                          takes any TB in [1, 128]; sk_stencil_iterate then
                          runs ceil(iterations / TB) launches.  five_point /
                          heat on the register-strip path (SK_LOAD_STRIPS,
                          or AUTO with TB > 4) take any TB in [1, 32], also
                          ceil(iterations / TB) launches.                    */
} sk_stencil_desc;

/* Launch one stencil pass over a W x H region, out-of-place, on `stream`
 * (a cudaStream_t; NULL = legacy default stream).  `d_in` points at row 0 of
 * the region; `rows_above` / `rows_below` further input rows are readable
 * beyond it (halo rows of a row shard, §8e) and are used as real data before
 * border substitution applies.  Replaces: simoracle::run
 * (simoracle.hpp:45, simoracle.cpp:122-141) for one sample. */
int sk_stencil_launch(const sk_stencil_desc* desc, const void* d_in, void* d_out,
                      int64_t width, int64_t height, int64_t pitch_in, int64_t pitch_out,
                      int64_t rows_above, int64_t rows_below, int32_t wc, int32_t wr,
                      void* stream);

/* User customising functions: a C++/CUDA caller compiles
 * the executor's kernel templates for its own functor (include/wgtb/
 * stencil_custom.cuh) and passes the resulting kernel handles here; geometry,
 * TMA descriptors, refusals and the launch are the library's.  Index [i] is
 * K = 1, 2, 4, 8 cells per work-item.  desc->op is ignored (the functor is
 * the op); borders, dtype, border mode and K are honoured. */
typedef struct {
  const void* tma[4];            /* k_stencil_tma<F, T, K, 1024>       */
  const void* explicit_load[4];  /* k_stencil_explicit<F, T, K, 1024>  */
} sk_kernel_table;

int sk_stencil_launch_custom(const sk_stencil_desc* desc, const sk_kernel_table* kernels,
                             const void* d_in, void* d_out, int64_t width, int64_t height,
                             int64_t pitch_in, int64_t pitch_out, int64_t rows_above,
                             int64_t rows_below, int32_t wc, int32_t wr, void* stream);

/* Iterated stencil: `iterations` generations ping-ponging between d_a
 * (input) and d_b, one launch per generation (or per TB generations when
 * desc->fused_iterations = TB).  The result lands in d_a after an even
 * number of launches, in d_b after an odd number; *result_in_b says which.
 * Same pitch for both buffers. */
int sk_stencil_iterate(const sk_stencil_desc* desc, void* d_a, void* d_b, int64_t width,
                       int64_t height, int64_t pitch, int32_t iterations, int32_t wc,
                       int32_t wr, void* stream, int32_t* result_in_b);

/* Row-sharded iterated stencil with the per-generation halo exchange over
 * NCCL (the "sk_halo_step(..., ncclComm_t)" of §8b).  This
 * rank owns `rows` rows of the global grid; d_a / d_b point at the first of
 * N halo rows above them and hold N + rows + S rows of `pitch` elements.
 * Per generation: ncclGroupStart; send the first S owned rows to rank-1 and
 * receive N halo rows from it; send the last N owned rows to rank+1 and
 * receive S halo rows from it; ncclGroupEnd - on an internal exchange
 * stream; the two boundary strips on an internal side stream behind the
 * exchange, beside the interior rows [N, rows-S) on `stream`, which then
 * joins the side stream.  Rank 0's north and rank nranks-1's south halos are
 * border cells (pad / nearest), so the ranks together compute exactly the
 * single-GPU result.  `comm` is an ncclComm_t of the NCCL loaded in the
 * process (resolved at run time; the library does not link NCCL), with
 * this process's `rank` of `nranks`; unused when nranks == 1.  One
 * generation per launch: fused_iterations <= 1, one-pass load paths
 * (SK_ENOTSUP otherwise).  *result_in_b as in sk_stencil_iterate.  The
 * single-GPU replacement for the reference's simulated run (simoracle.cpp:
 * 122-141) applied to an iterated multi-GPU step. */
int sk_stencil_iterate_nccl(const sk_stencil_desc* desc, void* d_a, void* d_b, int64_t width,
                            int64_t rows, int64_t pitch, int32_t iterations, int32_t wc, int32_t wr,
                            void* comm, int32_t rank, int32_t nranks, void* stream,
                            int32_t* result_in_b);

/* Zero-work legality probe for (wc, wr) on the current device.  Returns
 * SK_OK (legal), SK_OVERSIZED or SK_REFUSED.  Optional outputs: the
 * per-kernel maximum block size (cudaFuncAttributes.maxThreadsPerBlock,
 * replaces kernel_max_wgsize, simoracle.hpp:26), the shared-memory tile bytes
 * of one pipeline stage, and the load path a launch would take.  Replaces:
 * simoracle::is_refused (simoracle.hpp:34-35) and ProbeFn (tuner.hpp:17). */
int sk_stencil_probe(const sk_stencil_desc* desc, int64_t width, int64_t height,
                     int32_t wc, int32_t wr, int32_t* kernel_max, int64_t* tile_bytes,
                     int32_t* load_path);

/* Per-kernel maximum workgroup size for the descriptor (replaces
 * simoracle::kernel_max_wgsize, simoracle.cpp:62-70). */
int sk_kernel_max_wgsize(const sk_stencil_desc* desc, int32_t* kernel_max);

/* Timed samples of one pass (the sweep's "run", simoracle.cpp:122-141):
 * `warmup` untimed launches, then `samples` launches each bracketed by a
 * cudaEvent pair on an internal stream; when flush_l2 != 0 a buffer of
 * 2 x l2CacheSize is written and then read back (evicting the pass's data
 * and leaving clean lines, so no write-back debt lands in the pass) before every
 * sample.  ms_out[samples]. */
int sk_stencil_time(const sk_stencil_desc* desc, const void* d_in, void* d_out, int64_t width,
                    int64_t height, int64_t pitch, int32_t wc, int32_t wr, int32_t warmup,
                    int32_t samples, int32_t flush_l2, double* ms_out);

/* The streaming ceiling at a given size (no reference counterpart; the
 * denominator beside the measured HBM peak): `samples` copies of `bytes`
 * from d_in to d_out under exactly sk_stencil_time's harness (same stream,
 * events and L2 scrub).  kind 0 = cudaMemcpyAsync device-to-device, kind 1 =
 * a 16-B vector grid-stride copy kernel (16-B aligned, bytes % 16 == 0).
 * ms_out[samples]. */
int sk_copy_time(const void* d_in, void* d_out, int64_t bytes, int32_t kind, int32_t warmup,
                 int32_t samples, int32_t flush_l2, double* ms_out);

/* End-to-end call from HOST buffers (the plugin call a SkelCL user makes):
 * copies h_in (W*H dense) to the device, runs `iterations` passes, copies the
 * result to h_out.  Device buffers are cached per (size) inside the library. */
int sk_stencil_run_host(const sk_stencil_desc* desc, const void* h_in, void* h_out,
                        int64_t width, int64_t height, int32_t iterations, int32_t wc,
                        int32_t wr);

/* Streamed end-to-end jobs from HOST buffers (pinned for the copies to be
 * asynchronous): sk_stencil_submit_host enqueues H2D of h_in, `iterations`
 * passes and D2H into h_out on one of three internal slots (stream + device
 * buffers) and returns a ticket without waiting, so job j+1's H2D and job
 * j-1's D2H run on the copy engines while job j computes.  A submit waits
 * only for the job three tickets back (its slot's buffers).  sk_stencil_wait_host
 * blocks until job `ticket` has landed in its h_out.  Same results as
 * sk_stencil_run_host, which is the one-job-at-a-time form (both replace the
 * SkelCL user call on host data; the reference only
 * simulates it, simoracle.hpp:45). */
int sk_stencil_submit_host(const sk_stencil_desc* desc, const void* h_in, void* h_out,
                           int64_t width, int64_t height, int32_t iterations, int32_t wc,
                           int32_t wr, int64_t* ticket);
int sk_stencil_wait_host(int64_t ticket);

/* Device features (north-star subsystem 3): the DeviceDescriptor fields of
 * the reference (scenario.hpp:31-44) read from cudaDeviceProp instead of the
 * OpenCL device API. */
typedef struct {
  char name[128];          /* prop.name, sanitised (no ' ', '/', ',', '\n') */
  int32_t compute_units;   /* multiProcessorCount                          */
  int32_t frequency_mhz;   /* cudaDevAttrClockRate / 1000                  */
  int32_t local_mem_kb;    /* sharedMemPerBlockOptin / 1024                */
  int32_t global_cache_kb; /* l2CacheSize / 1024                           */
  int32_t global_mem_mb;   /* totalGlobalMem >> 20                         */
  int32_t device_max_wgsize; /* maxThreadsPerBlock                         */
  int32_t simd_width;      /* warpSize                                     */
  int32_t cc_major, cc_minor;
  int32_t mem_clock_mhz;
  int32_t mem_bus_width;
} sk_device_props;

int sk_device_features(int32_t device, sk_device_props* out);

/* Fill a device buffer with deterministic synthetic input (the reference
 * Rng stream, rng.hpp:34-72, so CPU and GPU inputs are identical): float
 * types get 2*uniform01()-1 or uniform01() (kind 0 / 1), int32 gets
 * uniform01() < 0.5 ? 1 : 0 (kind 2) or floor(256*uniform01()) (kind 3).
 * Generated on the host and copied. */
int sk_fill_host(int32_t dtype, int32_t kind, uint64_t seed, void* h_out, int64_t count);

/* Device-side bitwise comparison of two buffers (16-B aligned, size a
 * multiple of 16): *equal = 1 when identical.  Used by the sweep's
 * gold-standard check of every workgroup size. */
int sk_buffers_equal(const void* d_a, const void* d_b, int64_t bytes, int32_t* equal);

/* Last error text for the calling thread ("" if none). */
const char* sk_last_error(void);

/* Library version string. */
const char* sk_version(void);

/* ------------------------------------------------------------------------
 * Peer-memory halo exchange for row-sharded iterated stencils (SURVEY.md
 * §8e, the fused variant of the per-iteration ncclSend/ncclRecv; DESIGN.md
 * §7.1).  Each rank owns `rows` rows of a W-wide grid in two buffers A, B of
 * N + rows + S rows (north halo, owned rows, south halo; pitch elements per
 * row), and a control block of SK_HALO_CONTROL_BYTES zeroed device bytes.
 * The neighbours' buffers and control blocks are mapped into this process
 * (sk_ipc_import of handles the peers sk_ipc_export'ed, or plain pointers
 * when the "ranks" share one process).  Zero the control blocks and barrier
 * the ranks before the first call.
 * ---------------------------------------------------------------------- */
#define SK_HALO_CONTROL_BYTES 64

typedef struct {
  unsigned char handle[64]; /* cudaIpcMemHandle_t of the containing allocation */
  int64_t offset;           /* byte offset of the exported pointer inside it   */
} sk_ipc_handle;

/* Export / import a device pointer across processes (cudaIpc*MemHandle;
 * peer access is enabled lazily on import).  No reference counterpart: the
 * reference is single-device; the row-shard exchange is the north star's
 * addition. */
int sk_ipc_export(const void* d_ptr, sk_ipc_handle* out);
int sk_ipc_import(const sk_ipc_handle* h, void** d_ptr);
int sk_ipc_close(void* d_ptr);

typedef struct {
  void* north_a;         /* north neighbour's A / B buffers (its row 0 = its  */
  void* north_b;         /* first north-halo row); NULL on the first rank     */
  void* south_a;         /* south neighbour's A / B buffers; NULL on the last */
  void* south_b;
  void* north_control;   /* the neighbours' control blocks                    */
  void* south_control;
  int64_t north_rows;    /* rows owned by the north neighbour                 */
} sk_halo_peers;

/* `iterations` generations of a row shard with the halo exchange fused into
 * the boundary-strip pass: per generation, one k_halo_strips launch (acquire
 * the arrival flags, compute the max(N,S)-row top and bottom strips, store
 * them locally and into the neighbours' halo rows over the peer mapping,
 * publish the generation) and one interior launch of the tuned executor at
 * wc x wr - all on `stream`, no host synchronisation.  `epoch` is a host
 * counter every rank starts at 0 and passes to each call (updated in place).
 * The result lands in d_b when *result_in_b (odd iteration counts).  The
 * peers' *_a / *_b must be the neighbours' buffers in the roles d_a / d_b
 * play in this call (ranks ping-pong in lockstep: swap them together).
 * Replaces: the per-iteration exchange of the NCCL schedule
 * (paper_1511_02490_b200/distributed.py) - the reference has none (§8e).
 * Environment: SK_PEER_SCHEDULE=fused selects the opt-in one-pass kernel
 * with the exchange in its boundary tile-rows (refused for
 * peers on this device unless SK_PEER_ALLOW_SHARED is set - test use). */
int sk_stencil_iterate_peer(const sk_stencil_desc* desc, void* d_a, void* d_b, int64_t width,
                            int64_t rows, int64_t pitch, int32_t iterations, int32_t wc,
                            int32_t wr, const sk_halo_peers* peers, void* d_control,
                            int64_t* epoch, void* stream, int32_t* result_in_b);

#ifdef __cplusplus
}
#endif

#endif /* SK_STENCIL_H */
