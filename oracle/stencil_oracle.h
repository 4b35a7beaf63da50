/*
 * CPU oracle for the SkelCL-style stencil pattern — TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or the
 * timed CPU baseline.  The product path never calls it.
 *
 * PARITY STATUS: the stencil arithmetic is "parity unpinned" by the reference
 * in the strict sense — /root/reference ships no stencil implementation, no
 * golden grid and no known-answer test for stencil outputs (SURVEY.md §0.4,
 * SPEC.md:15).  This file restates the semantics of PAPER.md:91-100
 * (customising function over an N/S/E/W border region; out-of-matrix cells
 * replaced by a pad value or by the nearest in-matrix cell) with the
 * customising functions fixed in DESIGN.md §3, and is itself pinned by
 * analytic known answers (tests/test_oracle_kat.py: Game-of-Life still lifes,
 * oscillators and gliders, constant fields, delta responses, asymmetric ramps)
 * and by an independent numpy restatement (tests/golden/make_golden.py).
 */
#ifndef STENCIL_ORACLE_H
#define STENCIL_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors sk_stencil_desc field-for-field (include/sk_stencil.h) so a test
 * can hand the same descriptor to both sides. */
typedef struct {
  int32_t op, dtype;
  int32_t north, south, east, west;
  int32_t border_mode;
  double pad_value;
  int32_t complexity, instructions;
  int32_t load_path;        /* ignored */
  int32_t cells_per_thread; /* ignored */
  int32_t fused_iterations; /* ignored (one pass per call) */
} oracle_desc;

/* One pass over a W x H region (row pitch in elements); rows_above /
 * rows_below extra input rows are readable around it (row-shard halos).
 * threads <= 0 means one thread.  Returns 0 or -1 on a bad argument. */
int oracle_stencil(const oracle_desc* d, const void* in, void* out, int64_t width,
                   int64_t height, int64_t pitch_in, int64_t pitch_out, int64_t rows_above,
                   int64_t rows_below, int32_t threads);

/* `iterations` passes ping-ponging a -> b -> a ...; result in a when
 * iterations is even, in b when odd. */
int oracle_iterate(const oracle_desc* d, void* a, void* b, int64_t width, int64_t height,
                   int32_t iterations, int32_t threads);

/* Seeded synthetic input with the reference Rng stream (rng.hpp:34-72):
 * std::mt19937_64(seed), uniform01 = (x >> 11) * 2^-53; kind 0 -> 2u-1,
 * 1 -> u, 2 -> (u < 0.5), 3 -> floor(256u); cast to dtype (0 i32, 1 f32,
 * 2 f64).  Mirrors sk_fill_host so CPU-only code (the reference arm) can make
 * the bench's inputs without loading the product library. */
int oracle_fill(int32_t dtype, int32_t kind, uint64_t seed, void* out, int64_t count);

/* The CPU BASELINE (timed by bench.py; still test infrastructure): the same
 * arithmetic as oracle_stencil, but with the op switch hoisted out of the
 * interior so the compiler vectorises rows (gol/i32, heat/f32,
 * five_point/f32, boxmean/f32; every other op, the border rows and border
 * columns go through the per-cell restatement).  Bit-identical to
 * oracle_stencil (tests/test_oracle_kat.py).  No row-shard halos. */
int oracle_baseline_stencil(const oracle_desc* d, const void* in, void* out, int64_t width,
                            int64_t height, int32_t threads);

/* `iterations` baseline passes ping-ponging a <-> b (result as oracle_iterate). */
int oracle_baseline_iterate(const oracle_desc* d, void* a, void* b, int64_t width, int64_t height,
                            int32_t iterations, int32_t threads);

#ifdef __cplusplus
}
#endif

#endif
