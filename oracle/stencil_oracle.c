/*
 * CPU oracle for the SkelCL stencil pattern — TEST INFRASTRUCTURE ONLY
 * (see stencil_oracle.h for the import rule and the parity status).
 *
 * Direct restatement, one output cell at a time:
 *   out[r][c] = F(region)  with region(dr, dc) = fetch(r + dr, c + dc),
 *   dr in [-north, south] (north = smaller row index), dc in [-west, east],
 * and fetch substituting the pad value or the clamped (nearest) cell outside
 * the readable rows [-rows_above, H + rows_below) / columns [0, W)
 * (PAPER.md:91-100).  No tiling, no shared state: the GPU executor's tiles,
 * TMA boxes and shared-memory fix-ups are what this checks.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared -pthread (oracle/Makefile);
 * no FMA contraction so float expressions round exactly as written.
 */
#include "stencil_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

enum { OP_FIVE_POINT, OP_HEAT, OP_GOL, OP_BOXMEAN, OP_GAUSSIAN, OP_SOBEL, OP_NMS,
       OP_THRESHOLD, OP_SYNTHETIC };
enum { DT_I32, DT_F32, DT_F64 };

typedef struct {
  const oracle_desc* d;
  const char* in;
  char* out;
  int64_t W, H, pin, pout, above, below;
  int64_t r_begin, r_end;
  double gw[21 * 21];      /* unused (kept for layout) */
  double gb[21];           /* gaussian 1-D weights C(2g,j)/2^(2g) */
  long long giw[21 * 21];  /* gaussian weights, int kernels    */
} job;

static int64_t clamp64(int64_t v, int64_t lo, int64_t hi) {
  return v < lo ? lo : (v > hi ? hi : v);
}

/* Readable-window fetch with border substitution, as double / float /
 * int32 views of the same element. */
#define DEFINE_FETCH(NAME, T)                                                     \
  static T NAME(const job* j, int64_t r, int64_t c) {                             \
    const T* in = (const T*)j->in;                                                \
    int64_t lo = -j->above, hi = j->H - 1 + j->below;                             \
    if (r >= lo && r <= hi && c >= 0 && c < j->W) return in[r * j->pin + c];     \
    if (j->d->border_mode == 0) return (T)j->d->pad_value;                        \
    return in[clamp64(r, lo, hi) * j->pin + clamp64(c, 0, j->W - 1)];             \
  }
DEFINE_FETCH(fetch_f32, float)
DEFINE_FETCH(fetch_f64, double)
DEFINE_FETCH(fetch_i32, int32_t)

static long long binom(int n, int k) {
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

static int alu_iters(const oracle_desc* d) {
  if (d->op != OP_SYNTHETIC) return 0;
  return d->complexity ? d->instructions / 4 : d->instructions / 32;
}

/* ---------------------------------------------------------------- float32 */
static float cell_f32(const job* j, int64_t r, int64_t c) {
  const oracle_desc* d = j->d;
#define V(dr, dc) fetch_f32(j, r + (dr), c + (dc))
  switch (d->op) {
    case OP_FIVE_POINT: {
      float s = V(-1, 0) + V(1, 0);
      s = s + V(0, 1);
      s = s + V(0, -1);
      s = s + V(0, 0);
      return s * 0.2f;
    }
    case OP_HEAT: {
      float u = V(0, 0);
      float lap = V(-1, 0) + V(1, 0);
      lap = lap + V(0, 1);
      lap = lap + V(0, -1);
      lap = lap - 4.0f * u;
      return u + 0.2f * lap;
    }
    case OP_GOL: {
      int n = 0;
      for (int dr = -1; dr <= 1; ++dr)
        for (int dc = -1; dc <= 1; ++dc)
          if ((dr || dc) && V(dr, dc) != 0.0f) ++n;
      int alive = V(0, 0) != 0.0f;
      return (n == 3 || (alive && n == 2)) ? 1.0f : 0.0f;
    }
    case OP_BOXMEAN: { /* sum of row sums (west->east), rows north->south */
      float s = 0.0f;
      for (int dr = -d->north; dr <= d->south; ++dr) {
        float row = V(dr, -d->west);
        for (int dc = -d->west + 1; dc <= d->east; ++dc) row = row + V(dr, dc);
        s = dr == -d->north ? row : s + row;
      }
      return s / (float)((d->north + d->south + 1) * (d->east + d->west + 1));
    }
    case OP_GAUSSIAN: { /* separable: row pass west->east, then rows north->south */
      int g = d->north;
      float s = 0.0f;
      for (int i = -g; i <= g; ++i) {
        float row = (float)j->gb[0] * V(i, -g);
        for (int k = -g + 1; k <= g; ++k) {
          float p = (float)j->gb[k + g] * V(i, k);
          row = row + p;
        }
        float t = (float)j->gb[i + g] * row;
        s = i == -g ? t : s + t;
      }
      return s;
    }
    case OP_SOBEL: {
      float ex = V(-1, 1) + 2.0f * V(0, 1);
      ex = ex + V(1, 1);
      float wx = V(-1, -1) + 2.0f * V(0, -1);
      wx = wx + V(1, -1);
      float gx = ex - wx;
      float sy = V(1, -1) + 2.0f * V(1, 0);
      sy = sy + V(1, 1);
      float ny = V(-1, -1) + 2.0f * V(-1, 0);
      ny = ny + V(-1, 1);
      float gy = sy - ny;
      float m2 = gx * gx;
      m2 = m2 + gy * gy;
      return sqrtf(m2);
    }
    case OP_NMS: {
      float m = V(-1, -1);
      const int nb[7][2] = {{-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
      for (int k = 0; k < 7; ++k) {
        float x = V(nb[k][0], nb[k][1]);
        m = x > m ? x : m;
      }
      float ce = V(0, 0);
      return ce >= m ? ce : 0.0f;
    }
    case OP_THRESHOLD:
      return V(0, 0) > 0.5f ? 1.0f : 0.0f;
    case OP_SYNTHETIC: {
      float s = 0.0f;
      for (int dr = -d->north; dr <= d->south; ++dr) s = s + V(dr, 0);
      for (int dc = -d->west; dc <= -1; ++dc) s = s + V(0, dc);
      for (int dc = 1; dc <= d->east; ++dc) s = s + V(0, dc);
      float x = s / (float)(d->north + d->south + 1 + d->east + d->west);
      for (int k = 0, it = alu_iters(d); k < it; ++k) {
        x = x * 0.999f;
        x = x + 0.001f;
      }
      return x;
    }
  }
#undef V
  return 0.0f;
}

/* ---------------------------------------------------------------- float64 */
static double cell_f64(const job* j, int64_t r, int64_t c) {
  const oracle_desc* d = j->d;
#define V(dr, dc) fetch_f64(j, r + (dr), c + (dc))
  switch (d->op) {
    case OP_FIVE_POINT: {
      double s = V(-1, 0) + V(1, 0);
      s = s + V(0, 1);
      s = s + V(0, -1);
      s = s + V(0, 0);
      return s * 0.2;
    }
    case OP_HEAT: {
      double u = V(0, 0);
      double lap = V(-1, 0) + V(1, 0);
      lap = lap + V(0, 1);
      lap = lap + V(0, -1);
      lap = lap - 4.0 * u;
      return u + 0.2 * lap;
    }
    case OP_GOL: {
      int n = 0;
      for (int dr = -1; dr <= 1; ++dr)
        for (int dc = -1; dc <= 1; ++dc)
          if ((dr || dc) && V(dr, dc) != 0.0) ++n;
      int alive = V(0, 0) != 0.0;
      return (n == 3 || (alive && n == 2)) ? 1.0 : 0.0;
    }
    case OP_BOXMEAN: { /* sum of row sums (west->east), rows north->south */
      double s = 0.0;
      for (int dr = -d->north; dr <= d->south; ++dr) {
        double row = V(dr, -d->west);
        for (int dc = -d->west + 1; dc <= d->east; ++dc) row = row + V(dr, dc);
        s = dr == -d->north ? row : s + row;
      }
      return s / (double)((d->north + d->south + 1) * (d->east + d->west + 1));
    }
    case OP_GAUSSIAN: { /* separable: row pass west->east, then rows north->south */
      int g = d->north;
      double s = 0.0;
      for (int i = -g; i <= g; ++i) {
        double row = j->gb[0] * V(i, -g);
        for (int k = -g + 1; k <= g; ++k) {
          double p = j->gb[k + g] * V(i, k);
          row = row + p;
        }
        double t = j->gb[i + g] * row;
        s = i == -g ? t : s + t;
      }
      return s;
    }
    case OP_SOBEL: {
      double ex = V(-1, 1) + 2.0 * V(0, 1);
      ex = ex + V(1, 1);
      double wx = V(-1, -1) + 2.0 * V(0, -1);
      wx = wx + V(1, -1);
      double gx = ex - wx;
      double sy = V(1, -1) + 2.0 * V(1, 0);
      sy = sy + V(1, 1);
      double ny = V(-1, -1) + 2.0 * V(-1, 0);
      ny = ny + V(-1, 1);
      double gy = sy - ny;
      double m2 = gx * gx;
      m2 = m2 + gy * gy;
      return sqrt(m2);
    }
    case OP_NMS: {
      double m = V(-1, -1);
      const int nb[7][2] = {{-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
      for (int k = 0; k < 7; ++k) {
        double x = V(nb[k][0], nb[k][1]);
        m = x > m ? x : m;
      }
      double ce = V(0, 0);
      return ce >= m ? ce : 0.0;
    }
    case OP_THRESHOLD:
      return V(0, 0) > 0.5 ? 1.0 : 0.0;
    case OP_SYNTHETIC: {
      double s = 0.0;
      for (int dr = -d->north; dr <= d->south; ++dr) s = s + V(dr, 0);
      for (int dc = -d->west; dc <= -1; ++dc) s = s + V(0, dc);
      for (int dc = 1; dc <= d->east; ++dc) s = s + V(0, dc);
      double x = s / (double)(d->north + d->south + 1 + d->east + d->west);
      for (int k = 0, it = alu_iters(d); k < it; ++k) {
        x = x * 0.999;
        x = x + 0.001;
      }
      return x;
    }
  }
#undef V
  return 0.0;
}

/* ------------------------------------------------------------------ int32 */
/* Integer kernels accumulate in 64 bits with wrap-around (unsigned) so the
 * result is defined for any input. */
static long long wadd(long long a, long long b) {
  return (long long)((unsigned long long)a + (unsigned long long)b);
}
static long long wmul(long long a, long long b) {
  return (long long)((unsigned long long)a * (unsigned long long)b);
}

static int32_t cell_i32(const job* j, int64_t r, int64_t c) {
  const oracle_desc* d = j->d;
#define V(dr, dc) ((long long)fetch_i32(j, r + (dr), c + (dc)))
  switch (d->op) {
    case OP_FIVE_POINT:
      return (int32_t)((V(-1, 0) + V(1, 0) + V(0, 1) + V(0, -1) + V(0, 0)) / 5);
    case OP_HEAT: {
      long long u = V(0, 0);
      long long lap = V(-1, 0) + V(1, 0) + V(0, 1) + V(0, -1) - 4 * u;
      return (int32_t)(u + lap / 5);
    }
    case OP_GOL: {
      int n = 0;
      for (int dr = -1; dr <= 1; ++dr)
        for (int dc = -1; dc <= 1; ++dc)
          if ((dr || dc) && V(dr, dc) != 0) ++n;
      int alive = V(0, 0) != 0;
      return (n == 3 || (alive && n == 2)) ? 1 : 0;
    }
    case OP_BOXMEAN: {
      long long s = 0;
      for (int dr = -d->north; dr <= d->south; ++dr)
        for (int dc = -d->west; dc <= d->east; ++dc) s = wadd(s, V(dr, dc));
      return (int32_t)(s / ((d->north + d->south + 1) * (d->east + d->west + 1)));
    }
    case OP_GAUSSIAN: {
      int g = d->north, n = 2 * g + 1;
      long long s = 0;
      for (int i = -g; i <= g; ++i)
        for (int k = -g; k <= g; ++k) s = wadd(s, wmul(j->giw[(i + g) * n + (k + g)], V(i, k)));
      return (int32_t)(s >> (4 * g));
    }
    case OP_SOBEL: {
      long long gx = (V(-1, 1) + 2 * V(0, 1) + V(1, 1)) - (V(-1, -1) + 2 * V(0, -1) + V(1, -1));
      long long gy = (V(1, -1) + 2 * V(1, 0) + V(1, 1)) - (V(-1, -1) + 2 * V(-1, 0) + V(-1, 1));
      return (int32_t)((gx < 0 ? -gx : gx) + (gy < 0 ? -gy : gy));
    }
    case OP_NMS: {
      long long m = V(-1, -1);
      const int nb[7][2] = {{-1, 0}, {-1, 1}, {0, -1}, {0, 1}, {1, -1}, {1, 0}, {1, 1}};
      for (int k = 0; k < 7; ++k) {
        long long x = V(nb[k][0], nb[k][1]);
        m = x > m ? x : m;
      }
      long long ce = V(0, 0);
      return (int32_t)(ce >= m ? ce : 0);
    }
    case OP_THRESHOLD:
      return V(0, 0) > 0 ? 1 : 0;
    case OP_SYNTHETIC: {
      long long s = 0;
      for (int dr = -d->north; dr <= d->south; ++dr) s = wadd(s, V(dr, 0));
      for (int dc = -d->west; dc <= -1; ++dc) s = wadd(s, V(0, dc));
      for (int dc = 1; dc <= d->east; ++dc) s = wadd(s, V(0, dc));
      uint32_t x = (uint32_t)(int32_t)(s / (d->north + d->south + 1 + d->east + d->west));
      for (int k = 0, it = alu_iters(d); k < it; ++k) x = x * 1664525u + 1013904223u;
      return (int32_t)x;
    }
  }
#undef V
  return 0;
}

static void* run_rows(void* arg) {
  job* j = (job*)arg;
  for (int64_t r = j->r_begin; r < j->r_end; ++r) {
    for (int64_t c = 0; c < j->W; ++c) {
      switch (j->d->dtype) {
        case DT_F32: ((float*)j->out)[r * j->pout + c] = cell_f32(j, r, c); break;
        case DT_F64: ((double*)j->out)[r * j->pout + c] = cell_f64(j, r, c); break;
        default: ((int32_t*)j->out)[r * j->pout + c] = cell_i32(j, r, c); break;
      }
    }
  }
  return NULL;
}

static int check_desc(const oracle_desc* d) {
  if (!d || d->op < 0 || d->op > OP_SYNTHETIC || d->dtype < 0 || d->dtype > DT_F64) return -1;
  if (d->north < 0 || d->south < 0 || d->east < 0 || d->west < 0) return -1;
  if (d->op == OP_GAUSSIAN && (d->north < 1 || d->north > 10)) return -1;
  return 0;
}

/* ------------------------------------------------------------ input fill */
/* std::mt19937_64 (the reference Rng engine, include/wgtune/rng.hpp:34-72). */
typedef struct {
  uint64_t mt[312];
  int i;
} mt64;

static void mt64_seed(mt64* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int k = 1; k < 312; ++k)
    m->mt[k] = 6364136223846793005ULL * (m->mt[k - 1] ^ (m->mt[k - 1] >> 62)) + (uint64_t)k;
  m->i = 312;
}

static uint64_t mt64_next(mt64* m) {
  if (m->i >= 312) {
    for (int k = 0; k < 312; ++k) {
      uint64_t x = (m->mt[k] & 0xFFFFFFFF80000000ULL) | (m->mt[(k + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ULL;
      m->mt[k] = m->mt[(k + 156) % 312] ^ xa;
    }
    m->i = 0;
  }
  uint64_t x = m->mt[m->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}

int oracle_fill(int32_t dtype, int32_t kind, uint64_t seed, void* out, int64_t count) {
  if (!out || count < 0 || dtype < DT_I32 || dtype > DT_F64 || kind < 0 || kind > 3) return -1;
  mt64* m = (mt64*)malloc(sizeof(mt64));
  if (!m) return -1;
  mt64_seed(m, seed);
  for (int64_t i = 0; i < count; ++i) {
    double u = (double)(mt64_next(m) >> 11) * 0x1.0p-53;
    double v = kind == 0 ? 2.0 * u - 1.0 : kind == 1 ? u : kind == 2 ? (u < 0.5 ? 1.0 : 0.0)
                                                                     : floor(256.0 * u);
    if (dtype == DT_I32) ((int32_t*)out)[i] = (int32_t)v;
    else if (dtype == DT_F32) ((float*)out)[i] = (float)v;
    else ((double*)out)[i] = v;
  }
  free(m);
  return 0;
}

/* ------------------------------------------------------- CPU baseline path */
/* Interior rows with the op switch hoisted: plain loops over a row that gcc
 * vectorises (avx2 clone where the host has it).  Same expressions, same
 * order, no contraction: bit-identical to cell_*. */
#define SK_CLONES __attribute__((target_clones("avx2", "default")))

SK_CLONES static void row_gol_i32(const int32_t* up, const int32_t* mid, const int32_t* dn,
                                  int32_t* out, int64_t c0, int64_t c1) {
  for (int64_t c = c0; c < c1; ++c) {
    int n = (up[c - 1] != 0) + (up[c] != 0) + (up[c + 1] != 0) + (mid[c - 1] != 0) +
            (mid[c + 1] != 0) + (dn[c - 1] != 0) + (dn[c] != 0) + (dn[c + 1] != 0);
    int alive = mid[c] != 0;
    out[c] = (n == 3) | (alive & (n == 2));
  }
}

SK_CLONES static void row_heat_f32(const float* up, const float* mid, const float* dn, float* out,
                                   int64_t c0, int64_t c1) {
  for (int64_t c = c0; c < c1; ++c) {
    float u = mid[c];
    float lap = up[c] + dn[c];
    lap = lap + mid[c + 1];
    lap = lap + mid[c - 1];
    lap = lap - 4.0f * u;
    out[c] = u + 0.2f * lap;
  }
}

SK_CLONES static void row_five_f32(const float* up, const float* mid, const float* dn, float* out,
                                   int64_t c0, int64_t c1) {
  for (int64_t c = c0; c < c1; ++c) {
    float s = up[c] + dn[c];
    s = s + mid[c + 1];
    s = s + mid[c - 1];
    s = s + mid[c];
    out[c] = s * 0.2f;
  }
}

/* boxmean f32 over rows r-N..r+S: each row summed west->east, the row sums
 * north->south, then one division (cell_f32's OP_BOXMEAN order). */
SK_CLONES static void row_boxmean_f32(const float* in, int64_t pitch, const oracle_desc* d,
                                      float* out, float* acc, float* row, int64_t c0, int64_t c1) {
  const float cnt = (float)((d->north + d->south + 1) * (d->east + d->west + 1));
  for (int dr = -d->north; dr <= d->south; ++dr) {
    const float* p = in + dr * pitch;
    for (int64_t c = c0; c < c1; ++c) row[c] = p[c - d->west];
    for (int dc = -d->west + 1; dc <= d->east; ++dc)
      for (int64_t c = c0; c < c1; ++c) row[c] = row[c] + p[c + dc];
    if (dr == -d->north)
      for (int64_t c = c0; c < c1; ++c) acc[c] = row[c];
    else
      for (int64_t c = c0; c < c1; ++c) acc[c] = acc[c] + row[c];
  }
  for (int64_t c = c0; c < c1; ++c) out[c] = acc[c] / cnt;
}

static int fast_op(const oracle_desc* d) {
  int unit = d->north == 1 && d->south == 1 && d->east == 1 && d->west == 1;
  if (d->op == OP_GOL && d->dtype == DT_I32 && unit) return 1;
  if (d->op == OP_HEAT && d->dtype == DT_F32 && unit) return 2;
  if (d->op == OP_FIVE_POINT && d->dtype == DT_F32 && unit) return 3;
  if (d->op == OP_BOXMEAN && d->dtype == DT_F32) return 4;
  return 0;
}

static void cell_store(const job* j, int64_t r, int64_t c) {
  switch (j->d->dtype) {
    case DT_F32: ((float*)j->out)[r * j->pout + c] = cell_f32(j, r, c); break;
    case DT_F64: ((double*)j->out)[r * j->pout + c] = cell_f64(j, r, c); break;
    default: ((int32_t*)j->out)[r * j->pout + c] = cell_i32(j, r, c); break;
  }
}

static void* run_rows_baseline(void* arg) {
  job* j = (job*)arg;
  const oracle_desc* d = j->d;
  const int kind = fast_op(d);
  const int64_t cl = d->west, ch = j->W - d->east; /* interior columns [cl, ch) */
  float *acc = NULL, *row = NULL;
  if (kind == 4) {
    acc = (float*)malloc(sizeof(float) * (size_t)j->W);
    row = (float*)malloc(sizeof(float) * (size_t)j->W);
  }
  for (int64_t r = j->r_begin; r < j->r_end; ++r) {
    const int interior = kind && (kind != 4 || (acc && row)) && r - d->north >= 0 &&
                         r + d->south <= j->H - 1 && ch > cl;
    if (!interior) {
      for (int64_t c = 0; c < j->W; ++c) cell_store(j, r, c);
      continue;
    }
    for (int64_t c = 0; c < cl; ++c) cell_store(j, r, c);
    for (int64_t c = ch; c < j->W; ++c) cell_store(j, r, c);
    if (kind == 1) {
      const int32_t* m = (const int32_t*)j->in + r * j->pin;
      row_gol_i32(m - j->pin, m, m + j->pin, (int32_t*)j->out + r * j->pout, cl, ch);
    } else if (kind == 2 || kind == 3) {
      const float* m = (const float*)j->in + r * j->pin;
      float* o = (float*)j->out + r * j->pout;
      if (kind == 2) row_heat_f32(m - j->pin, m, m + j->pin, o, cl, ch);
      else row_five_f32(m - j->pin, m, m + j->pin, o, cl, ch);
    } else {
      row_boxmean_f32((const float*)j->in + r * j->pin, j->pin, d, (float*)j->out + r * j->pout,
                      acc, row, cl, ch);
    }
  }
  free(acc);
  free(row);
  return NULL;
}

static int run_jobs(const oracle_desc* d, const void* in, void* out, int64_t width,
                    int64_t height, int64_t pitch_in, int64_t pitch_out, int64_t rows_above,
                    int64_t rows_below, int32_t threads, void* (*fn)(void*)) {
  if (check_desc(d) || !in || !out || width < 1 || height < 1) return -1;
  if (pitch_in < width || pitch_out < width || rows_above < 0 || rows_below < 0) return -1;
  int nt = threads < 1 ? 1 : threads;
  if (nt > height) nt = (int)height;
  job base;
  memset(&base, 0, sizeof base);
  base.d = d;
  base.in = (const char*)in;
  base.out = (char*)out;
  base.W = width;
  base.H = height;
  base.pin = pitch_in;
  base.pout = pitch_out;
  base.above = rows_above < d->north ? rows_above : d->north;
  base.below = rows_below < d->south ? rows_below : d->south;
  if (d->op == OP_GAUSSIAN) {
    int g = d->north, n = 2 * g + 1;
    for (int i = 0; i < n; ++i)
      for (int k = 0; k < n; ++k) {
        long long cij = binom(2 * g, i) * binom(2 * g, k);
        base.giw[i * n + k] = cij;
        base.gw[i * n + k] = ldexp((double)cij, -4 * g);
      }
    for (int i = 0; i < n; ++i) base.gb[i] = ldexp((double)binom(2 * g, i), -2 * g);
  }
  job* jobs = (job*)malloc(sizeof(job) * (size_t)nt);
  pthread_t* tids = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nt);
  if (!jobs || !tids) {
    free(jobs);
    free(tids);
    return -1;
  }
  for (int t = 0; t < nt; ++t) {
    jobs[t] = base;
    jobs[t].r_begin = height * t / nt;
    jobs[t].r_end = height * (t + 1) / nt;
  }
  for (int t = 1; t < nt; ++t) pthread_create(&tids[t], NULL, fn, &jobs[t]);
  fn(&jobs[0]);
  for (int t = 1; t < nt; ++t) pthread_join(tids[t], NULL);
  free(jobs);
  free(tids);
  return 0;
}

int oracle_stencil(const oracle_desc* d, const void* in, void* out, int64_t width,
                   int64_t height, int64_t pitch_in, int64_t pitch_out, int64_t rows_above,
                   int64_t rows_below, int32_t threads) {
  return run_jobs(d, in, out, width, height, pitch_in, pitch_out, rows_above, rows_below, threads,
                  run_rows);
}

int oracle_baseline_stencil(const oracle_desc* d, const void* in, void* out, int64_t width,
                            int64_t height, int32_t threads) {
  return run_jobs(d, in, out, width, height, width, width, 0, 0, threads, run_rows_baseline);
}

int oracle_baseline_iterate(const oracle_desc* d, void* a, void* b, int64_t width, int64_t height,
                            int32_t iterations, int32_t threads) {
  void* src = a;
  void* dst = b;
  for (int i = 0; i < iterations; ++i) {
    int rc = oracle_baseline_stencil(d, src, dst, width, height, threads);
    if (rc) return rc;
    void* t = src;
    src = dst;
    dst = t;
  }
  return 0;
}

int oracle_iterate(const oracle_desc* d, void* a, void* b, int64_t width, int64_t height,
                   int32_t iterations, int32_t threads) {
  void* src = a;
  void* dst = b;
  for (int i = 0; i < iterations; ++i) {
    int rc = oracle_stencil(d, src, dst, width, height, width, width, 0, 0, threads);
    if (rc) return rc;
    void* t = src;
    src = dst;
    dst = t;
  }
  return 0;
}
