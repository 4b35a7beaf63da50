/* CPU reference of generated kernel 'synthetic-17-15' (build with -ffp-contract=off). */
typedef struct { const float* in; long W, H; int mode; float pad; } grid_t;
static float tap(const grid_t* g, long r, long c) {
  if (r < 0 || r >= g->H || c < 0 || c >= g->W) {
    if (g->mode == 0) return g->pad;
    r = r < 0 ? 0 : (r >= g->H ? g->H - 1 : r);
    c = c < 0 ? 0 : (c >= g->W ? g->W - 1 : c);
  }
  return g->in[r * g->W + c];
}
static float cell(const grid_t* g, long r, long c) {
    float acc = tap(g, r + (0), c + (0));
    unsigned h = 2166136261u;
    acc = (acc + tap(g, r + (-8), c + (0)));
    acc = (acc + tap(g, r + (6), c + (0)));
    acc = (acc + tap(g, r + (0), c + (2)));
    acc = (acc + tap(g, r + (0), c + (-10)));
    acc = (acc + tap(g, r + (-2), c + (-3)));
    acc = (acc + tap(g, r + (4), c + (2)));
    acc = (acc + tap(g, r + (-7), c + (-4)));
    acc = (acc + tap(g, r + (-7), c + (2)));
    acc = (acc + tap(g, r + (-3), c + (-6)));
    acc = (acc + tap(g, r + (0), c + (2)));
    acc = (acc + tap(g, r + (4), c + (1)));
    acc = (acc + tap(g, r + (0), c + (-2)));
    acc = (acc + tap(g, r + (4), c + (-5)));
    acc = (acc + tap(g, r + (2), c + (-9)));
    acc = (acc + tap(g, r + (1), c + (-8)));
    acc = (acc + tap(g, r + (-3), c + (0)));
    acc = (acc + tap(g, r + (4), c + (-2)));
    acc = (acc + tap(g, r + (6), c + (-5)));
    acc = (acc + tap(g, r + (-8), c + (-7)));
    acc = (acc + tap(g, r + (0), c + (1)));
    acc = (acc + tap(g, r + (-8), c + (2)));
    acc = (acc + tap(g, r + (6), c + (1)));
    acc = (acc + tap(g, r + (-6), c + (-8)));
    acc = (acc + tap(g, r + (-5), c + (2)));
    acc = (acc + tap(g, r + (-5), c + (2)));
    acc = (acc + tap(g, r + (-1), c + (1)));
    acc = (acc + tap(g, r + (-4), c + (-10)));
    acc = (acc + tap(g, r + (-8), c + (-1)));
    acc = (acc + tap(g, r + (-2), c + (1)));
    acc = (acc + tap(g, r + (2), c + (-10)));
    acc = (acc + tap(g, r + (-7), c + (-7)));
    acc = (acc + tap(g, r + (-6), c + (0)));
    acc = (acc + tap(g, r + (-5), c + (-7)));
    acc = (acc + tap(g, r + (-3), c + (0)));
    acc = (acc + tap(g, r + (0), c + (-5)));
    acc = (acc + tap(g, r + (0), c + (-3)));
    acc = (acc + tap(g, r + (6), c + (-8)));
    acc = (acc + tap(g, r + (-3), c + (2)));
    acc = (acc + tap(g, r + (-6), c + (1)));
    acc = (acc + tap(g, r + (0), c + (-4)));
    acc = (acc + tap(g, r + (-3), c + (-3)));
    acc = (acc + tap(g, r + (2), c + (-2)));
    acc = (acc + tap(g, r + (-6), c + (-5)));
    acc = (acc + tap(g, r + (-2), c + (1)));
    acc = (acc + tap(g, r + (-2), c + (-9)));
    h = h * 3608416015u;
    h ^= h >> 13;
    h += 12494428u;
    if (acc > 1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    if (acc > -1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 925225585u;
    h ^= h >> 13;
    h = h * 2815068943u;
    h += 3165775u;
    h ^= h >> 13;
    if (acc > -1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h ^= h >> 13;
    if (acc > 0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 1019854787u;
    if (acc > 0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 3887098943u;
    if (acc > 0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 3048789u;
    h += 13227098u;
    h += 12445648u;
    if (acc > -0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 2387733403u;
    h += 12479862u;
    h = h * 514276671u;
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
