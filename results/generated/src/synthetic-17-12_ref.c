/* CPU reference of generated kernel 'synthetic-17-12' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (-23), c + (0)));
    acc = (acc + tap(g, r + (28), c + (0)));
    acc = (acc + tap(g, r + (0), c + (18)));
    acc = (acc + tap(g, r + (0), c + (-22)));
    acc = (acc + tap(g, r + (4), c + (4)));
    acc = (acc + tap(g, r + (26), c + (12)));
    acc = (acc + tap(g, r + (1), c + (13)));
    acc = (acc + tap(g, r + (-17), c + (-18)));
    acc = (acc + tap(g, r + (-15), c + (15)));
    acc = (acc + tap(g, r + (14), c + (15)));
    acc = (acc + tap(g, r + (-2), c + (0)));
    acc = (acc + tap(g, r + (-22), c + (15)));
    acc = (acc + tap(g, r + (-4), c + (-22)));
    acc = (acc + tap(g, r + (-3), c + (18)));
    acc = (acc + tap(g, r + (15), c + (-21)));
    acc = (acc + tap(g, r + (12), c + (14)));
    acc = (acc + tap(g, r + (21), c + (12)));
    acc = (acc + tap(g, r + (-14), c + (-20)));
    acc = (acc + tap(g, r + (-17), c + (-2)));
    acc = (acc + tap(g, r + (-4), c + (17)));
    acc = (acc + tap(g, r + (28), c + (15)));
    acc = (acc + tap(g, r + (-3), c + (6)));
    acc = (acc + tap(g, r + (-21), c + (1)));
    acc = (acc + tap(g, r + (15), c + (-12)));
    acc = (acc + tap(g, r + (4), c + (12)));
    h ^= h >> 13;
    h = h * 3025069249u;
    if (acc > 0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 10819720u;
    h += 16198744u;
    h ^= h >> 13;
    h ^= h >> 13;
    h = h * 178591057u;
    h = h * 250762815u;
    if (acc > -0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 2999102u;
    if (acc > -0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 2509971763u;
    if (acc > -1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
