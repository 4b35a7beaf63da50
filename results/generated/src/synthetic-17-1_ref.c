/* CPU reference of generated kernel 'synthetic-17-1' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (-7), c + (0)));
    acc = (acc + tap(g, r + (14), c + (0)));
    acc = (acc + tap(g, r + (0), c + (21)));
    acc = (acc + tap(g, r + (0), c + (-24)));
    acc = (acc + tap(g, r + (-6), c + (21)));
    acc = (acc + tap(g, r + (10), c + (8)));
    acc = (acc + tap(g, r + (2), c + (14)));
    acc = (acc + tap(g, r + (14), c + (-10)));
    acc = (acc + tap(g, r + (12), c + (6)));
    acc = (acc + tap(g, r + (4), c + (-24)));
    acc = (acc + tap(g, r + (11), c + (4)));
    acc = (acc + tap(g, r + (-7), c + (0)));
    acc = (acc + tap(g, r + (-2), c + (-3)));
    acc = (acc + tap(g, r + (-5), c + (-7)));
    acc = (acc + tap(g, r + (4), c + (-4)));
    acc = (acc + tap(g, r + (-3), c + (7)));
    acc = (acc + tap(g, r + (14), c + (-6)));
    acc = (acc + tap(g, r + (-2), c + (19)));
    acc = (acc + tap(g, r + (-7), c + (16)));
    acc = (acc + tap(g, r + (-4), c + (3)));
    acc = (acc + tap(g, r + (12), c + (-4)));
    acc = (acc + tap(g, r + (-3), c + (20)));
    acc = (acc + tap(g, r + (-3), c + (16)));
    acc = (acc + tap(g, r + (14), c + (4)));
    acc = (acc + tap(g, r + (-7), c + (-22)));
    acc = (acc + tap(g, r + (6), c + (1)));
    acc = (acc + tap(g, r + (4), c + (-11)));
    acc = (acc + tap(g, r + (-7), c + (21)));
    acc = (acc + tap(g, r + (8), c + (-3)));
    acc = (acc + tap(g, r + (9), c + (-22)));
    acc = (acc + tap(g, r + (14), c + (-20)));
    acc = (acc + tap(g, r + (3), c + (-5)));
    acc = (acc + tap(g, r + (5), c + (0)));
    h = h * 478063181u;
    if (acc > 0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    if (acc > 0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 12896132u;
    if (acc > -0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 43908721u;
    h += 6597397u;
    if (acc > -0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 2740606289u;
    if (acc > -0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h = h * 2810901767u;
    h += 9879292u;
    if (acc > -0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h ^= h >> 13;
    if (acc > 1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 6238193u;
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
