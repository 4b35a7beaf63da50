/* CPU reference of generated kernel 'synthetic-17-0' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (-21), c + (0)));
    acc = (acc + tap(g, r + (3), c + (0)));
    acc = (acc + tap(g, r + (0), c + (29)));
    acc = (acc + tap(g, r + (0), c + (-27)));
    acc = (acc + tap(g, r + (-15), c + (25)));
    acc = (acc + tap(g, r + (-12), c + (-3)));
    acc = (acc + tap(g, r + (1), c + (19)));
    acc = (acc + tap(g, r + (-4), c + (29)));
    acc = (acc + tap(g, r + (-18), c + (28)));
    acc = (acc + tap(g, r + (-20), c + (-27)));
    acc = (acc + tap(g, r + (-5), c + (27)));
    acc = (acc + tap(g, r + (-15), c + (-2)));
    acc = (acc + tap(g, r + (-13), c + (16)));
    acc = (acc + tap(g, r + (-3), c + (-7)));
    acc = (acc + tap(g, r + (2), c + (-14)));
    acc = (acc + tap(g, r + (-5), c + (-2)));
    acc = (acc + tap(g, r + (-12), c + (-8)));
    acc = (acc + tap(g, r + (-6), c + (-15)));
    acc = (acc + tap(g, r + (-21), c + (-10)));
    acc = (acc + tap(g, r + (-11), c + (0)));
    acc = (acc + tap(g, r + (-5), c + (16)));
    acc = (acc + tap(g, r + (-8), c + (-15)));
    acc = (acc + tap(g, r + (-19), c + (11)));
    acc = (acc + tap(g, r + (-5), c + (-21)));
    acc = (acc + tap(g, r + (-7), c + (-10)));
    acc = (acc + tap(g, r + (0), c + (23)));
    acc = (acc + tap(g, r + (-6), c + (-6)));
    acc = (acc + tap(g, r + (-7), c + (29)));
    acc = (acc + tap(g, r + (-4), c + (-4)));
    acc = (acc + tap(g, r + (-9), c + (9)));
    acc = (acc + tap(g, r + (1), c + (12)));
    acc = (acc + tap(g, r + (-17), c + (27)));
    acc = (acc + tap(g, r + (0), c + (-10)));
    acc = (acc + tap(g, r + (3), c + (-15)));
    acc = (acc + tap(g, r + (2), c + (-19)));
    acc = (acc + tap(g, r + (-7), c + (18)));
    acc = (acc + tap(g, r + (0), c + (10)));
    acc = (acc + tap(g, r + (-14), c + (7)));
    h = h * 38384829u;
    h += 239644u;
    h = h * 2699274937u;
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 3202919943u;
    h += 13996789u;
    h ^= h >> 13;
    h = h * 1695602839u;
    if (acc > -0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 8559275u;
    h += 9009894u;
    h ^= h >> 13;
    h += 11937129u;
    h = h * 3299188923u;
    if (acc > 0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h ^= h >> 13;
    h = h * 1516224233u;
    if (acc > 1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h ^= h >> 13;
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
