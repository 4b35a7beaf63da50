/* CPU reference of generated kernel 'synthetic-17-8' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (3), c + (0)));
    acc = (acc + tap(g, r + (0), c + (13)));
    acc = (acc + tap(g, r + (0), c + (-11)));
    acc = (acc + tap(g, r + (3), c + (12)));
    acc = (acc + tap(g, r + (-3), c + (-9)));
    acc = (acc + tap(g, r + (-1), c + (9)));
    acc = (acc + tap(g, r + (2), c + (-2)));
    acc = (acc + tap(g, r + (-4), c + (-1)));
    acc = (acc + tap(g, r + (-8), c + (-10)));
    acc = (acc + tap(g, r + (-3), c + (9)));
    acc = (acc + tap(g, r + (-2), c + (-7)));
    acc = (acc + tap(g, r + (-4), c + (-7)));
    acc = (acc + tap(g, r + (-6), c + (-4)));
    acc = (acc + tap(g, r + (-8), c + (8)));
    acc = (acc + tap(g, r + (-6), c + (2)));
    acc = (acc + tap(g, r + (-8), c + (4)));
    acc = (acc + tap(g, r + (-3), c + (-3)));
    acc = (acc + tap(g, r + (-7), c + (-4)));
    acc = (acc + tap(g, r + (-1), c + (-5)));
    acc = (acc + tap(g, r + (-4), c + (4)));
    acc = (acc + tap(g, r + (-2), c + (-3)));
    acc = (acc + tap(g, r + (-3), c + (3)));
    acc = (acc + tap(g, r + (-2), c + (-3)));
    h += 7073340u;
    h = h * 2260532039u;
    h ^= h >> 13;
    h = h * 2143133189u;
    if (acc > 0.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 5088810u;
    h += 8204398u;
    h = h * 4051928767u;
    h ^= h >> 13;
    h += 15790155u;
    if (acc > -0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h = h * 4092053631u;
    h ^= h >> 13;
    if (acc > 0.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 304383197u;
    h += 12785365u;
    h = h * 142237903u;
    h ^= h >> 13;
    h ^= h >> 13;
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
