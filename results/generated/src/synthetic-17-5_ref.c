/* CPU reference of generated kernel 'synthetic-17-5' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (-19), c + (0)));
    acc = (acc + tap(g, r + (30), c + (0)));
    acc = (acc + tap(g, r + (0), c + (14)));
    acc = (acc + tap(g, r + (0), c + (-24)));
    acc = (acc + tap(g, r + (-15), c + (-14)));
    acc = (acc + tap(g, r + (19), c + (6)));
    acc = (acc + tap(g, r + (-16), c + (-5)));
    acc = (acc + tap(g, r + (-3), c + (-5)));
    acc = (acc + tap(g, r + (-13), c + (-18)));
    acc = (acc + tap(g, r + (14), c + (-4)));
    acc = (acc + tap(g, r + (7), c + (-8)));
    acc = (acc + tap(g, r + (-1), c + (-14)));
    acc = (acc + tap(g, r + (1), c + (-17)));
    acc = (acc + tap(g, r + (5), c + (-18)));
    acc = (acc + tap(g, r + (17), c + (12)));
    acc = (acc + tap(g, r + (-19), c + (-21)));
    acc = (acc + tap(g, r + (25), c + (12)));
    acc = (acc + tap(g, r + (0), c + (-12)));
    acc = (acc + tap(g, r + (4), c + (-22)));
    acc = (acc + tap(g, r + (20), c + (6)));
    acc = (acc + tap(g, r + (21), c + (-14)));
    acc = (acc + tap(g, r + (-17), c + (1)));
    acc = (acc + tap(g, r + (29), c + (-4)));
    acc = (acc + tap(g, r + (13), c + (-10)));
    acc = (acc + tap(g, r + (11), c + (-19)));
    acc = (acc + tap(g, r + (-12), c + (-22)));
    acc = (acc + tap(g, r + (16), c + (13)));
    acc = (acc + tap(g, r + (-9), c + (-15)));
    acc = (acc + tap(g, r + (18), c + (-19)));
    acc = (acc + tap(g, r + (1), c + (-6)));
    acc = (acc + tap(g, r + (30), c + (-15)));
    acc = (acc + tap(g, r + (26), c + (12)));
    acc = (acc + tap(g, r + (25), c + (1)));
    acc = (acc + tap(g, r + (-17), c + (3)));
    acc = (acc + tap(g, r + (-9), c + (-2)));
    acc = (acc + tap(g, r + (-16), c + (9)));
    acc = (acc + tap(g, r + (11), c + (-19)));
    acc = (acc + tap(g, r + (30), c + (4)));
    acc = (acc + tap(g, r + (26), c + (1)));
    acc = (acc + tap(g, r + (7), c + (-16)));
    acc = (acc + tap(g, r + (-9), c + (9)));
    acc = (acc + tap(g, r + (-12), c + (11)));
    acc = (acc + tap(g, r + (-19), c + (-12)));
    acc = (acc + tap(g, r + (26), c + (6)));
    h ^= h >> 13;
    h = h * 1126470991u;
    if (acc > -0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 13744698u;
    if (acc > 0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h = h * 3506133431u;
    h ^= h >> 13;
    if (acc > 0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 8858525u;
    h ^= h >> 13;
    h += 7584970u;
    h ^= h >> 13;
    h = h * 2029920263u;
    h = h * 3534441363u;
    if (acc > 0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 16488206u;
    if (acc > -0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 5740933u;
    h = h * 1397641321u;
    h ^= h >> 13;
    h += 2576550u;
    if (acc > 1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h += 15138912u;
    h ^= h >> 13;
    h = h * 943280561u;
    h = h * 3644965085u;
    h = h * 1003153359u;
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 10674412u;
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
