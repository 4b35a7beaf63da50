/* CPU reference of generated kernel 'synthetic-17-2' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (-6), c + (0)));
    acc = (acc + tap(g, r + (29), c + (0)));
    acc = (acc + tap(g, r + (0), c + (28)));
    acc = (acc + tap(g, r + (0), c + (-17)));
    acc = (acc + tap(g, r + (12), c + (16)));
    acc = (acc + tap(g, r + (23), c + (1)));
    acc = (acc + tap(g, r + (25), c + (-4)));
    acc = (acc + tap(g, r + (19), c + (14)));
    acc = (acc + tap(g, r + (29), c + (-8)));
    acc = (acc + tap(g, r + (14), c + (22)));
    acc = (acc + tap(g, r + (15), c + (-14)));
    acc = (acc + tap(g, r + (-4), c + (26)));
    acc = (acc + tap(g, r + (-2), c + (3)));
    acc = (acc + tap(g, r + (-4), c + (24)));
    acc = (acc + tap(g, r + (8), c + (1)));
    acc = (acc + tap(g, r + (28), c + (26)));
    acc = (acc + tap(g, r + (18), c + (-10)));
    acc = (acc + tap(g, r + (9), c + (-3)));
    acc = (acc + tap(g, r + (14), c + (19)));
    acc = (acc + tap(g, r + (18), c + (17)));
    acc = (acc + tap(g, r + (27), c + (20)));
    acc = (acc + tap(g, r + (22), c + (27)));
    acc = (acc + tap(g, r + (25), c + (10)));
    acc = (acc + tap(g, r + (16), c + (7)));
    acc = (acc + tap(g, r + (-3), c + (-11)));
    acc = (acc + tap(g, r + (-2), c + (-2)));
    acc = (acc + tap(g, r + (13), c + (-7)));
    acc = (acc + tap(g, r + (6), c + (15)));
    acc = (acc + tap(g, r + (21), c + (25)));
    acc = (acc + tap(g, r + (13), c + (15)));
    acc = (acc + tap(g, r + (23), c + (12)));
    acc = (acc + tap(g, r + (23), c + (8)));
    acc = (acc + tap(g, r + (8), c + (12)));
    h += 5294242u;
    h += 8682510u;
    h += 12941646u;
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 3149905901u;
    if (acc > -0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 3239627u;
    h ^= h >> 13;
    h += 6184718u;
    h ^= h >> 13;
    if (acc > 0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h ^= h >> 13;
    if (acc > 0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 2354964u;
    h ^= h >> 13;
    if (acc > 0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 2411951325u;
    h += 1763681u;
    h = h * 4112452607u;
    h = h * 3204506977u;
    h ^= h >> 13;
    if (acc > 0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 3021958799u;
    h = h * 2322392851u;
    h = h * 1520085491u;
    if (acc > 0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 1802922399u;
    h ^= h >> 13;
    if (acc > -0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
