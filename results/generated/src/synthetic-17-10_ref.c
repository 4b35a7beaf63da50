/* CPU reference of generated kernel 'synthetic-17-10' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (11), c + (0)));
    acc = (acc + tap(g, r + (0), c + (18)));
    acc = (acc + tap(g, r + (0), c + (-10)));
    acc = (acc + tap(g, r + (-6), c + (16)));
    acc = (acc + tap(g, r + (1), c + (18)));
    acc = (acc + tap(g, r + (5), c + (11)));
    acc = (acc + tap(g, r + (11), c + (12)));
    acc = (acc + tap(g, r + (-4), c + (8)));
    acc = (acc + tap(g, r + (8), c + (-1)));
    acc = (acc + tap(g, r + (-6), c + (13)));
    acc = (acc + tap(g, r + (1), c + (-8)));
    acc = (acc + tap(g, r + (-6), c + (12)));
    acc = (acc + tap(g, r + (9), c + (13)));
    acc = (acc + tap(g, r + (-3), c + (-10)));
    acc = (acc + tap(g, r + (3), c + (6)));
    acc = (acc + tap(g, r + (0), c + (9)));
    acc = (acc + tap(g, r + (-3), c + (8)));
    acc = (acc + tap(g, r + (-6), c + (-2)));
    acc = (acc + tap(g, r + (1), c + (5)));
    acc = (acc + tap(g, r + (4), c + (-9)));
    acc = (acc + tap(g, r + (-4), c + (18)));
    acc = (acc + tap(g, r + (10), c + (15)));
    acc = (acc + tap(g, r + (8), c + (5)));
    acc = (acc + tap(g, r + (0), c + (9)));
    acc = (acc + tap(g, r + (10), c + (-1)));
    acc = (acc + tap(g, r + (10), c + (8)));
    acc = (acc + tap(g, r + (9), c + (5)));
    acc = (acc + tap(g, r + (10), c + (6)));
    acc = (acc + tap(g, r + (11), c + (14)));
    acc = (acc + tap(g, r + (7), c + (2)));
    acc = (acc + tap(g, r + (6), c + (5)));
    acc = (acc + tap(g, r + (6), c + (-8)));
    acc = (acc + tap(g, r + (9), c + (-8)));
    acc = (acc + tap(g, r + (10), c + (-2)));
    acc = (acc + tap(g, r + (-3), c + (-3)));
    acc = (acc + tap(g, r + (2), c + (14)));
    acc = (acc + tap(g, r + (8), c + (10)));
    acc = (acc + tap(g, r + (9), c + (0)));
    acc = (acc + tap(g, r + (11), c + (0)));
    acc = (acc + tap(g, r + (10), c + (-8)));
    acc = (acc + tap(g, r + (-4), c + (14)));
    acc = (acc + tap(g, r + (-6), c + (-6)));
    acc = (acc + tap(g, r + (5), c + (11)));
    acc = (acc + tap(g, r + (11), c + (-9)));
    acc = (acc + tap(g, r + (6), c + (-2)));
    acc = (acc + tap(g, r + (9), c + (-6)));
    h ^= h >> 13;
    h ^= h >> 13;
    if (acc > -0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h += 16365725u;
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 2726446513u;
    h = h * 3381417557u;
    if (acc > -0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 14301923u;
    if (acc > 0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h ^= h >> 13;
    if (acc > 0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 3546616061u;
    h = h * 3686355507u;
    h += 11755622u;
    h += 8225529u;
    h = h * 3127261499u;
    h = h * 7204439u;
    if (acc > 0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h += 2147845u;
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
