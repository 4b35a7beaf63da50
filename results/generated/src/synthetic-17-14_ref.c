/* CPU reference of generated kernel 'synthetic-17-14' (build with -ffp-contract=off). */
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
    acc = (acc + tap(g, r + (-9), c + (0)));
    acc = (acc + tap(g, r + (15), c + (0)));
    acc = (acc + tap(g, r + (0), c + (18)));
    acc = (acc + tap(g, r + (0), c + (-9)));
    acc = (acc + tap(g, r + (6), c + (1)));
    acc = (acc + tap(g, r + (2), c + (0)));
    acc = (acc + tap(g, r + (-7), c + (-6)));
    acc = (acc + tap(g, r + (-2), c + (4)));
    acc = (acc + tap(g, r + (10), c + (-7)));
    acc = (acc + tap(g, r + (10), c + (2)));
    acc = (acc + tap(g, r + (8), c + (-1)));
    acc = (acc + tap(g, r + (-9), c + (4)));
    acc = (acc + tap(g, r + (9), c + (2)));
    acc = (acc + tap(g, r + (12), c + (15)));
    acc = (acc + tap(g, r + (-9), c + (3)));
    acc = (acc + tap(g, r + (-7), c + (12)));
    acc = (acc + tap(g, r + (0), c + (11)));
    acc = (acc + tap(g, r + (9), c + (10)));
    acc = (acc + tap(g, r + (11), c + (12)));
    acc = (acc + tap(g, r + (12), c + (0)));
    acc = (acc + tap(g, r + (7), c + (2)));
    acc = (acc + tap(g, r + (-9), c + (5)));
    acc = (acc + tap(g, r + (9), c + (17)));
    acc = (acc + tap(g, r + (5), c + (11)));
    acc = (acc + tap(g, r + (0), c + (13)));
    if (acc > -0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    h ^= h >> 13;
    if (acc > 0.875f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 2363140221u;
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 3890504933u;
    h ^= h >> 13;
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 1238453427u;
    if (acc > 0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 14753292u;
    h += 14088752u;
    if (acc > -0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.125f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.75f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > -0.375f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h = h * 3246405247u;
    h = h * 1031371369u;
    if (acc > -0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.25f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h ^= h >> 13;
    if (acc > -1.0f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    if (acc > 0.5f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    h += 12934025u;
    h += 6479115u;
    h ^= h >> 13;
    if (acc > 0.625f) acc = (acc * 0.5f); else acc = (acc + 0.25f);
    return (acc + ((float)(h & 255u) * 0.0009765625f));
}
void gen_grid(const float* in, float* out, long W, long H, int mode, float pad) {
  grid_t g = {in, W, H, mode, pad};
  for (long r = 0; r < H; ++r)
    for (long c = 0; c < W; ++c) out[r * W + c] = cell(&g, r, c);
}
