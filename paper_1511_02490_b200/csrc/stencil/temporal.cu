// Host side of the temporally blocked paths: the
// bit-plane Game of Life (pack -> k_gol_strips x ceil(iterations / TB) ->
// unpack) and the register-strip cross stencils (k_cross_strips), their
// legality plans and launches.  Called from launch() / sk_stencil_iterate /
// sk_stencil_probe (launch.cu) and the peer schedules (peer.cu).
#include "launch_internal.cuh"

namespace sk {
namespace detail {

// ------------------------------------------------------- bit-plane (gol)
KernelPtr pack_kernel(int dtype) {
  switch (dtype) {
    case SK_INT32: return gol_pack_i32();
    case SK_FLOAT32: return gol_pack_f32();
    default: return gol_pack_f64();
  }
}
KernelPtr unpack_kernel(int dtype) {
  switch (dtype) {
    case SK_INT32: return gol_unpack_i32();
    case SK_FLOAT32: return gol_unpack_f32();
    default: return gol_unpack_f64();
  }
}

// Rows per lane of the strip kernel: the descriptor's K in {8, 16, 32}, or 16.
int strip_rows(const sk_stencil_desc& d) { return d.cells_per_thread > 0 ? d.cells_per_thread : 16; }

// Legality and geometry of one k_gol_strips launch advancing `tb`
// generations of a packed W x H grid whose readable rows are [lo, hi].
int make_strips_plan(const sk_stencil_desc& d, long long W, long long H, long long lo,
                     long long hi, int wc, int wr, int tb, StripPlan* plan) {
  if (W < 1 || H < 1 || W > (1LL << 30) || H > (1LL << 30)) return fail(SK_EINVAL, "bad dims %lldx%lld", W, H);
  if (wc < 1 || wr < 1) return fail(SK_EINVAL, "bad workgroup %dx%d", wc, wr);
  if (tb < 1 || tb > kMaxBitsTB) return fail(SK_EINVAL, "bad generation count %d", tb);
  DeviceInfo info;
  int dev = 0;
  if (int rc = current_device_info(&info, &dev)) return rc;
  const int R = strip_rows(d);
  plan->kernel = gol_strips(R);
  if (!plan->kernel) return fail(SK_EINVAL, "bit-plane rows per work-item must be 8, 16 or 32");
  KernelAttr attr;
  if (int rc = kernel_attr(dev, plan->kernel, info, &attr)) return rc;
  plan->kernel_max = std::min(info.max_threads, attr.max_threads);
  const long long threads = static_cast<long long>(wc) * wr;
  if (threads > plan->kernel_max) {
    return fail(SK_OVERSIZED, "workgroup %dx%d exceeds the effective maximum %d", wc, wr,
                plan->kernel_max);
  }
  plan->threads = static_cast<int>((threads + 31) / 32 * 32);
  const int nwarps = plan->threads / 32;
  StripGeom& g = plan->g;
  g.W = static_cast<int>(W);
  g.H = static_cast<int>(H);
  g.lo = static_cast<int>(lo);
  g.hi = static_cast<int>(hi);
  g.nwords = static_cast<int>((W + 31) / 32);
  g.tb = tb;
  g.hw = (tb + 31) / 32;
  g.ow = 32 - 2 * g.hw;
  g.th = nwarps * R - 2 * tb;
  if (g.th < 1 || g.ow < 1) {
    return fail(SK_REFUSED, "a %d-row x 32-word tile cannot hold %d halo generations", nwarps * R, tb);
  }
  g.tiles_x = (g.nwords + g.ow - 1) / g.ow;
  g.tiles_y = static_cast<int>((H + g.th - 1) / g.th);
  g.mode = d.border_mode;
  const double padv = d.pad_value;
  const bool pad_alive = d.dtype == SK_INT32 ? static_cast<int32_t>(padv) != 0
                         : d.dtype == SK_FLOAT32 ? static_cast<float>(padv) != 0.0f
                                                 : padv != 0.0;
  g.padword = pad_alive ? 0xffffffffu : 0u;
  plan->tile_bytes = static_cast<long long>(nwarps) * R * 32 * 4;  // bit tile in registers
  plan->smem = (2 * nwarps * 64 + 64) * 4;
  if (plan->smem > attr.max_dyn_smem) return fail(SK_REFUSED, "exchange area exceeds shared memory");
  if (occupancy(dev, plan->kernel, plan->threads, plan->smem) < 1) {
    return fail(SK_REFUSED, "no resident block possible for %dx%d", wc, wr);
  }
  plan->grid = static_cast<long long>(g.tiles_x) * g.tiles_y;
  if (plan->grid >= (1LL << 31)) return fail(SK_REFUSED, "grid of %lld tiles too large", plan->grid);
  return SK_OK;
}

// `iterations` generations of gol on the bit-plane path: pack (T -> bits,
// rows [-above, H + below) when the generations fit one launch), then
// ceil(iterations / TB) strip launches ping-ponging two packed grids, then
// unpack into `out`.  Halo rows are only meaningful for a single launch
// (iterations <= TB), as for sk_stencil_launch on a row shard.
int run_bits(const sk_stencil_desc& d, const void* in, void* out, long long W, long long H,
             long long pitch_in, long long pitch_out, long long above, long long below, int wc,
             int wr, int iterations, int TB, cudaStream_t stream) {
  if (pitch_in < W || pitch_out < W) return fail(SK_EINVAL, "pitch smaller than width");
  TB = std::max(1, TB);
  const long long a = iterations <= TB ? std::min<long long>(above, iterations) : 0;
  const long long b = iterations <= TB ? std::min<long long>(below, iterations) : 0;
  StripPlan first;
  if (int rc = make_strips_plan(d, W, H, -a, H - 1 + b, wc, wr, std::max(1, std::min(TB, iterations)),
                                &first)) {
    return rc;
  }
  if (iterations == 0) return SK_OK;
  const long long pw = (first.g.nwords + 3) / 4 * 4;  // 16-B packed rows
  // Packed ping-pong grids, allocated stream-ordered on the caller's stream
  // and freed on it when this call's launches are enqueued: concurrent calls
  // on different streams (streamed host jobs, user streams) never share them.
  StreamBits bits(stream);
  if (int rc = bits.alloc(static_cast<size_t>(pw * (H + a + b)) * 4)) return rc;
  void* P[2] = {bits.p[0], bits.p[1]};
  DeviceInfo info;
  if (int rc = current_device_info(&info)) return rc;
  const int cvt_grid = 4 * info.sms * 8;  // 8 warps per block, grid-stride
  {  // pack rows [-a, H + b) of `in` into P[0]
    const void* base = static_cast<const char*>(in) - a * pitch_in * static_cast<long long>(dtype_size(d.dtype));
    int row0 = 0, rows = static_cast<int>(H + a + b), w = static_cast<int>(W);
    long long pi = pitch_in, pwl = pw;
    void* args[] = {&base, &pi, &row0, &rows, &w, &P[0], &pwl};
    if (int rc = launch_checked(pack_kernel(d.dtype), dim3(cvt_grid), dim3(256), args, 0, stream)) return rc;
  }
  int cur = 0, done = 0;
  for (bool firstl = true; done < iterations; firstl = false) {
    const int tb = std::min(TB, iterations - done);
    StripPlan plan;
    if (int rc = make_strips_plan(d, W, H, firstl ? -a : 0, firstl ? H - 1 + b : H - 1, wc, wr, tb, &plan)) {
      return rc;
    }
    plan.g.pw_in = pw;
    plan.g.pw_out = pw;
    const uint32_t* src = static_cast<const uint32_t*>(P[cur]) + (firstl ? a * pw : 0);
    uint32_t* dst = static_cast<uint32_t*>(P[1 - cur]);
    void* args[] = {&src, &dst, &plan.g};
    if (int rc = launch_pdl_checked(plan.kernel, dim3(static_cast<unsigned>(plan.grid)), dim3(plan.threads),
                                    args, plan.smem, stream)) {
      return rc;
    }
    cur = 1 - cur;
    done += tb;
  }
  {  // unpack P[cur] rows [0, H) into `out`
    const void* src = P[cur];
    long long pwl = pw, po = pitch_out;
    int rows = static_cast<int>(H), w = static_cast<int>(W);
    int vec = (pitch_out % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
    void* args[] = {&src, &pwl, &rows, &w, &out, &po, &vec};
    if (int rc = launch_checked(unpack_kernel(d.dtype), dim3(cvt_grid), dim3(256), args, 0, stream)) return rc;
  }
  return SK_OK;
}

// ------------------------------------------- register strips (cross ops)
KernelPtr cross_kernel(const sk_stencil_desc& d, int R) {
  switch (d.dtype) {
    case SK_INT32: return cross_strips_i32(d, R);
    case SK_FLOAT32: return cross_strips_f32(d, R);
    default: return cross_strips_f64(d, R);
  }
}

// Rows per lane of the cross-strip kernel: the descriptor's K in {4, 8, 16},
// or 8 (4 for float64, whose 8-row strips spill) - two resident blocks per SM.
int cross_rows(const sk_stencil_desc& d) {
  return d.cells_per_thread > 0 ? d.cells_per_thread : (d.dtype == SK_FLOAT64 ? 4 : 8);
}

// Legality and geometry of one k_cross_strips launch advancing `tb`
// generations of a W x H region whose readable input rows are [lo, hi].
int make_cross_plan(const sk_stencil_desc& d, long long W, long long H, long long pitch_in,
                    long long pitch_out, long long lo, long long hi, int wc, int wr, int tb,
                    const void* in, const void* out, CrossPlan* plan) {
  if (W < 1 || H < 1 || W > (1LL << 30) || H > (1LL << 30)) return fail(SK_EINVAL, "bad dims %lldx%lld", W, H);
  if (pitch_in < W || pitch_out < W) return fail(SK_EINVAL, "pitch smaller than width");
  if (wc < 1 || wr < 1) return fail(SK_EINVAL, "bad workgroup %dx%d", wc, wr);
  if (tb < 1 || tb > kMaxStripsTB) return fail(SK_EINVAL, "bad generation count %d", tb);
  DeviceInfo info;
  int dev = 0;
  if (int rc = current_device_info(&info, &dev)) return rc;
  const int R = cross_rows(d);
  plan->kernel = cross_kernel(d, R);
  if (!plan->kernel) return fail(SK_EINVAL, "register-strip rows per work-item must be 4, 8 or 16");
  KernelAttr attr;
  if (int rc = kernel_attr(dev, plan->kernel, info, &attr)) return rc;
  plan->kernel_max = std::min(info.max_threads, attr.max_threads);
  const long long threads = static_cast<long long>(wc) * wr;
  if (threads > plan->kernel_max) {
    return fail(SK_OVERSIZED, "workgroup %dx%d exceeds the effective maximum %d", wc, wr,
                plan->kernel_max);
  }
  plan->threads = static_cast<int>((threads + 31) / 32 * 32);
  const int nwarps = plan->threads / 32;
  CrossGeom& g = plan->g;
  g.pitch_in = pitch_in;
  g.pitch_out = pitch_out;
  g.W = static_cast<int>(W);
  g.H = static_cast<int>(H);
  g.lo = static_cast<int>(lo);
  g.hi = static_cast<int>(hi);
  g.tb = tb;
  g.hl = (tb + 3) / 4;
  g.oc = 4 * (32 - 2 * g.hl);
  g.th = nwarps * R - 2 * tb;
  if (g.th < 1 || g.oc < 4) {
    return fail(SK_REFUSED, "a %d-row x 128-column tile cannot hold %d halo generations", nwarps * R, tb);
  }
  g.tiles_x = static_cast<int>((W + g.oc - 1) / g.oc);
  g.tiles_y = static_cast<int>((H + g.th - 1) / g.th);
  g.mode = d.border_mode;
  const size_t es = dtype_size(d.dtype);
  g.vec = (pitch_in % 4 == 0) && (pitch_out % 4 == 0) &&
          (reinterpret_cast<uintptr_t>(in) % (4 * es) == 0) &&
          (reinterpret_cast<uintptr_t>(out) % (4 * es) == 0);
  plan->tile_bytes = static_cast<long long>(nwarps) * R * 128 * static_cast<long long>(es);  // in registers
  plan->smem = static_cast<int>(2 * nwarps * 64 * 4 * es);
  if (plan->smem > attr.max_dyn_smem) return fail(SK_REFUSED, "exchange area exceeds shared memory");
  if (occupancy(dev, plan->kernel, plan->threads, plan->smem) < 1) {
    return fail(SK_REFUSED, "no resident block possible for %dx%d", wc, wr);
  }
  plan->grid = static_cast<long long>(g.tiles_x) * g.tiles_y;
  if (plan->grid >= (1LL << 31)) return fail(SK_REFUSED, "grid of %lld tiles too large", plan->grid);
  return SK_OK;
}

template <typename T>
int launch_cross_typed(const sk_stencil_desc& d, const CrossPlan& plan, const void* in, void* out,
                       cudaStream_t stream) {
  OpParams<T> p;
  fill_params<T>(d, &p);
  T pad = static_cast<T>(d.pad_value);
  const T* tin = static_cast<const T*>(in);
  T* tout = static_cast<T*>(out);
  void* args[] = {&tin, &tout, const_cast<CrossGeom*>(&plan.g), &pad, &p};
  return launch_pdl_checked(plan.kernel, dim3(static_cast<unsigned>(plan.grid)), dim3(plan.threads), args,
                            plan.smem, stream);
}

// One k_cross_strips launch: `tb` generations from `in` (row 0 of the region,
// `above` / `below` readable halo rows) into `out`.
int run_cross(const sk_stencil_desc& d, const void* in, void* out, long long W, long long H,
              long long pitch_in, long long pitch_out, long long above, long long below, int wc,
              int wr, int tb, cudaStream_t stream) {
  CrossPlan plan;
  if (int rc = make_cross_plan(d, W, H, pitch_in, pitch_out, -above, H - 1 + below, wc, wr, tb, in,
                               out, &plan)) {
    return rc;
  }
  switch (d.dtype) {
    case SK_INT32: return launch_cross_typed<int32_t>(d, plan, in, out, stream);
    case SK_FLOAT32: return launch_cross_typed<float>(d, plan, in, out, stream);
    default: return launch_cross_typed<double>(d, plan, in, out, stream);
  }
}

}  // namespace detail
}  // namespace sk
