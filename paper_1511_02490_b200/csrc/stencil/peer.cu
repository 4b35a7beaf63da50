// Host side of the peer-memory halo exchange for row-sharded iterated
// stencils: CUDA IPC mapping, the one-generation
// schedule (strips kernel with fused put + signal, interior on a side lane;
// or the opt-in PEER one-pass kernel) and the temporally blocked schedule of
// the register-strip path.
#include "launch_internal.cuh"

namespace sk {
namespace detail {

// Fork/join lane of a caller's stream for the peer schedule: the interior
// launch of a generation runs on `side` while the caller's stream runs the
// boundary strips (which may wait on a neighbour's flag).  Keyed by (device,
// caller stream): ranks sharing a process each bring their own stream, and
// one shared side stream would serialise their interiors into a cycle.
struct SideLane {
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
std::map<std::pair<int, cudaStream_t>, SideLane> g_side;

int side_lane(cudaStream_t st, SideLane** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SK_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_mu);
  SideLane& l = g_side[{dev, st}];
  if (!l.side) {
    if (cudaStreamCreateWithFlags(&l.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&l.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&l.join, cudaEventDisableTiming) != cudaSuccess) {
      return fail(SK_ECUDA, "side stream/event creation failed");
    }
  }
  *out = &l;
  return SK_OK;
}

// ------------------------------------------- peer-memory halo exchange
KernelPtr halo_kernel(const sk_stencil_desc& d) {
  switch (d.dtype) {
    case SK_INT32: return halo_strips_i32(d);
    case SK_FLOAT32: return halo_strips_f32(d);
    default: return halo_strips_f64(d);
  }
}
// True when a (peer) device pointer lives on the current device.
bool peer_on_device(const void* p) {
  int dev = 0;
  cudaPointerAttributes a;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.device == dev;
}

KernelPtr peer_tma_kernel(const sk_stencil_desc& d, int K) {
  switch (d.dtype) {
    case SK_INT32: return peer_tma_i32(d, K);
    case SK_FLOAT32: return peer_tma_f32(d, K);
    default: return peer_tma_f64(d, K);
  }
}

KernelPtr halo_put_kernel(int dtype) {
  switch (dtype) {
    case SK_INT32: return halo_put_i32();
    case SK_FLOAT32: return halo_put_f32();
    default: return halo_put_f64();
  }
}

template <typename T>
int launch_halo_strips(const sk_stencil_desc& d, const void* src, void* dst, void* peer_n,
                       void* peer_s, const long long* flag_n, const long long* flag_s,
                       long long* pflag_n, long long* pflag_s, unsigned* done, const HaloGeom& g,
                       int grid_x, cudaStream_t stream) {
  OpParams<T> p;
  fill_params<T>(d, &p);
  T pad = static_cast<T>(d.pad_value);
  void* args[] = {const_cast<void**>(&src), &dst, &peer_n, &peer_s, const_cast<long long**>(&flag_n),
                  const_cast<long long**>(&flag_s), &pflag_n, &pflag_s, &done,
                  const_cast<HaloGeom*>(&g), &pad, &p};
  return launch_checked(halo_kernel(d), dim3(grid_x, 2), dim3(256), args, 0, stream);
}

// Temporally blocked peer schedule (register-strip path, TB generations per
// exchange).  The shard buffers carry TB-deep halos: TB*N rows above, TB*S
// below.  Per launch k (generations (k-1)TB+1 .. kTB, the last one shorter):
//   k_halo_wait   acquire the neighbours' state-(k-1) halos (value B + k);
//   strips        k_cross_strips over the top / bottom m = TB*max(N,S) rows;
//   k_halo_put    their first TB*S / last TB*N rows into the neighbours' halos,
//                 publish B + k + 1 (last block, release.sys);
//   interior      k_cross_strips over rows [m, rows - m), owned rows only.
// Same one-flag-per-direction argument as the one-generation schedule: the
// neighbour publishes state k only after its launch-k strip pass - the last
// reader of the halo rows overwritten by launch k+1's put - has run.
int iterate_peer_strips(const sk_stencil_desc& d, void* d_a, void* d_b, int64_t width, int64_t rows,
                        int64_t pitch, int32_t iterations, int32_t wc, int32_t wr,
                        const sk_halo_peers& peers, void* d_control, int64_t* epoch,
                        cudaStream_t st, int32_t* result_in_b) {
  const int TB = d.fused_iterations;
  const int Nh = TB * d.north, Sh = TB * d.south;
  const int m = std::max(Nh, Sh);
  if (width < 1 || pitch < width || rows < 2LL * m + std::max(Nh, Sh)) {
    return fail(SK_EINVAL, "shard of %lld rows cannot hold %d-generation strips of %d rows",
                (long long)rows, TB, m);
  }
  if ((peers.north_a == nullptr) != (peers.north_b == nullptr) ||
      (peers.north_a == nullptr) != (peers.north_control == nullptr) ||
      (peers.south_a == nullptr) != (peers.south_b == nullptr) ||
      (peers.south_a == nullptr) != (peers.south_control == nullptr)) {
    return fail(SK_EINVAL, "incomplete peer mapping");
  }
  const bool has_n = peers.north_a != nullptr, has_s = peers.south_a != nullptr;
  if (has_n && peers.north_rows < 2LL * m) return fail(SK_EINVAL, "bad north_rows");
  const size_t es = dtype_size(d.dtype);
  const long long row_bytes = pitch * static_cast<long long>(es);
  long long* ctl = static_cast<long long*>(d_control);
  const long long* flag_n = has_n ? ctl + 0 : nullptr;
  const long long* flag_s = has_s ? ctl + 1 : nullptr;
  unsigned* done = reinterpret_cast<unsigned*>(ctl + 2);
  long long* pflag_n = has_n ? static_cast<long long*>(peers.north_control) + 1 : nullptr;
  long long* pflag_s = has_s ? static_cast<long long*>(peers.south_control) + 0 : nullptr;
  DeviceInfo info;
  int dev = 0;
  if (int rc = current_device_info(&info, &dev)) return rc;

  HaloGeom g{};
  g.pitch = pitch;
  g.W = static_cast<int>(width);
  g.h = static_cast<int>(rows);
  g.north_rows = Sh;
  g.south_rows = Nh;
  g.north_off = has_n ? (Nh + peers.north_rows) * pitch : 0;
  g.south_off = 0;
  g.mode = d.border_mode;
  const long long B = *epoch;
  const long long inner = rows - 2LL * m;

  // Resolve every kernel before the first launch (lazy loading; see the
  // one-generation schedule).
  {
    KernelAttr ka;
    if (int rc = kernel_attr(dev, halo_wait(), info, &ka)) return rc;
    if (int rc = kernel_attr(dev, halo_put_kernel(d.dtype), info, &ka)) return rc;
    CrossPlan cp;
    const char* a0 = static_cast<const char*>(d_a) + Nh * row_bytes;
    if (int rc = make_cross_plan(d, width, m, pitch, pitch, -Nh, m - 1 + Sh, wc, wr, TB, a0, a0, &cp)) return rc;
    if (int rc = make_cross_plan(d, width, inner, pitch, pitch, -Nh, inner - 1 + Sh, wc, wr, TB, a0, a0, &cp)) {
      return rc;
    }
  }
  const int put_grid = static_cast<int>(std::max<long long>(
      1, std::min<long long>((static_cast<long long>(Nh + Sh) * width + 255) / 256, 4LL * info.sms)));
  auto put = [&](const void* src_rows, void* pn, void* ps, long long wait, long long signal) {
    g.wait_value = wait;
    g.signal_value = signal;
    void* args[] = {const_cast<void**>(&src_rows), &pn, &ps, const_cast<long long**>(&flag_n),
                    const_cast<long long**>(&flag_s), &pflag_n, &pflag_s, &done, &g};
    return launch_checked(halo_put_kernel(d.dtype), dim3(put_grid), dim3(256), args, 0, st);
  };
  // state-0 halos
  if (int rc = put(static_cast<const char*>(d_a) + Nh * row_bytes, peers.north_a, peers.south_a, B, B + 1)) {
    return rc;
  }
  void* src = d_a;
  void* dst = d_b;
  int launches = 0;
  for (int done_gens = 0; done_gens < iterations; ++launches) {
    const int tb = std::min(TB, iterations - done_gens);
    const long long k = launches + 1;
    {
      long long value = B + k;
      void* args[] = {const_cast<long long**>(&flag_n), const_cast<long long**>(&flag_s), &value};
      if (int rc = launch_checked(halo_wait(), dim3(1), dim3(32), args, 0, st)) return rc;
    }
    const char* s0 = static_cast<const char*>(src) + Nh * row_bytes;
    char* d0 = static_cast<char*>(dst) + Nh * row_bytes;
    // top strip: reads the north halo (if any) and TB*S owned rows below it
    if (int rc = run_cross(d, s0, d0, width, m, pitch, pitch, has_n ? Nh : 0, Sh, wc, wr, tb, st)) return rc;
    // bottom strip
    if (int rc = run_cross(d, s0 + (rows - m) * row_bytes, d0 + (rows - m) * row_bytes, width, m, pitch,
                           pitch, Nh, has_s ? Sh : 0, wc, wr, tb, st)) {
      return rc;
    }
    void* pn = has_n ? (k & 1 ? peers.north_b : peers.north_a) : nullptr;
    void* ps = has_s ? (k & 1 ? peers.south_b : peers.south_a) : nullptr;
    if (int rc = put(d0, pn, ps, B + k, B + k + 1)) return rc;
    if (inner > 0) {
      if (int rc = run_cross(d, s0 + m * row_bytes, d0 + m * row_bytes, width, inner, pitch, pitch, Nh, Sh,
                             wc, wr, tb, st)) {
        return rc;
      }
    }
    done_gens += tb;
    std::swap(src, dst);
  }
  *epoch = B + launches + 1;
  if (result_in_b) *result_in_b = launches % 2;
  return SK_OK;
}

}  // namespace detail
}  // namespace sk

using namespace sk;
using namespace sk::detail;

extern "C" {

int sk_ipc_export(const void* d_ptr, sk_ipc_handle* out) {
  g_last_error.clear();
  if (!d_ptr || !out) return fail(SK_EINVAL, "null argument");
  CUdeviceptr base = 0;
  size_t size = 0;
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<GetRange>(nullptr);
    }
    return reinterpret_cast<GetRange>(fn);
  }();
  if (!get_range) return fail(SK_ECUDA, "cuMemGetAddressRange unavailable");
  if (get_range(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS) {
    return fail(SK_EINVAL, "pointer is not device memory");
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(SK_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) <= sizeof(out->handle), "IPC handle size");
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->handle, &h, sizeof(h));
  out->offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(d_ptr) - base);
  return SK_OK;
}

int sk_ipc_import(const sk_ipc_handle* h, void** d_ptr) {
  g_last_error.clear();
  if (!h || !d_ptr) return fail(SK_EINVAL, "null argument");
  cudaIpcMemHandle_t mh;
  std::memcpy(&mh, h->handle, sizeof(mh));
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(SK_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  *d_ptr = static_cast<char*>(base) + h->offset;
  return SK_OK;
}

int sk_ipc_close(void* d_ptr) {
  g_last_error.clear();
  // cudaIpcCloseMemHandle takes the mapped base; imported pointers carry an
  // offset, so resolve the containing mapping first.
  CUdeviceptr base = 0;
  size_t size = 0;
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess ||
      reinterpret_cast<GetRange>(fn)(&base, &size, reinterpret_cast<CUdeviceptr>(d_ptr)) != CUDA_SUCCESS) {
    cudaGetLastError();
    return fail(SK_EINVAL, "pointer is not a mapped device allocation");
  }
  cudaError_t e = cudaIpcCloseMemHandle(reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(SK_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return SK_OK;
}

int sk_stencil_iterate_peer(const sk_stencil_desc* desc, void* d_a, void* d_b, int64_t width,
                            int64_t rows, int64_t pitch, int32_t iterations, int32_t wc,
                            int32_t wr, const sk_halo_peers* peers, void* d_control,
                            int64_t* epoch, void* stream, int32_t* result_in_b) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  const sk_stencil_desc& d = *desc;
  if (!d_a || !d_b || !peers || !d_control || !epoch) return fail(SK_EINVAL, "null argument");
  if (iterations < 0) return fail(SK_EINVAL, "negative iterations");
  if (uses_strips(d) && d.fused_iterations > 1) {
    return iterate_peer_strips(d, d_a, d_b, width, rows, pitch, iterations, wc, wr, *peers,
                               d_control, epoch, static_cast<cudaStream_t>(stream), result_in_b);
  }
  if (d.fused_iterations > 1 || uses_bits(d) || uses_strips(d)) {
    return fail(SK_ENOTSUP, "the peer-exchange schedule fuses generations only on the register-strip path");
  }
  const int N = d.north, S = d.south;
  const int m = std::max(N, S);
  if (width < 1 || pitch < width || rows < std::max(m, 1)) {
    return fail(SK_EINVAL, "shard of %lld rows cannot hold halos of N=%d, S=%d", (long long)rows, N, S);
  }
  if ((peers->north_a == nullptr) != (peers->north_b == nullptr) ||
      (peers->north_a == nullptr) != (peers->north_control == nullptr) ||
      (peers->south_a == nullptr) != (peers->south_b == nullptr) ||
      (peers->south_a == nullptr) != (peers->south_control == nullptr)) {
    return fail(SK_EINVAL, "incomplete peer mapping");
  }
  if (peers->north_a && peers->north_rows < std::max(m, 1)) return fail(SK_EINVAL, "bad north_rows");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool has_n = peers->north_a != nullptr, has_s = peers->south_a != nullptr;
  const size_t es = dtype_size(d.dtype);
  const long long row_bytes = pitch * static_cast<long long>(es);
  long long* ctl = static_cast<long long*>(d_control);
  const long long* flag_n = has_n ? ctl + 0 : nullptr;  // north halo arrivals (from p-1)
  const long long* flag_s = has_s ? ctl + 1 : nullptr;  // south halo arrivals (from p+1)
  unsigned* done = reinterpret_cast<unsigned*>(ctl + 2);
  // I deliver the north neighbour's SOUTH halo (its flag 1) and the south
  // neighbour's NORTH halo (its flag 0).
  long long* pflag_n = has_n ? static_cast<long long*>(peers->north_control) + 1 : nullptr;
  long long* pflag_s = has_s ? static_cast<long long*>(peers->south_control) + 0 : nullptr;
  DeviceInfo info;
  if (int rc = current_device_info(&info)) return rc;

  HaloGeom g{};
  g.pitch = pitch;
  g.W = static_cast<int>(width);
  g.h = static_cast<int>(rows);
  g.above = has_n ? N : 0;
  g.below = has_s ? S : 0;
  g.m = m;
  g.north_rows = S;
  g.south_rows = N;
  g.north_off = has_n ? (N + peers->north_rows) * pitch : 0;
  g.south_off = 0;
  g.mode = d.border_mode;
  const long long B = *epoch;

  // Resolve every kernel of the schedule before the first launch.  With CUDA
  // lazy loading, loading a module may wait for the context's running
  // kernels; a strip pass spinning on a peer whose launches this thread has
  // not issued yet (ranks sharing one process) would then never finish.
  {
    int dev = 0;
    if (int rc = current_device_info(&info, &dev)) return rc;
    KernelAttr ka;
    if (int rc = kernel_attr(dev, halo_kernel(d), info, &ka)) return rc;
    if (int rc = kernel_attr(dev, halo_put_kernel(d.dtype), info, &ka)) return rc;
    if (rows - 2LL * m > 0) {
      Plan plan;
      const char* a0 = static_cast<const char*>(d_a) + (N + m) * row_bytes;
      if (int rc = make_plan(d, width, rows - 2LL * m, pitch, pitch, N, S, wc, wr, a0, &plan)) return rc;
    }
  }

  // Fused path: one launch per generation of the one-pass TMA kernel with
  // the exchange folded into its boundary tile-rows (k_stencil_tma<..., PEER>),
  // when the TMA plan applies and every mirrored row lies in the first / last
  // tile-row.  Otherwise the strips + interior schedule below.
  // Opt-in (SK_PEER_SCHEDULE=fused).  Measured on one B200, one rank, GoL
  // 8192^2 at 128x8: the PEER instantiation executes 8.9 % more instructions
  // (the boundary-row remap and checks on every tile) and runs 104.5 us per
  // generation against 91.5 us for the plain one-pass kernel, worse than the
  // strips schedule (+7 %).  It is also persistent: its boundary blocks hold
  // their SMs while they wait for a neighbour's flag, so ranks sharing a GPU
  // can starve each other - never chosen for peers on this device.
  Plan fplan;
  KernelPtr peer_k = nullptr;
  const char* sched = std::getenv("SK_PEER_SCHEDULE");
  const bool shared_gpu = (has_n && peer_on_device(peers->north_a)) || (has_s && peer_on_device(peers->south_a));
  const bool forced = sched && std::strcmp(sched, "fused") == 0;
  if (forced && (!shared_gpu || std::getenv("SK_PEER_ALLOW_SHARED"))) {
    int dev = 0;
    current_device_info(&info, &dev);
    const char* a0 = static_cast<const char*>(d_a) + N * row_bytes;
    sk_stencil_desc scalar = d;  // the PEER kernels are scalar work-items
    if (scalar.load_path == SK_LOAD_AUTO) scalar.load_path = SK_LOAD_TMA;
    if (m > 0 && make_plan(scalar, width, rows, pitch, pitch, g.above, g.below, wc, wr, a0, &fplan) == SK_OK &&
        fplan.tma && !fplan.driver_handle && fplan.g.tile_rows >= m) {
      KernelPtr k = peer_tma_kernel(d, fplan.g.K);
      KernelAttr ka;
      if (k && kernel_attr(dev, k, info, &ka) == SK_OK && fplan.threads <= ka.max_threads &&
          fplan.smem <= ka.max_dyn_smem && occupancy(dev, k, fplan.threads, fplan.smem) >= 1) {
        peer_k = k;
      }
    }
    g_last_error.clear();
  }

  // generation 0 halos: put the initial boundary rows, publish B + 1
  {
    g.wait_value = B;
    g.signal_value = B + 1;
    const void* src = static_cast<const char*>(d_a) + N * row_bytes;
    void* pn = peers->north_a;
    void* ps = peers->south_a;
    const long long cells = static_cast<long long>(S + N) * width;
    const int grid = static_cast<int>(std::max<long long>(1, std::min<long long>((cells + 255) / 256, 4LL * info.sms)));
    void* args[] = {const_cast<void**>(&src), &pn, &ps, const_cast<long long**>(&flag_n),
                    const_cast<long long**>(&flag_s), &pflag_n, &pflag_s, &done, &g};
    if (int rc = launch_checked(halo_put_kernel(d.dtype), dim3(grid), dim3(256), args, 0, st)) return rc;
  }
  const int strip_grid = static_cast<int>(
      std::max<long long>(1, std::min<long long>((static_cast<long long>(m) * width + 255) / 256, 2LL * info.sms)));
  if (peer_k) {
    Plan pl = fplan;
    pl.kernel = peer_k;
    PeerTile& pt = pl.g.peer;
    pt.flag_n = flag_n;
    pt.flag_s = flag_s;
    pt.north_off = g.north_off;
    pt.south_off = 0;
    pt.north_rows = S;
    pt.south_rows = N;
    pt.pflag_n = pflag_n;
    pt.pflag_s = pflag_s;
    pt.done = done;
    pt.boundary_tiles = pl.g.tiles_x * (pl.g.tiles_y >= 2 ? 2 : 1);
    const long long total_rows = rows + pl.g.above + pl.g.below;
    void* src = d_a;
    void* dst = d_b;
    for (int gen = 1; gen <= iterations; ++gen) {
      pt.wait_value = B + gen;
      pt.signal_value = B + gen + 1;
      pt.peer_n = has_n ? (gen & 1 ? peers->north_b : peers->north_a) : nullptr;
      pt.peer_s = has_s ? (gen & 1 ? peers->south_b : peers->south_a) : nullptr;
      const void* s0 = static_cast<const char*>(src) + N * row_bytes;
      void* d0 = static_cast<char*>(dst) + N * row_bytes;
      int rc;
      switch (d.dtype) {
        case SK_INT32: rc = launch_typed<int32_t>(d, pl, s0, d0, pl.g.above, total_rows, st); break;
        case SK_FLOAT32: rc = launch_typed<float>(d, pl, s0, d0, pl.g.above, total_rows, st); break;
        default: rc = launch_typed<double>(d, pl, s0, d0, pl.g.above, total_rows, st);
      }
      if (rc) return rc;
      std::swap(src, dst);
    }
    *epoch = B + iterations + 1;
    if (result_in_b) *result_in_b = iterations % 2;
    return SK_OK;
  }

  // Per generation the strips (caller's stream) and the interior (side
  // stream) run concurrently; a fork/join event pair orders generation g+1
  // after both halves of generation g (each half reads the other's rows).
  const long long inner = rows - 2LL * m;
  SideLane* lane = nullptr;
  if (inner > 0 && m > 0) {
    if (int rc = side_lane(st, &lane)) return rc;
  }
  void* src = d_a;
  void* dst = d_b;
  for (int gen = 1; gen <= iterations; ++gen) {
    g.wait_value = B + gen;
    g.signal_value = B + gen + 1;
    void* pn = has_n ? (gen & 1 ? peers->north_b : peers->north_a) : nullptr;
    void* ps = has_s ? (gen & 1 ? peers->south_b : peers->south_a) : nullptr;
    const void* s0 = static_cast<const char*>(src) + N * row_bytes;
    void* d0 = static_cast<char*>(dst) + N * row_bytes;
    cudaStream_t ist = st;
    if (lane) {
      cudaEventRecord(lane->fork, st);
      cudaStreamWaitEvent(lane->side, lane->fork, 0);
      ist = lane->side;
    }
    if (m > 0) {
      int rc;
      switch (d.dtype) {
        case SK_INT32:
          rc = launch_halo_strips<int32_t>(d, s0, d0, pn, ps, flag_n, flag_s, pflag_n, pflag_s, done, g, strip_grid, st);
          break;
        case SK_FLOAT32:
          rc = launch_halo_strips<float>(d, s0, d0, pn, ps, flag_n, flag_s, pflag_n, pflag_s, done, g, strip_grid, st);
          break;
        default:
          rc = launch_halo_strips<double>(d, s0, d0, pn, ps, flag_n, flag_s, pflag_n, pflag_s, done, g, strip_grid, st);
      }
      if (rc) return rc;
    }
    // interior rows [m, rows - m) read only owned rows (m >= N, S)
    if (inner > 0) {
      if (int rc = launch(d, static_cast<const char*>(s0) + m * row_bytes, static_cast<char*>(d0) + m * row_bytes,
                          width, inner, pitch, pitch, N, S, wc, wr, ist)) {
        return rc;
      }
    }
    if (lane) {
      cudaEventRecord(lane->join, lane->side);
      cudaStreamWaitEvent(st, lane->join, 0);
    }
    std::swap(src, dst);
  }
  *epoch = B + iterations + 1;
  if (result_in_b) *result_in_b = iterations % 2;
  return SK_OK;
}

}  // extern "C"
