// Host side of the B200 stencil executor: geometry, legality (refusal),
// TMA tensor-map cache, kernel dispatch and the extern "C" ABI declared in
// include/sk_stencil.h.
//
// Legality mirrors the reference's constraint model (space.hpp:38-51,
// simoracle.cpp:62-88) with real device facts instead of simulated ones:
//   oversized  <=> wc*wr > min(maxThreadsPerBlock, cudaFuncAttributes.maxThreadsPerBlock)
//   refused    <=> the staged tile does not fit the opt-in shared memory, no
//                  block can be resident, or the launch reports a
//                  (non-sticky) configuration/resource error.
#include <cstdarg>
#include <numeric>
#include <cmath>
#include <cstdio>
#include <random>
#include <set>
#include <thread>

#include "launch_internal.cuh"

namespace sk {
namespace detail {

thread_local std::string g_last_error;  // declared in launch_internal.cuh

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

// Launch-time errors that leave the context usable and mean "this
// configuration cannot run" -> refused parameter.  Only
// the two resource/config errors qualify: the dynamic shared-memory
// attribute is raised to the opt-in maximum when the kernel's attributes are
// first read, so cudaErrorInvalidValue at launch is a bad argument (a bug),
// reported as SK_EINVAL rather than hidden as a refused size.
bool is_config_error(cudaError_t e) {
  return e == cudaErrorInvalidConfiguration || e == cudaErrorLaunchOutOfResources;
}

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SK_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}

// Persistent grid size.  CTA b visits tiles b, b + G, b + 2G, ... of the
// row-major tile list, so its tile columns stay in one residue class modulo
// d = gcd(G, tiles_x).  G = occupancy x 148 SMs is a multiple of 148 = 4 x 37:
// at tiles_x = 74 or 37 (heat 16384^2 at 56 x wr or 224 x 4) every tile of
// the CTAs in column 0 and column tiles_x-1 is an edge tile (border fix-up,
// two block barriers, bounds-checked stores) and the launch waits for them:
// 1.7-2.1x the neighbouring sizes in the sweep.  Dropping a few CTAs from the
// grid to reach d <= 2 spreads the edge columns over every CTA's cycle; the
// cost is at most 1/G of the resident slots.  SK_GRID_BALANCE=0 disables it.
int balanced_grid(int grid, int tiles_x) {
  static const bool on = [] {
    const char* e = std::getenv("SK_GRID_BALANCE");
    return !(e && e[0] == '0');
  }();
  if (!on || tiles_x <= 2) return grid;
  int best = grid, best_d = std::gcd(grid, tiles_x);
  for (int G = grid - 1; best_d > 2 && G >= std::max(1, grid - 32); --G) {
    const int dd = std::gcd(G, tiles_x);
    if (dd < best_d) {
      best = G;
      best_d = dd;
    }
  }
  return best;
}

cudaError_t launch_tma(const void* kernel, dim3 grid, dim3 block, void** args, int smem, cudaStream_t stream) {
  if (!pdl_enabled()) return cudaLaunchKernel(kernel, grid, block, args, smem, stream);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, kernel, args);
}

int launch_pdl_checked(const void* kernel, dim3 grid, dim3 block, void** args, int smem, cudaStream_t stream) {
  const cudaError_t e = launch_tma(kernel, grid, block, args, smem, stream);
  return e == cudaSuccess ? SK_OK : launch_error(e);
}

int launch_error(cudaError_t e) {
  if (is_config_error(e)) {
    cudaGetLastError();
    return fail(SK_REFUSED, "launch refused: %s", cudaGetErrorString(e));
  }
  if (e == cudaErrorInvalidValue) {
    cudaGetLastError();
    return fail(SK_EINVAL, "launch rejected an argument: %s", cudaGetErrorString(e));
  }
  return fail(SK_ECUDA, "launch failed: %s", cudaGetErrorString(e));
}

size_t dtype_size(int dtype) { return dtype == SK_FLOAT64 ? 8 : 4; }

std::mutex g_mu;
std::map<int, DeviceInfo> g_devices;

int current_device_info(DeviceInfo* out, int* dev_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return fail(SK_ECUDA, "cudaGetDevice: %s", cudaGetErrorString(e));
  if (dev_out) *dev_out = dev;
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_devices.find(dev);
  if (it == g_devices.end()) {
    DeviceInfo d;
    cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&d.max_threads, cudaDevAttrMaxThreadsPerBlock, dev);
    cudaDeviceGetAttribute(&d.smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&d.smem_per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
    cudaDeviceGetAttribute(&d.l2_bytes, cudaDevAttrL2CacheSize, dev);
    e = cudaGetLastError();
    if (e != cudaSuccess || d.sms == 0) {
      return fail(SK_ECUDA, "device attribute query failed: %s", cudaGetErrorString(e));
    }
    it = g_devices.emplace(dev, d).first;
  }
  *out = it->second;
  return SK_OK;
}

long long floor_div(long long a, long long b) {
  long long q = a / b;
  return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
long long ceil_div(long long a, long long b) { return -floor_div(-a, b); }

// Cells per work-item: the descriptor's value, or AUTO = the largest of
// {8, 4, 2, 1} keeping the tile at most 64 output rows (and no taller than
// the grid needs).
int cells_per_thread(const sk_stencil_desc& d, int wr, long long H) {
  if (d.cells_per_thread > 0) return d.cells_per_thread;
  int k = 8;
  while (k > 1 && (static_cast<long long>(wr) * k > 64 || static_cast<long long>(wr) * k > H)) k /= 2;
  return k;
}

// ------------------------------------------------------------ op parameters
// ------------------------------------------------------- descriptor checks

// Game of Life takes the bit-plane kernel when asked to, or under AUTO once
// generations are fused - unless the descriptor asks for a per-cell work-item
// shape (K = 1, 2 or 4 cells) with TB = 2 or 4, which only the per-cell fused
// kernel has (that kernel also stays reachable through SK_LOAD_TMA).
bool uses_bits(const sk_stencil_desc& d) {
  if (d.op != SK_OP_GOL) return false;
  if (d.load_path == SK_LOAD_BITPLANE) return true;
  if (d.load_path != SK_LOAD_AUTO || d.fused_iterations <= 1) return false;
  const int k = d.cells_per_thread;
  const bool per_cell_k = k == 1 || k == 2 || k == 4;
  const bool per_cell_tb = d.fused_iterations == 2 || d.fused_iterations == 4;
  return !(per_cell_k && per_cell_tb);
}

// five_point / heat with unit borders take the register-strip kernel when
// asked to, or under AUTO for TB > 4 (beyond the per-cell fused kernel).
bool uses_strips(const sk_stencil_desc& d) {
  if (d.op != SK_OP_FIVE_POINT && d.op != SK_OP_HEAT) return false;
  if (d.north != 1 || d.south != 1 || d.east != 1 || d.west != 1) return false;
  return d.load_path == SK_LOAD_STRIPS || (d.load_path == SK_LOAD_AUTO && d.fused_iterations > 4);
}

int validate_desc(const sk_stencil_desc* d) {
  if (!d) return fail(SK_EINVAL, "null descriptor");
  if (d->op < 0 || d->op >= SK_OP_COUNT) return fail(SK_EINVAL, "bad op %d", d->op);
  if (d->dtype < SK_INT32 || d->dtype > SK_FLOAT64) return fail(SK_EINVAL, "bad dtype %d", d->dtype);
  if (d->border_mode != SK_BORDER_PAD && d->border_mode != SK_BORDER_NEAREST) {
    return fail(SK_EINVAL, "bad border mode %d", d->border_mode);
  }
  if (d->load_path < SK_LOAD_AUTO || d->load_path > SK_LOAD_VECTOR) {
    return fail(SK_EINVAL, "bad load path %d", d->load_path);
  }
  if (d->load_path == SK_LOAD_VECTOR && d->fused_iterations > 1) {
    return fail(SK_ENOTSUP, "the vector path runs one generation per launch (fused_iterations <= 1)");
  }
  if (d->load_path == SK_LOAD_BITPLANE && d->op != SK_OP_GOL) {
    return fail(SK_ENOTSUP, "the bit-plane path is Game of Life only");
  }
  for (int b : {d->north, d->south, d->east, d->west}) {
    if (b < 0 || b > 64) return fail(SK_EINVAL, "border values must be in [0, 64]");
  }
  if (d->load_path == SK_LOAD_STRIPS && !uses_strips(*d)) {
    return fail(SK_ENOTSUP, "the register-strip path is five_point / heat with N=S=E=W=1 only");
  }
  if (uses_strips(*d)) {
    if (d->cells_per_thread != 0 && d->cells_per_thread != 4 && d->cells_per_thread != 8 &&
        d->cells_per_thread != 16) {
      return fail(SK_EINVAL, "register-strip cells_per_thread (rows per work-item) must be 0, 4, 8 or 16");
    }
    if (d->fused_iterations < 0 || d->fused_iterations > kMaxStripsTB) {
      return fail(SK_EINVAL, "register-strip fused_iterations must be in [0, %d]", kMaxStripsTB);
    }
  } else if (uses_bits(*d)) {
    if (d->cells_per_thread != 0 && d->cells_per_thread != 8 && d->cells_per_thread != 16 &&
        d->cells_per_thread != 32) {
      return fail(SK_EINVAL, "bit-plane cells_per_thread (rows per work-item) must be 0, 8, 16 or 32");
    }
  } else if (d->load_path == SK_LOAD_VECTOR) {
    if (d->cells_per_thread != 0 && d->cells_per_thread != 1 && d->cells_per_thread != 2 &&
        d->cells_per_thread != 4 && d->cells_per_thread != 8 && d->cells_per_thread != 16) {
      return fail(SK_EINVAL, "vector cells_per_thread (rows per work-item) must be 0 (auto), 1, 2, 4, 8 or 16");
    }
  } else if (d->cells_per_thread != 0 && d->cells_per_thread != 1 && d->cells_per_thread != 2 &&
      d->cells_per_thread != 4 && d->cells_per_thread != 8) {
    return fail(SK_EINVAL, "cells_per_thread must be 0 (auto), 1, 2, 4 or 8");
  }
  if (uses_strips(*d)) {
    // checked above
  } else if (uses_bits(*d)) {
    if (d->fused_iterations < 0 || d->fused_iterations > kMaxBitsTB) {
      return fail(SK_EINVAL, "bit-plane fused_iterations must be in [0, %d]", kMaxBitsTB);
    }
  } else if (d->fused_iterations != 0 && d->fused_iterations != 1 && d->fused_iterations != 2 &&
             d->fused_iterations != 4) {
    return fail(SK_EINVAL, "fused_iterations must be 0, 1, 2 or 4");
  }
  int need = 0;
  switch (d->op) {
    case SK_OP_FIVE_POINT: case SK_OP_HEAT: case SK_OP_GOL: case SK_OP_SOBEL: case SK_OP_NMS:
      need = 1;
      break;
    case SK_OP_GAUSSIAN:
      if (d->north < 1 || d->north > 10 || d->south != d->north || d->east != d->north ||
          d->west != d->north) {
        return fail(SK_EINVAL, "gaussian needs equal borders g in [1, 10]");
      }
      break;
    case SK_OP_SYNTHETIC:
      if (d->instructions < 1) return fail(SK_EINVAL, "synthetic needs instructions >= 1");
      break;
    default:
      break;
  }
  if (need && (d->north < need || d->south < need || d->east < need || d->west < need)) {
    return fail(SK_EINVAL, "op %d needs borders >= %d in every direction", d->op, need);
  }
  return SK_OK;
}

// --------------------------------------------------------- kernel registry
KernelPtr fused_for_desc(const sk_stencil_desc& d, int K, int TB) {
  switch (d.dtype) {
    case SK_INT32: return fused_i32(d, K, TB);
    case SK_FLOAT32: return fused_f32(d, K, TB);
    default: return fused_f64(d, K, TB);
  }
}

KernelPtr vector_for_desc(const sk_stencil_desc& d, int K) {
  switch (d.dtype) {
    case SK_INT32: return vector_i32(d, K);
    case SK_FLOAT32: return vector_f32(d, K);
    default: return vector_f64(d, K);
  }
}

KernelPair kernels_for_desc(const sk_stencil_desc& d, int K) {
  switch (d.dtype) {
    case SK_INT32: return kernels_i32(d, K);
    case SK_FLOAT32: return kernels_f32(d, K);
    default: return kernels_f64(d, K);
  }
}

// ------------------------------------------------ driver API (custom kernels)
// Custom-functor kernels are registered in the CALLER's CUDA runtime, so they
// arrive as driver CUfunction handles and are queried/launched with the
// driver API (process-wide, context-shared).
struct DriverApi {
  CUresult (*func_get_attribute)(int*, CUfunction_attribute, CUfunction) = nullptr;
  CUresult (*func_set_attribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*occupancy)(int*, CUfunction, int, size_t) = nullptr;
  CUresult (*launch)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                     unsigned, CUstream, void**, void**) = nullptr;
  bool ok = false;
};

const DriverApi& driver() {
  static DriverApi api = [] {
    DriverApi a;
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess;
    };
    a.ok = get("cuFuncGetAttribute", reinterpret_cast<void**>(&a.func_get_attribute)) &&
           get("cuFuncSetAttribute", reinterpret_cast<void**>(&a.func_set_attribute)) &&
           get("cuOccupancyMaxActiveBlocksPerMultiprocessor", reinterpret_cast<void**>(&a.occupancy)) &&
           get("cuLaunchKernel", reinterpret_cast<void**>(&a.launch));
    cudaGetLastError();
    return a;
  }();
  return api;
}

// Per-(device, kernel) attributes: kernel max threads and the opt-in smem
// attribute, set once.
std::map<std::pair<int, KernelPtr>, KernelAttr> g_kattr;



int kernel_attr(int dev, KernelPtr k, const DeviceInfo& info, KernelAttr* out,
                bool is_driver) {
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, k);
  auto it = g_kattr.find(key);
  if (it == g_kattr.end() && is_driver) {
    const DriverApi& api = driver();
    if (!api.ok) return fail(SK_ECUDA, "driver entry points unavailable");
    CUfunction f = reinterpret_cast<CUfunction>(const_cast<void*>(k));
    int max_threads = 0, static_smem = 0;
    if (api.func_get_attribute(&max_threads, CU_FUNC_ATTRIBUTE_MAX_THREADS_PER_BLOCK, f) != CUDA_SUCCESS ||
        api.func_get_attribute(&static_smem, CU_FUNC_ATTRIBUTE_SHARED_SIZE_BYTES, f) != CUDA_SUCCESS) {
      return fail(SK_EINVAL, "custom kernel handle is not a valid CUfunction");
    }
    KernelAttr a;
    a.max_threads = max_threads;
    a.max_dyn_smem = info.smem_optin - static_smem;
    if (api.func_set_attribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, a.max_dyn_smem) !=
        CUDA_SUCCESS) {
      return fail(SK_ECUDA, "cuFuncSetAttribute failed on custom kernel");
    }
    it = g_kattr.emplace(key, a).first;
  }
  if (it == g_kattr.end()) {
    cudaFuncAttributes fa;
    cudaError_t e = cudaFuncGetAttributes(&fa, k);
    if (e != cudaSuccess) {
      return fail(SK_ECUDA, "cudaFuncGetAttributes: %s", cudaGetErrorString(e));
    }
    KernelAttr a;
    a.max_threads = fa.maxThreadsPerBlock;
    a.max_dyn_smem = info.smem_optin - static_cast<int>(fa.sharedSizeBytes);
    e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, a.max_dyn_smem);
    if (e != cudaSuccess) {
      return fail(SK_ECUDA, "cudaFuncSetAttribute: %s", cudaGetErrorString(e));
    }
    it = g_kattr.emplace(key, a).first;
  }
  *out = it->second;
  return SK_OK;
}

std::map<std::tuple<int, KernelPtr, int, int>, int> g_occ;

int occupancy(int dev, KernelPtr k, int threads, int smem, bool is_driver) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_occ.find({dev, k, threads, smem});
    if (it != g_occ.end()) return it->second;
  }
  int n = 0;
  if (is_driver) {
    CUfunction f = reinterpret_cast<CUfunction>(const_cast<void*>(k));
    if (!driver().ok || driver().occupancy(&n, f, threads, static_cast<size_t>(smem)) != CUDA_SUCCESS) n = 0;
  } else if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k, threads, smem) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  g_occ[{dev, k, threads, smem}] = n;
  return n;
}

// ------------------------------------------------------------ tensor maps
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<EncodeTiledFn>(nullptr);
    }
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

std::map<MapKey, CUtensorMap> g_maps;

// L2 fill granularity of the tile loads (SK_L2_PROMO=0/64/128/256 for A/B).
CUtensorMapL2promotion l2_promotion() {
  static const CUtensorMapL2promotion p = [] {
    const char* e = std::getenv("SK_L2_PROMO");
    const int v = e ? std::atoi(e) : 256;
    return v == 0     ? CU_TENSOR_MAP_L2_PROMOTION_NONE
           : v == 64  ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                      : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  return p;
}

int tensor_map(const MapKey& key, CUtensorMap* out) {
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_maps.find(key);
    if (it != g_maps.end()) {
      *out = it->second;
      return SK_OK;
    }
  }
  EncodeTiledFn fn = encode_fn();
  if (!fn) return fail(SK_ECUDA, "cuTensorMapEncodeTiled unavailable");
  CUtensorMapDataType dt = key.dtype == SK_INT32     ? CU_TENSOR_MAP_DATA_TYPE_INT32
                           : key.dtype == SK_FLOAT32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                                     : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(key.w), static_cast<cuuint64_t>(key.h)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(key.pitch) * dtype_size(key.dtype)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(key.box_w), static_cast<cuuint32_t>(key.box_h)};
  cuuint32_t estr[2] = {1, 1};
  CUtensorMap m;
  CUresult r = fn(&m, dt, 2, const_cast<void*>(key.base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, l2_promotion(),
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(SK_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_maps.size() > 4096) g_maps.clear();
  g_maps[key] = m;
  *out = m;
  return SK_OK;
}

// ------------------------------------------------------------------ plan
// Builds the launch plan; returns SK_OK, SK_OVERSIZED, SK_REFUSED or an error.
// `in` may be null for a probe (TMA eligibility then assumes aligned buffers).
int k_index(int K) { return K == 1 ? 0 : K == 2 ? 1 : K == 4 ? 2 : 3; }

int make_plan(const sk_stencil_desc& d, long long W, long long H, long long pitch_in,
              long long pitch_out, long long above, long long below, int wc, int wr,
              const void* in, Plan* plan, const sk_kernel_table* custom) {
  if (W < 1 || H < 1 || W > (1LL << 30) || H > (1LL << 30)) {
    return fail(SK_EINVAL, "bad dims %lldx%lld", W, H);
  }
  if (pitch_in < W || pitch_out < W) return fail(SK_EINVAL, "pitch smaller than width");
  if (wc < 1 || wr < 1) return fail(SK_EINVAL, "bad workgroup %dx%d", wc, wr);
  DeviceInfo info;
  int dev = 0;
  if (int rc = current_device_info(&info, &dev)) return rc;
  const int K = cells_per_thread(d, wr, H);
  KernelPair kp = custom ? KernelPair{custom->tma[k_index(K)], custom->explicit_load[k_index(K)]}
                         : kernels_for_desc(d, K);
  if (!kp.tma || !kp.explicit_) return fail(SK_EINVAL, "kernel table has no entry for K=%d", K);
  const bool drv = custom != nullptr;
  plan->driver_handle = drv;
  // temporal blocking: TB generations per launch (TMA path only)
  const int TB = (!drv && d.fused_iterations > 1) ? d.fused_iterations : 1;
  // Vector work-items (vector.cuh): V = 16 B of cells per work-item row.
  // SK_LOAD_VECTOR demands them; AUTO takes them for one-pass launches of
  // ops that have a vector form whenever the tile fits one TMA box and the
  // buffers are 16-B aligned (the scalar TMA kernel otherwise).
  bool vec_path = false;
  int V = 1;
  if (!drv && TB == 1 && (d.load_path == SK_LOAD_VECTOR || d.load_path == SK_LOAD_AUTO)) {
    KernelPtr vk = vector_for_desc(d, K);
    if (!vk && d.load_path == SK_LOAD_VECTOR) {
      return fail(SK_ENOTSUP, "no vector kernel for op %d with border (%d,%d,%d,%d)", d.op, d.north,
                  d.south, d.east, d.west);
    }
    if (vk) {
      const int es_ = static_cast<int>(dtype_size(d.dtype));
      const int vec_ = 16 / es_;
      const long long lw_ = static_cast<long long>(wc) * vec_ + d.east + d.west;
      const long long box_w = (lw_ + ((-d.west) & (vec_ - 1)) + vec_ - 1) / vec_ * vec_;
      const bool aligned = (pitch_in * es_) % 16 == 0 && (pitch_out * es_) % 16 == 0 &&
                           (in == nullptr || reinterpret_cast<uintptr_t>(in) % 16 == 0);
      // AUTO also needs the block to fit the vector kernel's own thread bound
      KernelAttr va;
      if (int rc = kernel_attr(dev, vk, info, &va)) return rc;
      const bool fits = static_cast<long long>(wc) * wr <= va.max_threads;
      if (d.load_path == SK_LOAD_VECTOR || (box_w <= 256 && aligned && fits)) {
        vec_path = true;
        V = vec_;
        kp.tma = vk;
      }
    }
  }
  if (TB > 1) {
    kp.tma = fused_for_desc(d, K, TB);
    if (!kp.tma) return fail(SK_ENOTSUP, "no fused (TB=%d) kernel for op %d", TB, d.op);
  }
  KernelAttr a_tma, a_exp;
  if (int rc = kernel_attr(dev, kp.tma, info, &a_tma, drv)) return rc;
  if (int rc = kernel_attr(dev, kp.explicit_, info, &a_exp, drv)) return rc;
  // halo of the loaded box: TB border regions
  const int eN = TB * d.north, eS = TB * d.south, eE = TB * d.east, eW = TB * d.west;

  const long long threads = static_cast<long long>(wc) * wr;
  const size_t es = dtype_size(d.dtype);
  Geom& g = plan->g;
  g.W = static_cast<int>(W);
  g.H = static_cast<int>(H);
  g.pitch_in = pitch_in;
  g.pitch_out = pitch_out;
  g.above = static_cast<int>(std::min<long long>(above, eN));
  g.below = static_cast<int>(std::min<long long>(below, eS));
  g.N = eN;
  g.S = eS;
  g.E = eE;
  g.Wb = eW;
  g.TB = TB;
  g.bN = d.north;
  g.bS = d.south;
  g.bE = d.east;
  g.bW = d.west;
  g.wc = wc;
  g.wr = wr;
  g.K = K;
  g.V = V;
  g.tile_cols = wc * V;
  const int tc = g.tile_cols;
  g.tile_rows = wr * K;
  g.lw = tc + eE + eW;
  const int vec = static_cast<int>(16 / es);
  g.vec = vec;
  // Box width: the logical tile plus the largest 16-B alignment offset any
  // tile can have (constant when wc is a multiple of vec).
  const int max_off = (tc % vec == 0) ? ((-eW) & (vec - 1)) : vec - 1;
  g.tile_w = (g.lw + max_off + vec - 1) / vec * vec;
  g.tile_h = g.tile_rows + eN + eS;
  g.tiles_x = static_cast<int>((W + tc - 1) / tc);
  g.tiles_y = static_cast<int>((H + g.tile_rows - 1) / g.tile_rows);
  // Interior tiles: read only inside the readable window and store in range.
  g.ex_lo = static_cast<int>(ceil_div(eW, tc));
  g.ex_hi = static_cast<int>(floor_div(W - tc - eE, tc));
  g.ey_lo = static_cast<int>(ceil_div(std::max<long long>(0, eN - g.above), g.tile_rows));
  g.ey_hi = static_cast<int>(floor_div(H + g.below - eS - g.tile_rows, g.tile_rows));
  g.mode = d.border_mode;
  g.pad_is_zero = d.pad_value == 0.0 && !std::signbit(d.pad_value);
  plan->tile_bytes = static_cast<long long>(g.lw) * g.tile_h * static_cast<long long>(es);

  // TMA eligibility: box width <= 256 elements, 16-B aligned base and pitch.
  bool tma_ok = g.tile_w <= 256 && (pitch_in * es) % 16 == 0 &&
                (in == nullptr || (reinterpret_cast<uintptr_t>(in) % 16) == 0) &&
                static_cast<long long>(g.tiles_x) * g.tiles_y < (1LL << 31);
  bool use_tma = d.load_path == SK_LOAD_TMA || (d.load_path == SK_LOAD_AUTO && tma_ok);
  if (TB > 1) {
    if (!tma_ok) return fail(SK_ENOTSUP, "fused iterations need the TMA path (tile_w %d)", g.tile_w);
    use_tma = true;
  }
  if (d.load_path == SK_LOAD_TMA && !tma_ok) {
    return fail(SK_ENOTSUP, "TMA path not possible for this tile/buffer (tile_w %d)", g.tile_w);
  }
  if (vec_path) {
    if (g.tile_w > 256) {
      return fail(SK_REFUSED, "vector tile %d columns wide exceeds one TMA box (256)", g.tile_w);
    }
    if (!tma_ok || (pitch_out * es) % 16 != 0) {
      return fail(SK_ENOTSUP, "the vector path needs 16-B aligned input and pitches");
    }
    use_tma = true;
  }
  const KernelAttr& attr = use_tma ? a_tma : a_exp;
  plan->kernel_max = std::min(info.max_threads, attr.max_threads);
  plan->threads = static_cast<int>(threads);
  if (threads > plan->kernel_max) {
    return fail(SK_OVERSIZED, "workgroup %dx%d exceeds the effective maximum %d", wc, wr,
                plan->kernel_max);
  }
  plan->tma = use_tma;
  plan->kernel = use_tma ? kp.tma : kp.explicit_;

  if (!use_tma) {
    long long smem = static_cast<long long>(g.tile_w) * g.tile_h * static_cast<long long>(es);
    if (smem > attr.max_dyn_smem) {
      return fail(SK_REFUSED, "tile %lld B exceeds shared memory %d B", smem, attr.max_dyn_smem);
    }
    g.stages = 1;
    g.stage_bytes = static_cast<int>(smem);
    g.box_h = g.tile_h;
    g.nchunks = 1;
    plan->smem = static_cast<int>(smem);
    if (occupancy(dev, plan->kernel, plan->threads, plan->smem, drv) < 1) {
      return fail(SK_REFUSED, "no resident block possible for %dx%d", wc, wr);
    }
    plan->grid = g.tiles_x * g.tiles_y;  // one block per tile
    return SK_OK;
  }

  // Boxes of <= 256 rows; a multiple of 8 rows keeps every box's shared
  // destination 128-B aligned (tile_w * es is a 16-B multiple).
  g.nchunks = (g.tile_h + 255) / 256;
  g.box_h = (g.tile_h + g.nchunks - 1) / g.nchunks;
  if (g.nchunks > 1) g.box_h = (g.box_h + 7) / 8 * 8;
  // fused kernels read up to K-1 rows past a generation region: slack rows
  const int slack = TB > 1 ? K : 0;
  long long stage = static_cast<long long>(g.tile_w) * (g.box_h * g.nchunks + slack) *
                    static_cast<long long>(es);
  stage = (stage + 127) / 128 * 128;
  long long scratch = 0;
  if (TB > 1) {
    g.sp = wc + (TB - 1) * (d.east + d.west);
    const long long rows = g.tile_rows + static_cast<long long>(TB - 1) * (d.north + d.south) + K;
    g.scratch_elems = static_cast<int>((g.sp * rows + 31) / 32 * 32);
    scratch = 2LL * g.scratch_elems * static_cast<long long>(es);
  } else {
    g.sp = 0;
    g.scratch_elems = 0;
  }
  if (stage + scratch + 128 > attr.max_dyn_smem) {
    return fail(SK_REFUSED, "tile %lld B exceeds shared memory %d B", stage + scratch,
                attr.max_dyn_smem);
  }
  g.stage_bytes = static_cast<int>(stage);
  // Ring depth: as deep as the per-block share of the SM's shared memory
  // allows at the thread-limited occupancy, between 2 and 8 stages.
  int occ2 = occupancy(dev, plan->kernel, plan->threads,
                       static_cast<int>(std::min<long long>(2 * stage + scratch + 128, attr.max_dyn_smem)),
                       drv);
  int blocks = std::max(1, occ2);
  long long share = (static_cast<long long>(info.smem_per_sm) / blocks) - 1024 - 128 - scratch;
  int stages = static_cast<int>(std::clamp<long long>(share / stage, 1, 8));
  while (stages > 1 && stage * stages + scratch + 128 > attr.max_dyn_smem) --stages;
  // A/B knobs (unset: the policy above): SK_MIN_STAGES deepens the ring at the
  // cost of resident blocks; SK_RING_LAG sets the refill lag (prefetch depth
  // = stages - lag tiles).
  static const int min_stages = [] {
    const char* e = std::getenv("SK_MIN_STAGES");
    return e ? std::atoi(e) : 0;
  }();
  static const int ring_lag = [] {
    const char* e = std::getenv("SK_RING_LAG");
    return e ? std::atoi(e) : 0;
  }();
  if (min_stages > stages && stage * min_stages + scratch + 128 <= attr.max_dyn_smem) stages = min_stages;
  // A two-stage ring has no slack: the refill of tile i+1 waits for the
  // slowest warp of tile i-1.  When the share policy leaves at most two
  // resident blocks with two stages each, one block with a three-stage ring
  // (lag 2: one tile ahead plus one stage of slack) is faster: heat 16384^2
  // vector 48x8 393 -> 357 us, 40x8 400 -> 352 (profiles/r04_landscape_ab.jsonl).
  // Only the light 3x3 / cross ops: the box mean's 28 instructions per cell
  // need the second block's warps (36x8 27.7 -> 34.9 us with one block;
  // landscape A/B in profiles/r04_landscape_ab.jsonl).
  static const bool deep_ring = [] {
    const char* e = std::getenv("SK_DEEP_RING");
    return !(e && e[0] == '0');
  }();
  const bool light_op = d.op == SK_OP_HEAT || d.op == SK_OP_FIVE_POINT || d.op == SK_OP_GOL;
  if (deep_ring && light_op && min_stages == 0 && TB == 1 && stages < 3 && blocks <= 2 &&
      stage * 3 + scratch + 128 <= attr.max_dyn_smem) {
    stages = 3;
  }
  g.stages = stages;
  g.lag = ring_lag > 0 ? std::min(ring_lag, std::max(1, stages - 1)) : 0;
  plan->smem = static_cast<int>(stage * stages + scratch + 16 * stages);  // + full/empty barriers
  int occ = occupancy(dev, plan->kernel, plan->threads, plan->smem, drv);
  if (occ < 1) return fail(SK_REFUSED, "no resident block possible for %dx%d", wc, wr);
  long long ntiles = static_cast<long long>(g.tiles_x) * g.tiles_y;
  plan->grid = static_cast<int>(std::min<long long>(ntiles, static_cast<long long>(occ) * info.sms));
  if (plan->grid < ntiles) plan->grid = balanced_grid(plan->grid, g.tiles_x);
  return SK_OK;
}

int launch_driver(const Plan& plan, dim3 grid, dim3 block, void** args, cudaStream_t stream) {
  CUfunction f = reinterpret_cast<CUfunction>(const_cast<void*>(plan.kernel));
  CUresult r = driver().launch(f, grid.x, grid.y, grid.z, block.x, block.y, block.z,
                               static_cast<unsigned>(plan.smem), reinterpret_cast<CUstream>(stream), args,
                               nullptr);
  if (r == CUDA_SUCCESS) return SK_OK;
  if (r == CUDA_ERROR_LAUNCH_OUT_OF_RESOURCES) {
    return fail(SK_REFUSED, "launch refused (driver error %d)", static_cast<int>(r));
  }
  if (r == CUDA_ERROR_INVALID_VALUE) {
    return fail(SK_EINVAL, "launch rejected an argument (driver error %d)", static_cast<int>(r));
  }
  return fail(SK_ECUDA, "custom kernel launch failed (driver error %d)", static_cast<int>(r));
}

int launch_checked(KernelPtr k, dim3 grid, dim3 block, void** args, int smem, cudaStream_t stream) {
  cudaError_t e = cudaLaunchKernel(k, grid, block, args, smem, stream);
  if (e == cudaSuccess) return SK_OK;
  return launch_error(e);
}

int launch(const sk_stencil_desc& d, const void* in, void* out, long long W, long long H,
           long long pitch_in, long long pitch_out, long long above, long long below, int wc,
           int wr, cudaStream_t stream, const sk_kernel_table* custom) {
  if (!custom && uses_strips(d)) {
    return run_cross(d, in, out, W, H, pitch_in, pitch_out, above, below, wc, wr,
                     std::max(1, d.fused_iterations), stream);
  }
  if (!custom && uses_bits(d)) {
    const int tb = std::max(1, d.fused_iterations);
    return run_bits(d, in, out, W, H, pitch_in, pitch_out, above, below, wc, wr, tb, tb, stream);
  }
  Plan plan;
  if (int rc = make_plan(d, W, H, pitch_in, pitch_out, above, below, wc, wr, in, &plan, custom)) {
    return rc;
  }
  if (plan.g.V > 1 && d.load_path == SK_LOAD_AUTO && reinterpret_cast<uintptr_t>(out) % 16 != 0) {
    // AUTO chose vector work-items, but their 16-B row stores need an
    // aligned output: take the scalar TMA kernel instead
    sk_stencil_desc scalar = d;
    scalar.load_path = SK_LOAD_TMA;
    if (int rc = make_plan(scalar, W, H, pitch_in, pitch_out, above, below, wc, wr, in, &plan, custom)) {
      return rc;
    }
  }
  long long used_above = plan.g.above;
  long long total_rows = H + plan.g.above + plan.g.below;
  switch (d.dtype) {
    case SK_INT32:
      return launch_typed<int32_t>(d, plan, in, out, used_above, total_rows, stream);
    case SK_FLOAT32:
      return launch_typed<float>(d, plan, in, out, used_above, total_rows, stream);
    default:
      return launch_typed<double>(d, plan, in, out, used_above, total_rows, stream);
  }
}

// ------------------------------------------------------------- scratch
struct Scratch {
  void* flush = nullptr;
  size_t flush_bytes = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* host_in = nullptr;
  void* host_out = nullptr;
  void* dev_a = nullptr;
  void* dev_b = nullptr;
  size_t dev_bytes = 0;
  void* diff = nullptr;
  std::vector<cudaEvent_t> events;
  // streamed host jobs (sk_stencil_submit_host): three slots, each with its
  // own stream, device ping-pong buffers and completion event, so job j+1's
  // H2D, job j's passes and job j-1's D2H can all be in flight at once
  struct Slot {
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    void* a = nullptr;
    void* b = nullptr;
    size_t bytes = 0;
    long long ticket = -1;  // job in flight (or last completed)
    int status = SK_OK;
  } slots[3];
  long long next_ticket = 0;
};
// Per (device, calling thread): the timing stream, event pool, flush buffer
// and e2e staging buffers are never shared between threads (reentrant ABI).
std::map<std::pair<int, std::thread::id>, Scratch> g_scratch;

int scratch(Scratch** out) {
  DeviceInfo info;
  int dev = 0;
  if (int rc = current_device_info(&info, &dev)) return rc;
  std::lock_guard<std::mutex> lk(g_mu);
  Scratch& s = g_scratch[{dev, std::this_thread::get_id()}];
  if (!s.stream) {
    if (cudaStreamCreate(&s.stream) != cudaSuccess || cudaEventCreate(&s.ev0) != cudaSuccess ||
        cudaEventCreate(&s.ev1) != cudaSuccess) {
      return fail(SK_ECUDA, "stream/event creation failed");
    }
    s.flush_bytes = static_cast<size_t>(info.l2_bytes) * 2;
    if (cudaMalloc(&s.flush, s.flush_bytes) != cudaSuccess ||
        cudaMemset(s.flush, 0, s.flush_bytes) != cudaSuccess) {
      return fail(SK_ECUDA, "L2 flush buffer allocation failed");
    }
  }
  *out = &s;
  return SK_OK;
}

int StreamBits::alloc(size_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SK_ECUDA, "cudaGetDevice failed");
  {
    static std::mutex mu;
    static std::set<int> retained;
    std::lock_guard<std::mutex> lk(mu);
    if (!retained.count(dev)) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
      retained.insert(dev);
    }
  }
  for (void*& q : p) {
    if (cudaMallocAsync(&q, bytes, stream) != cudaSuccess) {
      q = nullptr;
      return fail(SK_ECUDA, "bit-grid allocation failed (%zu B)", bytes);
    }
  }
  return SK_OK;
}

StreamBits::~StreamBits() {
  for (void* q : p) {
    if (q) cudaFreeAsync(q, stream);
  }
}

// L2 scrub between timed samples, second half: READ back the 2 x L2 buffer
// the memset just wrote, so the next pass finds none of its input in L2 and
// the cache holds clean lines only - the scrub's (and the previous pass's)
// dirty lines are written back here, not during the next timed pass.  (A
// memset alone left ~2 x L2 of dirty lines whose write-back was charged to
// the pass: +6 us on the 32 us config-4 pass.)
__global__ void k_l2_scrub(const uint4* __restrict__ p, long long n, unsigned* sink) {
  unsigned acc = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint4 v = p[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9e3779b9u && n < 0) *sink = acc;  // never true: keeps the loads
}

// Word-wise device comparison; *diff counts differing 16-B words.
__global__ void k_count_diff(const uint4* __restrict__ a, const uint4* __restrict__ b, long long n,
                             unsigned long long* diff) {
  unsigned long long local = 0;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint4 x = a[i], y = b[i];
    local += (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
  }
  if (local) atomicAdd(diff, local);
}

}  // namespace detail
}  // namespace sk

// ======================================================================= ABI
namespace sk {
namespace detail {

// The one-pass generation loop of sk_stencil_iterate: TB generations per
// fused launch, the remainder one pass at a time, ping-ponging a / b.
int iterate_direct(const sk_stencil_desc& d, void* d_a, void* d_b, long long W, long long H, long long pitch,
                   int iterations, int wc, int wr, cudaStream_t stream, int* launches) {
  const int TB = d.fused_iterations > 1 ? d.fused_iterations : 1;
  sk_stencil_desc one = d;
  one.fused_iterations = 0;
  void* src = d_a;
  void* dst = d_b;
  int n = 0;
  for (int done = 0; done < iterations; ++n) {
    const bool fuse = TB > 1 && iterations - done >= TB;
    if (int rc = launch(fuse ? d : one, src, dst, W, H, pitch, pitch, 0, 0, wc, wr, stream)) return rc;
    done += fuse ? TB : 1;
    std::swap(src, dst);
  }
  *launches = n;
  return SK_OK;
}

// CUDA-graph replay of that loop.  Generations are taken in chunks of 64
// (an even number of launches for TB = 1, 2 or 4, so every chunk starts and
// ends in d_a) plus a remainder; each chunk shape is a cache entry keyed by
// (descriptor, buffers, shape, block, generations, device).  An entry's
// first call runs directly (it validates the launch and fills the plan /
// tensor-map caches), its second call runs directly and then captures the
// same launches (private stream, thread-local capture: capturing runs
// nothing) into an executable graph, and later calls launch the graph: one
// host call per chunk and graph-node launch latency instead of a host launch
// per generation (GoL 1024^2: 5.2 -> 3.2 us per generation,
// scripts/launch_overhead_probe.py).  One-off loops never pay for a capture.
// SK_GRAPHS=0 disables it; a capture that fails is remembered (the entry
// stays direct).
struct GraphEntry {
  int calls = 0;
  bool failed = false;
  cudaGraphExec_t exec = nullptr;
  int launches = 0;
};
std::mutex g_graph_mu;
std::map<std::string, GraphEntry> g_graphs;
constexpr int kGraphMinIterations = 4;
constexpr int kGraphChunk = 64;
constexpr std::size_t kGraphCacheMax = 256;

std::string graph_key(const sk_stencil_desc& d, const void* a, const void* b, long long W, long long H,
                      long long pitch, int iterations, int wc, int wr, int dev) {
  char buf[320];
  std::snprintf(buf, sizeof buf, "%d,%d,%d,%d,%d,%d,%d,%a,%d,%d,%d,%d,%d|%p,%p|%lld,%lld,%lld|%d,%d,%d|%d", d.op,
                d.dtype, d.north, d.south, d.east, d.west, d.border_mode, d.pad_value, d.complexity,
                d.instructions, d.load_path, d.cells_per_thread, d.fused_iterations, a, b, W, H, pitch, iterations,
                wc, wr, dev);
  return buf;
}

bool graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("SK_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return on;
}

// `iterations` generations from d_a through the cache entry of that shape.
int cached_loop(const sk_stencil_desc& d, void* d_a, void* d_b, long long W, long long H, long long pitch,
                int iterations, int wc, int wr, int dev, cudaStream_t stream, int* launches) {
  if (iterations < kGraphMinIterations) {
    return iterate_direct(d, d_a, d_b, W, H, pitch, iterations, wc, wr, stream, launches);
  }
  const std::string key = graph_key(d, d_a, d_b, W, H, pitch, iterations, wc, wr, dev);
  int calls = 0;
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    GraphEntry& e = g_graphs[key];
    if (e.exec) {
      const cudaError_t err = cudaGraphLaunch(e.exec, stream);
      if (err != cudaSuccess) return fail(SK_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(err));
      *launches = e.launches;
      return SK_OK;
    }
    calls = e.failed ? 0 : ++e.calls;
  }
  if (int rc = iterate_direct(d, d_a, d_b, W, H, pitch, iterations, wc, wr, stream, launches)) return rc;
  if (calls != 2) return SK_OK;
  // second identical call: capture it for the next ones
  GraphEntry made;
  cudaStream_t cap = nullptr;
  cudaGraph_t graph = nullptr;
  bool ok = cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking) == cudaSuccess &&
            cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    int n = 0;
    const int rc = iterate_direct(d, d_a, d_b, W, H, pitch, iterations, wc, wr, cap, &n);
    const bool ended = cudaStreamEndCapture(cap, &graph) == cudaSuccess;
    ok = rc == SK_OK && ended && graph != nullptr && n == *launches &&
         cudaGraphInstantiate(&made.exec, graph, 0) == cudaSuccess;
    made.launches = n;
  }
  if (graph) cudaGraphDestroy(graph);
  if (cap) cudaStreamDestroy(cap);
  cudaGetLastError();  // a failed capture leaves nothing sticky behind
  g_last_error.clear();
  std::lock_guard<std::mutex> lk(g_graph_mu);
  if (g_graphs.size() >= kGraphCacheMax) {
    for (auto& kv : g_graphs) {
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    }
    g_graphs.clear();
  }
  GraphEntry& e = g_graphs[key];
  if (ok) {
    e.exec = made.exec;
    e.launches = made.launches;
  } else {
    if (made.exec) cudaGraphExecDestroy(made.exec);
    e.failed = true;
  }
  return SK_OK;
}

int graph_iterate(const sk_stencil_desc& d, void* d_a, void* d_b, long long W, long long H, long long pitch,
                  int iterations, int wc, int wr, cudaStream_t stream, int* launches) {
  if (iterations < kGraphMinIterations || !graphs_enabled()) {
    return iterate_direct(d, d_a, d_b, W, H, pitch, iterations, wc, wr, stream, launches);
  }
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SK_ECUDA, "cudaGetDevice failed");
  int total = 0, n = 0;
  const int full = iterations / kGraphChunk, rem = iterations % kGraphChunk;
  for (int c = 0; c < full; ++c) {  // each chunk ends in d_a (even launch count)
    if (int rc = cached_loop(d, d_a, d_b, W, H, pitch, kGraphChunk, wc, wr, dev, stream, &n)) return rc;
    total += n;
  }
  if (rem > 0) {
    if (int rc = cached_loop(d, d_a, d_b, W, H, pitch, rem, wc, wr, dev, stream, &n)) return rc;
    total += n;
  }
  *launches = total;
  return SK_OK;
}

}  // namespace detail
}  // namespace sk

using namespace sk;
using namespace sk::detail;

extern "C" {

const char* sk_last_error(void) { return g_last_error.c_str(); }

const char* sk_version(void) { return "sk_stencil 0.1 sm_100a"; }

int sk_stencil_launch(const sk_stencil_desc* desc, const void* d_in, void* d_out, int64_t width,
                      int64_t height, int64_t pitch_in, int64_t pitch_out, int64_t rows_above,
                      int64_t rows_below, int32_t wc, int32_t wr, void* stream) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (!d_in || !d_out) return fail(SK_EINVAL, "null buffer");
  if (rows_above < 0 || rows_below < 0) return fail(SK_EINVAL, "negative halo rows");
  return launch(*desc, d_in, d_out, width, height, pitch_in, pitch_out, rows_above, rows_below,
                wc, wr, static_cast<cudaStream_t>(stream));
}

int sk_stencil_launch_custom(const sk_stencil_desc* desc, const sk_kernel_table* kernels,
                             const void* d_in, void* d_out, int64_t width, int64_t height,
                             int64_t pitch_in, int64_t pitch_out, int64_t rows_above,
                             int64_t rows_below, int32_t wc, int32_t wr, void* stream) {
  g_last_error.clear();
  if (!kernels) return fail(SK_EINVAL, "null kernel table");
  if (!desc) return fail(SK_EINVAL, "null descriptor");
  sk_stencil_desc d = *desc;
  d.op = SK_OP_BOXMEAN;  // the functor is the op; no op-specific border rule
  if (int rc = validate_desc(&d)) return rc;
  desc = &d;
  if (!d_in || !d_out) return fail(SK_EINVAL, "null buffer");
  if (rows_above < 0 || rows_below < 0) return fail(SK_EINVAL, "negative halo rows");
  return launch(*desc, d_in, d_out, width, height, pitch_in, pitch_out, rows_above, rows_below,
                wc, wr, static_cast<cudaStream_t>(stream), kernels);
}

int sk_stencil_iterate(const sk_stencil_desc* desc, void* d_a, void* d_b, int64_t width,
                       int64_t height, int64_t pitch, int32_t iterations, int32_t wc,
                       int32_t wr, void* stream, int32_t* result_in_b) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (!d_a || !d_b) return fail(SK_EINVAL, "null buffer");
  if (iterations < 0) return fail(SK_EINVAL, "negative iterations");
  void* src = d_a;
  void* dst = d_b;
  int launches = 0;
  const int TB = desc->fused_iterations > 1 ? desc->fused_iterations : 1;
  if (uses_bits(*desc)) {
    // Bit-plane gol: pack, ceil(iterations / TB) strip launches, unpack into
    // d_b (d_a is left as the input).
    if (int rc = run_bits(*desc, d_a, d_b, width, height, pitch, pitch, 0, 0, wc, wr, iterations,
                          TB, static_cast<cudaStream_t>(stream))) {
      return rc;
    }
    if (result_in_b) *result_in_b = iterations > 0;
    return SK_OK;
  }
  if (uses_strips(*desc)) {
    // Register strips: ceil(iterations / TB) launches, the last one shorter.
    for (int done = 0; done < iterations; ++launches) {
      const int tb = std::min(TB, iterations - done);
      if (int rc = run_cross(*desc, src, dst, width, height, pitch, pitch, 0, 0, wc, wr, tb,
                             static_cast<cudaStream_t>(stream))) {
        return rc;
      }
      done += tb;
      std::swap(src, dst);
    }
    if (result_in_b) *result_in_b = (launches % 2) == 1;
    return SK_OK;
  }
  // one-pass (and per-cell fused) generations: replayed from a CUDA graph
  // when this exact loop ran before (graph_iterate), else launched directly
  const int rc = graph_iterate(*desc, d_a, d_b, width, height, pitch, iterations, wc, wr,
                               static_cast<cudaStream_t>(stream), &launches);
  if (rc != SK_OK) return rc;
  if (result_in_b) *result_in_b = (launches % 2) == 1;
  return SK_OK;
}

int sk_stencil_probe(const sk_stencil_desc* desc, int64_t width, int64_t height, int32_t wc,
                     int32_t wr, int32_t* kernel_max, int64_t* tile_bytes, int32_t* load_path) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (uses_strips(*desc)) {
    CrossPlan cp;
    int rc = make_cross_plan(*desc, width, height, width, width, 0, height - 1, wc, wr,
                             std::max(1, desc->fused_iterations), nullptr, nullptr, &cp);
    if (kernel_max) *kernel_max = cp.kernel_max;
    if (tile_bytes) *tile_bytes = cp.tile_bytes;
    if (load_path) *load_path = SK_LOAD_STRIPS;
    return rc;
  }
  if (uses_bits(*desc)) {
    StripPlan sp;
    int rc = make_strips_plan(*desc, width, height, 0, height - 1, wc, wr,
                              std::max(1, desc->fused_iterations), &sp);
    if (kernel_max) *kernel_max = sp.kernel_max;
    if (tile_bytes) *tile_bytes = sp.tile_bytes;
    if (load_path) *load_path = SK_LOAD_BITPLANE;
    return rc;
  }
  Plan plan;
  int rc = make_plan(*desc, width, height, width, width, 0, 0, wc, wr, nullptr, &plan);
  if (kernel_max) *kernel_max = plan.kernel_max;
  if (tile_bytes) *tile_bytes = plan.tile_bytes;
  if (load_path) *load_path = plan.g.V > 1 ? SK_LOAD_VECTOR : plan.tma ? SK_LOAD_TMA : SK_LOAD_EXPLICIT;
  return rc;
}

int sk_kernel_max_wgsize(const sk_stencil_desc* desc, int32_t* kernel_max) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (!kernel_max) return fail(SK_EINVAL, "null output");
  if (uses_strips(*desc)) {
    CrossPlan cp;
    int rc = make_cross_plan(*desc, 64, 64, 64, 64, 0, 63, 2, 2, 1, nullptr, nullptr, &cp);
    if (rc == SK_OK || rc == SK_REFUSED || rc == SK_OVERSIZED) {
      *kernel_max = cp.kernel_max;
      return SK_OK;
    }
    return rc;
  }
  if (uses_bits(*desc)) {
    StripPlan sp;
    int rc = make_strips_plan(*desc, 64, 64, 0, 63, 2, 2, 1, &sp);
    if (rc == SK_OK || rc == SK_REFUSED || rc == SK_OVERSIZED) {
      *kernel_max = sp.kernel_max;
      return SK_OK;
    }
    return rc;
  }
  Plan plan;
  // A 2x2 block on a small grid is always within the maxima; the plan
  // carries the per-kernel maximum of the path AUTO would take.
  int rc = make_plan(*desc, 64, 64, 64, 64, 0, 0, 2, 2, nullptr, &plan);
  if (rc == SK_OK || rc == SK_REFUSED || rc == SK_OVERSIZED) {
    *kernel_max = plan.kernel_max;
    return SK_OK;
  }
  return rc;
}

namespace {

int ensure_events(Scratch* s, int samples) {
  for (int i = static_cast<int>(s->events.size()); i < 2 * samples; ++i) {
    cudaEvent_t ev;
    if (cudaEventCreate(&ev) != cudaSuccess) return fail(SK_ECUDA, "cudaEventCreate failed");
    s->events.push_back(ev);
  }
  return SK_OK;
}

// write 2 x L2 (evicts everything), then read it back (the written lines
// leave dirty during this read, not during the timed pass)
int scrub_l2(Scratch* s, int sample) {
  cudaMemsetAsync(s->flush, sample & 0xff, s->flush_bytes, s->stream);
  DeviceInfo info;
  if (int rc = current_device_info(&info)) return rc;
  k_l2_scrub<<<info.sms * 4, 512, 0, s->stream>>>(static_cast<const uint4*>(s->flush),
                                                 static_cast<long long>(s->flush_bytes / 16),
                                                 static_cast<unsigned*>(s->flush));
  return SK_OK;
}

int collect_samples(Scratch* s, int samples, double* ms_out) {
  cudaError_t e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return fail(SK_ECUDA, "timing stream failed: %s", cudaGetErrorString(e));
  for (int i = 0; i < samples; ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, s->events[2 * i], s->events[2 * i + 1]);
    ms_out[i] = ms;
  }
  return SK_OK;
}

}  // namespace

int sk_stencil_time(const sk_stencil_desc* desc, const void* d_in, void* d_out, int64_t width,
                    int64_t height, int64_t pitch, int32_t wc, int32_t wr, int32_t warmup,
                    int32_t samples, int32_t flush_l2, double* ms_out) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (!d_in || !d_out || (samples > 0 && !ms_out)) return fail(SK_EINVAL, "null argument");
  Scratch* s = nullptr;
  if (int rc = scratch(&s)) return rc;
  for (int i = 0; i < warmup; ++i) {
    if (int rc = launch(*desc, d_in, d_out, width, height, pitch, pitch, 0, 0, wc, wr, s->stream)) {
      return rc;
    }
  }
  // All samples are enqueued back to back (flush, event, pass, event) and
  // synchronised once; each sample is its own event pair on the stream.
  if (int rc = ensure_events(s, samples)) return rc;
  for (int i = 0; i < samples; ++i) {
    if (flush_l2) {
      if (int rc = scrub_l2(s, i)) return rc;
    }
    cudaEventRecord(s->events[2 * i], s->stream);
    if (int rc = launch(*desc, d_in, d_out, width, height, pitch, pitch, 0, 0, wc, wr, s->stream)) {
      cudaStreamSynchronize(s->stream);
      return rc;
    }
    cudaEventRecord(s->events[2 * i + 1], s->stream);
  }
  return collect_samples(s, samples, ms_out);
}

// The streaming ceiling the one-pass kernel is held to at a given size: a
// copy of the same bytes (read + write once), 16-B vector grid-stride loop.
__global__ void k_copy_ceiling(const uint4* __restrict__ src, uint4* __restrict__ dst, long long n) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    dst[i] = src[i];
  }
}

int sk_copy_time(const void* d_in, void* d_out, int64_t bytes, int32_t kind, int32_t warmup,
                 int32_t samples, int32_t flush_l2, double* ms_out) {
  g_last_error.clear();
  if (!d_in || !d_out || bytes < 16 || (samples > 0 && !ms_out)) return fail(SK_EINVAL, "bad argument");
  if (kind != 0 && kind != 1) return fail(SK_EINVAL, "kind must be 0 (cudaMemcpyAsync) or 1 (copy kernel)");
  if (kind == 1 && ((reinterpret_cast<uintptr_t>(d_in) | reinterpret_cast<uintptr_t>(d_out) | bytes) & 15)) {
    return fail(SK_EINVAL, "the copy kernel needs 16-B aligned buffers and a multiple of 16 bytes");
  }
  Scratch* s = nullptr;
  if (int rc = scratch(&s)) return rc;
  DeviceInfo info;
  if (int rc = current_device_info(&info)) return rc;
  auto copy = [&] {
    if (kind == 0) {
      cudaMemcpyAsync(d_out, d_in, static_cast<size_t>(bytes), cudaMemcpyDeviceToDevice, s->stream);
    } else {
      k_copy_ceiling<<<info.sms * 4, 512, 0, s->stream>>>(static_cast<const uint4*>(d_in),
                                                         static_cast<uint4*>(d_out), bytes / 16);
    }
  };
  for (int i = 0; i < warmup; ++i) copy();
  if (int rc = ensure_events(s, samples)) return rc;
  for (int i = 0; i < samples; ++i) {
    if (flush_l2) {
      if (int rc = scrub_l2(s, i)) return rc;
    }
    cudaEventRecord(s->events[2 * i], s->stream);
    copy();
    cudaEventRecord(s->events[2 * i + 1], s->stream);
  }
  return collect_samples(s, samples, ms_out);
}

int sk_stencil_run_host(const sk_stencil_desc* desc, const void* h_in, void* h_out,
                        int64_t width, int64_t height, int32_t iterations, int32_t wc,
                        int32_t wr) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (!h_in || !h_out) return fail(SK_EINVAL, "null host buffer");
  if (width < 1 || height < 1) return fail(SK_EINVAL, "bad dims");
  Scratch* s = nullptr;
  if (int rc = scratch(&s)) return rc;
  size_t bytes = static_cast<size_t>(width) * height * dtype_size(desc->dtype);
  if (s->dev_bytes < bytes) {
    cudaFree(s->dev_a);
    cudaFree(s->dev_b);
    s->dev_a = s->dev_b = nullptr;
    s->dev_bytes = 0;
    if (cudaMalloc(&s->dev_a, bytes) != cudaSuccess || cudaMalloc(&s->dev_b, bytes) != cudaSuccess) {
      return fail(SK_ECUDA, "device buffer allocation failed (%zu B)", bytes);
    }
    s->dev_bytes = bytes;
  }
  cudaMemcpyAsync(s->dev_a, h_in, bytes, cudaMemcpyHostToDevice, s->stream);
  int32_t in_b = 0;
  if (int rc = sk_stencil_iterate(desc, s->dev_a, s->dev_b, width, height, width, iterations, wc,
                                  wr, s->stream, &in_b)) {
    return rc;
  }
  cudaMemcpyAsync(h_out, in_b ? s->dev_b : s->dev_a, bytes, cudaMemcpyDeviceToHost, s->stream);
  cudaError_t e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return fail(SK_ECUDA, "run_host failed: %s", cudaGetErrorString(e));
  return SK_OK;
}

int sk_stencil_submit_host(const sk_stencil_desc* desc, const void* h_in, void* h_out,
                           int64_t width, int64_t height, int32_t iterations, int32_t wc,
                           int32_t wr, int64_t* ticket) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (!h_in || !h_out || !ticket) return fail(SK_EINVAL, "null argument");
  if (width < 1 || height < 1) return fail(SK_EINVAL, "bad dims");
  Scratch* s = nullptr;
  if (int rc = scratch(&s)) return rc;
  const long long t = s->next_ticket;
  Scratch::Slot& sl = s->slots[t % 3];
  if (!sl.stream) {
    if (cudaStreamCreateWithFlags(&sl.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) != cudaSuccess) {
      return fail(SK_ECUDA, "slot stream/event creation failed");
    }
  }
  // the slot's previous job (ticket t - 3) must be finished before its
  // buffers are reused: a host wait only when the caller runs ahead
  if (sl.ticket >= 0) {
    cudaError_t e = cudaEventSynchronize(sl.done);
    if (e != cudaSuccess) return fail(SK_ECUDA, "previous job failed: %s", cudaGetErrorString(e));
  }
  const size_t bytes = static_cast<size_t>(width) * height * dtype_size(desc->dtype);
  if (sl.bytes < bytes) {
    cudaFree(sl.a);
    cudaFree(sl.b);
    sl.a = sl.b = nullptr;
    sl.bytes = 0;
    if (cudaMalloc(&sl.a, bytes) != cudaSuccess || cudaMalloc(&sl.b, bytes) != cudaSuccess) {
      return fail(SK_ECUDA, "device buffer allocation failed (%zu B)", bytes);
    }
    sl.bytes = bytes;
  }
  cudaMemcpyAsync(sl.a, h_in, bytes, cudaMemcpyHostToDevice, sl.stream);
  int32_t in_b = 0;
  if (int rc = sk_stencil_iterate(desc, sl.a, sl.b, width, height, width, iterations, wc, wr,
                                  sl.stream, &in_b)) {
    return rc;
  }
  cudaMemcpyAsync(h_out, in_b ? sl.b : sl.a, bytes, cudaMemcpyDeviceToHost, sl.stream);
  cudaError_t e = cudaEventRecord(sl.done, sl.stream);
  if (e != cudaSuccess) return fail(SK_ECUDA, "submit failed: %s", cudaGetErrorString(e));
  sl.ticket = t;
  s->next_ticket = t + 1;
  *ticket = t;
  return SK_OK;
}

int sk_stencil_wait_host(int64_t ticket) {
  g_last_error.clear();
  Scratch* s = nullptr;
  if (int rc = scratch(&s)) return rc;
  if (ticket < 0 || ticket >= s->next_ticket) return fail(SK_EINVAL, "unknown ticket %lld", (long long)ticket);
  Scratch::Slot& sl = s->slots[ticket % 3];
  if (sl.ticket != ticket) {
    // the slot has moved on: a later submit already waited for this job
    return ticket < sl.ticket ? SK_OK : fail(SK_EINVAL, "ticket %lld not in flight", (long long)ticket);
  }
  cudaError_t e = cudaEventSynchronize(sl.done);
  if (e != cudaSuccess) return fail(SK_ECUDA, "job %lld failed: %s", (long long)ticket, cudaGetErrorString(e));
  return SK_OK;
}

int sk_device_features(int32_t device, sk_device_props* out) {
  g_last_error.clear();
  if (!out) return fail(SK_EINVAL, "null output");
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return fail(SK_ECUDA, "cudaGetDeviceProperties: %s", cudaGetErrorString(e));
  std::memset(out, 0, sizeof(*out));
  // Stable across boxes (scenario ids embed it): the marketing name only;
  // identical GPUs are the same tuning device.
  std::string name = std::string(p.name);
  for (char& ch : name) {
    if (ch == '/' || ch == ',' || ch == '\n' || ch == ' ') ch = '-';
  }
  std::snprintf(out->name, sizeof out->name, "%s", name.c_str());
  int clock_khz = 0, mem_khz = 0;
  cudaDeviceGetAttribute(&clock_khz, cudaDevAttrClockRate, device);
  cudaDeviceGetAttribute(&mem_khz, cudaDevAttrMemoryClockRate, device);
  out->compute_units = p.multiProcessorCount;
  out->frequency_mhz = clock_khz / 1000;
  out->local_mem_kb = static_cast<int32_t>(p.sharedMemPerBlockOptin / 1024);
  out->global_cache_kb = p.l2CacheSize / 1024;
  out->global_mem_mb = static_cast<int32_t>(p.totalGlobalMem >> 20);
  out->device_max_wgsize = p.maxThreadsPerBlock;
  out->simd_width = p.warpSize;
  out->cc_major = p.major;
  out->cc_minor = p.minor;
  out->mem_clock_mhz = mem_khz / 1000;
  out->mem_bus_width = p.memoryBusWidth;
  return SK_OK;
}

int sk_buffers_equal(const void* d_a, const void* d_b, int64_t bytes, int32_t* equal) {
  g_last_error.clear();
  if (!d_a || !d_b || !equal || bytes < 0) return fail(SK_EINVAL, "bad compare arguments");
  if (bytes % 16 != 0 || reinterpret_cast<uintptr_t>(d_a) % 16 || reinterpret_cast<uintptr_t>(d_b) % 16) {
    return fail(SK_EINVAL, "compare needs 16-B aligned buffers and sizes");
  }
  Scratch* s = nullptr;
  if (int rc = scratch(&s)) return rc;
  if (!s->diff && cudaMalloc(&s->diff, sizeof(unsigned long long)) != cudaSuccess) {
    return fail(SK_ECUDA, "cudaMalloc(diff)");
  }
  cudaMemsetAsync(s->diff, 0, sizeof(unsigned long long), s->stream);
  const long long words = bytes / 16;
  DeviceInfo info;
  current_device_info(&info);
  const int grid = static_cast<int>(std::min<long long>((words + 255) / 256, 4LL * info.sms));
  if (grid > 0) {
    k_count_diff<<<grid, 256, 0, s->stream>>>(static_cast<const uint4*>(d_a),
                                              static_cast<const uint4*>(d_b), words,
                                              static_cast<unsigned long long*>(s->diff));
  }
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, s->diff, sizeof h, cudaMemcpyDeviceToHost, s->stream);
  cudaError_t e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) return fail(SK_ECUDA, "compare failed: %s", cudaGetErrorString(e));
  *equal = h == 0;
  return SK_OK;
}

int sk_fill_host(int32_t dtype, int32_t kind, uint64_t seed, void* h_out, int64_t count) {
  g_last_error.clear();
  if (!h_out || count < 0) return fail(SK_EINVAL, "bad fill arguments");
  std::mt19937_64 eng(seed);  // the reference Rng engine (rng.hpp:34-72)
  auto u01 = [&]() { return static_cast<double>(eng() >> 11) * 0x1.0p-53; };
  for (int64_t i = 0; i < count; ++i) {
    double u = u01();
    double v = kind == 0 ? 2.0 * u - 1.0 : kind == 1 ? u : kind == 2 ? (u < 0.5 ? 1.0 : 0.0)
                                                                      : std::floor(256.0 * u);
    switch (dtype) {
      case SK_INT32: static_cast<int32_t*>(h_out)[i] = static_cast<int32_t>(v); break;
      case SK_FLOAT32: static_cast<float*>(h_out)[i] = static_cast<float>(v); break;
      case SK_FLOAT64: static_cast<double*>(h_out)[i] = v; break;
      default: return fail(SK_EINVAL, "bad dtype");
    }
  }
  return SK_OK;
}

}  // extern "C"
