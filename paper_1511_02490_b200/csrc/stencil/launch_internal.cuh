// Internal interface of the host side (launch.cu, temporal.cu, peer.cu):
// device facts, legality and launch plans, the tensor-map cache, kernel
// dispatch, per-thread scratch.  Not part of the C-ABI.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <type_traits>

#include "cross_strips.cuh"
#include "gol_bits.cuh"
#include "halo.cuh"
#include "kernels.cuh"
#include "registry.cuh"
#include "sk_stencil.h"

namespace sk {
namespace detail {

// ---------------------------------------------------------------- errors
extern thread_local std::string g_last_error;  // sk_last_error()
extern std::mutex g_mu;                        // guards every cache below
int fail(int code, const char* fmt, ...);
bool is_config_error(cudaError_t e);
// Status for a failed launch: SK_REFUSED / SK_EINVAL / SK_ECUDA.
int launch_error(cudaError_t e);
// A one-pass TMA kernel launched with programmatic stream serialization
// (PDL): its prologue may overlap the previous kernel's tail; the kernel
// waits (griddepcontrol.wait) before any global access.  SK_PDL=0 disables.
cudaError_t launch_tma(const void* kernel, dim3 grid, dim3 block, void** args, int smem, cudaStream_t stream);
// The same for kernels that execute griddepcontrol.wait before their first
// global access (the register-strip and bit-plane kernels), with the launch
// status mapped like launch_checked.
int launch_pdl_checked(const void* kernel, dim3 grid, dim3 block, void** args, int smem, cudaStream_t stream);
size_t dtype_size(int dtype);

// ---------------------------------------------------------- device facts
struct DeviceInfo {
  int sms = 0;
  int max_threads = 0;
  int smem_optin = 0;
  int smem_per_sm = 0;
  int l2_bytes = 0;
};

int current_device_info(DeviceInfo* out, int* dev_out = nullptr);

// ------------------------------------------------------------ descriptors
constexpr int kMaxBitsTB = 128;   // bit-plane GoL generations per launch
constexpr int kMaxStripsTB = 32;  // register-strip generations per launch
bool uses_bits(const sk_stencil_desc& d);
bool uses_strips(const sk_stencil_desc& d);
int validate_desc(const sk_stencil_desc* d);
int cells_per_thread(const sk_stencil_desc& d, int wr, long long H);

// Per-(device, kernel) attributes: kernel max threads and the opt-in smem
// attribute, set once.
struct KernelAttr {
  int max_threads = 0;
  int max_dyn_smem = 0;
};
int kernel_attr(int dev, KernelPtr k, const DeviceInfo& info, KernelAttr* out, bool is_driver = false);
int occupancy(int dev, KernelPtr k, int threads, int smem, bool is_driver = false);
int launch_checked(KernelPtr k, dim3 grid, dim3 block, void** args, int smem, cudaStream_t stream);

// ------------------------------------------------------------ tensor maps
struct MapKey {
  int dev;
  const void* base;
  int dtype;
  long long w, h, pitch;
  int box_w, box_h;
  bool operator<(const MapKey& o) const {
    return std::tie(dev, base, dtype, w, h, pitch, box_w, box_h) <
           std::tie(o.dev, o.base, o.dtype, o.w, o.h, o.pitch, o.box_w, o.box_h);
  }
};
int tensor_map(const MapKey& key, CUtensorMap* out);

// ------------------------------------------------------ one-pass launches
struct Plan {
  Geom g{};
  KernelPtr kernel = nullptr;
  bool driver_handle = false;  // kernel is a CUfunction of a custom functor
  bool tma = false;
  int threads = 0;
  int smem = 0;
  int grid = 0;
  int kernel_max = 0;
  long long tile_bytes = 0;
};

int make_plan(const sk_stencil_desc& d, long long W, long long H, long long pitch_in,
              long long pitch_out, long long above, long long below, int wc, int wr,
              const void* in, Plan* plan, const sk_kernel_table* custom = nullptr);
int launch_driver(const Plan& plan, dim3 grid, dim3 block, void** args, cudaStream_t stream);
// One launch of `desc` (any path: one-pass, fused, bit-plane, strips).
int launch(const sk_stencil_desc& d, const void* in, void* out, long long W, long long H,
           long long pitch_in, long long pitch_out, long long above, long long below, int wc,
           int wr, cudaStream_t stream, const sk_kernel_table* custom = nullptr);

// ------------------------------------------- temporal paths (temporal.cu)
struct StripPlan {
  StripGeom g{};
  KernelPtr kernel = nullptr;
  int threads = 0;     // launched: wc*wr rounded up to whole warps
  int smem = 0;
  long long grid = 0;
  int kernel_max = 0;
  long long tile_bytes = 0;
};
int make_strips_plan(const sk_stencil_desc& d, long long W, long long H, long long lo,
                     long long hi, int wc, int wr, int tb, StripPlan* plan);
int run_bits(const sk_stencil_desc& d, const void* in, void* out, long long W, long long H,
             long long pitch_in, long long pitch_out, long long above, long long below, int wc,
             int wr, int iterations, int TB, cudaStream_t stream);

struct CrossPlan {
  CrossGeom g{};
  KernelPtr kernel = nullptr;
  int threads = 0;
  int smem = 0;
  long long grid = 0;
  int kernel_max = 0;
  long long tile_bytes = 0;
};
int make_cross_plan(const sk_stencil_desc& d, long long W, long long H, long long pitch_in,
                    long long pitch_out, long long lo, long long hi, int wc, int wr, int tb,
                    const void* in, const void* out, CrossPlan* plan);
int run_cross(const sk_stencil_desc& d, const void* in, void* out, long long W, long long H,
              long long pitch_in, long long pitch_out, long long above, long long below, int wc,
              int wr, int tb, cudaStream_t stream);

// --------------------------------------------- per-thread scratch (launch.cu)
// Packed ping-pong grids of the bit-plane path, grown as needed.
// Two packed bit grids of the bit-plane path, stream-ordered
// (cudaMallocAsync / cudaFreeAsync on `stream`, from the device's default
// pool, which is set to retain its memory so repeated calls do not remap).
struct StreamBits {
  cudaStream_t stream;
  void* p[2] = {nullptr, nullptr};
  explicit StreamBits(cudaStream_t s) : stream(s) {}
  int alloc(size_t bytes);
  ~StreamBits();
  StreamBits(const StreamBits&) = delete;
  StreamBits& operator=(const StreamBits&) = delete;
};

// ------------------------------------------------------- op parameters
inline long long binom(int n, int k) {
  long long r = 1;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

template <typename T>
inline void fill_params(const sk_stencil_desc& d, OpParams<T>* p) {
  std::memset(p, 0, sizeof(*p));
  p->north = d.north;
  p->south = d.south;
  p->east = d.east;
  p->west = d.west;
  p->complexity = d.complexity;
  // Synthetic kernels: instruction budget -> dependent ALU steps per cell
  // (DESIGN.md §3.9): heavy (synthetic-b) instructions/4, light instructions/32.
  p->alu_iters = d.op == SK_OP_SYNTHETIC ? (d.complexity ? d.instructions / 4 : d.instructions / 32)
                                         : 0;
  if (d.op == SK_OP_GAUSSIAN) {
    const int g = d.north;
    p->gauss_radius = g;
    for (int j = 0; j <= 2 * g; ++j) {
      const long long c = binom(2 * g, j);
      if constexpr (std::is_same_v<T, int32_t>) {
        p->gauss_b[j] = c;
      } else {
        p->gauss_b[j] = static_cast<T>(std::ldexp(static_cast<double>(c), -2 * g));
      }
    }
  }
}

// ------------------------------------------------ typed one-pass launch
template <typename T>
inline int launch_typed(const sk_stencil_desc& d, const Plan& plan, const void* in, void* out,
                 long long above_rows, long long H_total_rows, cudaStream_t stream) {
  OpParams<T> p;
  fill_params<T>(d, &p);
  T pad = static_cast<T>(d.pad_value);
  if (plan.g.V > 1 && ((reinterpret_cast<uintptr_t>(out) % 16) != 0 ||
                       (plan.g.pitch_out * static_cast<long long>(sizeof(T))) % 16 != 0)) {
    return fail(SK_EINVAL, "the vector path stores 16 B per row: output and its pitch must be 16-B aligned");
  }
  dim3 block(plan.g.wc, plan.g.wr, 1);
  cudaError_t e;
  if (plan.tma) {
    int dev = 0;
    cudaGetDevice(&dev);
    MapKey key{dev,
               static_cast<const char*>(in) -
                   above_rows * plan.g.pitch_in * static_cast<long long>(sizeof(T)),
               d.dtype,
               plan.g.W,
               H_total_rows,
               plan.g.pitch_in,
               plan.g.tile_w,
               plan.g.box_h};
    CUtensorMap map;
    if (int rc = tensor_map(key, &map)) return rc;
    void* args[] = {&map, &out, const_cast<Geom*>(&plan.g), &pad, &p};
    if (plan.driver_handle) return launch_driver(plan, dim3(plan.grid), block, args, stream);
    e = launch_tma(plan.kernel, dim3(plan.grid), block, args, plan.smem, stream);
  } else {
    const T* tin = static_cast<const T*>(in);
    T* tout = static_cast<T*>(out);
    void* args[] = {&tin, &tout, const_cast<Geom*>(&plan.g), &pad, &p};
    if (plan.driver_handle) {
      return launch_driver(plan, dim3(plan.g.tiles_x * plan.g.tiles_y), block, args, stream);
    }
    e = cudaLaunchKernel(plan.kernel, dim3(plan.g.tiles_x * plan.g.tiles_y), block, args,
                         plan.smem, stream);
  }
  if (e != cudaSuccess) return launch_error(e);
  return SK_OK;
}


}  // namespace detail
}  // namespace sk
