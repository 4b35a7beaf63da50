// NCCL halo exchange for row-sharded iterated stencils, behind the C-ABI
// (sk_stencil_iterate_nccl, include/sk_stencil.h).
//
// Each rank owns `rows` consecutive rows of the global grid and holds them
// in two ping-pong buffers of N + rows + S rows (N north halo rows, S south).
// Per generation:
//   comm stream    : [wait: previous generation complete]
//                    ncclGroupStart
//                      send first S owned rows -> rank-1, recv N halo rows <- rank-1
//                      send last  N owned rows -> rank+1, recv S halo rows <- rank+1
//                    ncclGroupEnd
//   compute stream : interior rows [N, rows-S)  (needs no halo; overlaps the exchange)
//                    [wait: exchange]  north strip [0, N), south strip [rows-S, rows)
// Global edges (rank 0's north, rank n-1's south) are border cells of the
// stencil's border mode, exactly as in a single-GPU pass.  Row-major rows
// are contiguous, so halo messages are the raw row spans (no packing).
//
// NCCL is resolved at run time (dlopen "libnccl.so.2"): the caller's
// communicator must come from the NCCL already loaded in the process (torch's,
// or the one a C++ host links), and the stencil library does not link NCCL.
#include <dlfcn.h>

#include <cstddef>
#include <map>
#include <mutex>
#include <thread>

#include "launch_internal.cuh"

namespace sk {
namespace detail {
namespace {

// The slice of nccl.h this file uses (ABI-stable since NCCL 2.7).
using nccl_result = int;  // ncclSuccess = 0
constexpr int kNcclUint8 = 1;
using FnGroup = nccl_result (*)();
using FnSend = nccl_result (*)(const void*, size_t, int, int, void*, cudaStream_t);
using FnRecv = nccl_result (*)(void*, size_t, int, int, void*, cudaStream_t);
using FnErr = const char* (*)(nccl_result);

struct Nccl {
  FnGroup group_start = nullptr, group_end = nullptr;
  FnSend send = nullptr;
  FnRecv recv = nullptr;
  FnErr error_string = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's NCCL
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return x;
    x.group_start = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupStart"));
    x.group_end = reinterpret_cast<FnGroup>(dlsym(h, "ncclGroupEnd"));
    x.send = reinterpret_cast<FnSend>(dlsym(h, "ncclSend"));
    x.recv = reinterpret_cast<FnRecv>(dlsym(h, "ncclRecv"));
    x.error_string = reinterpret_cast<FnErr>(dlsym(h, "ncclGetErrorString"));
    x.ok = x.group_start && x.group_end && x.send && x.recv;
    return x;
  }();
  return n;
}

// Per (device, calling thread): the exchange stream and its two events.
struct CommStream {
  cudaStream_t stream = nullptr;  // the exchange
  cudaStream_t side = nullptr;    // the south strip, beside the north strip
  cudaEvent_t ready = nullptr, halo = nullptr, south = nullptr;
};
std::mutex g_comm_mu;
std::map<std::pair<int, std::thread::id>, CommStream> g_comm;

int comm_stream(CommStream** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(SK_ECUDA, "cudaGetDevice failed");
  std::lock_guard<std::mutex> lk(g_comm_mu);
  CommStream& c = g_comm[{dev, std::this_thread::get_id()}];
  if (!c.stream) {
    if (cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&c.side, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.ready, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.halo, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.south, cudaEventDisableTiming) != cudaSuccess) {
      return fail(SK_ECUDA, "exchange stream/event creation failed");
    }
  }
  *out = &c;
  return SK_OK;
}

int nccl_check(nccl_result r, const char* what) {
  if (r == 0) return SK_OK;
  const Nccl& n = nccl();
  return fail(SK_ECUDA, "%s failed: %s", what, n.error_string ? n.error_string(r) : "NCCL error");
}

}  // namespace
}  // namespace detail
}  // namespace sk

using namespace sk::detail;

extern "C" int sk_stencil_iterate_nccl(const sk_stencil_desc* desc, void* d_a, void* d_b, int64_t width,
                                       int64_t rows, int64_t pitch, int32_t iterations, int32_t wc,
                                       int32_t wr, void* comm, int32_t rank, int32_t nranks, void* stream,
                                       int32_t* result_in_b) {
  g_last_error.clear();
  if (int rc = validate_desc(desc)) return rc;
  if (!d_a || !d_b) return fail(SK_EINVAL, "null buffer");
  if (iterations < 0 || width < 1 || rows < 1 || pitch < width) return fail(SK_EINVAL, "bad shard geometry");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(SK_EINVAL, "rank %d of %d", rank, nranks);
  if (nranks > 1 && !comm) return fail(SK_EINVAL, "null NCCL communicator");
  if (desc->fused_iterations > 1 || uses_bits(*desc) || uses_strips(*desc)) {
    return fail(SK_ENOTSUP, "the NCCL schedule exchanges one generation of halo per launch "
                            "(fused_iterations <= 1, one-pass load paths)");
  }
  const int N = desc->north, S = desc->south;
  if (rows < static_cast<int64_t>(N) + S) {
    return fail(SK_EINVAL, "a shard of %lld rows cannot source %d + %d halo rows", static_cast<long long>(rows), N, S);
  }
  static const Nccl none{};
  const Nccl& n = nranks > 1 ? nccl() : none;  // one rank: no exchange, NCCL never loaded
  if (nranks > 1 && !n.ok) return fail(SK_ENOTSUP, "libnccl.so.2 not loadable: %s", dlerror());
  CommStream* cs = nullptr;
  if (int rc = comm_stream(&cs)) return rc;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t es = dtype_size(desc->dtype);
  const long long rb = pitch * static_cast<long long>(es);  // bytes per row
  const bool has_n = rank > 0, has_s = rank < nranks - 1;
  sk_stencil_desc one = *desc;
  one.fused_iterations = 0;

  char* src = static_cast<char*>(d_a);
  char* dst = static_cast<char*>(d_b);
  auto row = [&](char* base, long long r) { return base + (N + r) * rb; };  // owned row r
  const int swc = es == 8 ? 124 : 62;
  const bool strips = N > 0 || S > 0;
  for (int it = 0; it < iterations; ++it) {
    // generation start: src is complete on the caller's stream
    if (cudaEventRecord(cs->ready, st) != cudaSuccess) return fail(SK_ECUDA, "generation ordering failed");
    if (nranks > 1) {
      if (cudaStreamWaitEvent(cs->stream, cs->ready, 0) != cudaSuccess) {
        return fail(SK_ECUDA, "exchange ordering failed");
      }
      if (int rc = nccl_check(n.group_start(), "ncclGroupStart")) return rc;
      int rc = SK_OK;
      if (has_n && rc == SK_OK) {
        if (S > 0) rc = nccl_check(n.send(row(src, 0), static_cast<size_t>(S * rb), kNcclUint8, rank - 1, comm, cs->stream), "ncclSend");
        if (rc == SK_OK && N > 0) rc = nccl_check(n.recv(row(src, -N), static_cast<size_t>(N * rb), kNcclUint8, rank - 1, comm, cs->stream), "ncclRecv");
      }
      if (has_s && rc == SK_OK) {
        if (N > 0) rc = nccl_check(n.send(row(src, rows - N), static_cast<size_t>(N * rb), kNcclUint8, rank + 1, comm, cs->stream), "ncclSend");
        if (rc == SK_OK && S > 0) rc = nccl_check(n.recv(row(src, rows), static_cast<size_t>(S * rb), kNcclUint8, rank + 1, comm, cs->stream), "ncclRecv");
      }
      const int rc_end = nccl_check(n.group_end(), "ncclGroupEnd");
      if (rc != SK_OK) return rc;
      if (rc_end != SK_OK) return rc_end;
      if (cudaEventRecord(cs->halo, cs->stream) != cudaSuccess) return fail(SK_ECUDA, "exchange event failed");
    }
    // Boundary strips on the side stream, behind the halo (or the generation
    // start at one rank), queued before the interior so their few CTAs are
    // resident beside the persistent interior grid instead of after it.
    if (strips && cudaStreamWaitEvent(cs->side, nranks > 1 ? cs->halo : cs->ready, 0) != cudaSuccess) {
      return fail(SK_ECUDA, "strip ordering failed");
    }
    if (N > 0) {
      if (int rc = launch(one, row(src, 0), row(dst, 0), width, N, pitch, pitch, has_n ? N : 0, S, swc, 1, cs->side)) {
        return rc;
      }
    }
    if (S > 0) {
      if (int rc = launch(one, row(src, rows - S), row(dst, rows - S), width, S, pitch, pitch, N, has_s ? S : 0,
                          swc, 1, cs->side)) {
        return rc;
      }
    }
    const long long inner = rows - N - S;
    if (inner > 0) {
      if (int rc = launch(one, row(src, N), row(dst, N), width, inner, pitch, pitch, N, S, wc, wr, st)) return rc;
    }
    if (strips && (cudaEventRecord(cs->south, cs->side) != cudaSuccess ||
                   cudaStreamWaitEvent(st, cs->south, 0) != cudaSuccess)) {
      return fail(SK_ECUDA, "strip join failed");
    }
    std::swap(src, dst);
  }
  if (result_in_b) *result_in_b = (iterations % 2) == 1;
  return SK_OK;
}
