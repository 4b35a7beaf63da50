// Test double for NCCL point-to-point, for exercising the NCCL halo schedule
// (sk_stencil_iterate_nccl) with several ranks on ONE GPU, where real NCCL
// refuses two ranks on the same device.  Built with soname libnccl.so.2 so
// the stencil library's dlopen("libnccl.so.2", RTLD_NOLOAD) finds it.
// Ranks are threads of one process; a communicator is a (rank, world) pair.
//
// Semantics kept from NCCL: inside ncclGroupStart/End a rank posts sends and
// receives; ncclGroupEnd returns once its receives are enqueued on its
// stream (each ordered after the matching send was posted on the sender's
// stream) and its sends' source buffers may be reused only after the
// receiver's copies - the sender's stream waits for them.  Matching is FIFO
// per (sender, receiver) pair.  Test infrastructure only.
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <deque>
#include <map>
#include <mutex>
#include <vector>

namespace {

struct Msg {
  const void* src;
  size_t bytes;
  cudaEvent_t posted;                 // recorded on the sender's stream
  cudaEvent_t copied = nullptr;       // recorded on the receiver's stream
  bool done = false;
};

struct World {
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<Msg*>> inbox;  // (from, to)
};

struct Comm {
  int rank, nranks;
  World* world;
};

struct Op {
  bool send;
  void* buf;
  size_t bytes;
  int peer;
  Comm* comm;
  cudaStream_t stream;
};
thread_local std::vector<Op> t_group;
thread_local int t_depth = 0;

int run_group() {
  std::vector<Msg*> mine;
  // 1. post sends
  for (Op& o : t_group) {
    if (!o.send) continue;
    Msg* m = new Msg{o.buf, o.bytes, nullptr};
    cudaEventCreateWithFlags(&m->posted, cudaEventDisableTiming);
    cudaEventRecord(m->posted, o.stream);
    {
      std::lock_guard<std::mutex> lk(o.comm->world->mu);
      o.comm->world->inbox[{o.comm->rank, o.peer}].push_back(m);
    }
    o.comm->world->cv.notify_all();
    mine.push_back(m);
  }
  // 2. receives: wait for the matching send, copy on this rank's stream
  for (Op& o : t_group) {
    if (o.send) continue;
    World* w = o.comm->world;
    Msg* m = nullptr;
    {
      std::unique_lock<std::mutex> lk(w->mu);
      auto& q = w->inbox[{o.peer, o.comm->rank}];
      w->cv.wait(lk, [&] { return !q.empty(); });
      m = q.front();
      q.pop_front();
    }
    if (m->bytes != o.bytes) return 5;  // ncclInvalidUsage
    cudaStreamWaitEvent(o.stream, m->posted, 0);
    cudaMemcpyAsync(o.buf, m->src, o.bytes, cudaMemcpyDeviceToDevice, o.stream);
    cudaEvent_t c;
    cudaEventCreateWithFlags(&c, cudaEventDisableTiming);
    cudaEventRecord(c, o.stream);
    {
      std::lock_guard<std::mutex> lk(w->mu);
      m->copied = c;
      m->done = true;
    }
    w->cv.notify_all();
  }
  // 3. the sender's stream may not run ahead of the receivers' copies
  for (size_t i = 0, k = 0; i < t_group.size(); ++i) {
    Op& o = t_group[i];
    if (!o.send) continue;
    Msg* m = mine[k++];
    World* w = o.comm->world;
    std::unique_lock<std::mutex> lk(w->mu);
    w->cv.wait(lk, [&] { return m->done; });
    lk.unlock();
    cudaStreamWaitEvent(o.stream, m->copied, 0);
    cudaStreamSynchronize(o.stream);  // events of this message can go
    cudaEventDestroy(m->posted);
    cudaEventDestroy(m->copied);
    delete m;
  }
  t_group.clear();
  return 0;
}

}  // namespace

extern "C" {

// Test entry point: communicators for `nranks` thread-ranks of one world.
void fake_nccl_make_comms(int nranks, void** comms) {
  World* w = new World;
  for (int r = 0; r < nranks; ++r) comms[r] = new Comm{r, nranks, w};
}

int ncclGroupStart() {
  ++t_depth;
  return 0;
}

int ncclGroupEnd() {
  if (--t_depth > 0) return 0;
  return run_group();
}

int ncclSend(const void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t stream) {
  if (dtype != 1) return 4;  // this double only carries bytes (ncclUint8)
  t_group.push_back({true, const_cast<void*>(buf), count, peer, static_cast<Comm*>(comm), stream});
  return t_depth > 0 ? 0 : run_group();
}

int ncclRecv(void* buf, size_t count, int dtype, int peer, void* comm, cudaStream_t stream) {
  if (dtype != 1) return 4;
  t_group.push_back({false, buf, count, peer, static_cast<Comm*>(comm), stream});
  return t_depth > 0 ? 0 : run_group();
}

const char* ncclGetErrorString(int r) { return r == 0 ? "no error" : "fake NCCL error"; }

}  // extern "C"
