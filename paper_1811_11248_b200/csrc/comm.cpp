// NCCL for the multi-GPU factor: one communicator per handle, loaded with
// dlopen at hs_create time only when world_size > 1, so the single-GPU library has no NCCL
// dependency and a process that already carries torch's NCCL reuses that copy (libnccl.so.2
// resolves to the already-loaded library; HS_NCCL_LIB overrides the path).
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>
#include <string>

#include "runtime.h"

namespace hs {

namespace {

struct NcclApi {
  void* so = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

const NcclApi& nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.so) return g_nccl;
  const char* env = std::getenv("HS_NCCL_LIB");
  for (const char* path : {env, "libnccl.so.2", "libnccl.so"}) {
    if (!path) continue;
    g_nccl.so = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.so) break;
  }
  if (!g_nccl.so) fail(HS_E_NCCL, std::string("cannot load NCCL: ") + dlerror());
  auto sym = [](const char* n) {
    void* p = dlsym(g_nccl.so, n);
    if (!p) fail(HS_E_NCCL, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))sym("ncclGetUniqueId");
  g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))sym("ncclCommInitRank");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))sym("ncclCommDestroy");
  g_nccl.AllReduce = (decltype(g_nccl.AllReduce))sym("ncclAllReduce");
  g_nccl.Send = (decltype(g_nccl.Send))sym("ncclSend");
  g_nccl.Recv = (decltype(g_nccl.Recv))sym("ncclRecv");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))sym("ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))sym("ncclGroupEnd");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))sym("ncclGetErrorString");
  return g_nccl;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) fail(HS_E_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

}  // namespace

void nccl_unique_id(void* out128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out128, &id, sizeof id);
}

// ---- the transport interface used by the factor ------------------------------------------
struct Comm {
  int world = 1, rank = 0;
  virtual ~Comm() {}
  virtual void allreduce_sum_i32(int32_t* d_buf, size_t n, cudaStream_t st) = 0;
  virtual void allreduce_sum_f64(double* d_buf, size_t n, cudaStream_t st) = 0;
  virtual void group_start() = 0;
  virtual void group_end(cudaStream_t st) = 0;
  virtual void send(const double* d, size_t n, int peer, cudaStream_t st) = 0;
  virtual void recv(double* d, size_t n, int peer, cudaStream_t st) = 0;
};

namespace {

struct NcclComm : Comm {
  ncclComm_t c = nullptr;
  ~NcclComm() override {
    if (c && g_nccl.so) g_nccl.CommDestroy(c);
  }
  void allreduce_sum_i32(int32_t* d_buf, size_t n, cudaStream_t st) override {
    if (n) check(nccl().AllReduce(d_buf, d_buf, n, ncclInt32, ncclSum, c, st), "ncclAllReduce");
  }
  void allreduce_sum_f64(double* d_buf, size_t n, cudaStream_t st) override {
    if (n) check(nccl().AllReduce(d_buf, d_buf, n, ncclFloat64, ncclSum, c, st), "ncclAllReduce");
  }
  void group_start() override { check(nccl().GroupStart(), "ncclGroupStart"); }
  void group_end(cudaStream_t) override { check(nccl().GroupEnd(), "ncclGroupEnd"); }
  void send(const double* d, size_t n, int peer, cudaStream_t st) override {
    if (n) check(nccl().Send(d, n, ncclFloat64, peer, c, st), "ncclSend");
  }
  void recv(double* d, size_t n, int peer, cudaStream_t st) override {
    if (n) check(nccl().Recv(d, n, ncclFloat64, peer, c, st), "ncclRecv");
  }
};

}  // namespace

// ---- loopback transport: P ranks as P host threads of one process on one device ----------
// Test harness for the multi-GPU factor on a single GPU (tests/test_gpu_dist.py): the
// exchanges become device-to-device copies ordered by CUDA events between the ranks'
// streams, so no kernel ever waits on another rank's kernel.  Blocking points (the
// all-reduce and the end of a send/recv group) meet at a host barrier.
struct LoopWorld {
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  struct Msg {
    const double* src;
    double* dst;
    size_t n;
    int from, to;
  };
  std::vector<std::vector<Msg>> sends, recvs;   // per rank, posted in the current group
  std::vector<cudaEvent_t> ev_send, ev_done;    // per rank
  std::vector<std::vector<int32_t>> red;        // per rank all-reduce contributions
  std::vector<std::vector<double>> redf;
  explicit LoopWorld(int w) : world(w), sends(w), recvs(w), ev_send(w, nullptr), ev_done(w, nullptr), red(w), redf(w) {
    for (int r = 0; r < w; ++r) {
      HS_CUDA(cudaEventCreateWithFlags(&ev_send[r], cudaEventDisableTiming));
      HS_CUDA(cudaEventCreateWithFlags(&ev_done[r], cudaEventDisableTiming));
    }
  }
  ~LoopWorld() {
    for (auto e : ev_send) cudaEventDestroy(e);
    for (auto e : ev_done) cudaEventDestroy(e);
  }
  void barrier() {   // a rank that failed never arrives: give up instead of hanging the test
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else if (!cv.wait_for(lk, std::chrono::seconds(60), [&] { return gen != g; })) {
      fail(HS_E_INTERNAL, "loopback: barrier timed out (another rank failed)");
    }
  }
};

namespace {

struct LoopComm : Comm {
  LoopWorld* w = nullptr;
  std::vector<LoopWorld::Msg> my_send, my_recv;
  void allreduce_sum_i32(int32_t* d_buf, size_t n, cudaStream_t st) override {
    std::vector<int32_t> v(n);
    HS_CUDA(cudaMemcpyAsync(v.data(), d_buf, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    w->red[rank] = v;
    w->barrier();
    std::vector<int32_t> sum(n, 0);
    for (int r = 0; r < world; ++r)
      for (size_t i = 0; i < n; ++i) sum[i] += w->red[r][i];
    w->barrier();   // everybody has read the contributions
    HS_CUDA(cudaMemcpyAsync(d_buf, sum.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaStreamSynchronize(st));
  }
  void allreduce_sum_f64(double* d_buf, size_t n, cudaStream_t st) override {   // sum in rank order
    std::vector<double> v(n);
    HS_CUDA(cudaMemcpyAsync(v.data(), d_buf, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    w->redf[rank] = v;
    w->barrier();
    std::vector<double> sum(n, 0.0);
    for (int r = 0; r < world; ++r)
      for (size_t i = 0; i < n; ++i) sum[i] += w->redf[r][i];
    w->barrier();
    HS_CUDA(cudaMemcpyAsync(d_buf, sum.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaStreamSynchronize(st));
  }
  void group_start() override {
    my_send.clear();
    my_recv.clear();
  }
  void send(const double* d, size_t n, int peer, cudaStream_t) override {
    if (n) my_send.push_back({d, nullptr, n, rank, peer});
  }
  void recv(double* d, size_t n, int peer, cudaStream_t) override {
    if (n) my_recv.push_back({nullptr, d, n, peer, rank});
  }
  void group_end(cudaStream_t st) override {
    // 1. post: the send buffers are complete at this point of my stream
    HS_CUDA(cudaEventRecord(w->ev_send[rank], st));
    w->sends[rank] = my_send;
    w->barrier();
    // 2. pull every message addressed to me (pairwise in posting order), after its sender
    std::vector<size_t> next(world, 0);
    for (auto& r : my_recv) {
      auto& box = w->sends[r.from];
      size_t& k = next[r.from];
      while (k < box.size() && box[k].to != rank) ++k;
      if (k == box.size()) fail(HS_E_INTERNAL, "loopback: receive without a matching send");
      if (box[k].n != r.n) fail(HS_E_INTERNAL, "loopback: message size mismatch");
      HS_CUDA(cudaStreamWaitEvent(st, w->ev_send[r.from], 0));
      HS_CUDA(cudaMemcpyAsync(r.dst, box[k].src, sizeof(double) * r.n, cudaMemcpyDeviceToDevice, st));
      ++k;
    }
    for (int from = 0; from < world; ++from) {   // every send to me must have been received
      for (size_t k = next[from]; k < w->sends[from].size(); ++k)
        if (w->sends[from][k].to == rank) fail(HS_E_INTERNAL, "loopback: send without a matching receive");
    }
    HS_CUDA(cudaEventRecord(w->ev_done[rank], st));
    w->barrier();
    // 3. my send buffers may be reused only after the receivers' copies
    for (int to = 0; to < world; ++to)
      if (to != rank) HS_CUDA(cudaStreamWaitEvent(st, w->ev_done[to], 0));
    w->barrier();   // the events of this group are consumed before the next group re-records them
  }
};

}  // namespace

Comm* comm_init(int world, int rank, const void* id128) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  auto* c = new NcclComm();
  c->world = world;
  c->rank = rank;
  try {
    check(nccl().CommInitRank(&c->c, world, id, rank), "ncclCommInitRank");
  } catch (...) {
    delete c;
    throw;
  }
  return c;
}

Comm* comm_loopback(LoopWorld* w, int rank) {
  auto* c = new LoopComm();
  c->w = w;
  c->world = w->world;
  c->rank = rank;
  return c;
}

LoopWorld* loop_world_create(int world) { return new LoopWorld(world); }
void loop_world_destroy(LoopWorld* w) { delete w; }
int loop_world_size(LoopWorld* w) { return w->world; }

void comm_destroy(Comm* c) { delete c; }

void comm_allreduce_sum_i32(Comm* c, int32_t* d_buf, size_t n, cudaStream_t st) {
  if (n) c->allreduce_sum_i32(d_buf, n, st);
}
void comm_allreduce_sum_f64(Comm* c, double* d_buf, size_t n, cudaStream_t st) {
  if (n) c->allreduce_sum_f64(d_buf, n, st);
}
void comm_group_start(Comm* c) { c->group_start(); }
void comm_group_end(Comm* c, cudaStream_t st) { c->group_end(st); }
void comm_send_f64(Comm* c, const double* d, size_t n, int peer, cudaStream_t st) { c->send(d, n, peer, st); }
void comm_recv_f64(Comm* c, double* d, size_t n, int peer, cudaStream_t st) { c->recv(d, n, peer, st); }

}  // namespace hs
