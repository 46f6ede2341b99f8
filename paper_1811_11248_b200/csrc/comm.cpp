// NCCL for the multi-GPU factor: one communicator per handle, loaded with
// dlopen at hs_create time only when world_size > 1, so the single-GPU library has no NCCL
// dependency and a process that already carries torch's NCCL reuses that copy (libnccl.so.2
// resolves to the already-loaded library; HS_NCCL_LIB overrides the path).
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <mutex>
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

void* comm_init(int world, int rank, const void* id128) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclComm_t c = nullptr;
  check(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank");
  return c;
}

void comm_destroy(void* c) {
  if (c && g_nccl.so) g_nccl.CommDestroy((ncclComm_t)c);
}

void comm_allreduce_sum_i32(void* c, int32_t* d_buf, size_t n, cudaStream_t st) {
  if (n) check(nccl().AllReduce(d_buf, d_buf, n, ncclInt32, ncclSum, (ncclComm_t)c, st), "ncclAllReduce");
}

void comm_group_start() { check(nccl().GroupStart(), "ncclGroupStart"); }
void comm_group_end() { check(nccl().GroupEnd(), "ncclGroupEnd"); }

void comm_send_f64(void* c, const double* d, size_t n, int peer, cudaStream_t st) {
  if (n) check(nccl().Send(d, n, ncclFloat64, peer, (ncclComm_t)c, st), "ncclSend");
}
void comm_recv_f64(void* c, double* d, size_t n, int peer, cudaStream_t st) {
  if (n) check(nccl().Recv(d, n, ncclFloat64, peer, (ncclComm_t)c, st), "ncclRecv");
}

}  // namespace hs
