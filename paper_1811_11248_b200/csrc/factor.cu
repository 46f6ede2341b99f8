// hs_factor — host driver of Algorithm 1 on one B200.
//
// Per level l = 0 .. L_top-1 and per batch of independent clusters (schedule from
// hs_analyze), the runtime plans descriptors on the host and launches
//   pack (copy2d) -> POTRF -> TRSM (deferred compression) -> CPQR+rotation
//   -> [one D2H of the batch's ranks]
//   -> Schur update (ordered per target tile) + write-back (copy2d, identity)
// then assembles the parent level's blocks (A_c) and finally factors the dense top
// (P:626-628).  The elimination record (G, V, tau, C) stays in device memory for the
// apply, whose plan (descriptors) is built alongside and replayed as a CUDA graph.
#include <algorithm>
#include <atomic>
#include <cuda.h>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <functional>
#include <future>
#include <memory>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <unordered_map>

#include "runtime.h"

namespace hs {

void* DevCache::alloc(size_t bytes) {
  const size_t c = size_class(std::max<size_t>(bytes, 1));
  void* p = nullptr;
  auto it = bins.find(c);
  if (it != bins.end() && !it->second.empty()) {
    p = it->second.back();
    it->second.pop_back();
    cached -= c;
  } else {
    cudaError_t e = cudaMalloc(&p, c);
    if (e == cudaErrorMemoryAllocation) {   // give the cache back to the driver and retry once
      cudaGetLastError();
      trim();
      e = cudaMalloc(&p, c);
    }
    if (e == cudaErrorMemoryAllocation && vmm && vmm->rec) {   // then spill completed factor records
      cudaGetLastError();
      while (e == cudaErrorMemoryAllocation && vmm->rec->spill(c + ((size_t)1 << 30))) {
        cudaGetLastError();
        vmm->trim();
        e = cudaMalloc(&p, c);
      }
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      size_t fb = 0, tb = 0;
      cudaMemGetInfo(&fb, &tb);
      cudaGetLastError();
      fail(e == cudaErrorMemoryAllocation ? HS_E_OOM : HS_E_CUDA,
           std::string("device allocation of ") + std::to_string(c) + " bytes: " + cudaGetErrorString(e) +
               " (cache in use " + std::to_string(in_use >> 20) + " MB, VMM chunks " +
               std::to_string(vmm ? (vmm->created * vmm->chunk) >> 20 : 0) + " MB, device free " +
               std::to_string(fb >> 20) + " MB)");
    }
  }
  live[p] = c;
  in_use += c;
  peak = std::max(peak, in_use);
  return p;
}
void DevCache::free(void* p) {
  if (!p) return;
  auto it = live.find(p);
  if (it == live.end()) return;
  bins[it->second].push_back(p);
  cached += it->second;
  in_use -= it->second;
  live.erase(it);
}
void DevCache::trim() {
  if (vmm) vmm->trim();
  if (!cached) return;
  cudaDeviceSynchronize();
  for (auto& b : bins)
    for (void* p : b.second) cudaFree(p);
  bins.clear();
  cached = 0;
}

// ---- CUDA VMM through the driver entry points (no link-time dependency on libcuda) -------
namespace {
struct DriverVmm {
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  DriverVmm() {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
        *fn = nullptr;
    };
    get("cuMemCreate", (void**)&create);
    get("cuMemRelease", (void**)&release);
    get("cuMemAddressReserve", (void**)&reserve);
    get("cuMemAddressFree", (void**)&addr_free);
    get("cuMemMap", (void**)&map);
    get("cuMemUnmap", (void**)&unmap);
    get("cuMemSetAccess", (void**)&set_access);
    get("cuMemGetAllocationGranularity", (void**)&granularity);
  }
  void need() const {
    if (!create || !release || !reserve || !addr_free || !map || !unmap || !set_access || !granularity)
      fail(HS_E_CUDA, "CUDA virtual memory management entry points unavailable");
  }
};
const DriverVmm& drv() {
  static DriverVmm d;
  d.need();
  return d;
}
void cu_check(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return;
  fail(r == CUDA_ERROR_OUT_OF_MEMORY ? HS_E_OOM : HS_E_CUDA, std::string(what) + " failed (CUresult " + std::to_string((int)r) + ")");
}
CUmemAllocationProp chunk_prop(int device) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  return prop;
}
}  // namespace

// HS_PROFILE: host time in the VMM calls (take = reuse / cuMemCreate incl. spills, map, access, unmap)
double g_vmm_t[4] = {0, 0, 0, 0};
long long g_vmm_n[4] = {0, 0, 0, 0};
static inline double vmm_now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
void VmmPool::init(int dev) {
  if (device == dev && chunk) return;
  device = dev;
  const CUmemAllocationProp prop = chunk_prop(dev);
  size_t g = 0;
  cu_check(drv().granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity");
  const char* ce = std::getenv("HS_VMM_CHUNK_MB");   // 1 GB chunks (A/B vs 256 MB: profiles/r02fin_c4_chunk*.json)
  const size_t want = (size_t)(ce ? std::max(2, std::atoi(ce)) : 1024) << 20;
  chunk = (want + g - 1) / g * g;
}
unsigned long long VmmPool::take() {
  const double t0 = vmm_now();
  struct Acc {
    double t0;
    ~Acc() {
      g_vmm_t[0] += vmm_now() - t0;
      ++g_vmm_n[0];
    }
  } acc{t0};
  if (!idle.empty()) {
    const unsigned long long h = idle.back();
    idle.pop_back();
    return h;
  }
  const CUmemAllocationProp prop = chunk_prop(device);
  CUmemGenericAllocationHandle h = 0;
  CUresult r = drv().create(&h, chunk, &prop, 0);
  if (r == CUDA_ERROR_OUT_OF_MEMORY && dc) {   // give cached blocks back to the driver and retry once
    dc->trim();
    r = drv().create(&h, chunk, &prop, 0);
  }
  if (r == CUDA_ERROR_OUT_OF_MEMORY && rec && rec->spill(chunk)) {   // a spilled record chunk's memory
    if (!idle.empty()) {
      const unsigned long long hh = idle.back();
      idle.pop_back();
      return hh;
    }
    r = drv().create(&h, chunk, &prop, 0);
  }
  cu_check(r, "cuMemCreate (block store chunk)");
  ++created;
  return (unsigned long long)h;
}
void VmmPool::trim() {
  for (unsigned long long h : idle) drv().release((CUmemGenericAllocationHandle)h);
  created -= idle.size();
  idle.clear();
}
char* VmmPool::take_host() {
  if (!host_idle.empty()) {
    char* p = host_idle.back();
    host_idle.pop_back();
    return p;
  }
  char* p = nullptr;
  HS_CUDA(cudaHostAlloc((void**)&p, chunk, cudaHostAllocDefault));
  return p;
}
VmmPool::~VmmPool() {
  trim();
  for (char* p : host_idle) cudaFreeHost(p);
  host_idle.clear();
}

// ---- factor records in a spillable virtual range (runtime.h) --------------------------------
void RecSpace::init(VmmPool* p, size_t reserve_bytes, cudaStream_t stream) {
  release();
  pool = p;
  st = stream;
  const size_t cb = pool->chunk;
  vbytes = (reserve_bytes + cb - 1) / cb * cb;
  base = vmm_reserve(vbytes);
  handle.assign(vbytes / cb, 0ull);
  host.assign(vbytes / cb, nullptr);
  pre.assign(vbytes / cb, nullptr);
  pre_ev.assign(vbytes / cb, nullptr);
  top = frontier = pin_lo = pin_hi = 0;
  n_spilled = bytes_spilled = bytes_restored = 0;
  t_spill = t_restore = 0.0;
  pre_bytes = pre_used = 0;
  pre_budget = 0;
  const char* e = std::getenv("HS_REC_PRECOPY");   // 0: off; else the previous factor's spill + 1 GB
  if (!(e && std::atoi(e) == 0) && pool->last_spilled > 0) pre_budget = pool->last_spilled + ((size_t)1 << 30);
}
void RecSpace::precopy(cudaStream_t side) {
  if (!active() || pre_budget == 0) return;
  const size_t cb = pool->chunk;
  bool started = false;
  for (size_t i = 0; i < handle.size() && (i + 1) * cb <= frontier && pre_bytes < pre_budget; ++i) {
    if (!handle[i] || host[i] || pre[i] || ((i + 1) * cb > pin_lo && i * cb < pin_hi)) continue;
    if (!started) {   // the copies start after every writer queued so far (main and side stream)
      if (!cst) HS_CUDA(cudaStreamCreateWithFlags(&cst, cudaStreamNonBlocking));
      cudaEvent_t ev;
      HS_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      HS_CUDA(cudaEventRecord(ev, st));
      HS_CUDA(cudaStreamWaitEvent(cst, ev, 0));
      if (side) {
        HS_CUDA(cudaEventRecord(ev, side));
        HS_CUDA(cudaStreamWaitEvent(cst, ev, 0));
      }
      HS_CUDA(cudaEventDestroy(ev));
      started = true;
    }
    pre[i] = pool->take_host();
    HS_CUDA(cudaMemcpyAsync(pre[i], (const void*)(uintptr_t)(base + i * cb), cb, cudaMemcpyDeviceToHost, cst));
    HS_CUDA(cudaEventCreateWithFlags(&pre_ev[i], cudaEventDisableTiming));
    HS_CUDA(cudaEventRecord(pre_ev[i], cst));
    pre_bytes += cb;
  }
}
static void drop_precopy(RecSpace& R, size_t i) {   // the chunk's pre-copy is not needed (any more)
  if (R.pre_ev[i]) {
    cudaEventSynchronize(R.pre_ev[i]);
    cudaEventDestroy(R.pre_ev[i]);
    R.pre_ev[i] = nullptr;
  }
  if (R.pre[i]) {
    R.pool->give_host(R.pre[i]);
    R.pre[i] = nullptr;
  }
}
void* RecSpace::alloc(size_t bytes) {
  const size_t cb = pool->chunk;
  const size_t off = (top + 255) & ~size_t(255), end = off + std::max<size_t>(bytes, 8);
  if (end > vbytes) fail(HS_E_OOM, "factor records exceed the device memory (record space of " + std::to_string(vbytes) + " bytes)");
  for (size_t i = off / cb; i < (end + cb - 1) / cb; ++i) {
    if (handle[i]) continue;
    const unsigned long long hd = pool->take();   // may spill chunks below the frontier (not this one)
    vmm_map(base + i * cb, hd, cb, pool->device);
    handle[i] = hd;
  }
  top = end;
  return (void*)(uintptr_t)(base + off);
}
void RecSpace::level_start() {
  const size_t cb = pool->chunk;
  top = (top + cb - 1) / cb * cb;
  frontier = top;
}
size_t RecSpace::spill(size_t bytes) {
  const size_t cb = pool->chunk;
  std::vector<size_t> pick;
  size_t got = 0;
  for (size_t i = 0; i < handle.size() && (i + 1) * cb <= frontier && got < bytes; ++i)
    if (handle[i] && !((i + 1) * cb > pin_lo && i * cb < pin_hi)) {
      pick.push_back(i);
      got += cb;
    }
  if (pick.empty()) return 0;
  const auto t0 = std::chrono::steady_clock::now();
  bool copy = false;
  for (size_t i : pick) copy |= pre[i] == nullptr;
  if (copy) HS_CUDA(cudaDeviceSynchronize());   // every writer of a completed record has finished
  for (size_t i : pick) {
    if (pre[i]) {   // pre-copied on the copy stream: wait for that copy only
      HS_CUDA(cudaEventSynchronize(pre_ev[i]));
      HS_CUDA(cudaEventDestroy(pre_ev[i]));
      pre_ev[i] = nullptr;
      host[i] = pre[i];
      pre[i] = nullptr;
      pre_used += cb;
      continue;
    }
    host[i] = pool->take_host();
    HS_CUDA(cudaMemcpyAsync(host[i], (const void*)(uintptr_t)(base + i * cb), cb, cudaMemcpyDeviceToHost, st));
  }
  if (copy) HS_CUDA(cudaStreamSynchronize(st));
  for (size_t i : pick) {
    vmm_unmap(base + i * cb, cb);
    pool->give(handle[i]);
    handle[i] = 0;
  }
  n_spilled += pick.size();
  bytes_spilled += got;
  t_spill += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return got;
}
void RecSpace::restore() {
  if (!active()) return;
  const size_t cb = pool->chunk;
  for (size_t i = 0; i < pre.size(); ++i) drop_precopy(*this, i);   // pre-copies never spilled
  pool->last_spilled = bytes_spilled;
  const auto t0 = std::chrono::steady_clock::now();
  bool any = false;
  for (size_t i = 0; i < host.size(); ++i)
    if (host[i]) {
      const unsigned long long hd = pool->take();
      vmm_map(base + i * cb, hd, cb, pool->device);
      handle[i] = hd;
      HS_CUDA(cudaMemcpyAsync((void*)(uintptr_t)(base + i * cb), host[i], cb, cudaMemcpyHostToDevice, st));
      bytes_restored += cb;
      any = true;
    }
  if (!any) return;
  HS_CUDA(cudaStreamSynchronize(st));
  for (size_t i = 0; i < host.size(); ++i)
    if (host[i]) {
      pool->give_host(host[i]);
      host[i] = nullptr;
    }
  t_restore += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}
void RecSpace::release() {
  if (!base) return;
  cudaDeviceSynchronize();   // the apply / a failed factor's kernels may still read the records
  const size_t cb = pool->chunk;
  try {
    for (size_t i = 0; i < pre.size(); ++i) drop_precopy(*this, i);
    if (cst) {
      cudaStreamDestroy(cst);
      cst = nullptr;
    }
    for (size_t i = 0; i < handle.size(); ++i) {
      if (handle[i]) {
        vmm_unmap(base + i * cb, cb);
        pool->give(handle[i]);
        handle[i] = 0;
      }
      if (host[i]) {
        pool->give_host(host[i]);
        host[i] = nullptr;
      }
    }
    vmm_free_range(base, vbytes);
  } catch (...) {
  }
  if (pool && pool->rec == this) pool->rec = nullptr;
  base = 0;
  vbytes = top = frontier = pin_lo = pin_hi = 0;
}
unsigned long long vmm_reserve(size_t bytes) {
  CUdeviceptr p = 0;
  cu_check(drv().reserve(&p, bytes, 0, 0, 0), "cuMemAddressReserve");
  return (unsigned long long)p;
}
void vmm_free_range(unsigned long long base, size_t bytes) { drv().addr_free((CUdeviceptr)base, bytes); }
void vmm_map(unsigned long long va, unsigned long long handle, size_t bytes, int device) {
  cu_check(drv().map((CUdeviceptr)va, bytes, 0, (CUmemGenericAllocationHandle)handle, 0), "cuMemMap");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu_check(drv().set_access((CUdeviceptr)va, bytes, &acc, 1), "cuMemSetAccess");
}
// one cuMemMap per chunk, then one cuMemSetAccess over each contiguous run of new mappings
static void vmm_map_run(unsigned long long va0, const unsigned long long* handles, size_t n, size_t cb, int device) {
  double t0 = vmm_now();
  for (size_t i = 0; i < n; ++i)
    cu_check(drv().map((CUdeviceptr)(va0 + i * cb), cb, 0, (CUmemGenericAllocationHandle)handles[i], 0), "cuMemMap");
  g_vmm_t[1] += vmm_now() - t0;
  g_vmm_n[1] += (long long)n;
  t0 = vmm_now();
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  cu_check(drv().set_access((CUdeviceptr)va0, n * cb, &acc, 1), "cuMemSetAccess");
  g_vmm_t[2] += vmm_now() - t0;
  ++g_vmm_n[2];
}
void vmm_unmap(unsigned long long va, size_t bytes) {
  const double t0 = vmm_now();
  cu_check(drv().unmap((CUdeviceptr)va, bytes), "cuMemUnmap");
  g_vmm_t[3] += vmm_now() - t0;
  ++g_vmm_n[3];
}

void DevScratch::ensure(size_t bytes) {
  if (bytes <= cap) return;
  dc->free(d);
  d = nullptr;
  cap = DevCache::size_class(std::max(bytes, cap * 2));
  d = (char*)dc->alloc(cap);
}
DevScratch::~DevScratch() {
  if (d && dc) dc->free(d);
}
void HostStage::ensure(size_t bytes) {
  if (bytes <= cap) return;
  if (h) cudaFreeHost(h);
  h = nullptr;
  cap = std::max(bytes, cap * 2);
  HS_CUDA(cudaMallocHost(&h, cap));
}
HostStage::~HostStage() {
  if (h) cudaFreeHost(h);
}

namespace {

struct BlockStore {
  double* d = nullptr;
  std::vector<int32_t> cap;
  std::vector<std::vector<std::pair<int32_t, int64_t>>> rows;   // p -> sorted (q <= p, offset)
  std::vector<int64_t> rowbeg;   // [n + 1] first offset of row p's blocks (rows are contiguous, ascending)
  size_t total = 0;
  cudaStream_t st = nullptr;
  DevCache* dc = nullptr;
  // VMM backing: one virtual range of nchunk chunks; handle[i] != 0 while chunk i is mapped
  VmmPool* pool = nullptr;
  size_t vbytes = 0;
  std::vector<unsigned long long> handle;

  // dp/level (multi-GPU): keep only the blocks this rank holds (it owns p or q)
  BlockStore() = default;
  BlockStore(const BlockStore&) = delete;
  BlockStore& operator=(const BlockStore&) = delete;
  BlockStore& operator=(BlockStore&&) = default;   // the moved-from store must be forget()-ed
  ~BlockStore() {   // error paths: wait for the store's users, then give the chunks back
    if (!d && !d_ptr) return;
    if (st) cudaStreamSynchronize(st);
    try {
      release();
    } catch (...) {
    }
  }
  void build(const std::vector<int32_t>& caps, const Adj& edges, cudaStream_t stream, DevCache* cache, VmmPool* vp,
             const DistPlan* dp = nullptr, int level = 0) {
    reserve(caps, edges, stream, cache, vp, dp, level);
    map_bytes(0, total * sizeof(double));
  }
  // layout + virtual range, nothing mapped yet
  void reserve(const std::vector<int32_t>& caps, const Adj& edges, cudaStream_t stream, DevCache* cache, VmmPool* vp,
               const DistPlan* dp = nullptr, int level = 0) {
    st = stream;
    dc = cache;
    pool = vp;
    layout(caps, edges, dp, level);
    if (!total) return;
    // map/unmap cost milliseconds per chunk: stores that fit comfortably twice come from the
    // caching allocator, only the large ones (C4-sized) are VMM-backed
    static const size_t vmm_min = [] {
      const char* e = std::getenv("HS_VMM_MIN_GB");
      return (size_t)(e ? std::atof(e) * 1e9 : 24e9);
    }();
    if (total * sizeof(double) < vmm_min) {
      pool = nullptr;
      d = (double*)dc->alloc(total * sizeof(double));
      return;
    }
    const size_t cb = pool->chunk;
    vbytes = (total * sizeof(double) + cb - 1) / cb * cb;
    d = (double*)(uintptr_t)vmm_reserve(vbytes);
    handle.assign(vbytes / cb, 0ull);
  }
  // map (and zero) every chunk overlapping the byte range [b0, b1) that is not mapped yet
  void map_bytes(size_t b0, size_t b1) {
    if (!total || b1 <= b0) return;
    if (!pool) {   // cache-backed: zero exactly the range
      b1 = std::min(b1, total * sizeof(double));
      if (b1 > b0) HS_CUDA(cudaMemsetAsync((char*)d + b0, 0, b1 - b0, st));
      return;
    }
    const size_t cb = pool->chunk;
    size_t i0 = b0 / cb, i1 = (std::min(b1, vbytes) + cb - 1) / cb;
    for (size_t i = i0; i < i1;) {
      if (handle[i]) {
        ++i;
        continue;
      }
      size_t j = i;
      for (; j < i1 && !handle[j]; ++j) handle[j] = pool->take();
      vmm_map_run((unsigned long long)(uintptr_t)d + i * cb, &handle[i], j - i, cb, pool->device);
      HS_CUDA(cudaMemsetAsync((char*)d + i * cb, 0, (j - i) * cb, st));
      i = j;
    }
  }
  // unmap every chunk lying entirely below byte b (its users must have completed)
  void unmap_below(size_t b) {
    if (!total || !pool) return;
    const size_t cb = pool->chunk;
    for (size_t i = 0; i < handle.size() && (i + 1) * cb <= b; ++i)
      if (handle[i]) {
        vmm_unmap((unsigned long long)(uintptr_t)d + i * cb, cb);
        pool->give(handle[i]);
        handle[i] = 0;
      }
  }
  std::vector<std::vector<std::pair<int32_t, int64_t>>> cols;   // q -> sorted (p > q, offset)
  void layout(const std::vector<int32_t>& caps, const Adj& edges, const DistPlan* dp = nullptr, int level = 0) {
    cap = caps;
    const int n = (int)caps.size();
    rows.assign(n, {});
    cols.assign(n, {});
    int64_t off = 0;
    rowbeg.assign(n + 1, 0);
    for (int p = 0; p < n; ++p) {
      rowbeg[p] = off;
      for (int32_t q : edges[p])
        if (q < p && (!dp || dp->holds(level, p, q))) {
          rows[p].push_back({q, off});
          cols[q].push_back({p, off});
          off += (int64_t)caps[p] * caps[q];
        }
      if (!dp || dp->own(level, p)) {
        rows[p].push_back({p, off});
        off += (int64_t)caps[p] * caps[p];
      }
    }
    rowbeg[n] = off;
    total = (size_t)off;
  }
  int64_t off(int32_t p, int32_t q) const {   // p >= q
    const auto& r = rows[p];
    auto it = std::lower_bound(r.begin(), r.end(), std::make_pair(q, (int64_t)-1));
    if (it == r.end() || it->first != q) return -1;
    return it->second;
  }
  bool has(int32_t p, int32_t q) const { return p >= q ? off(p, q) >= 0 : off(q, p) >= 0; }
  // offsets of the blocks (s, q), q in `list` (ascending, q != s), -1 where absent: one
  // merge over row s (q < s) and column s (q > s) instead of a search per block
  void row_offsets(int32_t s, const std::vector<int32_t>& list, std::vector<int64_t>& out) const {
    const auto& R = rows[s];
    const auto& K = cols[s];
    size_t i = 0, j = 0;
    for (int32_t q : list) {
      if (q < s) {
        while (i < R.size() && R[i].first < q) ++i;
        out.push_back(i < R.size() && R[i].first == q ? R[i].second : -1);
      } else {
        while (j < K.size() && K[j].first < q) ++j;
        out.push_back(j < K.size() && K[j].first == q ? K[j].second : -1);
      }
    }
  }
  // block (s, q) from a row_offsets() entry, as get() returns it
  void at(int32_t s, int32_t q, int64_t o, double*& ptr, int32_t& ld, int32_t& trans) const {
    ptr = d + o;
    ld = q < s ? cap[q] : cap[s];
    trans = q < s ? 0 : 1;
  }
  // A(p, q) as (pointer, ld, trans): A(p,q)[i][j] = trans ? ptr[j*ld + i] : ptr[i*ld + j]
  void get(int32_t p, int32_t q, double*& ptr, int32_t& ld, int32_t& trans) const {
    if (p >= q) {
      const int64_t o = off(p, q);
      if (o < 0) fail(HS_E_INTERNAL, "block store: missing block");
      ptr = d + o;
      ld = cap[q];
      trans = 0;
    } else {
      const int64_t o = off(q, p);
      if (o < 0) fail(HS_E_INTERNAL, "block store: missing block");
      ptr = d + o;
      ld = cap[p];
      trans = 1;
    }
  }
  // device copy of the directory for the Schur kernel's target lookup
  int64_t* d_ptr = nullptr;
  int32_t* d_q = nullptr;
  int64_t* d_off = nullptr;
  int32_t* d_cap = nullptr;
  // the directory through one pinned staging buffer, no host synchronisation: the staging is
  // rewritten only at the next level transition, after the stream has drained
  void upload_dir(HostStage& hst) {
    const int n = (int)cap.size();
    size_t nq = 0;
    for (int p = 0; p < n; ++p) nq += rows[p].size();
    const size_t o_ptr = 0, o_off = o_ptr + 8 * (size_t)(n + 1), o_q = o_off + 8 * std::max<size_t>(nq, 1),
                 o_cap = o_q + ((4 * std::max<size_t>(nq, 1) + 7) & ~size_t(7)), tot = o_cap + 4 * (size_t)std::max(n, 1);
    hst.ensure(tot);
    int64_t* ptr = (int64_t*)(hst.h + o_ptr);
    int64_t* off = (int64_t*)(hst.h + o_off);
    int32_t* qq = (int32_t*)(hst.h + o_q);
    int32_t* cp = (int32_t*)(hst.h + o_cap);
    size_t k = 0;
    ptr[0] = 0;
    for (int p = 0; p < n; ++p) {
      for (const auto& e : rows[p]) {
        qq[k] = e.first;
        off[k] = e.second;
        ++k;
      }
      ptr[p + 1] = (int64_t)k;
    }
    for (int p = 0; p < n; ++p) cp[p] = cap[p];
    char* dev = (char*)dc->alloc(tot);
    HS_CUDA(cudaMemcpyAsync(dev, hst.h, tot, cudaMemcpyHostToDevice, st));
    d_ptr = (int64_t*)(dev + o_ptr);
    d_off = (int64_t*)(dev + o_off);
    d_q = (int32_t*)(dev + o_q);
    d_cap = (int32_t*)(dev + o_cap);
  }
  BlockDir dir() const { return BlockDir{d, (int64_t)total, d_ptr, d_q, d_off, d_cap}; }
  // the store's users must have completed (the callers synchronise the stream first)
  void release() {
    if (d && pool) {
      unmap_below(vbytes);
      vmm_free_range((unsigned long long)(uintptr_t)d, vbytes);
    } else if (d) {
      dc->free(d);
    }
    if (d_ptr) dc->free(d_ptr);   // one allocation holds the whole directory
    forget();
  }
  void forget() {
    handle.clear();
    vbytes = 0;
    d = nullptr;
    d_ptr = nullptr;
    d_q = nullptr;
    d_off = nullptr;
    d_cap = nullptr;
  }
};

// Per-kernel-class device time (CUDA events on the library stream), collected at the
// batch's rank read-back, which already synchronises: a = [gather|potrf|trsm|cpqr],
// b = [schur|write-back] of the previous batch.
struct PhaseTimer {
  cudaEvent_t a[5], b[3];
  bool b_pending = false;
  // Each event record costs ~2-3 us of stream time per batch, so phases are timed only on
  // request: HS_PHASE_EVENTS=all brackets every phase, =cpqr only the CPQR kernel.
  int level = [] {
    const char* e = std::getenv("HS_PHASE_EVENTS");
    if (!e) return std::getenv("HS_PROFILE") ? 2 : 0;
    return std::strcmp(e, "all") == 0 ? 2 : std::strcmp(e, "cpqr") == 0 ? 1 : 0;
  }();
  bool on = level == 2;
  void rec(cudaEvent_t e, cudaStream_t st) {
    if (on || (level == 1 && (e == a[3] || e == a[4]))) HS_CUDA(cudaEventRecord(e, st));
  }
  PhaseTimer() {
    for (auto& e : a) HS_CUDA(cudaEventCreate(&e));
    for (auto& e : b) HS_CUDA(cudaEventCreate(&e));
  }
  ~PhaseTimer() {
    for (auto& e : a) cudaEventDestroy(e);
    for (auto& e : b) cudaEventDestroy(e);
  }
  static double el(cudaEvent_t x, cudaEvent_t y) {
    float ms = 0.f;
    HS_CUDA(cudaEventElapsedTime(&ms, x, y));
    return ms * 1e-3;
  }
  void collect_b(hs_factor_stats_t& S) {
    if (!b_pending || !on) return;
    HS_CUDA(cudaEventSynchronize(b[2]));
    S.t_phase_s[4] += el(b[0], b[1]);
    S.t_phase_s[5] += el(b[1], b[2]);
    b_pending = false;
  }
  void collect_a(hs_factor_stats_t& S) {   // (the ranks are published before a[4]: wait for it)
    if (on || level == 1) HS_CUDA(cudaEventSynchronize(a[4]));
    if (on)
      for (int k = 0; k < 4; ++k) S.t_phase_s[k] += el(a[k], a[k + 1]);
    else if (level == 1)
      S.t_phase_s[3] += el(a[3], a[4]);
  }
  void collect(hs_factor_stats_t& S) {   // after a synchronising point
    collect_a(S);
    collect_b(S);
  }
};

// [chunk_lo(n, T, t), chunk_lo(n, T, t + 1)): the t-th of T contiguous chunks of [0, n)
inline int chunk_lo(int n, int T, int t) { return (int)((int64_t)n * t / T); }
// Host threads for planning n clusters of a batch (HS_PLAN_THREADS overrides; 1 = sequential)
int plan_threads(int n) {
  static const int hw = [] {
    const char* e = std::getenv("HS_PLAN_THREADS");
    if (e) return std::max(1, std::atoi(e));
    return std::max(1, std::min(8, (int)std::thread::hardware_concurrency() / 2));
  }();
  return std::max(1, std::min(hw, n / 128));
}
// Persistent host worker threads for the batch planning (spawning threads per batch costs
// more than the planning they would share).  run(T, fn) calls fn(t) for t = 1 .. T-1 on the
// workers and fn(0) on the caller, and returns when all are done; the first exception is
// rethrown on the caller.  Calls from several host threads are serialised.
class PlanPool {
 public:
  static PlanPool& get() {
    static PlanPool pool;
    return pool;
  }
  void run(int T, const std::function<void(int)>& fn) {
    if (T <= 1) {
      fn(0);
      return;
    }
    std::lock_guard<std::mutex> call(call_mu_);
    {
      std::lock_guard<std::mutex> lk(mu_);
      while ((int)th_.size() < T - 1) th_.emplace_back([this] { loop(); });
      job_ = &fn;
      next_ = 1;
      ntask_ = T;
      pending_ = T - 1;
      err_ = nullptr;
      ++gen_;
    }
    cv_.notify_all();
    std::exception_ptr e0;
    try {
      fn(0);
    } catch (...) {
      e0 = std::current_exception();
    }
    std::unique_lock<std::mutex> lk(mu_);
    done_.wait(lk, [&] { return pending_ == 0; });
    job_ = nullptr;
    if (e0) std::rethrow_exception(e0);
    if (err_) std::rethrow_exception(err_);
  }
  ~PlanPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }

 private:
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || (gen_ != seen && next_ < ntask_); });
      if (stop_) return;
      seen = gen_;
      while (next_ < ntask_) {
        const int t = next_++;
        const std::function<void(int)>* job = job_;
        lk.unlock();
        std::exception_ptr e;
        try {
          (*job)(t);
        } catch (...) {
          e = std::current_exception();
        }
        lk.lock();
        if (e && !err_) err_ = e;
        if (--pending_ == 0) done_.notify_one();
      }
    }
  }
  std::mutex call_mu_, mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> th_;
  const std::function<void(int)>* job_ = nullptr;
  int next_ = 0, ntask_ = 0, pending_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
  std::exception_ptr err_;
};

// fn(b0, b1, t) over the T contiguous chunks of [0, n) on the planning pool
template <class F>
void par_chunks(int n, int T, F&& fn) {
  if (T <= 1) {
    fn(0, n, 0);
    return;
  }
  PlanPool::get().run(T, [&](int t) { fn(chunk_lo(n, T, t), chunk_lo(n, T, t + 1), t); });
}

// the batch vectors, kept across batches so that their storage is reused (no allocation, no
// first-touch page faults per batch)
struct BatchVecs {
  std::vector<int32_t> cnt[6];
  std::vector<CopyItem> gather, wb;
  std::vector<CluItem> clu;
  std::vector<TrsmItem> trsm, rot;
  std::vector<FusedItem> fci;
  std::vector<ScaleTile> fz;
  std::vector<FusedSeg> fseg;
  std::vector<SchurSrc> srcs;
  std::vector<NbCol> nbc;
  std::vector<SchurTile2> tiles;
  std::vector<PatchItem> patch;
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Per-batch workspace whose last reader runs on the side stream (k_form_T): returned to the
// cache only once the side-stream event recorded after that reader has completed.
struct DeferredFree {
  DevCache* dc = nullptr;
  std::vector<std::pair<cudaEvent_t, std::vector<void*>>> q;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t take() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e;
    HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
  }
  void push(cudaEvent_t e, std::vector<void*> ptrs) { q.push_back({e, std::move(ptrs)}); }
  void drain(bool wait) {
    size_t k = 0;
    for (; k < q.size(); ++k) {
      if (wait) HS_CUDA(cudaEventSynchronize(q[k].first));
      else if (cudaEventQuery(q[k].first) != cudaSuccess) break;
      for (void* p : q[k].second) dc->free(p);
      pool.push_back(q[k].first);
    }
    cudaGetLastError();   // a not-ready query is not an error
    q.erase(q.begin(), q.begin() + k);
  }
  ~DeferredFree() {
    for (auto& e : q) cudaEventSynchronize(e.first);
    for (auto& e : q)
      for (void* p : e.second) dc->free(p);
    for (auto& e : q) pool.push_back(e.first);
    for (cudaEvent_t e : pool) cudaEventDestroy(e);
  }
};

// Bump allocator for the persistent C_s records of a factor: slabs from the cache.
struct Slab {
  DevCache* dc = nullptr;
  RecSpace* rec = nullptr;   // active: slabs from the factor's record space
  std::vector<double*>* owned = nullptr;
  double* cur = nullptr;
  int64_t left = 0;
  double* get(int64_t words) {
    words = (words + 3) & ~int64_t(3);
    if (words > left) {
      const int64_t sz = std::max<int64_t>(words, (int64_t)8 << 20);   // >= 64 MB
      if (rec && rec->active()) {   // exact: a record is complete once its writer is queued
        return (double*)rec->alloc(sizeof(double) * words);
      } else {
        cur = (double*)dc->alloc(sizeof(double) * sz);
        owned->push_back(cur);
      }
      left = sz;
    }
    double* p = cur;
    cur += words;
    left -= words;
    return p;
  }
};

// n(s) neighbour-pair -> target block pointer tables of one level, built on the device once
// per level (the Schur tiles index them instead of searching the directory per tile).
struct LevelPairs {
  DevCache* dc = nullptr;
  double** pairs = nullptr;
  char* meta = nullptr;
  std::vector<int64_t> poff;
  template <class BS>
  void build(const Level& lev, const BS& bs, DevCache& cache, Upload& up, cudaStream_t st) {
    dc = &cache;
    const int n = lev.nclus;
    std::vector<int64_t> hptr(n + 1, 0), row_cl;
    std::vector<int32_t> hq;
    poff.assign(n + 1, 0);
    for (int s = 0; s < n; ++s) {
      const int64_t nn = (int64_t)lev.H[s].size();
      hptr[s + 1] = hptr[s] + nn;
      poff[s + 1] = poff[s] + nn * (nn + 1) / 2;
      hq.insert(hq.end(), lev.H[s].begin(), lev.H[s].end());
      for (int64_t a = 0; a < nn; ++a) row_cl.push_back(s);
    }
    if (poff[n] == 0) return;
    pairs = (double**)dc->alloc(sizeof(double*) * poff[n]);
    up.reset();
    const size_t iP = up.add(hptr), iQ = up.add(hq), iO = up.add(poff), iR = up.add(row_cl);
    up.stage.ensure(up.total);
    up.dev.ensure(up.total);
    up.copy_in(iP, hptr); up.copy_in(iQ, hq); up.copy_in(iO, poff); up.copy_in(iR, row_cl);
    up.send(st);
    launch_level_pairs(up.dptr<int64_t>(iP), up.dptr<int32_t>(iQ), up.dptr<int64_t>(iO), n, (int64_t)row_cl.size(),
                       up.dptr<int64_t>(iR), pairs, bs.dir(), st);
    HS_CUDA(cudaStreamSynchronize(st));   // the staging buffers are reused by the first batch
  }
  ~LevelPairs() {
    if (pairs) dc->free(pairs);
  }
};

void check_status(DevStatus* d_status, DevStatus* h_status, cudaStream_t st) {
  HS_CUDA(cudaMemcpyAsync(h_status, d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  HS_CUDA(cudaStreamSynchronize(st));
  if (h_status->flag) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "NOT_SPD: Cholesky breakdown at level %d cluster %d pivot %d value %.17g (P:283)",
                  h_status->level, h_status->cluster, h_status->pivot, h_status->value);
    fail(HS_E_NOT_SPD, buf);
  }
}

}  // namespace
}  // namespace hs

hs_factor_s::~hs_factor_s() {
  using namespace hs;
  if (!h) return;
  // the apply operators are formed on the side stream: make sure that work is done before
  // the arenas go back to the cache (the factor joined it, but a failed factor may not have)
  if (h->side) cudaStreamSynchronize(h->side);
  DevCache* dc = &h->cache;
  auto fr = [dc](void* p) { dc->free(p); };
  fr(d_vals); fr(d_top);   // d_rowptr, d_colind, d_perm are borrowed from the analysis
  for (auto& l : lv) {
    fr(l.arena);
    fr(l.iarena);
    for (double* p : l.wchunks) fr(p);
    for (double* p : l.cchunks) fr(p);
  }
  for (auto& p : ap.lv) {
    fr(p.d_src); fr(p.d_ftask); fr(p.d_ftgt); fr(p.d_btask); fr(p.d_bnb); fr(p.d_pull); fr(p.d_post_cl); fr(p.d_ctb); fr(p.d_bcl); fr(p.d_cinv);
  }
  fr(ap.d_y); fr(ap.d_yf); fr(ap.d_xb); fr(ap.d_parts); fr(ap.d_ctr); fr(ap.d_contrib);
  if (ap.graph) cudaGraphExecDestroy(ap.graph);
  fr(d_r); fr(d_z); fr(d_p); fr(d_q); fr(d_x); fr(d_b); fr(d_red);
  if (h_red) cudaFreeHost(h_red);
}

namespace hs {

// Pattern-only device data, computed once per analysis and cached in it: the CSR pattern,
// the permutation, the map of every CSR entry into the level-0 block store and the
// transpose map used by the on-device symmetry check.
static void ensure_device_pattern(Analysis* an, int device, cudaStream_t st, const DistPlan& dp, DevCache* dc) {
  if (an->dev == device && an->d_rowptr && an->map_world == dp.world && an->map_rank == dp.rank) {
    if (an->d_map) return;
    if (!an->h_map.empty()) return;   // large pattern: each factor stages the maps itself (factor_create)
  }
  if (an->dev >= 0 && an->dev != device) fail(HS_E_INVALID_ARG, "factor: analysis already bound to another device");
  if (an->d_rowptr) {   // cached for another (world, rank): rebuild
    HS_CUDA(cudaStreamSynchronize(st));
    for (void* p : {(void*)an->d_rowptr, (void*)an->d_colind, (void*)an->d_perm, (void*)an->d_map, (void*)an->d_tmap})
      if (p) cudaFree(p);
    an->d_rowptr = nullptr; an->d_colind = nullptr; an->d_perm = nullptr; an->d_map = nullptr; an->d_tmap = nullptr;
    if (an->maps_pinned) {
      cudaHostUnregister(an->h_map.data());
      cudaHostUnregister(an->h_tmap.data());
      an->maps_pinned = false;
    }
    an->h_map.clear();
    an->h_tmap.clear();
  }
  const bool dist = dp.world > 1;
  const int64_t n = an->n, nnz = an->rowptr[n];
  const int nleaf0 = (int)(an->leaf_off.size() - 1);
  std::vector<int32_t> cap(nleaf0);
  for (int c = 0; c < nleaf0; ++c) cap[c] = (int32_t)(an->leaf_off[c + 1] - an->leaf_off[c]);
  BlockStore layout;
  layout.layout(cap, an->L_top > 0 ? an->levels[0].Ffinal : an->H_top, dist && an->L_top > 0 ? &dp : nullptr, 0);
  std::vector<int32_t> leaf_of(n);
  for (int c = 0; c < nleaf0; ++c)
    for (int64_t k = an->leaf_off[c]; k < an->leaf_off[c + 1]; ++k) leaf_of[k] = c;
  std::vector<int64_t> map(nnz, -1), tmap(nnz);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t pi = an->iperm[i];
    const int32_t p = leaf_of[pi];
    for (int64_t k = an->rowptr[i]; k < an->rowptr[i + 1]; ++k) {
      const int64_t j = an->colind[k];
      const int32_t* b = an->colind.data() + an->rowptr[j];
      const int32_t* e = an->colind.data() + an->rowptr[j + 1];
      tmap[k] = an->rowptr[j] + (std::lower_bound(b, e, (int32_t)i) - b);
      const int64_t pj = an->iperm[j];
      const int32_t q = leaf_of[pj];
      if (p < q) continue;
      const int64_t o = layout.off(p, q);
      if (o < 0) {
        if (dist) continue;   // a block this rank does not hold
        fail(HS_E_INTERNAL, "factor: level-0 block missing");
      }
      map[k] = o + (pi - an->leaf_off[p]) * cap[q] + (pj - an->leaf_off[q]);
    }
  }
  HS_CUDA(cudaMalloc(&an->d_rowptr, sizeof(int64_t) * (n + 1)));
  HS_CUDA(cudaMalloc(&an->d_colind, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  HS_CUDA(cudaMalloc(&an->d_perm, sizeof(int64_t) * n));
  HS_CUDA(cudaMalloc(&an->d_map, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
  HS_CUDA(cudaMalloc(&an->d_tmap, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
  HS_CUDA(cudaMemcpyAsync(an->d_rowptr, an->rowptr.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaMemcpyAsync(an->d_colind, an->colind.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaMemcpyAsync(an->d_perm, an->perm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaMemcpyAsync(an->d_map, map.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaMemcpyAsync(an->d_tmap, tmap.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaStreamSynchronize(st));
  if (!dist && nnz * 16 >= ((int64_t)2 << 30)) {
    an->h_map = std::move(map);
    an->h_tmap = std::move(tmap);
    // pinned: a factor that stages them copies at full PCIe speed (unregistered by hs_analysis_destroy)
    an->maps_pinned = cudaHostRegister(an->h_map.data(), sizeof(int64_t) * nnz, cudaHostRegisterDefault) == cudaSuccess &&
                      cudaHostRegister(an->h_tmap.data(), sizeof(int64_t) * nnz, cudaHostRegisterDefault) == cudaSuccess;
    cudaGetLastError();
  }
  an->dev = device;
  an->map_world = dp.world;
  an->map_rank = dp.rank;
}

hs_factor_s* factor_create(hs_handle_s* h, const Analysis* an_c, const double* values, const hs_factor_opts& opt) {
  if (opt.eps < 0 || !std::isfinite(opt.eps)) fail(HS_E_INVALID_ARG, "factor: eps must be finite and >= 0");
  if (opt.dc != 0 && opt.dc != 1) fail(HS_E_INVALID_ARG, "factor: dc must be 0 or 1");
  const bool nodc = opt.dc == 0;   // NEXT f1: the original LoRaSp step (nodc.cu)
  Analysis* an = const_cast<Analysis*>(an_c);   // the device pattern cache lives in the analysis
  const int64_t n = an->n, nnz = an->rowptr[n];
  cudaStream_t st = h->stream;
  const DistPlan DP = make_plan(*an, h->world, h->rank);
  ensure_device_pattern(an, h->device, st, DP, &h->cache);
  auto* f = new hs_factor_s();
  std::unique_ptr<hs_factor_s> guard(f);
  f->h = h;
  f->an = an;
  f->opt = opt;
  f->keep_records = std::getenv("HS_KEEP_RECORDS") != nullptr;
  double t_plan = 0.0;
  double t_rank_wait = 0.0;   // host blocked on the previous batch's ranks (HS_PROFILE)
  double t_launch = 0.0;      // host time issuing a batch's uploads and kernels (HS_PROFILE)
  double t_apply_plan = 0.0;  // apply planning (host worker)
  std::future<void> plan_prev;  // the chain of per-level apply-plan tasks (joined before upload)
  double t_sub[4] = {0, 0, 0, 0};
  double t_fh[6] = {0, 0, 0, 0, 0, 0};   // first-half planning: shapes + column maps, items, upload staging
  double t_trans = 0.0;   // host planning breakdown (HS_PROFILE): schur, write-back, apply, tail
  double t_tr[4] = {0, 0, 0, 0};   // level transition: block store build, upload_dir, arena alloc, release
  double t_as[5] = {0, 0, 0, 0, 0};   // assembly loop: map, items, upload + launch, sync, unmap
  cudaEvent_t ev0, ev1;
  HS_CUDA(cudaEventCreate(&ev0));
  HS_CUDA(cudaEventCreate(&ev1));
  HS_CUDA(cudaEventRecord(ev0, st));
  std::vector<std::pair<const char*, double>> tl{{"start", now_s()}};   // host timeline (HS_PROFILE)
  f->d_rowptr = an->d_rowptr;      // borrowed from the analysis
  f->d_colind = an->d_colind;
  f->d_perm = an->d_perm;
  DevCache& dc = h->cache;
  h->vmm.init(h->device);   // physical chunks of the block stores
  h->vmm.dc = &dc;
  dc.vmm = &h->vmm;
  f->d_vals = (double*)dc.alloc(sizeof(double) * std::max<int64_t>(nnz, 1));
  HS_CUDA(cudaMemcpyAsync(f->d_vals, values, sizeof(double) * nnz,
                          opt.values_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));

  DevStatus h_status{};
  DevStatus* d_status = (DevStatus*)dc.alloc(sizeof(DevStatus));
  std::unique_ptr<void, std::function<void(void*)>> status_guard(d_status, [&dc](void* p) { dc.free(p); });
  HS_CUDA(cudaMemsetAsync(d_status, 0, sizeof(DevStatus), st));
  // numerical symmetry of the values (A SPD, A_ns = A_sn^T), checked on the device
  // the level-0 scatter map and the transpose map: the analysis's device copies, or (large
  // patterns whose maps a record-space factor dropped) staged from the host copies into the
  // handle's cache for this factor's symmetry check and scatter only
  const int64_t* d_map = an->d_map;
  const int64_t* d_tmap = an->d_tmap;
  int64_t *stage_map = nullptr, *stage_tmap = nullptr;
  if (!d_map) {
    if (an->h_map.empty()) fail(HS_E_INTERNAL, "factor: level-0 scatter map missing");
    stage_map = (int64_t*)dc.alloc(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
    stage_tmap = (int64_t*)dc.alloc(sizeof(int64_t) * std::max<int64_t>(nnz, 1));
    HS_CUDA(cudaMemcpyAsync(stage_map, an->h_map.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(stage_tmap, an->h_tmap.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
    d_map = stage_map;
    d_tmap = stage_tmap;
  }
  launch_symcheck(f->d_vals, d_tmap, nnz, &d_status->pivot, st);
  HS_CUDA(cudaMemcpyAsync(&h_status, d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  HS_CUDA(cudaStreamSynchronize(st));
  if (h_status.pivot) fail(HS_E_NOT_SYMMETRIC, "factor: values are not symmetric");
  HS_CUDA(cudaMemsetAsync(d_status, 0, sizeof(DevStatus), st));

  tl.push_back({"values + symmetry check", now_s()});
  // ---- level-0 blocks from the permuted CSR ------------------------------------------------
  const int nleaf0 = (int)(an->leaf_off.size() - 1);
  std::vector<int32_t> cap(nleaf0);
  for (int c = 0; c < nleaf0; ++c) cap[c] = (int32_t)(an->leaf_off[c + 1] - an->leaf_off[c]);
  BlockStore bs;
  bs.build(cap, an->L_top > 0 ? an->levels[0].Ffinal : an->H_top, st, &dc, &h->vmm,
           h->world > 1 && an->L_top > 0 ? &DP : nullptr, 0);   // mapped and zeroed
  launch_scatter(f->d_vals, d_map, nnz, bs.d, st);
  if (stage_map) {   // stream-ordered reuse by the factor's later allocations
    dc.free(stage_map);
    dc.free(stage_tmap);
  }
  if (an->L_top > 0) bs.upload_dir(h->dirstage);

  Upload& upA = h->upA;   // persistent per handle: pinned staging is allocated once
  Upload& upB = h->upB;
  upA.dev.dc = &dc;
  upB.dev.dc = &dc;
  h->upC.dev.dc = &dc;
  int32_t* d_rank = nullptr;
  int32_t* h_rank = nullptr;
  int max_batch = 1;
  for (const auto& lev : an->levels)
    for (const auto& B : lev.batches) max_batch = std::max(max_batch, (int)B.size());
  d_rank = (int32_t*)dc.alloc(sizeof(int32_t) * max_batch);
  std::unique_ptr<void, std::function<void(void*)>> rank_guard(d_rank, [&dc](void* p) { dc.free(p); });
  // dpatch: ranks + status published by k_publish into mapped pinned memory (host spins on seq);
  // the pinned buffers live in the handle (allocating them costs milliseconds per factor)
  if (h->pub_cap < max_batch) {
    if (h->h_rank) cudaFreeHost(h->h_rank);
    if (h->pub) cudaFreeHost(h->pub);
    h->h_rank = nullptr;
    h->pub = nullptr;
    h->pub_cap = 0;
    HS_CUDA(cudaMallocHost(&h->h_rank, sizeof(int32_t) * max_batch));
    HS_CUDA(cudaHostAlloc(&h->pub, sizeof(RankPub) + sizeof(int32_t) * max_batch, cudaHostAllocMapped));
    h->pub_cap = max_batch;
  }
  h_rank = h->h_rank;
  RankPub* pub = (RankPub*)h->pub;
  RankPub* pub_dev = nullptr;
  HS_CUDA(cudaHostGetDevicePointer((void**)&pub_dev, pub, 0));
  pub->seq = 0;
  int32_t pub_seq = 0;

  hs_factor_stats_t& S = f->stats;
  PhaseTimer pt;
  DeferredFree deferred;
  deferred.dc = &dc;
  ApplyPlan& ap = f->ap;
  int64_t vbase = 0;
  f->lv.resize(an->L_top);
  ap.lv.resize(an->L_top);

  const bool prof = std::getenv("HS_PROFILE") != nullptr;
  // A/B switches for the previous CPQR kernels (single CTA / cluster with per-thread columns)
  const bool no_fused = std::getenv("HS_NO_FUSED_POTRF_TRSM") != nullptr;   // separate gather/POTRF/TRSM
  const bool no_dwb = std::getenv("HS_NO_DIRECT_WB") != nullptr;            // write-back pass instead
  // ---- multi-GPU (dist.cpp; protocol of oracle/dist.py) ---------------------
  // Rank g eliminates the clusters of its subdomains and stores only the blocks it holds
  // (it owns an endpoint).  Phase-I batches are local; before phase II and at the level end
  // the kept ranks are all-reduced; after each phase-II batch the owner of s sends B_s (rows
  // [0, r) = coarse rows, the fine n-rows = C_s) to the owners of n(s) u w(s), which apply
  // the Schur update and the write-back to the blocks they hold.  The factor records (T_s,
  // C_s) and the top blocks are gathered to rank 0, which builds the apply (v1: the apply and
  // PCG run on rank 0).
  const bool dist = h->world > 1;
  const bool plan_apply = !dist;   // world > 1: the distributed solve's plan instead (dsolve.cu)
  auto own = [&](int lv, int c) { return !dist || DP.own(lv, c); };
  // Single GPU, DC: the second half of a batch is patched with the kept ranks on the device
  // (k_patch) and launched right behind the first half; the host reads the ranks back one
  // batch later, while that second half runs (HS_HOST_PATCH=1: synchronous host patch).
  const bool dpatch = !dist && !nodc && std::getenv("HS_HOST_PATCH") == nullptr;
  int32_t* d_ired = nullptr;   // int32 all-reduce scratch
  int32_t* h_ired = nullptr;
  size_t ired_cap = 0;
  auto allreduce_i32 = [&](std::vector<int32_t>& v) {   // in place, sum over ranks (blocking)
    if (v.empty()) return;
    if (v.size() > ired_cap) {
      if (d_ired) dc.free(d_ired);
      if (h_ired) cudaFreeHost(h_ired);
      ired_cap = std::max(v.size(), 2 * ired_cap);
      d_ired = (int32_t*)dc.alloc(sizeof(int32_t) * ired_cap);
      HS_CUDA(cudaMallocHost(&h_ired, sizeof(int32_t) * ired_cap));
    }
    std::memcpy(h_ired, v.data(), sizeof(int32_t) * v.size());
    HS_CUDA(cudaMemcpyAsync(d_ired, h_ired, sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice, st));
    comm_allreduce_sum_i32(h->comm, d_ired, v.size(), st);
    HS_CUDA(cudaMemcpyAsync(h_ired, d_ired, sizeof(int32_t) * v.size(), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    std::memcpy(v.data(), h_ired, sizeof(int32_t) * v.size());
  };
  std::unique_ptr<void, std::function<void(void*)>> ired_guard((void*)1, [&](void*) {
    if (d_ired) dc.free(d_ired);
    if (h_ired) cudaFreeHost(h_ired);
  });

  // per-level device time (P:1013-1019 report the per-level factor cost): events at the
  // level boundaries, read once the factor is done
  std::vector<cudaEvent_t> lev_ev(an->L_top + 1);
  for (auto& e : lev_ev) HS_CUDA(cudaEventCreate(&e));
  std::unique_ptr<void, std::function<void(void*)>> lev_ev_guard((void*)1, [&](void*) {
    for (auto& e : lev_ev) cudaEventDestroy(e);
  });
  std::vector<double> lev_flops(an->L_top + 1, 0.0);
  BatchVecs rc;   // the batch vectors, reused batch after batch
  // Large factors (the level-0 store is VMM-backed, C4-sized) keep their records in a record
  // space whose completed chunks spill to pinned host memory when a later level's store does
  // not fit beside them (RecSpace, runtime.h).  HS_RECSPACE=0/1 forces it off/on; "force"
  // also spills every completed level at its end (tests the spill/restore path on small cases).
  const char* rs_env = std::getenv("HS_RECSPACE");
  const bool rec_force = rs_env && std::strcmp(rs_env, "force") == 0;
  if (!dist && !nodc && an->L_top > 0 && (rs_env ? std::strcmp(rs_env, "0") != 0 : bs.pool != nullptr)) {
    size_t fr_b = 0, tot_b = 0;
    HS_CUDA(cudaMemGetInfo(&fr_b, &tot_b));
    f->rec.init(&h->vmm, tot_b, st);
    h->vmm.rec = &f->rec;
    if (!an->h_map.empty()) {   // the level-0 scatter and the symmetry check are done with them
      HS_CUDA(cudaStreamSynchronize(st));
      cudaFree(an->d_map);
      cudaFree(an->d_tmap);
      an->d_map = an->d_tmap = nullptr;
    }
  }
  tl.push_back({"level-0 store + setup", now_s()});
  for (int l = 0; l < an->L_top; ++l) {
    HS_CUDA(cudaEventRecord(lev_ev[l], st));
    lev_flops[l] = S.flops;
    const Level& lev = an->levels[l];
    LevelRT& L = f->lv[l];
    const double lv_t0 = now_s(), lv_plan0 = t_plan;
    double lv_ph0[8];
    std::memcpy(lv_ph0, S.t_phase_s, sizeof lv_ph0);
    L.nclus = lev.nclus;
    L.cap = cap;
    L.rank.assign(lev.nclus, 0);
    L.kn.assign(lev.nclus, 0);
    L.kw.assign(lev.nclus, 0);
    L.ldB.assign(lev.nclus, 0);
    L.ldc.assign(lev.nclus, 0);
    L.voff.assign(lev.nclus + 1, 0);
    for (int c = 0; c < lev.nclus; ++c) L.voff[c + 1] = L.voff[c] + cap[c];
    L.vlen = L.voff[lev.nclus];
    ap.vbase.push_back(vbase);
    vbase += L.vlen;
    // ---- level arena (persistent): T_s (cap^2) and the pivots of the owned clusters -------
    std::vector<int64_t> oX(lev.nclus, -1), oP(lev.nclus, 0);
    int64_t off = 0, ioff = 0;
    for (int s = 0; s < lev.nclus; ++s) {
      const int64_t m = cap[s];
      if (m > MAX_M) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "factor: cluster %d at level %d has %lld DOFs > %d (not supported yet)", s,
                      l, (long long)m, MAX_M);
        fail(HS_E_UNSUPPORTED, buf);
      }
      if (!own(l, s)) continue;
      oX[s] = off; off += (m * m + 3) & ~int64_t(3);   // T_s (apply operator), 32-byte aligned
      oP[s] = ioff; ioff += m;
    }
    L.arena_bytes = (size_t)off * sizeof(double);
    const double ta0 = now_s();
    if (f->rec.active()) {   // written batch after batch: not spillable before the level ends
      f->rec.level_start();
      L.arena = (double*)f->rec.alloc(L.arena_bytes);
      f->rec.pin_lo = (uintptr_t)L.arena - f->rec.base;
      f->rec.level_start();
      f->rec.pin_hi = f->rec.top;
    } else {
      L.arena = (double*)dc.alloc(std::max<size_t>(L.arena_bytes, 8));
    }
    L.iarena = (int32_t*)dc.alloc(std::max<size_t>(sizeof(int32_t) * ioff, 4));
    t_tr[2] += now_s() - ta0;
    if (prof) {
      size_t fb = 0, tb = 0;
      HS_CUDA(cudaMemGetInfo(&fb, &tb));
      std::fprintf(stderr, "[hs profile] level %d start: store %.1f GB, T_s arena %.1f GB, cache in use %.1f GB, "
                   "VMM chunks %.1f GB, records %.1f GB (%.1f GB spilled), device free %.1f GB\n", l,
                   bs.total * 8.0 / 1e9, L.arena_bytes / 1e9, dc.in_use / 1e9, h->vmm.created * (double)h->vmm.chunk / 1e9,
                   f->rec.top / 1e9, f->rec.bytes_spilled / 1e9, fb / 1e9);
    }
    L.G.assign(lev.nclus, nullptr); L.V.assign(lev.nclus, nullptr); L.tau.assign(lev.nclus, nullptr);
    L.B.assign(lev.nclus, nullptr); L.nu.assign(lev.nclus, nullptr); L.C.assign(lev.nclus, nullptr);
    L.piv.assign(lev.nclus, nullptr); L.T.assign(lev.nclus, nullptr);
    Slab cslab;
    cslab.dc = &dc;
    cslab.owned = &L.cchunks;
    cslab.rec = &f->rec;
    for (int s = 0; s < lev.nclus; ++s)
      if (oX[s] >= 0) {
        L.piv[s] = L.iarena + oP[s];
        L.T[s] = L.arena + oX[s];
      }
    // neighbour-pair target tables of the level (pattern-only; k_level_pairs)
    LevelPairs lp;   // built below for the levels that run the batch pipeline
    std::vector<int32_t> live = cap;
    std::vector<uint8_t> done(lev.nclus, 0);   // eliminated (rank known here)
    // support-restricted level 0 (support.cpp): B_s of a level-0 cluster holds
    // only the structurally nonzero columns of its blocks (single GPU, direct write-back path)
    const bool khat_lv = l == 0 && dpatch && !no_dwb && !no_fused && !f->keep_records &&
                         std::getenv("HS_NO_KHAT") == nullptr;
    const int32_t* d_sup = nullptr;   // the supports on the device
    if (khat_lv) {
      build_l0_support(*an);
      d_sup = l0_support_device(*an, h->device);
    }
    L.khat = khat_lv;
    std::vector<int32_t> fkn(lev.nclus, 0), fkw(lev.nclus, 0);   // B_s's n/w widths (flop counts)
    // store offsets of row s's blocks, [w(s) ..., n(s) ...] (computed once per cluster)
    std::vector<std::vector<int64_t>> roff(lev.nclus);
    auto row_offs = [&](int32_t s) -> const std::vector<int64_t>& {
      auto& v = roff[s];
      if (v.empty() && !(lev.w[s].empty() && lev.H[s].empty())) {
        v.reserve(lev.w[s].size() + lev.H[s].size());
        bs.row_offsets(s, lev.w[s], v);
        bs.row_offsets(s, lev.H[s], v);
      }
      return v;
    };
    std::vector<uint64_t> wave_mask(lev.nclus, 0);
    // all-reduce of the kept ranks of the eliminated clusters (dist): owners contribute
    auto sync_ranks = [&](const std::vector<uint8_t>& elim) {
      std::vector<int32_t> v(lev.nclus, 0);
      for (int s = 0; s < lev.nclus; ++s)
        if (own(l, s) && elim[s]) v[s] = L.rank[s];
      allreduce_i32(v);
      for (int s = 0; s < lev.nclus; ++s)
        if (elim[s] && !own(l, s)) {
          L.rank[s] = v[s];
          live[s] = v[s];
          done[s] = 1;
        }
    };

    // the batch whose ranks are still on their way to the host (dpatch): (s, m) of its clusters
    std::vector<std::pair<int32_t, int32_t>> pend_cl;
    bool pend_active = false;
    // dpatch: C_s is written into a per-batch region sized for m rows (the rank is not known
    // when the batch is planned) and compacted to its K = m - r rows in the persistent slab
    // once the host reads the ranks (the Schur waves that read it are queued before the copy)
    double* ctmp = nullptr;          // the planned batch's region
    double* pend_ctmp = nullptr;     // the pending batch's region
    bool pend_in_arena = false;      // ... carved from the level's workspace arena
    auto finish_pending = [&]() {
      if (!pend_active) return;
      pend_active = false;
      const double tw0 = now_s();
      for (uint64_t spin = 0; pub->seq != pub_seq; ++spin)
        if ((spin & 0xFFFF) == 0xFFFF) {   // the stream faulted: report instead of spinning
          const cudaError_t e = cudaStreamQuery(st);
          if (e != cudaSuccess && e != cudaErrorNotReady) HS_CUDA(e);
        }
      std::atomic_thread_fence(std::memory_order_acquire);
      t_rank_wait += now_s() - tw0;
      if (pub->flag) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "NOT_SPD: Cholesky breakdown at level %d cluster %d pivot %d value %.17g (P:283)",
                      pub->level, pub->cluster, pub->pivot, pub->value);
        fail(HS_E_NOT_SPD, buf);
      }
      pt.collect_a(S);
      for (size_t bi = 0; bi < pend_cl.size(); ++bi) {
        const int32_t s = pend_cl[bi].first, m = pend_cl[bi].second;
        const int32_t r = m == 0 ? 0 : pub->rank[bi];
        L.rank[s] = r;
        live[s] = r;
        done[s] = 1;
        if (m == 0) continue;
        const int32_t K = m - r, kn = fkn[s], kw = fkw[s];
        S.max_m = std::max(S.max_m, m);
        S.max_rank = std::max(S.max_rank, r);
        double fq = 0.0;
        for (int j = 0; j < r; ++j) fq += 4.0 * (m - j) * (double)(kw - j) + 4.0 * (m - j) * (double)kn;
        S.flops += fq + (double)K * kn * (kn + 1);
        S.flops_phase[3] += fq;
        S.flops_phase[4] += (double)K * kn * (kn + 1);
      }
      if (pend_ctmp) {   // compact the batch's C_s: K x kn each into the persistent slab
        std::vector<CopyItem> cc;
        for (size_t bi = 0; bi < pend_cl.size(); ++bi) {
          const int32_t s = pend_cl[bi].first, m = pend_cl[bi].second;
          if (!L.C[s]) continue;
          const int32_t K = m - L.rank[s], kn = L.ldc[s];
          if (K <= 0 || kn <= 0) {
            L.C[s] = nullptr;
            continue;
          }
          double* dst = cslab.get((int64_t)K * kn);
          cc.push_back(CopyItem{L.C[s], dst, kn, kn, K, kn, 0, 0});
          L.C[s] = dst;
        }
        split_copies(cc);
        Upload& upC = h->upC;
        upC.reset();
        const size_t iC = upC.add(cc);
        upC.stage.ensure(upC.total);
        upC.dev.ensure(upC.total);
        upC.copy_in(iC, cc);
        upC.send(st);
        launch_copy2d(upC.dptr<CopyItem>(iC), (int)cc.size(), st);
        if (!pend_in_arena) dc.free(pend_ctmp);   // stream-ordered reuse: later users are queued after the copy
        pend_ctmp = nullptr;
        if (f->rec.active()) f->rec.frontier = f->rec.top;   // these C_s are complete (spillable)
      }
    };

    int64_t level_dofs = 0;
    for (int32_t c : cap) level_dofs += c;
    // ---- a level of small clusters: one device-planned kernel per wave (small.cu) ---------
    bool small = !dist && !nodc && dpatch && !f->keep_records && level_dofs > 0 &&
                 std::getenv("HS_NO_SMALL_LEVELS") == nullptr;
    std::vector<int64_t> kn_cap(lev.nclus, 0), kw_cap(lev.nclus, 0);
    int small_k = 1, small_m = 1, small_nseg = 1, small_np = 1;
    for (int s = 0; s < lev.nclus && small; ++s) {
      for (int32_t q : lev.H[s]) kn_cap[s] += cap[q];
      for (int32_t q : lev.w[s]) kw_cap[s] += cap[q];
      const int nn = (int)lev.H[s].size();
      small = cap[s] <= SMALL_M && kn_cap[s] + kw_cap[s] <= SMALL_K;
      small_m = std::max(small_m, cap[s]);
      small_k = std::max<int>(small_k, (int)(kn_cap[s] + kw_cap[s]));
      small_nseg = std::max<int>(small_nseg, nn + (int)lev.w[s].size());   // raw entries (empty ones included)
      small_np = std::max(small_np, nn * (nn + 1) / 2);
    }
    if (small) {
      const int n = lev.nclus;
      std::vector<int32_t> nptr(n + 1, 0), nidx, wptr(n + 1, 0), widx, items;
      for (int c = 0; c < n; ++c) {
        nidx.insert(nidx.end(), lev.H[c].begin(), lev.H[c].end());
        widx.insert(widx.end(), lev.w[c].begin(), lev.w[c].end());
        nptr[c + 1] = (int32_t)nidx.size();
        wptr[c + 1] = (int32_t)widx.size();
      }
      // waves: the clusters of a batch without a common neighbour (Schur targets disjoint)
      std::vector<std::pair<int32_t, int32_t>> waves;   // (first, count) into items
      std::vector<uint64_t> mask(n, 0);
      for (const auto& Bt : lev.batches) {
        std::vector<std::vector<int32_t>> wv;
        std::vector<int32_t> touched;
        for (int32_t c : Bt) {
          uint64_t used = 0;
          for (int32_t q : lev.H[c]) used |= mask[q];
          int w = 0;
          while (w < 64 && ((used >> w) & 1ull)) ++w;
          if (w == 64) w = 64 + (int)wv.size();   // overflow: a wave of its own
          if ((int)wv.size() <= w) wv.resize(w + 1);
          wv[w].push_back(c);
          if (w < 64)
            for (int32_t q : lev.H[c]) {
              if (!mask[q]) touched.push_back(q);
              mask[q] |= 1ull << w;
            }
        }
        for (int32_t q : touched) mask[q] = 0;
        for (auto& v : wv)
          if (!v.empty()) {
            waves.push_back({(int32_t)items.size(), (int32_t)v.size()});
            items.insert(items.end(), v.begin(), v.end());
          }
        S.n_batches++;
      }
      std::vector<int64_t> toff(n, 0), poff(n, 0), coff(n, 0);
      int64_t ctot = 0;
      for (int c = 0; c < n; ++c) {
        toff[c] = oX[c] < 0 ? 0 : oX[c];
        poff[c] = oP[c];
        coff[c] = ctot;
        ctot += ((int64_t)cap[c] * kn_cap[c] + 3) & ~int64_t(3);
      }
      double* cbase = (double*)dc.alloc(sizeof(double) * std::max<int64_t>(ctot, 4));
      L.cchunks.push_back(cbase);
      int32_t* dint = (int32_t*)dc.alloc(sizeof(int32_t) * (4 * (size_t)n + 1));   // live rank kn kw
      upA.reset();
      const size_t iNP = upA.add(nptr), iNI = upA.add(nidx), iWP = upA.add(wptr), iWI = upA.add(widx),
                   iIT = upA.add(items), iLV = upA.add(cap), iTO = upA.add(toff), iPO = upA.add(poff),
                   iCO = upA.add(coff);
      upA.stage.ensure(upA.total);
      upA.dev.ensure(upA.total);
      upA.copy_in(iNP, nptr); upA.copy_in(iNI, nidx); upA.copy_in(iWP, wptr); upA.copy_in(iWI, widx);
      upA.copy_in(iIT, items); upA.copy_in(iLV, cap); upA.copy_in(iTO, toff); upA.copy_in(iPO, poff);
      upA.copy_in(iCO, coff);
      upA.send(st);
      HS_CUDA(cudaMemcpyAsync(dint, upA.dptr<int32_t>(iLV), sizeof(int32_t) * n, cudaMemcpyDeviceToDevice, st));
      SmallArgs sa{};
      sa.dir = bs.dir();
      sa.nptr = upA.dptr<int32_t>(iNP); sa.nidx = upA.dptr<int32_t>(iNI);
      sa.wptr = upA.dptr<int32_t>(iWP); sa.widx = upA.dptr<int32_t>(iWI);
      sa.live = dint; sa.rank = dint + n; sa.kn = dint + 2 * n; sa.kw = dint + 3 * n;
      sa.T = L.arena; sa.toff = upA.dptr<int64_t>(iTO);
      sa.piv = L.iarena; sa.poff = upA.dptr<int64_t>(iPO);
      sa.C = cbase; sa.coff = upA.dptr<int64_t>(iCO);
      sa.items = upA.dptr<int32_t>(iIT);
      sa.status = d_status;
      sa.eps = opt.eps; sa.relative = opt.eps_relative ? 1 : 0; sa.level = l;
      sa.m_max = small_m; sa.k_max = small_k; sa.nseg_max = small_nseg; sa.npair_max = small_np;
      pt.rec(pt.a[3], st);
      for (const auto& w : waves) launch_elim_small(sa, w.first, w.second, st);
      pt.rec(pt.a[4], st);
      std::vector<int32_t> back(3 * (size_t)n);
      HS_CUDA(cudaMemcpyAsync(back.data(), dint + n, sizeof(int32_t) * 3 * n, cudaMemcpyDeviceToHost, st));
      HS_CUDA(cudaMemcpyAsync(&h_status, d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
      HS_CUDA(cudaStreamSynchronize(st));
      dc.free(dint);
      if (h_status.flag == 1) {
        char buf[256];
        std::snprintf(buf, sizeof buf, "NOT_SPD: Cholesky breakdown at level %d cluster %d pivot %d value %.17g (P:283)",
                      h_status.level, h_status.cluster, h_status.pivot, h_status.value);
        fail(HS_E_NOT_SPD, buf);
      }
      if (h_status.flag) fail(HS_E_INTERNAL, "small-cluster level: a block of the schedule is missing");
      if (pt.on) S.t_phase_s[3] += PhaseTimer::el(pt.a[3], pt.a[4]);
      for (int c = 0; c < n; ++c) {
        const int32_t m = cap[c], r = back[c], kn = back[n + c], kw = back[2 * n + c];
        L.rank[c] = r;
        L.kn[c] = kn;
        L.kw[c] = kw;
        L.ldB[c] = kn + kw;
        L.ldc[c] = kn;
        live[c] = r;
        done[c] = 1;
        L.C[c] = (m > r && kn > 0) ? cbase + coff[c] : nullptr;
        if (m == 0) continue;
        const int32_t K = m - r;
        S.max_m = std::max(S.max_m, m);
        S.max_rank = std::max(S.max_rank, r);
        double fq = 0.0;
        for (int j = 0; j < r; ++j) fq += 4.0 * (m - j) * (double)(kw - j) + 4.0 * (m - j) * (double)kn;
        const double all = (double)m * m * m / 3.0 + (double)m * m * (kn + kw) + fq + (double)K * kn * (kn + 1);
        S.flops += all;
        S.flops_phase[3] += all;   // the fused small-cluster kernel is timed as one phase (entry 3)
      }
    }
    if (!small) lp.build(lev, bs, dc, upA, st);   // n(s)-pair target tables of the Schur tiles
    // Batches whose workspace (G, G^-1, V, B_s, the C_s region; bounded with the level-start
    // sizes) exceeds the budget run as consecutive sub-batches: a batch is an independent set,
    // so its clusters' eliminations commute and each Schur target still receives its updates
    // in source order (C4 on one GPU: a level-2 batch would need ~30 GB of workspace next to
    // a ~130 GB block store).  HS_BATCH_WS_GB sets the budget (default 12 GB).
    struct SubBatch { size_t bidx; size_t b0, b1; };
    std::vector<SubBatch> subs;
    {
      static const double ws_cap = [] {
        const char* e = std::getenv("HS_BATCH_WS_GB");
        return (e ? std::atof(e) : 12.0) * 1e9;
      }();
      double ws_budget = ws_cap;
      if (f->rec.active()) {   // a quarter of what the store, the arena and the resident data leave
        size_t fb = 0, tb = 0;
        HS_CUDA(cudaMemGetInfo(&fb, &tb));
        const double resident = 12.0 * nnz + 24.0 * n + (an->d_map ? 16.0 * nnz : 0.0);
        const double left = (double)tb - 8.0 * bs.total - (double)L.arena_bytes - (double)dc.in_use - resident;
        ws_budget = std::min(ws_cap, std::max(1e9, 0.25 * left));
      }
      for (size_t bidx = 0; bidx < (small ? 0 : lev.batches.size()); ++bidx) {
        const auto& Bt = lev.batches[bidx];
        size_t b0 = 0;
        double acc = 0.0;
        for (size_t i = 0; i < Bt.size(); ++i) {
          const int32_t c = Bt[i];
          const double m = cap[c];
          double kk = 0.0;
          for (int32_t q : lev.H[c]) kk += cap[q];
          for (int32_t q : lev.w[c]) kk += cap[q];
          const double w = 8.0 * (3 * m * m + 2 * m + kk + 2 * m * kk);
          if (!dist && i > b0 && acc + w > ws_budget) {
            subs.push_back({bidx, b0, i});
            b0 = i;
            acc = 0.0;
          }
          acc += w;
        }
        subs.push_back({bidx, b0, Bt.size()});
      }
    }
    // Record-space factors (C4-sized, device memory nearly full): one workspace arena per level,
    // sized by the largest sub-batch's bound (level-start sizes), from which every batch carves
    // its G / G^-1 / V / B_s, C_s region and CPQR scratch -- per-batch allocations of changing
    // sizes would miss the cache and trim it (a device synchronisation) batch after batch
    double* lvl_ws = nullptr;
    int64_t lvl_ws_words = 0;
    if (f->rec.active() && !dist && !subs.empty()) {
      for (const auto& sb : subs) {
        int64_t w = 0;
        for (size_t i = sb.b0; i < sb.b1; ++i) {
          const int32_t c = lev.batches[sb.bidx][i];
          const int64_t m = cap[c];
          int64_t kn = 0, kw = 0;
          for (int32_t q : lev.H[c]) kn += cap[q];
          for (int32_t q : lev.w[c]) kw += cap[q];
          w += 3 * m * m + m + kw + m * (kn + kw) + 12 + m * kn + 4;
          const int64_t g = (int64_t)std::max(cpqr_global_words((int)m, (int)kw, (int)m),
                                              cpqr_global_words((int)m, (int)kw, MAX_M));
          if (g) w += g + 4;
        }
        lvl_ws_words = std::max(lvl_ws_words, w + 16);
      }
      lvl_ws = (double*)dc.alloc(sizeof(double) * lvl_ws_words);
    }
    std::vector<int32_t> sub_cl;
    for (size_t ib = 0; ib < subs.size(); ++ib) {
      const size_t bidx = subs[ib].bidx;
      sub_cl.assign(lev.batches[bidx].begin() + subs[ib].b0, lev.batches[bidx].begin() + subs[ib].b1);
      const auto& Bt = sub_cl;
      if (level_dofs == 0) break;   // every cluster is empty: nothing to eliminate on this level
      const bool phase2 = (int)bidx >= lev.nphase1;
      if (dist && phase2 && (int)bidx == lev.nphase1) {   // the phase-I ranks of every owner
        std::vector<uint8_t> ph1(lev.nclus, 0);
        for (int b = 0; b < lev.nphase1; ++b)
          for (int32_t s : lev.batches[b]) ph1[s] = 1;
        sync_ranks(ph1);
      }
      finish_pending();   // the previous batch's ranks (its second half may still be running)
      const double tp0 = now_s();
      // shapes of every cluster of the batch from the current live sizes
      for (int32_t s : Bt) {
        int32_t kn = 0, kw = 0;
        for (int32_t q : lev.H[s]) kn += live[q];
        for (int32_t q : lev.w[s]) kw += live[q];
        L.kn[s] = kn; L.kw[s] = kw; L.ldB[s] = kn + kw; L.ldc[s] = kn;
      }
      CluItem* d_clu_batch = nullptr;   // this batch's cluster items on the device (upA)
      std::vector<int32_t> Bo;   // the batch's clusters eliminated here
      for (int32_t s : Bt)
        if (own(l, s)) Bo.push_back(s);
      const int nb = (int)Bo.size();
      auto& gather = rc.gather;
      auto& clu = rc.clu;
      auto& trsm = rc.trsm;
      auto& rot = rc.rot;
      auto& fci = rc.fci;   // gather-free Cholesky + inverse per cluster
      auto& fz = rc.fz;     // the scaling per 64-column tile of a cluster (fci index)
      auto& fseg = rc.fseg;
      gather.clear(); trsm.clear(); rot.clear(); fci.clear(); fz.clear(); fseg.clear();
      clu.assign(nb, CluItem{});
      int max_m = 1;
      for (int bi = 0; bi < nb; ++bi) max_m = std::max(max_m, live[Bo[bi]]);
      const bool fused = !nodc && max_m <= CI_MAX_M && !no_fused;
      // direct write-back: CPQR / k_rotate_n write row s's coarse blocks, I_r and C_s
      // themselves (no write-back pass); needs the device patch and CPQR v3
      const bool dwb = fused && dpatch && !no_dwb;
      std::vector<int32_t> seg0v(nb, 0);
      // the widths of B_s: dense, or (khat) the supported columns of each block (the segments
      // point into the analysis's device copy of the supports, d_sup)
      const bool khat = khat_lv && dwb;
      std::vector<int32_t> bkn(nb), bkw(nb);
      std::vector<std::vector<int32_t>> nlen(nb);   // compressed width of each q of n(s)
      std::vector<std::vector<int64_t>> nsup(nb);   // its supported columns in su.idx (-1: dense)
      const L0Support& su = an->l0s;
      for (int bi = 0; bi < nb; ++bi) {
        const int32_t s = Bo[bi];
        bkn[bi] = L.kn[s];
        bkw[bi] = L.kw[s];
        if (!khat) continue;
        int64_t e = su.sptr[s], x = su.iptr[s];
        bkn[bi] = bkw[bi] = 0;
        nlen[bi].reserve(lev.H[s].size());
        nsup[bi].reserve(lev.H[s].size());
        for (int pass = 0; pass < 2; ++pass)
          for (int32_t q : (pass == 0 ? lev.w[s] : lev.H[s])) {
            const int32_t ln = su.len[e++];
            if ((ln < 0) != (done[q] != 0)) fail(HS_E_INTERNAL, "support: schedule mismatch");
            const int32_t c = ln < 0 ? live[q] : ln;
            if (pass == 0) {
              bkw[bi] += c;
            } else {
              bkn[bi] += c;
              nlen[bi].push_back(c);
              nsup[bi].push_back(ln < 0 ? -1 : x);
            }
            if (ln > 0) x += ln;
          }
        L.ldB[s] = bkn[bi] + bkw[bi];
        L.ldc[s] = bkn[bi];   // C_s on the supported n-columns
      }
      for (int bi = 0; bi < nb; ++bi) {
        fkn[Bo[bi]] = bkn[bi];
        fkw[Bo[bi]] = bkw[bi];
      }
      const double tfh1 = now_s();
      t_fh[0] += tfh1 - tp0;
      // batch workspace: G (m^2), V (m^2), tau (m), nu (kw), B (m x (kw + kn)) per cluster
      int64_t wsz = 0;
      std::vector<int64_t> wo(nb);
      for (int bi = 0; bi < nb; ++bi) {
        const int32_t s = Bo[bi];
        const int64_t m = live[s], kn = bkn[bi], kw = bkw[bi];
        wo[bi] = wsz;
        wsz += 3 * m * m + ((m + 3) & ~int64_t(3)) + ((kw + 3) & ~int64_t(3)) + ((m * (kn + kw) + 3) & ~int64_t(3));
      }
      // the batch's C_s region (dpatch: m rows each, compacted once the ranks are known)
      int64_t csz = 0;
      std::vector<int64_t> co(nb, -1);
      if (dpatch)
        for (int bi = 0; bi < nb; ++bi) {
          const int64_t m = live[Bo[bi]], kn = L.ldc[Bo[bi]];
          if (m > 0 && kn > 0) {
            co[bi] = csz;
            csz += (m * kn + 3) & ~int64_t(3);
          }
        }
      // CPQR global-memory scratch of the clusters whose w-block exceeds a 16-CTA cluster's
      // shared memory (freed once the batch's kernels are queued: stream-ordered reuse)
      int64_t gsz = 0;
      std::vector<int64_t> go(nb, -1);
      for (int bi = 0; bi < nb; ++bi) {
          const int64_t w = (int64_t)cpqr_global_words(live[Bo[bi]], bkw[bi], max_m);
          if (w) {
            go[bi] = gsz;
            gsz += (w + 3) & ~int64_t(3);
          }
        }
      double *ws = nullptr, *wtmp = nullptr;
      const int64_t wsz4 = (std::max<int64_t>(wsz, 4) + 3) & ~int64_t(3), csz4 = (csz + 3) & ~int64_t(3);
      const bool in_arena = nb && lvl_ws && wsz4 + csz4 + gsz <= lvl_ws_words;
      if (in_arena) {   // carved from the level's workspace arena (stream-ordered reuse)
        ws = lvl_ws;
        ctmp = csz ? lvl_ws + wsz4 : nullptr;
        wtmp = gsz ? lvl_ws + wsz4 + csz4 : nullptr;
      } else {
        ws = nb ? (double*)dc.alloc(sizeof(double) * std::max<int64_t>(wsz, 4)) : nullptr;
        ctmp = csz ? (double*)dc.alloc(sizeof(double) * csz) : nullptr;
        wtmp = gsz ? (double*)dc.alloc(sizeof(double) * gsz) : nullptr;
      }
      // the batch's items: the counts per cluster (sequential, cheap), then every cluster fills
      // its own ranges of the item lists on PT pooled host threads (the same lists as a
      // sequential pass)
      auto& cnt = rc.cnt;   // [6][nb + 1] prefix counts: segments, scale tiles, rotation tiles, fci, gathers, trsm
      for (auto& v : cnt) v.assign(nb + 1, 0);
      for (int bi = 0; bi < nb; ++bi) {
        const int32_t s = Bo[bi], m = live[s], kn = bkn[bi], kw = bkw[bi], ldB = L.ldB[s];
        int32_t c[6] = {0, 0, 0, 0, 0, 0};
        if (m > 0) {
          int64_t e = khat ? su.sptr[s] : 0;
          for (int pass = 0; pass < 2; ++pass)
            for (int32_t q : (pass == 0 ? lev.w[s] : lev.H[s])) {
              const int32_t ln = khat ? su.len[e++] : -1;
              const int32_t wq = ln >= 0 ? ln : live[q];
              if (live[q] > 0) {
                if (fused) c[0] += wq > 0;
                else ++c[4];
              }
            }
          const int32_t rw = rot_tile_cols(m, max_m), tw = nodc ? (m <= SMEM_M ? 64 : 32) : trsm_mma_tile_cols();
          if (fused) {
            c[1] = (ldB + 63) / 64;
            c[2] = (m + rw - 1) / rw;
            c[3] = 1;
          } else {
            c[4] += 1;
            c[5] = (ldB + tw - 1) / tw;
            if (!nodc) {   // G_s^{-1} as identity strips of the TRSM, T_s by the rotation
              c[5] += (m + tw - 1) / tw;
              c[2] = (m + rw - 1) / rw;
            }
          }
          if (kw > 0 || (dwb && kn > 0)) c[2] += (kn + rw - 1) / rw;
        }
        for (int k = 0; k < 6; ++k) cnt[k][bi + 1] = cnt[k][bi] + c[k];
      }
      fseg.resize(cnt[0][nb]); fz.resize(cnt[1][nb]); rot.resize(cnt[2][nb]); fci.resize(cnt[3][nb]);
      gather.resize(cnt[4][nb]); trsm.resize(cnt[5][nb]);
      const int PT = plan_threads(nb);
      std::vector<double> pfl(2 * PT, 0.0);
      const double tfa = now_s();
      t_fh[3] += tfa - tfh1;
      par_chunks(nb, PT, [&](int b0, int b1, int t) {
        for (int bi = b0; bi < b1; ++bi) {
          const int32_t s = Bo[bi];
          const int32_t m = live[s], kn = bkn[bi], kw = bkw[bi], ldB = L.ldB[s];
          int32_t isg = cnt[0][bi], itl = cnt[1][bi], irt = cnt[2][bi], igt = cnt[4][bi], itr = cnt[5][bi];
          const int32_t ci = cnt[3][bi];
          double* w0 = ws + wo[bi];
          L.G[s] = w0;
          L.V[s] = w0 + (int64_t)m * m;
          L.tau[s] = w0 + 2 * (int64_t)m * m;
          L.nu[s] = L.tau[s] + ((m + 3) & ~3);
          L.B[s] = L.nu[s] + ((kw + 3) & ~3);   // 32-byte aligned
          double* ginv = L.B[s] + (((int64_t)m * (kn + kw) + 3) & ~int64_t(3));   // G^{-1} (fused path)
          CluItem& it = clu[bi];
          it.G = L.G[s]; it.V = L.V[s]; it.tau = L.tau[s]; it.B = L.B[s]; it.piv = L.piv[s]; it.nu = L.nu[s];
          it.m = m; it.kw = kw; it.kn = kn; it.ldB = ldB; it.level = l; it.cluster = s;
          it.ldC = L.ldc[s];   // C_s: the record on B_s's n-columns
          it.kwd = khat ? L.kw[s] : -1;
          it.Wt = go[bi] >= 0 ? wtmp + go[bi] : nullptr;
          if (m == 0) continue;
          double* p; int32_t ld, tr;
          bs.get(s, s, p, ld, tr);
          // the store keeps the lower triangle of a diagonal block; dc = 0 rotates both sides
          // of A_ss, so it is gathered as the full symmetric block (copy mode 2)
          if (fused && tr) fail(HS_E_INTERNAL, "diagonal block stored transposed");
          const double* pss = p;
          const int32_t ldss = ld;
          if (!fused) gather[igt++] = CopyItem{p, L.G[s], ld, m, m, m, nodc ? 2 : tr, 0};
          const int32_t seg0 = isg;
          int32_t col = 0, dcol = 0;   // the block's first column in B_s / in the dense B_s
          const auto& ro = row_offs(s);
          size_t kq = 0;
          int64_t e = khat ? su.sptr[s] : 0, x = khat ? su.iptr[s] : 0;
          for (int pass = 0; pass < 2; ++pass)
            for (int32_t q : (pass == 0 ? lev.w[s] : lev.H[s])) {
              const int64_t o = ro[kq++];
              const int32_t ln = khat ? su.len[e++] : -1;   // >= 0: the supported columns at su.idx[x]
              const int32_t wq = ln >= 0 ? ln : live[q];
              const int32_t* sidx = ln >= 0 ? d_sup + x : nullptr;
              if (ln > 0) x += ln;
              if (live[q] > 0) {
                if (o < 0) fail(HS_E_INTERNAL, "gather: block of an owned row missing");
                bs.at(s, q, o, p, ld, tr);
                if (fused) {
                  if (wq > 0) fseg[isg++] = FusedSeg{p, sidx, ld, tr, col, wq, dcol, 0};
                } else {
                  gather[igt++] = CopyItem{p, L.B[s] + col, ld, ldB, m, live[q], tr, 0};
                }
              }
              col += wq;
              dcol += live[q];
            }
          const int32_t tw = nodc ? (m <= SMEM_M ? 64 : 32) : trsm_mma_tile_cols();   // the scaling kernel's strip width
          if (fused) {
            // segments are in column order: each tile takes the run of segments overlapping it
            int32_t sb = seg0;
            const int32_t se = isg;
            fci[ci] = FusedItem{pss, L.G[s], ginv, L.B[s], nullptr, m, ldss, ldB, kw, 0, 0, 0, 0, l, s, bi, 0};
            if (dwb) {
              seg0v[bi] = seg0;
              it.nseg = se - seg0;
              it.Dss = const_cast<double*>(pss);
              it.ldss = ldss;
              it.dwb = 1;
              it.keepB = f->keep_records ? 1 : 0;
              if (L.ldc[s] > 0) {
                L.C[s] = ctmp + co[bi];   // C_s = rows [r, m) of the rotated B_n (K <= m)
                it.Cout = L.C[s];
              }
            }
            for (int32_t c0 = 0; c0 < ldB; c0 += 64) {
              const int32_t nc = std::min(64, ldB - c0);
              while (sb < se && fseg[sb].col + fseg[sb].len <= c0) ++sb;
              int32_t sf = sb;
              while (sf < se && fseg[sf].col < c0 + nc) ++sf;
              fz[itl++] = ScaleTile{ci, c0, nc, sb, sf, 0};
            }
          } else {
            for (int32_t c0 = 0; c0 < ldB; c0 += tw) trsm[itr++] = TrsmItem{bi, c0, std::min(tw, ldB - c0), 0};
            if (!nodc)   // G_s^{-1} = the TRSM of the identity (k_trsm_mma strips, pad = 2)
              for (int32_t c0 = 0; c0 < m; c0 += tw) trsm[itr++] = TrsmItem{bi, c0, std::min(tw, m - c0), 2};
          }
          if (kw > 0 || (dwb && kn > 0)) {   // the n-columns are rotated by k_rotate_n
            const int32_t rw = rot_tile_cols(m, max_m);
            for (int32_t c0 = 0; c0 < kn; c0 += rw) rot[irt++] = TrsmItem{bi, c0, std::min(rw, kn - c0), 0};
          }
          if (fused || !nodc) {   // ... and so is G^{-1}: the apply operator T_s = Qᵀ G_s^{-1} (no k_form_T)
            it.Ginv = ginv;
            it.Tout = L.T[s];
            const int32_t rw = rot_tile_cols(m, max_m);
            for (int32_t c0 = 0; c0 < m; c0 += rw) rot[irt++] = TrsmItem{bi, c0, std::min(rw, m - c0), 1};
          }
          if (isg != cnt[0][bi + 1] || itl != cnt[1][bi + 1] || irt != cnt[2][bi + 1] || igt != cnt[4][bi + 1] ||
              itr != cnt[5][bi + 1])
            fail(HS_E_INTERNAL, "batch plan: item counts");
          pfl[2 * t] += (double)m * m * m / 3.0;
          pfl[2 * t + 1] += (double)m * m * ldB + (!fused && !nodc ? (double)m * m * m / 3.0 : 0.0);
        }
      });
      const double tfb = now_s();
      t_fh[4] += tfb - tfa;
      for (int t = 0; t < PT; ++t) {
        S.flops += pfl[2 * t] + pfl[2 * t + 1];
        S.flops_phase[1] += pfl[2 * t];
        S.flops_phase[2] += pfl[2 * t + 1];
      }
      // the first half's launches: at once (host patch), or (device patch) deferred until the
      // second half is planned, so that both uploads precede one uninterrupted kernel chain
      std::function<void(bool)> first_half_launch;   // argument: publish the ranks here
      const double tfh2 = now_s();
      t_fh[1] += tfh2 - tfh1;
      if (nb > 0) {
        split_copies(gather);
        upA.reset();
        std::vector<unsigned long long> nmax(nb, 0ull);
        const size_t iG = upA.add(gather), iC = upA.add(clu), iT = upA.add(trsm), iR = upA.add(rot),
                     iM = upA.add(nmax), iF = upA.add(fz), iS = upA.add(fseg), iI = upA.add(fci);
        upA.stage.ensure(upA.total);
        upA.dev.ensure(upA.total);
        for (int bi = 0; bi < nb; ++bi) clu[bi].nmax = upA.dptr<unsigned long long>(iM) + bi;
        for (auto& f : fci) f.nmax = upA.dptr<unsigned long long>(iM) + f.bi;   // R-floor slot
        for (int bi = 0; bi < nb; ++bi)
          if (clu[bi].dwb) clu[bi].seg = upA.dptr<FusedSeg>(iS) + seg0v[bi];
        upA.copy_in(iG, gather); upA.copy_in(iC, clu); upA.copy_in(iT, trsm); upA.copy_in(iR, rot);
        upA.copy_in(iM, nmax); upA.copy_in(iF, fz); upA.copy_in(iS, fseg); upA.copy_in(iI, fci);
        t_plan += now_s() - tp0;
        t_fh[2] += now_s() - tfh2;
        d_clu_batch = upA.dptr<CluItem>(iC);
        const size_t nfz = fz.size(), nfci = fci.size(), ngather = gather.size(), ntrsm = trsm.size(),
                     nrot = rot.size();
        first_half_launch = [&, iG, iC, iT, iR, iF, iS, iI, fused, max_m, nb, nfz, nfci, ngather, ntrsm, nrot,
                             clu](bool publish) {
          pt.rec(pt.a[0], st);
          if (fused) {   // Cholesky per cluster ("potrf"), scaling per tile ("trsm")
            pt.rec(pt.a[1], st);
            launch_chol(upA.dptr<FusedItem>(iI), (int)nfci, max_m, d_status, st);
            pt.rec(pt.a[2], st);
            launch_scale_tiles(upA.dptr<FusedItem>(iI), upA.dptr<ScaleTile>(iF), (int)nfz, upA.dptr<FusedSeg>(iS),
                               max_m, st);
          } else {
            launch_copy2d(upA.dptr<CopyItem>(iG), (int)ngather, st);
            pt.rec(pt.a[1], st);
            if (!nodc) launch_potrf(upA.dptr<CluItem>(iC), nb, max_m, d_status, st);
            pt.rec(pt.a[2], st);
            if (!nodc) launch_trsm_mma(upA.dptr<CluItem>(iC), upA.dptr<TrsmItem>(iT), (int)ntrsm, max_m, st);
            else launch_nmax(upA.dptr<CluItem>(iC), upA.dptr<TrsmItem>(iT), (int)ntrsm, st);   // R-floor
          }
          pt.rec(pt.a[3], st);
          launch_cpqr3(upA.dptr<CluItem>(iC), clu, opt.eps, opt.eps_relative, d_rank, st);
          // the ranks are final here: publish them before the rotation, so that the host plans
          // the next batch while the rotation and this batch's Schur update run
          if (dpatch && publish) launch_publish(d_rank, nb, d_status, pub_dev, ++pub_seq, st);
          launch_rotate_n(upA.dptr<CluItem>(iC), upA.dptr<TrsmItem>(iR), (int)nrot, max_m, d_rank, st);
          pt.rec(pt.a[4], st);
          if (!dpatch) HS_CUDA(cudaMemcpyAsync(h_rank, d_rank, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
        };
        if (!dpatch) {
          upA.send(st);
          first_half_launch(true);
          first_half_launch = nullptr;
        }
      } else {
        t_plan += now_s() - tp0;
      }
      // ---- pre-plan of the batch's second half while its first half runs: everything but
      // the kept ranks (patched after the read-back; a source whose rank turns out full is a
      // phantom whose tiles exit at once).  Remote clusters of a phase-II batch are planned if
      // this rank will receive their record.
      const double tpp = now_s();
      auto& srcs = rc.srcs;
      std::vector<int32_t> src_cl;
      auto& nbc = rc.nbc;
      srcs.clear();
      nbc.clear();
      std::vector<std::vector<SchurTile2>> waves;
      std::vector<int32_t> touched;
      auto& wb = rc.wb;
      wb.clear();
      std::vector<double*> id_ptr;
      std::vector<int32_t> id_ld, id_r;
      std::vector<FormTItem> ft;
      int ft_max_m = 0;
      struct Pend {
        int32_t s, k;
        bool mine;
        int64_t src, id, diag, ft;
        size_t wb_begin, wb_end;
      };
      std::vector<Pend> pend;
      std::vector<int32_t> live_at(Bt.size());
      for (size_t k = 0; k < Bt.size(); ++k) {
        const int32_t s = Bt[k];
        live_at[k] = live[s];
        const bool mine = own(l, s);
        if (!mine) {
          if (!(dist && phase2)) continue;
          const std::vector<int32_t> rc = receivers(*an, DP, l, s);
          if (!std::binary_search(rc.begin(), rc.end(), (int32_t)h->rank)) continue;
        }
        const int32_t m = live[s], kn = L.kn[s], ldB = L.ldB[s];
        if (m == 0) continue;
        const int32_t kc = khat ? bkn[k] : kn;   // the n-columns the Schur tiles run over
        Pend pd{s, (int32_t)k, mine, -1, -1, -1, -1, wb.size(), wb.size()};
        if (mine && !fused && nodc) {   // (dc: k_rotate_n forms T_s from G^{-1} of k_chol / k_trsm_mma)
          pd.ft = (int64_t)ft.size();
          ft.push_back(FormTItem{L.G[s], nullptr, L.V[s], L.tau[s], L.T[s], m, 0});
          ft_max_m = std::max(ft_max_m, m);
        }
        // neighbour column offsets inside the n-part
        const auto& ns = lev.H[s];
        std::vector<int32_t> noff(ns.size() + 1, 0);
        auto nwid = [&](size_t a) { return khat ? nlen[k][a] : live[ns[a]]; };
        for (size_t a = 0; a < ns.size(); ++a) noff[a + 1] = noff[a] + nwid(a);
        if (kc > 0) {
          // wave = lowest wave in which no earlier source shares a neighbour with s
          uint64_t used = 0;
          for (int32_t q : ns)
            if (live[q] > 0) used |= wave_mask[q];
          int w = 0;
          while (w < 63 && ((used >> w) & 1ull)) ++w;
          if ((used >> w) & 1ull) w = 63 + (int)waves.size();   // overflow: a wave of its own
          const uint64_t bit = w < 64 ? (1ull << w) : 0ull;
          SchurSrc sc{nullptr, dwb ? L.ldc[s] : ldB, 0, kc, (int32_t)nbc.size(), 0, 0};
          for (size_t a = 0; a < ns.size(); ++a)
            if (live[ns[a]] > 0) {
              if (nwid(a) > 0)
                nbc.push_back(NbCol{ns[a], noff[a], nwid(a), (int32_t)a,
                                    khat && nsup[k][a] >= 0 ? d_sup + nsup[k][a] : nullptr});
              if (!wave_mask[ns[a]]) touched.push_back(ns[a]);
              wave_mask[ns[a]] |= bit;
            }
          sc.nnb = (int32_t)nbc.size() - sc.nb_off;
          pd.src = (int64_t)srcs.size();
          srcs.push_back(sc);
          src_cl.push_back(s);
          if ((int)waves.size() <= w) waves.resize(w + 1);
          const int T = (kc + 63) / 64;
          for (int ti = 0; ti < T; ++ti)
            for (int tj = 0; tj <= ti; ++tj) waves[w].push_back(SchurTile2{(int32_t)pd.src, ti * 64, tj * 64, 0});
        }
        // write-back of row s: [I_r | coarse-w | coarse-n] into the blocks held here (rows r)
        double* p; int32_t ld, tr;
        if (mine && !dwb) {
          bs.get(s, s, p, ld, tr);
          if (nodc) {
            pd.diag = (int64_t)wb.size();
            wb.push_back(CopyItem{L.G[s], p, m, ld, 0, 0, 0, 0});   // A_cc - C_c^T C_c
          } else {
            pd.id = (int64_t)id_ptr.size();
            id_ptr.push_back(p); id_ld.push_back(ld); id_r.push_back(0);
          }
        }
        pd.wb_begin = wb.size();
        int32_t col = 0;
        const auto& ro = row_offs(s);
        size_t kq = 0;
        for (int pass = 0; pass < (dwb ? 0 : 2); ++pass)
          for (int32_t q : (pass == 0 ? lev.w[s] : lev.H[s])) {
            const int64_t o = ro[kq++];
            if (live[q] > 0 && o >= 0) {
              bs.at(s, q, o, p, ld, tr);
              const double* off = (const double*)(uintptr_t)col;   // + B_s once known
              if (!tr) wb.push_back(CopyItem{off, p, ldB, ld, 0, live[q], 0, 0});
              else wb.push_back(CopyItem{off, p, ldB, ld, live[q], 0, 1, 0});
            }
            col += live[q];
          }
        pd.wb_end = wb.size();
        pend.push_back(pd);
      }
      t_sub[0] += now_s() - tpp;
      if (nb > 0 && !dpatch) {
        check_status(d_status, &h_status, st);       // synchronises the stream
        pt.collect(S);
      }
      deferred.drain(false);
      const double tp1 = now_s();
      if (!dpatch)
        for (int bi = 0; bi < nb; ++bi) {
          const int32_t s = Bo[bi];
          L.rank[s] = live[s] == 0 ? 0 : h_rank[bi];
        }
      if (nodc && nb > 0) {
        // (U^T A_ss U) in G; L_f L_f^T = its fine block; C_c = L_f^{-1} G[r:, :r] in place,
        // C_n = L_f^{-1} (U^T A_sn)_f in B; [A_cc | A_cn] -= C_c^T [C_c | C_n]
        std::vector<CluItem> fine, fs;
        std::vector<TrsmItem> fst, cu;
        int fmax = 1;
        for (int bi = 0; bi < nb; ++bi) {
          const int32_t s = Bo[bi];
          const int32_t m = live[s], r = L.rank[s], K = m - r;
          if (K <= 0) continue;
          CluItem f0 = clu[bi];
          f0.G = L.G[s] + (int64_t)r * m + r;
          f0.m = K;
          f0.pad0 = m;            // ld of the fine block inside G
          f0.nmax = nullptr;
          fine.push_back(f0);
          fmax = std::max(fmax, K);
          const int32_t tw = K <= SMEM_M ? 64 : 32;
          CluItem a0 = f0;        // right-hand sides: G[r:, :r] (ld m) and B[r:, kw:] (ld ldB)
          a0.B = L.G[s] + (int64_t)r * m;
          a0.ldB = m;
          a0.kw = 0;
          CluItem b0 = f0;
          b0.B = L.B[s] + (int64_t)r * L.ldB[s] + L.kw[s];
          b0.ldB = L.ldB[s];
          b0.kw = 0;
          for (int rhs = 0; rhs < 2; ++rhs) {
            const int32_t nc_all = rhs == 0 ? r : L.kn[s];
            if (nc_all <= 0) continue;
            fs.push_back(rhs == 0 ? a0 : b0);
            for (int32_t c0 = 0; c0 < nc_all; c0 += tw)
              fst.push_back(TrsmItem{(int32_t)fs.size() - 1, c0, std::min(tw, nc_all - c0), 0});
          }
          for (int32_t c0 = 0; c0 < r + L.kn[s]; c0 += 256)
            cu.push_back(TrsmItem{bi, c0, std::min(256, r + L.kn[s] - c0), 0});
          S.flops += 4.0 * m * m * r + (double)K * K * K / 3.0 + (double)K * K * (r + L.kn[s]) +
                     2.0 * r * K * (r + L.kn[s]);
        }
        upB.reset();
        const size_t kF = upB.add(fine), kS = upB.add(fs), kT = upB.add(fst), kU = upB.add(cu);
        upB.stage.ensure(upB.total);
        upB.dev.ensure(upB.total);
        upB.copy_in(kF, fine); upB.copy_in(kS, fs); upB.copy_in(kT, fst); upB.copy_in(kU, cu);
        upB.send(st);
        launch_rot2(d_clu_batch, nb, max_m, d_rank, st);
        launch_potrf(upB.dptr<CluItem>(kF), (int)fine.size(), fmax, d_status, st);
        launch_trsm(upB.dptr<CluItem>(kS), upB.dptr<TrsmItem>(kT), (int)fst.size(), fmax, st);
        launch_coarse_update(d_clu_batch, upB.dptr<TrsmItem>(kU), (int)cu.size(), d_rank, st);
        check_status(d_status, &h_status, st);   // a fine block that is not SPD (Table 1: "may be indefinite")
      }
      // ---- phase II across GPUs: the batch's ranks, then the elimination records ---------
      std::vector<double*> rbuf(Bt.size(), nullptr);   // received B_s of remote clusters
      if (dist && phase2) {
        std::vector<int32_t> v(Bt.size(), 0);
        for (size_t k = 0; k < Bt.size(); ++k)
          if (own(l, Bt[k])) v[k] = L.rank[Bt[k]];
        allreduce_i32(v);
        for (size_t k = 0; k < Bt.size(); ++k) L.rank[Bt[k]] = v[k];
        comm_group_start(h->comm);
        for (size_t k = 0; k < Bt.size(); ++k) {
          const int32_t s = Bt[k];
          const size_t words = (size_t)live[s] * L.ldB[s];
          if (!words) continue;
          const std::vector<int32_t> rc = receivers(*an, DP, l, s);
          if (own(l, s)) {
            for (int32_t hdst : rc) comm_send_f64(h->comm, L.B[s], words, hdst, st);
          } else if (std::binary_search(rc.begin(), rc.end(), (int32_t)h->rank)) {
            rbuf[k] = (double*)dc.alloc(sizeof(double) * words);
            comm_recv_f64(h->comm, rbuf[k], words, DP.owner[l][s], st);
          }
        }
        comm_group_end(h->comm, st);
      }
      // ---- Schur update, write-back: patch the pre-planned records with the ranks ----------
      // dpatch: the patch items (target = section + index, resolved after the upload layout)
      struct PRef {
        PatchItem it;
        int sec;       // 0 srcs, 1 wb, 2 id_r, 3 ft
        size_t idx;
      };
      std::vector<PRef> prefs;
      if (dpatch) {
        if (nb != (int)Bt.size()) fail(HS_E_INTERNAL, "device patch: batch not fully owned");
        for (auto& pd : pend) {
          const int32_t s = pd.s;
          const double* Bs = L.B[s];
          const int32_t m = live_at[pd.k], kn = L.kn[s], kw = L.kw[s], ldB = L.ldB[s];
          PatchItem base{nullptr, Bs, pd.k, PK_SRC, m, ldB, kw, 0, 0, 0};
          if (pd.src >= 0) {
            srcs[pd.src].C = dwb ? L.C[s] : Bs + kw;
            srcs[pd.src].K = 0;
            PatchItem q = base;
            if (dwb) q.kind = PK_K;
            prefs.push_back({q, 0, (size_t)pd.src});
          }
          for (size_t i = pd.wb_begin; i < pd.wb_end; ++i) {
            CopyItem& c = wb[i];
            c.src = Bs + (uintptr_t)c.src;
            PatchItem q = base;
            q.kind = c.trans ? PK_COLS : PK_ROWS;
            prefs.push_back({q, 1, i});
          }
          if (pd.id >= 0) {
            PatchItem q = base;
            q.kind = PK_I32;
            prefs.push_back({q, 2, (size_t)pd.id});
          }
          if (pd.ft >= 0) {
            PatchItem q = base;
            q.kind = PK_FT;
            prefs.push_back({q, 3, (size_t)pd.ft});
          }
          if (kn > 0 && !dwb) {   // C_s = B_s[r:, kw:] into the batch region (K <= m rows)
            L.C[s] = ctmp + co[pd.k];
            const int32_t step = std::max(1, 16384 / kn);
            for (int32_t i0 = 0; i0 < m; i0 += step) {
              PatchItem q = base;
              q.kind = PK_CCOPY;
              q.i0 = i0;
              q.step = step;
              prefs.push_back({q, 1, wb.size()});
              wb.push_back(CopyItem{Bs + kw, L.C[s] + (int64_t)i0 * kn, ldB, kn, 0, kn, 0, 0});
            }
          }
        }
        pend_cl.clear();
        for (size_t k = 0; k < Bt.size(); ++k) pend_cl.emplace_back(Bt[k], live_at[k]);
        pend_active = nb > 0;
        pend_ctmp = ctmp;
        pend_in_arena = in_arena;
        ctmp = nullptr;
      }
      for (auto& pd : pend) {
        if (dpatch) break;
        const int32_t s = pd.s;
        const double* Bs = pd.mine ? L.B[s] : rbuf[pd.k];
        if (!pd.mine && !Bs) continue;
        const int32_t m = live_at[pd.k], kn = L.kn[s], kw = L.kw[s], ldB = L.ldB[s];
        const int32_t r = L.rank[s];
        const int32_t K = m - r;
        const double* C = Bs + (int64_t)r * ldB + kw;
        if (pd.src >= 0) {
          srcs[pd.src].C = C;
          srcs[pd.src].K = K;
        }
        for (size_t i = pd.wb_begin; i < pd.wb_end; ++i) {   // src holds the column offset
          CopyItem& c = wb[i];
          c.src = Bs + (uintptr_t)c.src;
          if (c.trans) c.cols = r;
          else c.rows = r;
        }
        if (pd.id >= 0) id_r[pd.id] = r;
        if (pd.diag >= 0) {   // dc = 0: the coarse block A_cc - C_c^T C_c
          wb[pd.diag].rows = r;
          wb[pd.diag].cols = r;
        }
        if (pd.ft >= 0) ft[pd.ft].r = r;
        if (pd.mine) {
          S.max_m = std::max(S.max_m, m);
          S.max_rank = std::max(S.max_rank, r);
          if (K > 0 && kn > 0) {
            L.C[s] = cslab.get((int64_t)K * kn);
            wb.push_back(CopyItem{C, L.C[s], ldB, kn, K, kn, 0, 0});
          }
          // algorithmic flops of CPQR (+ rotation of the n-columns) and Schur
          double fq = 0.0;
          for (int j = 0; j < r; ++j) fq += 4.0 * (m - j) * (double)(kw - j) + 4.0 * (m - j) * (double)kn;
          S.flops += fq + (double)K * kn * (kn + 1);
          S.flops_phase[3] += fq;
          S.flops_phase[4] += (double)K * kn * (kn + 1);
        }
      }
      t_sub[1] += now_s() - tp1;
      const double tq3 = now_s();
      for (int32_t q : touched) wave_mask[q] = 0;
      for (size_t k = 0; k < srcs.size(); ++k) srcs[k].pairs = lp.pairs + lp.poff[src_cl[k]];   // the level's pair tables
      auto& tiles = rc.tiles;
      tiles.clear();
      std::vector<int32_t> wave_off(1, 0);
      for (const auto& wv : waves) {
        tiles.insert(tiles.end(), wv.begin(), wv.end());
        wave_off.push_back((int32_t)tiles.size());
      }
      if (!dpatch)
        for (int32_t s : Bt)
          if (own(l, s) || (dist && phase2)) {   // the rank of s is known here
            live[s] = L.rank[s];
            done[s] = 1;
          }
      t_sub[3] += now_s() - tq3;
      const bool second = !srcs.empty() || !wb.empty() || !id_ptr.empty() || !ft.empty();
      if (second) {
        if (!dpatch) split_copies(wb);   // dpatch: item indices are patch targets (C copies pre-split)
        upB.reset();
        auto& patch = rc.patch;
        patch.assign(prefs.size(), PatchItem{});
        const size_t jT = upB.add(tiles), jS = upB.add(srcs), jN = upB.add(nbc), jW = upB.add(wb),
                     jP = upB.add(id_ptr), jL = upB.add(id_ld), jR = upB.add(id_r), jF = upB.add(ft),
                     jX = upB.add(patch);
        upB.stage.ensure(upB.total);
        upB.dev.ensure(upB.total);
        for (size_t i = 0; i < prefs.size(); ++i) {
          PatchItem q = prefs[i].it;
          const size_t x = prefs[i].idx;
          switch (prefs[i].sec) {
            case 0: q.target = upB.dptr<SchurSrc>(jS) + x; break;
            case 1: q.target = upB.dptr<CopyItem>(jW) + x; break;
            case 2: q.target = upB.dptr<int32_t>(jR) + x; break;
            default: q.target = upB.dptr<FormTItem>(jF) + x; break;
          }
          patch[i] = q;
        }
        upB.copy_in(jT, tiles); upB.copy_in(jS, srcs); upB.copy_in(jN, nbc); upB.copy_in(jW, wb);
        upB.copy_in(jP, id_ptr); upB.copy_in(jL, id_ld); upB.copy_in(jR, id_r); upB.copy_in(jF, ft);
        upB.copy_in(jX, patch);
        t_plan += now_s() - tp1;
        const double tl0 = now_s();
        if (first_half_launch) {   // device patch: both uploads, then the whole batch's kernels
          upA.send(st);
          upB.send(st);
          first_half_launch(true);
          first_half_launch = nullptr;
        } else {
          upB.send(st);
        }
        pt.collect_b(S);   // the previous batch's second-half events, before they are re-recorded
        pt.rec(pt.b[0], st);
        launch_patch(upB.dptr<PatchItem>(jX), (int)patch.size(), d_rank, st);
        for (size_t w = 0; w + 1 < wave_off.size(); ++w)
          launch_schur2(upB.dptr<SchurTile2>(jT) + wave_off[w], wave_off[w + 1] - wave_off[w],
                        upB.dptr<SchurSrc>(jS), upB.dptr<NbCol>(jN), bs.dir(), st);
        pt.rec(pt.b[1], st);
        launch_copy2d(upB.dptr<CopyItem>(jW), (int)wb.size(), st);
        launch_identity(upB.dptr<double*>(jP), upB.dptr<int32_t>(jL), upB.dptr<int32_t>(jR), (int)id_ptr.size(), st);
        pt.rec(pt.b[2], st);
        t_launch += now_s() - tl0;
        pt.b_pending = true;
        // apply operators T_s = U^T G^{-1} of the batch on the side stream (they are only
        // read by the apply): reads the workspace's G, V, tau, so the workspace (and the
        // items' own buffer) go back to the cache once the side stream has passed this point
        FormTItem* d_ft = nullptr;
        cudaEvent_t ev_ft = nullptr;
        if (!ft.empty()) {
          d_ft = (FormTItem*)dc.alloc(sizeof(FormTItem) * ft.size());
          // own copy of the items: upB's device buffer is rewritten by the next batch
          HS_CUDA(cudaMemcpyAsync(d_ft, upB.dptr<FormTItem>(jF), sizeof(FormTItem) * ft.size(),
                                  cudaMemcpyDeviceToDevice, st));
          HS_CUDA(cudaEventRecord(h->ev_fork, st));
          HS_CUDA(cudaStreamWaitEvent(h->side, h->ev_fork, 0));
          if (nodc) launch_form_T_nodc(d_ft, (int)ft.size(), ft_max_m, h->side);
          else launch_form_T(d_ft, (int)ft.size(), ft_max_m, h->side);
          ev_ft = deferred.take();
          HS_CUDA(cudaEventRecord(ev_ft, h->side));
        }
        if (f->keep_records) {
          if (ws) L.wchunks.push_back(ws);
          if (d_ft) deferred.push(ev_ft, {d_ft});
          ws = nullptr;
        } else if (ev_ft) {
          deferred.push(ev_ft, {ws, d_ft});
          ws = nullptr;
        }
      } else {
        t_plan += now_s() - tp1;
      }
      if (first_half_launch) {   // no second half (every cluster of the batch empty)
        upA.send(st);
        first_half_launch(true);
        first_half_launch = nullptr;
      }
      for (double* b : rbuf)
        if (b) dc.free(b);
      if (wtmp && !in_arena) dc.free(wtmp);   // the batch's CPQR is queued
      if (ws && !in_arena) {
        if (f->keep_records) L.wchunks.push_back(ws);
        else dc.free(ws);
      }
      if (!f->keep_records)
        for (int32_t s : Bo) L.G[s] = L.V[s] = L.tau[s] = L.nu[s] = L.B[s] = nullptr;
      S.n_batches++;
      if (const char* dd = std::getenv("HS_DEBUG_DUMP")) {   // debug aid: block store after every batch
        HS_CUDA(cudaStreamSynchronize(st));
        char path[512];
        std::snprintf(path, sizeof path, "%s/l%d_b%d.bin", dd, l, (int)bidx);
        FILE* fp = std::fopen(path, "wb");
        if (fp) {
          std::vector<double> host(bs.total);
          if (bs.total) HS_CUDA(cudaMemcpy(host.data(), bs.d, bs.total * sizeof(double), cudaMemcpyDeviceToHost));
          for (int p = 0; p < lev.nclus; ++p)
            for (const auto& qo : bs.rows[p]) {
              const int32_t q = qo.first;
              int32_t hdr[4] = {p, q, live[p], live[q]};
              std::fwrite(hdr, sizeof hdr, 1, fp);
              for (int i = 0; i < live[p]; ++i)
                std::fwrite(host.data() + qo.second + (int64_t)i * cap[q], sizeof(double), live[q], fp);
            }
          std::fclose(fp);
        }
      }
    }
    finish_pending();
    if (lvl_ws) dc.free(lvl_ws);   // stream-ordered: the level's kernels are queued
    if (f->rec.active()) {   // the level's records are complete (spillable)
      f->rec.pin_lo = f->rec.pin_hi = 0;
      f->rec.level_start();
      f->rec.precopy(h->side);
      if (rec_force) f->rec.spill(~size_t(0));
    }
    // ---- every rank learns every kept rank; the records go to rank 0 (dist) -----------------
    const double tp2 = now_s();
    if (dist) {
      std::vector<uint8_t> all(lev.nclus, 1);
      sync_ranks(all);
      // shapes at elimination of every cluster, now that every rank is known: during phase I
      // a remote interior cluster's neighbours' ranks were not known here
      std::vector<int32_t> lv2 = cap;
      for (const auto& Bt : lev.batches) {
        for (int32_t s : Bt) {
          int32_t kn = 0, kw = 0;
          for (int32_t q : lev.H[s]) kn += lv2[q];
          for (int32_t q : lev.w[s]) kw += lv2[q];
          L.kn[s] = kn; L.kw[s] = kw; L.ldB[s] = kn + kw; L.ldc[s] = kn;
        }
        for (int32_t s : Bt) lv2[s] = L.rank[s];
      }
      // the records (T_s, C_s) stay at their owners: the distributed solve (dsolve.cu)
      // applies them there; T_s is formed on the side stream, joined below
    }
    // ---- apply plan of the level (Algorithm 2), replayed in elimination order ---------------
    const int nP = lev.nclus / 2;
    std::vector<int32_t> capn(nP);
    for (int P = 0; P < nP; ++P) capn[P] = L.rank[2 * P] + L.rank[2 * P + 1];
    if (plan_apply) {
      // The apply plan of level l only reads this level's records: single GPU, it is built
      // on a host worker (chained after the previous level's) while the next level factors.
      auto plan_task = [l, &lev = lev, &L = L, &ap, capc = cap, capn, level_dofs, vb0 = ap.vbase[l], vbn0 = vbase,
                        nP, &t_apply_plan, su = &an->l0s, dsup = d_sup]() {
        ApplyLevelPlan& AP = ap.lv[l];
        AP.cinv.clear();
        AP.src.assign(lev.nclus, ApplySrc{});
        std::vector<int32_t> fev(lev.nclus, 0), lv2 = capc;
        std::vector<uint8_t> proc(lev.nclus, 0);
        std::vector<std::vector<PullSrc>> pre(lev.nclus), post(lev.nclus);
        int64_t slots = 0;   // contribution slots of the level
        std::vector<std::vector<BwdTask>> bwd_batches;
        std::vector<int64_t> foff(lev.nclus, 0);
        const double ta = now_s();
        std::vector<int32_t> bpos(lev.nclus, 0);   // batch index of each cluster
        for (size_t b = 0; b < lev.batches.size(); ++b)
          for (int32_t c : lev.batches[b]) bpos[c] = (int32_t)b;
        for (const auto& Bt : lev.batches) {
          if (level_dofs == 0) break;
          bwd_batches.emplace_back();
          std::vector<BwdTask>& bwd_tasks = bwd_batches.back();
          for (int32_t s : Bt) {
            const int32_t m = lv2[s], r = L.rank[s], K = m - r, kn = L.ldc[s];
            if (m == 0) continue;
            const auto& ns = lev.H[s];
            // q's columns of C_s: its live width, or (support-restricted level) the supported
            // columns of a neighbour not yet eliminated (su.idx: host inverse maps / device gathers)
            std::vector<int32_t> cw(ns.size()), noff(ns.size() + 1, 0);
            std::vector<int64_t> sx(ns.size(), -1);
            // (a cluster of a batch too large for the fused path keeps a dense record)
            const bool kh = L.khat && kn != L.kn[s];
            int64_t e = kh ? su->sptr[s] : 0, x = kh ? su->iptr[s] : 0;
            if (kh)
              for (size_t b = 0; b < lev.w[s].size(); ++b) {
                const int32_t ln = su->len[e++];
                if (ln > 0) x += ln;
              }
            for (size_t a = 0; a < ns.size(); ++a) {
              const int32_t ln = kh ? su->len[e++] : -1;
              cw[a] = ln >= 0 ? ln : lv2[ns[a]];
              if (ln >= 0) sx[a] = x;
              if (ln > 0) x += ln;
              noff[a + 1] = noff[a] + cw[a];
            }
            if (noff[ns.size()] != kn) fail(HS_E_INTERNAL, "apply plan: record width");
            // the cluster's record, its forward target tasks (targets grouped up to FWD_COLS
            // columns) and its backward column chunks
            ApplySrc& as = AP.src[s];
            as.T = L.T[s]; as.C = L.C[s]; as.ldC = kn; as.m = m; as.r = r; as.kn = kn;
            as.pre = fev[s]++;
            as.nb_begin = (int32_t)AP.bnb.size();
            // forward (pull form): s contributes to the unprocessed neighbours before their own
            // elimination (their pre lists) and to the coarse parts of the processed ones
            // afterwards (post lists); lists grow in elimination order
            as.tg_begin = (int32_t)AP.ctb.size();
            for (size_t a = 0; a < ns.size(); ++a) {
              const int32_t q = ns[a];
              if (lv2[q] == 0 || K == 0) continue;
              (proc[q] ? post[q] : pre[q]).push_back(PullSrc{slots, s, 0});
              const int32_t* inv = nullptr;   // (offset + 1 into AP.cinv until the upload)
              if (sx[a] >= 0) {
                const size_t base = AP.cinv.size();
                AP.cinv.resize(base + lv2[q], -1);
                for (int32_t j = 0; j < cw[a]; ++j) AP.cinv[base + su->idx[sx[a] + j]] = j;
                inv = (const int32_t*)(uintptr_t)(base + 1);
              }
              AP.ctb.push_back(Contrib{slots, noff[a], cw[a], q, proc[q] ? 0 : 1, lv2[q], 0, inv});
              slots += lv2[q];
              AP.bnb.push_back(BwdNb{nullptr, q, noff[a], cw[a], proc[q] ? 0 : 1, 0, 0,
                                     sx[a] >= 0 ? dsup + sx[a] : nullptr});
            }
            as.tg_end = (int32_t)AP.ctb.size();
            as.nb_end = (int32_t)AP.bnb.size();
            // produce order: the targets eliminated soonest first (T(s) produces the first
            // group itself, so the next cluster on the chain waits for one task, not two);
            // the order in which a target subtracts its contributions is its pre list's
            std::stable_sort(AP.ctb.begin() + as.tg_begin, AP.ctb.begin() + as.tg_end,
                             [&](const Contrib& x, const Contrib& y) {
                               const int32_t bx = x.pre ? bpos[x.q] : INT32_MAX, by = y.pre ? bpos[y.q] : INT32_MAX;
                               return bx < by;
                             });
            // T(s) with s's first contribution group, then the other groups (<= FWD_COLS
            // columns / 16 targets each) as tasks of their own
            if (as.tg_begin == as.tg_end) AP.ftask.push_back(FwdTask{s, as.tg_begin, as.tg_end, 1});
            for (int32_t g0 = as.tg_begin, first = 1; g0 < as.tg_end; first = 0) {
              int32_t g1 = g0, cols = 0;
              while (g1 < as.tg_end && (g1 == g0 || (cols + AP.ctb[g1].len <= FWD_COLS && g1 - g0 < 16)))
                cols += AP.ctb[g1++].len;
              AP.ftask.push_back(FwdTask{s, g0, g1, first});
              g0 = g1;
            }
            as.part = AP.parts;
            if (K > 0 && kn > 0 && as.nb_end > as.nb_begin) {
              // backward chunks by readiness: neighbours eliminated before s (final at the
              // level start), then the later ones latest-eliminated first (they finish first
              // in the reverse sweep); the last BWD_CRIT later neighbours — the critical path
              // of the sweep — get a chunk of their own, the rest are packed to BWD_COLS
              std::stable_sort(AP.bnb.begin() + as.nb_begin, AP.bnb.begin() + as.nb_end,
                               [&](const BwdNb& x, const BwdNb& y) {
                                 const int32_t kx = x.later ? INT32_MAX - bpos[x.q] : -1;
                                 const int32_t ky = y.later ? INT32_MAX - bpos[y.q] : -1;
                                 return kx < ky;
                               });
              int32_t nlater = 0;
              for (int32_t b = as.nb_begin; b < as.nb_end; ++b) nlater += AP.bnb[b].later;
              const int32_t crit0 = as.nb_end - std::min<int32_t>(nlater, BWD_CRIT);
              as.nchunk = 0;
              for (int32_t b0 = as.nb_begin; b0 < as.nb_end;) {
                int32_t b1 = b0, cols = 0;
                while (b1 < as.nb_end && (b1 == b0 || (b1 < crit0 && b0 < crit0 && cols + AP.bnb[b1].len <= BWD_COLS))) {
                  AP.bnb[b1].off = cols;
                  cols += AP.bnb[b1++].len;
                }
                bwd_tasks.push_back(BwdTask{s, b0, b1, cols, as.nchunk++, 0});
                b0 = b1;
              }
              AP.parts += (int64_t)as.nchunk * K;
            } else {
              as.nchunk = 1;
              bwd_tasks.push_back(BwdTask{s, 0, 0, 0, 0, 0});
            }
            foff[s] = ap.ftotal;
            ap.ftotal += K;
          }
          for (int32_t s : Bt) {
            lv2[s] = L.rank[s];
            proc[s] = 1;
          }
        }
        // vector positions (offsets into d_y / d_yf, made absolute at the end).  A cluster's
        // live segment is its level segment until it is eliminated, then its coarse rows
        // inside the parent's segment [coarse(2P); coarse(2P+1)].
        std::vector<int64_t> voffn(nP + 1, 0);
        for (int P = 0; P < nP; ++P) voffn[P + 1] = voffn[P] + capn[P];
        const int64_t vb = vb0, vbn = vbn0;   // this level's and the next level's vector bases
        auto lpos = [&](int32_t c) { return (double*)(uintptr_t)(vb + L.voff[c]); };
        auto ppos = [&](int32_t c) {
          return (double*)(uintptr_t)(vbn + voffn[c >> 1] + ((c & 1) ? L.rank[c - 1] : 0));
        };
        for (int32_t c = 0; c < lev.nclus; ++c) {
          ApplySrc& as = AP.src[c];
          if (as.m == 0) continue;
          as.y = lpos(c);
          as.x = lpos(c);
          as.yc = ppos(c);
          as.yf = (double*)(uintptr_t)foff[c];
        }
        for (auto& t : AP.ftgt) t.y = t.proc ? ppos(t.q) : lpos(t.q);
        for (auto& nbr : AP.bnb) nbr.x = (double*)(nbr.later ? lpos(nbr.q) : ppos(nbr.q));
        for (auto it = bwd_batches.rbegin(); it != bwd_batches.rend(); ++it)
          AP.btask.insert(AP.btask.end(), it->begin(), it->end());
        AP.contrib_off = ap.contrib_total;
        ap.contrib_total += slots;
        for (int32_t c = 0; c < lev.nclus; ++c) {
          ApplySrc& as = AP.src[c];
          as.pre_begin = (int32_t)AP.pull.size();
          AP.pull.insert(AP.pull.end(), pre[c].begin(), pre[c].end());
          as.pre_end = (int32_t)AP.pull.size();
          as.post_begin = (int32_t)AP.pull.size();
          AP.pull.insert(AP.pull.end(), post[c].begin(), post[c].end());
          as.post_end = (int32_t)AP.pull.size();
          if (!post[c].empty() && as.m > 0) AP.post_cl.push_back(c);
        }
        AP.ctr_off = ap.ctr_total;
        ap.ctr_total += 4 * (int64_t)lev.nclus + 2;
        ap.max_parts = std::max(ap.max_parts, AP.parts);
        // batch-synchronous sweeps (one launch per batch) where the batches are large: the
        // clusters of every batch, in order
        {
          int64_t nonempty = 0;
          bool fits = !lev.batches.empty();
          for (int32_t c = 0; c < lev.nclus; ++c) {
            const ApplySrc& as = AP.src[c];
            if (as.m == 0) continue;
            ++nonempty;
            fits = fits && as.tg_end - as.tg_begin <= BS_MAXG && as.kn <= BS_MAXCOLS;
          }
          AP.bsync = fits && nonempty >= 128 * (int64_t)lev.batches.size() && std::getenv("HS_APPLY_DEP") == nullptr;
          AP.bcl.clear();
          AP.boff.assign(1, 0);
          if (AP.bsync)
            for (const auto& Bt : lev.batches) {
              for (int32_t c : Bt)
                if (AP.src[c].m > 0) AP.bcl.push_back(c);
              AP.boff.push_back((int32_t)AP.bcl.size());
            }
        }
        t_apply_plan += now_s() - ta;
      };
      if (dist) {
        plan_task();
      } else {
        plan_prev = std::async(std::launch::async, [task = std::move(plan_task), prev = std::move(plan_prev)]() mutable {
          if (prev.valid()) prev.get();
          task();
        });
      }
    }
    // ---- end of level: A_c = parents of [coarse(2P); coarse(2P+1)] -----------------
    // The parent store is mapped group by group of parent rows while the consumed child rows'
    // chunks are unmapped: the two stores never coexist in full.
    const Adj& En = (l + 1 < an->L_top) ? an->levels[l + 1].Ffinal : an->H_top;
    BlockStore nbs;
    nbs.reserve(capn, En, st, &dc, &h->vmm, dist ? &DP : nullptr, l + 1);
    t_tr[0] += now_s() - tp2;
    // every stored child block (c >= d) lands in parent block (c/2, d/2) at offset
    // (c odd ? r(2P) : 0, d odd ? r(2Q) : 0); the upper child pair of a parent diagonal
    // block never occurs (c >= d), matching its lower-triangle semantics.  A rank holds
    // every child block of the parent blocks it holds (same owners).
    const int64_t group_words = std::max<int64_t>((int64_t)(2ull << 30) / 8, (int64_t)nbs.total / 16);
    pt.rec(pt.a[0], st);
    for (int32_t Pa = 0; Pa < nP;) {
      int32_t Pb = Pa + 1;
      while (Pb < nP && nbs.rowbeg[Pb + 1] - nbs.rowbeg[Pa] <= group_words) ++Pb;
      double ta = now_s();
      nbs.map_bytes((size_t)nbs.rowbeg[Pa] * sizeof(double), (size_t)nbs.rowbeg[Pb] * sizeof(double));
      t_as[0] += now_s() - ta;
      ta = now_s();
      std::vector<CopyItem> asmb;
      for (int32_t c = 2 * Pa; c < std::min(2 * Pb, lev.nclus); ++c) {
        if (L.rank[c] == 0) continue;
        const int32_t P = c >> 1;
        const auto& prow = nbs.rows[P];
        size_t pi = 0;
        for (const auto& dof : bs.rows[c]) {
          const int32_t d = dof.first;
          if (L.rank[d] == 0) continue;
          const int32_t Q = d >> 1;
          while (pi < prow.size() && prow[pi].first < Q) ++pi;   // d ascending -> Q ascending
          if (pi == prow.size() || prow[pi].first != Q) {
            if (dist) continue;   // a parent block this rank does not hold
            fail(HS_E_INTERNAL, "assembly: parent block missing");
          }
          const int32_t dld = capn[Q];
          const int32_t ro = (c & 1) ? L.rank[2 * P] : 0, co = (d & 1) ? L.rank[2 * Q] : 0;
          asmb.push_back(CopyItem{bs.d + dof.second, nbs.d + prow[pi].second + (int64_t)ro * dld + co, cap[d], dld,
                                  L.rank[c], L.rank[d], 0, 0});
        }
      }
      split_copies(asmb);
      t_as[1] += now_s() - ta;
      ta = now_s();
      upA.reset();
      const size_t iA = upA.add(asmb);
      upA.stage.ensure(upA.total);
      upA.dev.ensure(upA.total);
      upA.copy_in(iA, asmb);
      upA.send(st);
      launch_copy2d(upA.dptr<CopyItem>(iA), (int)asmb.size(), st);
      t_as[2] += now_s() - ta;
      if (bs.pool || Pb < nP) {   // VMM-backed: the consumed child rows can go (a group's staging is reused)
        ta = now_s();
        HS_CUDA(cudaStreamSynchronize(st));
        t_as[3] += now_s() - ta;
        ta = now_s();
        bs.unmap_below((size_t)bs.rowbeg[std::min(2 * Pb, lev.nclus)] * sizeof(double));
        t_as[4] += now_s() - ta;
      }
      Pa = Pb;
    }
    pt.rec(pt.a[1], st);
    t_plan += now_s() - tp2;
    t_trans += now_s() - tp2;
    // the child store goes back to the stream-ordered cache without a host sync (cache-backed);
    // a VMM-backed one is unmapped after the stream has drained
    if (pt.on || bs.pool) HS_CUDA(cudaStreamSynchronize(st));
    pt.collect_b(S);
    if (pt.on) S.t_phase_s[5] += PhaseTimer::el(pt.a[0], pt.a[1]);
    const double tr1 = now_s();
    bs.release();
    bs = std::move(nbs);
    nbs.forget();
    t_tr[3] += now_s() - tr1;
    if (l + 1 < an->L_top) bs.upload_dir(h->dirstage);
    t_tr[1] += now_s() - tr1;
    cap = capn;
    if (prof) {
      int64_t sm = 0, sr = 0, skn = 0, skw = 0, mx = 0;
      for (int s = 0; s < lev.nclus; ++s) {
        sm += L.cap[s]; sr += L.rank[s]; skn += L.kn[s]; skw += L.kw[s];
        mx = std::max<int64_t>(mx, L.kn[s] + L.kw[s]);
      }
      std::fprintf(stderr,
                   "[hs profile] level %d: %d clusters %zu batches wall %.1f ms plan %.1f ms | gather %.1f potrf %.1f "
                   "trsm %.1f cpqr %.1f schur %.1f wb %.1f ms | sum m %lld r %lld kn %lld kw %lld max ldB %lld | "
                   "cache in use %.1f GB (peak %.1f), store chunks %.1f GB\n",
                   l, lev.nclus, lev.batches.size(), 1e3 * (now_s() - lv_t0), 1e3 * (t_plan - lv_plan0),
                   1e3 * (S.t_phase_s[0] - lv_ph0[0]), 1e3 * (S.t_phase_s[1] - lv_ph0[1]),
                   1e3 * (S.t_phase_s[2] - lv_ph0[2]), 1e3 * (S.t_phase_s[3] - lv_ph0[3]),
                   1e3 * (S.t_phase_s[4] - lv_ph0[4]), 1e3 * (S.t_phase_s[5] - lv_ph0[5]), (long long)sm,
                   (long long)sr, (long long)skn, (long long)skw, (long long)mx, dc.in_use / 1e9, dc.peak / 1e9,
                   h->vmm.created * (double)h->vmm.chunk / 1e9);
    }
  }
  HS_CUDA(cudaEventRecord(lev_ev[an->L_top], st));
  lev_flops[an->L_top] = S.flops;
  tl.push_back({"levels", now_s()});
  // ---- top: dense Cholesky of all live DOFs, on rank 0 -------------------------
  {
    const int ntc = (int)cap.size();
    std::vector<int64_t> toff(ntc + 1, 0);
    for (int c = 0; c < ntc; ++c) toff[c + 1] = toff[c] + cap[c];
    const int64_t N = toff[ntc];
    f->ntop = N;
    f->top_sizes = cap;
    S.n_top = N;
    ap.vbase.push_back(vbase);
    vbase += N;
    const int Ltop = an->L_top;
    // the top blocks (P, Q) held by rank g with g owning P, in store order
    auto top_blocks = [&](int g) {
      std::vector<std::pair<int32_t, int32_t>> v;
      for (int P = 0; P < ntc; ++P) {
        if (dist && Ltop > 0 && DP.owner[Ltop][P] != g) continue;
        for (int32_t Q : an->H_top[P])
          if (Q < P) v.push_back({P, Q});
        v.push_back({P, P});
      }
      return v;
    };
    std::vector<std::pair<const double*, std::pair<int32_t, int32_t>>> src;   // rank 0: block data
    std::vector<double*> tbufs;
    if (N > 0 && dist && Ltop > 0) {
      if (h->rank != 0) {
        comm_group_start(h->comm);
        for (auto pq : top_blocks(h->rank)) {
          double* p; int32_t ld, tr;
          if (!bs.has(pq.first, pq.second)) continue;
          bs.get(pq.first, pq.second, p, ld, tr);
          comm_send_f64(h->comm, p, (size_t)cap[pq.first] * cap[pq.second], 0, st);
        }
        comm_group_end(h->comm, st);
        HS_CUDA(cudaStreamSynchronize(st));
      } else {
        comm_group_start(h->comm);
        for (int g = 1; g < h->world; ++g)
          for (auto pq : top_blocks(g)) {
            // rank g stores (P, Q) iff it holds it: it owns P here, and the block exists in H_top
            const size_t words = (size_t)cap[pq.first] * cap[pq.second];
            double* b = words ? (double*)dc.alloc(sizeof(double) * words) : nullptr;
            tbufs.push_back(b);
            comm_recv_f64(h->comm, b, words, g, st);
            src.push_back({b, pq});
          }
        comm_group_end(h->comm, st);
      }
    }
    if (N > 0 && (!dist || h->rank == 0)) {   // the top is factored on rank 0
      f->d_top = (double*)dc.alloc(sizeof(double) * N * N);
      HS_CUDA(cudaMemsetAsync(f->d_top, 0, sizeof(double) * N * N, st));
      for (int P = 0; P < ntc; ++P)
        for (const auto& qo : bs.rows[P])
          if (!dist || Ltop == 0 || DP.owner[Ltop][P] == 0) src.push_back({bs.d + qo.second, {P, qo.first}});
      std::vector<CopyItem> items;
      for (const auto& e : src) {
        const int32_t P = e.second.first, Q = e.second.second;
        if (cap[P] == 0 || cap[Q] == 0 || !e.first) continue;
        // diagonal blocks hold the lower triangle only: symmetrise them into A_top
        items.push_back(CopyItem{e.first, f->d_top + toff[P] * N + toff[Q], cap[Q], (int32_t)N, cap[P], cap[Q],
                                 P == Q ? 2 : 0, 0});
        if (P != Q)
          items.push_back(CopyItem{e.first, f->d_top + toff[Q] * N + toff[P], cap[Q], (int32_t)N, cap[Q], cap[P], 1, 0});
      }
      split_copies(items);
      upA.reset();
      const size_t iA = upA.add(items);
      upA.stage.ensure(upA.total);
      upA.dev.ensure(upA.total);
      upA.copy_in(iA, items);
      upA.send(st);
      launch_copy2d(upA.dptr<CopyItem>(iA), (int)items.size(), st);
      pt.rec(pt.a[0], st);
      dense_potrf(f->d_top, (int)N, (int)N, d_status, an->L_top, nullptr, st);
      pt.rec(pt.a[1], st);
      check_status(d_status, &h_status, st);
      if (pt.on) S.t_phase_s[6] += PhaseTimer::el(pt.a[0], pt.a[1]);
      S.flops += (double)N * N * N / 3.0;
      S.flops_phase[6] += (double)N * N * N / 3.0;
    }
    HS_CUDA(cudaStreamSynchronize(st));
    for (double* b : tbufs)
      if (b) dc.free(b);
    bs.release();
  }
  if (f->rec.active()) {   // the spilled records come back to the device (same addresses)
    f->rec.restore();
    h->vmm.rec = nullptr;
    if (prof || f->rec.n_spilled)
      std::fprintf(stderr, "[hs profile] record space: %.2f GB of records, %.2f GB spilled to the host in %.2f s "
                   "(%.2f GB of them pre-copied during earlier levels; %.2f GB pre-copied), %.2f GB restored in %.2f s\n",
                   f->rec.top / 1e9, f->rec.bytes_spilled / 1e9, f->rec.t_spill, f->rec.pre_used / 1e9,
                   f->rec.pre_bytes / 1e9, f->rec.bytes_restored / 1e9, f->rec.t_restore);
  }
  HS_CUDA(cudaEventRecord(h->ev_join, h->side));   // join the side stream (apply operators)
  HS_CUDA(cudaStreamWaitEvent(st, h->ev_join, 0));
  deferred.drain(true);
  HS_CUDA(cudaEventRecord(ev1, st));
  HS_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  HS_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  S.t_factor_s = ms * 1e-3;
  for (int l = 0; l < an->L_top && l < 32; ++l) {
    float lms = 0.f;
    HS_CUDA(cudaEventElapsedTime(&lms, lev_ev[l], lev_ev[l + 1]));
    S.t_level_s[l] = lms * 1e-3;
    S.flops_level[l] = lev_flops[l + 1] - lev_flops[l];
  }
  S.t_phase_s[7] = t_plan;
  if (std::getenv("HS_PROFILE"))
    std::fprintf(stderr, "[hs profile] host planning %.1f ms: schur+gather-side %.1f, write-back %.1f, apply %.1f, batch tail %.1f, level transitions %.1f\n",
                 1e3 * t_plan, 1e3 * t_sub[0], 1e3 * t_sub[1], 1e3 * t_sub[2], 1e3 * t_sub[3], 1e3 * t_trans);
  if (std::getenv("HS_PROFILE"))
    std::fprintf(stderr, "[hs profile] first-half planning: shapes + column maps %.1f ms, items %.1f ms (workspace %.1f, "
                 "%d threads %.1f), upload staging %.1f ms\n", 1e3 * t_fh[0], 1e3 * t_fh[1], 1e3 * t_fh[3],
                 plan_threads(1 << 20), 1e3 * t_fh[4], 1e3 * t_fh[2]);
  if (std::getenv("HS_PROFILE") || std::getenv("HS_RANK_WAIT"))
    std::fprintf(stderr, "[hs profile] host blocked on batch ranks: %.1f ms of %.1f ms; issuing uploads + kernels %.1f ms\n",
                 1e3 * t_rank_wait, ms, 1e3 * t_launch);
  if (std::getenv("HS_PROFILE"))
    std::fprintf(stderr, "[hs profile] device cache: in use %.2f GB, peak %.2f GB, cached %.2f GB\n", dc.in_use / 1e9,
                 dc.peak / 1e9, dc.cached / 1e9);
  if (std::getenv("HS_PROFILE"))
    std::fprintf(stderr, "[hs profile] level transitions: block store build %.1f ms, release+upload_dir (sync) %.1f ms "
                 "(release %.1f), arena alloc %.1f ms; assembly: map %.1f, items %.1f, upload+launch %.1f, "
                 "sync %.1f, unmap %.1f ms\n", 1e3 * t_tr[0], 1e3 * t_tr[1], 1e3 * t_tr[3], 1e3 * t_tr[2],
                 1e3 * t_as[0], 1e3 * t_as[1], 1e3 * t_as[2], 1e3 * t_as[3], 1e3 * t_as[4]);
  if (std::getenv("HS_PROFILE")) {
    std::fprintf(stderr, "[hs profile] VMM calls so far (chunk %.0f MB): take %.1f ms (%lld), map %.1f ms (%lld), "
                 "access %.1f ms (%lld runs), unmap %.1f ms (%lld)\n", h->vmm.chunk / 1048576.0, 1e3 * g_vmm_t[0],
                 g_vmm_n[0], 1e3 * g_vmm_t[1], g_vmm_n[1], 1e3 * g_vmm_t[2], g_vmm_n[2], 1e3 * g_vmm_t[3], g_vmm_n[3]);
    for (int i = 0; i < 4; ++i) g_vmm_t[i] = 0, g_vmm_n[i] = 0;
  }
  S.n_levels = an->L_top;
  // factor bytes read by the apply: T_s (m^2) and C_s ((m - r) kn) per cluster + top (N^2/2)
  double fb = 0.0;
  for (const auto& L : f->lv)
    for (int s = 0; s < L.nclus; ++s) {
      const double m = L.cap[s], r = L.rank[s];
      fb += 8.0 * (m * m + (m - r) * L.ldc[s]);
    }
  fb += 8.0 * (double)f->ntop * (f->ntop + 1) / 2;
  S.factor_bytes = fb;
  tl.push_back({"top + join", now_s()});
  // ---- device apply plan ----------------------------------------------------------------
  ap.vtotal = vbase;
  const double tj0 = now_s();
  if (plan_prev.valid()) plan_prev.get();   // every level's apply plan (rethrows a failure)
  if (std::getenv("HS_PROFILE"))
    std::fprintf(stderr, "[hs profile] apply planning on the host worker %.1f ms (main thread waited %.1f ms)\n",
                 1e3 * t_apply_plan, 1e3 * (now_s() - tj0));
  ap.d_y = (double*)dc.alloc(sizeof(double) * std::max<int64_t>(vbase, 1));
  ap.d_yf = (double*)dc.alloc(sizeof(double) * std::max<int64_t>(ap.ftotal, 1));
  ap.d_xb = (double*)dc.alloc(sizeof(double) * std::max<int64_t>(vbase, 1));
  ap.d_parts = (double*)dc.alloc(sizeof(double) * std::max<int64_t>(ap.max_parts, 1));
  ap.d_contrib = (double*)dc.alloc(sizeof(double) * std::max<int64_t>(ap.contrib_total, 1));
  ap.d_ctr = (int32_t*)dc.alloc(sizeof(int32_t) * std::max<int64_t>(ap.ctr_total, 1));
  auto up = [&](auto& vec, auto*& dptr) {
    using T = typename std::remove_reference<decltype(vec)>::type::value_type;
    if (vec.empty()) return;
    dptr = (T*)dc.alloc(sizeof(T) * vec.size());
    HS_CUDA(cudaMemcpyAsync(dptr, vec.data(), sizeof(T) * vec.size(), cudaMemcpyHostToDevice, st));
  };
  for (int l = 0; l < an->L_top; ++l) {   // offsets (stored as integers) -> absolute addresses
    ApplyLevelPlan& AP = ap.lv[l];
    for (auto& as : AP.src) {
      if (as.m == 0) continue;
      as.y = ap.d_y + (uintptr_t)as.y;
      as.x = ap.d_xb + (uintptr_t)as.x;
      as.xc = ap.d_xb + (uintptr_t)as.yc;
      as.yc = ap.d_y + (uintptr_t)as.yc;
      as.yf = ap.d_yf + (uintptr_t)as.yf;
    }
    for (auto& t : AP.ftgt) t.y = ap.d_y + (uintptr_t)t.y;
    for (auto& nbr : AP.bnb) nbr.x = ap.d_xb + (uintptr_t)nbr.x;
    up(AP.cinv, AP.d_cinv);
    for (auto& c : AP.ctb)
      if (c.inv) c.inv = AP.d_cinv + ((uintptr_t)c.inv - 1);
    up(AP.src, AP.d_src);
    up(AP.ftask, AP.d_ftask);
    up(AP.ftgt, AP.d_ftgt);
    up(AP.btask, AP.d_btask);
    up(AP.bnb, AP.d_bnb);
    up(AP.pull, AP.d_pull);
    up(AP.ctb, AP.d_ctb);
    up(AP.post_cl, AP.d_post_cl);
    up(AP.bcl, AP.d_bcl);
  }
  HS_CUDA(cudaStreamSynchronize(st));
  if (dist) dist_solve_build(f, DP);
  tl.push_back({"apply plan upload", now_s()});
  if (prof) {
    std::fprintf(stderr, "[hs profile] host timeline:");
    for (size_t i = 1; i < tl.size(); ++i) std::fprintf(stderr, " %s %.1f ms |", tl[i].first, 1e3 * (tl[i].second - tl[i - 1].second));
    std::fprintf(stderr, "\n");
  }
  return guard.release();
}

}  // namespace hs
