// Host runtime structures of libhsolve (handle, factor, apply plan).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <utility>
#include <string>
#include <unordered_map>
#include <vector>

#include "device.h"
#include "internal.h"


struct hs_analysis_s {
  hs::Analysis* an = nullptr;
};

namespace hs {

// Physical memory for the level block stores (CUDA virtual memory management).  A store
// reserves one contiguous virtual range (its kernels address blocks by offset from the
// base) and maps fixed-size physical chunks into it; the level transition maps the parent
// store chunk by chunk while it unmaps the consumed child chunks, so the two stores never
// coexist in full (C4: the level-0 store alone is ~90 GB).  Unmapped chunks are kept idle
// for the next store / factor and go back to the driver on OOM and at hs_destroy.
struct VmmPool {
  int device = -1;
  size_t chunk = 0;                      // bytes per physical chunk (granularity multiple)
  std::vector<unsigned long long> idle;  // CUmemGenericAllocationHandle
  size_t created = 0;                    // chunks alive (mapped or idle)
  struct DevCache* dc = nullptr;         // trimmed before retrying an allocation that failed
  struct RecSpace* rec = nullptr;        // the running factor's records: spilled to the host on OOM
  std::vector<char*> host_idle;          // pinned host chunks (spilled records), kept for the next factor
  size_t last_spilled = 0;               // bytes the previous factor on this handle spilled (pre-copy budget)
  void init(int dev);
  unsigned long long take();
  void give(unsigned long long h) { idle.push_back(h); }
  char* take_host();
  void give_host(char* p) { host_idle.push_back(p); }
  void trim();                           // release the idle chunks
  ~VmmPool();
};

// Persistent factor records (the T_s arenas and the C_s slabs of every level) of a large
// factor, in one virtual range backed by VmmPool chunks.  The records of completed levels
// are read only by the apply, after the factorization; when a block store or workspace does
// not fit beside them (C4 on one GPU: ~100 GB of records next to a ~100 GB level store), the
// oldest completed chunks are copied to pinned host memory and their physical memory goes to
// the pool.  After the last store is released every spilled chunk is mapped again at the
// SAME virtual address and copied back, so every record pointer (apply plan, exports) stays
// valid and the apply reads device memory only.
struct RecSpace {
  VmmPool* pool = nullptr;
  unsigned long long base = 0;
  size_t vbytes = 0, top = 0;
  size_t frontier = 0;                    // records below this byte offset are complete
  size_t pin_lo = 0, pin_hi = 0;          // except this range (the running level's T_s arena)
  std::vector<unsigned long long> handle; // physical chunk mapped at chunk i (0: none)
  std::vector<char*> host;                // pinned copy of a spilled chunk
  // pre-copies: completed chunks copied to pinned host memory on a copy stream while later
  // levels compute, so a spill of a pre-copied chunk is an event wait and an unmap (no device
  // synchronisation, no copy on the critical path); budget = what the previous factor spilled
  std::vector<char*> pre;                 // pinned copy in flight / done (valid once pre_ev[i] completed)
  std::vector<cudaEvent_t> pre_ev;
  cudaStream_t cst = nullptr;             // copy stream of the pre-copies
  size_t pre_bytes = 0, pre_used = 0, pre_budget = 0;
  cudaStream_t st = nullptr;
  size_t n_spilled = 0, bytes_spilled = 0, bytes_restored = 0;
  double t_spill = 0.0, t_restore = 0.0;
  void init(VmmPool* p, size_t reserve_bytes, cudaStream_t stream);
  void* alloc(size_t bytes);
  void level_start();                     // a level begins: everything allocated so far is complete
  size_t spill(size_t bytes);             // >= bytes of completed records to the host (syncs the device)
  void restore();                         // map and copy back every spilled chunk (stream-ordered)
  void precopy(cudaStream_t side);        // level end: pre-copy completed chunks up to the budget
  void release();
  bool active() const { return base != 0; }
  ~RecSpace() { release(); }
};
unsigned long long vmm_reserve(size_t bytes);                          // virtual range
void vmm_free_range(unsigned long long base, size_t bytes);
void vmm_map(unsigned long long va, unsigned long long handle, size_t bytes, int device);
void vmm_unmap(unsigned long long va, size_t bytes);

// Per-handle caching device allocator.  Every factor / apply / PCG buffer comes from here and
// goes back here: blocks are binned by size class (<= 25% rounding) and reused in host
// order.  All users of a handle's memory run on the handle's stream (the side stream is
// joined before a factor is returned), so reuse in host order is stream-ordered reuse.
// Memory goes back to the driver only on OOM (retry after a trim) and at hs_destroy;
// steady-state re-factoring therefore makes no driver allocation calls at all.
struct DevCache {
  std::map<size_t, std::vector<void*>> bins;
  std::unordered_map<void*, size_t> live;
  size_t cached = 0, in_use = 0, peak = 0;
  static size_t size_class(size_t b) {
    if (b <= 4096) return 4096;
    int k = 63 - __builtin_clzll((unsigned long long)b);   // 2^k <= b < 2^(k+1)
    const size_t q = size_t(1) << (k - 2);                  // quarter steps
    return (b + q - 1) / q * q;
  }
  void* alloc(size_t bytes);
  void free(void* p);
  void trim();        // return every cached block (and idle VMM chunk) to the driver (synchronises the device)
  VmmPool* vmm = nullptr;
  ~DevCache() {       // the handle is going away: also blocks leaked by a failed call
    trim();
    for (auto& kv : live) cudaFree(kv.first);
    live.clear();
  }
};

// device buffer that grows on demand (used for per-launch descriptor uploads)
struct DevScratch {
  char* d = nullptr;
  size_t cap = 0;
  DevCache* dc = nullptr;
  void ensure(size_t bytes);
  ~DevScratch();
};

// pinned host staging buffer
struct HostStage {
  char* h = nullptr;
  size_t cap = 0;
  size_t used = 0;
  void ensure(size_t bytes);
  ~HostStage();
};

// Uploads a set of host vectors into one device scratch region with one memcpy.  The
// pinned staging is double-buffered: the factor plans batch b+1 while batch b's second-half
// copy may still be queued (it waits for a batch's ranks, not for its second half), so
// reset() alternates between two buffers.  A buffer is rewritten two resets later, when the
// host has waited for an event behind its copy (the next batch's ranks): no event of its own.
struct Upload {
  HostStage stage, other;
  DevScratch dev;
  std::vector<std::pair<size_t, size_t>> parts;   // (offset, bytes)
  size_t total = 0;
  void reset() {
    parts.clear();
    total = 0;
    std::swap(stage.h, other.h);
    std::swap(stage.cap, other.cap);
    std::swap(stage.used, other.used);
  }
  template <class T>
  size_t add(const std::vector<T>& v) {
    const size_t off = (total + 255) & ~size_t(255);
    parts.push_back({off, v.size() * sizeof(T)});
    total = off + v.size() * sizeof(T);
    return parts.size() - 1;
  }
  template <class T>
  void copy_in(size_t idx, const std::vector<T>& v) {
    if (!v.empty()) std::memcpy(stage.h + parts[idx].first, v.data(), v.size() * sizeof(T));
  }
  template <class T>
  T* dptr(size_t idx) {
    return reinterpret_cast<T*>(dev.d + parts[idx].first);
  }
  void send(cudaStream_t st) {
    if (total) HS_CUDA(cudaMemcpyAsync(dev.d, stage.h, total, cudaMemcpyHostToDevice, st));
  }
};

struct LevelRT {
  int32_t nclus = 0;
  std::vector<int32_t> cap, rank, kn, kw, ldB;
  std::vector<int32_t> ldc;             // C_s's columns (= kn, or the supported ones on a support-restricted level)
  bool khat = false;                    // level 0 restricted to the supports (support.cpp)
  std::vector<int64_t> voff;            // apply-vector offsets (prefix sums of cap)
  int64_t vlen = 0;
  double* arena = nullptr;              // T_s of every cluster (persistent: the apply operators)
  int32_t* iarena = nullptr;            // pivots (persistent)
  // per-batch workspace G, V, tau, nu, B (freed after the batch unless HS_KEEP_RECORDS);
  // C_s compacted into per-batch chunks of the persistent factor
  std::vector<double*> G, V, tau, B, nu, T, C;
  std::vector<int32_t*> piv;
  std::vector<double*> wchunks, cchunks;
  size_t arena_bytes = 0;
};

// Apply plan of one level (Algorithm 2): per-cluster records, the forward task list in
// batch order and the backward task list in reverse batch order (solve_kernels.cu).
struct ApplyLevelPlan {
  std::vector<ApplySrc> src;            // by cluster id (m = 0: unused)
  std::vector<FwdTask> ftask;
  std::vector<FwdTgt> ftgt;
  std::vector<BwdTask> btask;
  std::vector<BwdNb> bnb;
  std::vector<PullSrc> pull;            // pre / post lists of every cluster
  std::vector<Contrib> ctb;             // contributions each source produces
  std::vector<int32_t> post_cl;
  int64_t contrib_off = 0;              // this level's slots in ApplyPlan::d_contrib
  int64_t ctr_off = 0;                  // counters: cnt[nclus] bcnt[nclus] done[nclus] ticket[2]
  int64_t parts = 0;                    // partial-sum doubles of the backward sweep
  ApplySrc* d_src = nullptr;
  FwdTask* d_ftask = nullptr;
  FwdTgt* d_ftgt = nullptr;
  BwdTask* d_btask = nullptr;
  BwdNb* d_bnb = nullptr;
  PullSrc* d_pull = nullptr;
  Contrib* d_ctb = nullptr;
  int32_t* d_post_cl = nullptr;
  std::vector<int32_t> cinv;            // support-restricted records: Contrib::inv maps
  int32_t* d_cinv = nullptr;
  // batch-synchronous sweeps (levels of large batches): the clusters of batch b are
  // bcl[boff[b], boff[b+1])
  bool bsync = false;
  std::vector<int32_t> bcl, boff;
  int32_t* d_bcl = nullptr;
};

struct ApplyPlan {
  std::vector<ApplyLevelPlan> lv;
  std::vector<int64_t> vbase;            // per level + top: offset of the level vector in d_y
  int64_t vtotal = 0, ftotal = 0, ctr_total = 0, max_parts = 0;
  double* d_y = nullptr;                 // the apply vector (all levels + top)
  double* d_yf = nullptr;                // fine parts y_f of every cluster (forward -> backward)
  double* d_xb = nullptr;                // backward result x (d_y's layout), reset to "empty" per apply
  double* d_parts = nullptr;
  double* d_contrib = nullptr;           // forward contributions (pull sweep), all levels
  int64_t contrib_total = 0;
  int32_t* d_ctr = nullptr;
  cudaGraphExec_t graph = nullptr;
  int64_t graph_kernels = 0;
};

}  // namespace hs

namespace hs {
// Multi-GPU transport (comm.cpp): NCCL (loaded only for world_size > 1), or the loopback
// test harness (P ranks as host threads on one device, copies ordered by events)
struct Comm;
struct LoopWorld;
void nccl_unique_id(void* out128);
Comm* comm_init(int world, int rank, const void* id128);
Comm* comm_loopback(LoopWorld* w, int rank);
LoopWorld* loop_world_create(int world);
void loop_world_destroy(LoopWorld* w);
int loop_world_size(LoopWorld* w);
void comm_destroy(Comm* c);
void comm_allreduce_sum_i32(Comm* c, int32_t* d_buf, size_t n, cudaStream_t st);
void comm_allreduce_sum_f64(Comm* c, double* d_buf, size_t n, cudaStream_t st);
void comm_group_start(Comm* c);
void comm_group_end(Comm* c, cudaStream_t st);
void comm_send_f64(Comm* c, const double* d, size_t n, int peer, cudaStream_t st);
void comm_recv_f64(Comm* c, double* d, size_t n, int peer, cudaStream_t st);
}  // namespace hs

namespace hs {
// Distributed solve (dsolve.cu): per-rank plan of the owner-computes Algorithm 2 and PCG.
struct DFwdItem {            // one owned cluster of a batch, forward
  const double* T;           // T_s (m x m, row-major)
  const double* C;           // C_s (K x kn, row-major)
  const double* y;           // y_s (level segment)
  double* yc;                // coarse part -> the parent's segment
  double* yf;                // fine part (kept for the backward sweep)
  double* slot;              // contributions C_s^T y_f (kn), or null
  int32_t m, r, kn, pad;
};
struct DAccItem {            // one owned target of a batch: y -= its contributions in source order
  double* y;
  int32_t len, s0, ns, pad;
};
struct DBwdItem {            // one owned cluster of a batch, backward
  const double* T;
  const double* C;
  const double* xc;          // coarse part (the parent's segment)
  const double* yf;
  double* x;                 // x_s (level segment)
  int32_t m, r, kn, nb0, nnb, pad;
};
struct DNb {                 // a neighbour's current x segment
  const double* x;
  int32_t len, pad;
};
struct DMsg {                // one message of a group: (device pointer, doubles, peer)
  double* ptr;
  int32_t len, peer;
};
struct DistBatch {
  int32_t level = 0, phase2 = 0;
  int32_t fwd0 = 0, nfwd = 0, acc0 = 0, nacc = 0, bwd0 = 0, nbwd = 0;
  std::vector<DMsg> fsend, frecv, bsend, brecv;
};
struct DevCache;
struct DistSolve {
  DevCache* dc = nullptr;
  std::vector<void*> owned;
  int rank = 0, world = 1;
  std::vector<int64_t> vbase;
  int64_t vtotal = 0;
  double *d_y = nullptr, *d_x = nullptr, *d_f = nullptr, *d_slot = nullptr;
  DFwdItem* d_fwd = nullptr;
  DAccItem* d_acc = nullptr;
  const double** d_accsrc = nullptr;
  DBwdItem* d_bwd = nullptr;
  DNb* d_nb = nullptr;
  int max_m = 0, max_kn = 0;
  std::vector<DistBatch> batches;
  std::vector<DMsg> top;              // per top cluster: (unused, size, owner)
  std::vector<int64_t> top_off;
  // PCG
  int64_t r0 = 0, r1 = 0, nloc = 0, nghost = 0, nnz_loc = 0;
  std::vector<int64_t> range_lo, range_hi;   // every rank's owned permuted range
  std::vector<DMsg> hsend, hrecv;
  std::vector<int64_t> hsend_off, hrecv_off;
  int64_t* d_lrow = nullptr;
  int32_t* d_lcol = nullptr;
  int64_t* d_vidx = nullptr;
  int32_t* d_sidx = nullptr;
  double *d_lval = nullptr, *d_xext = nullptr, *d_sbuf = nullptr;
  double *d_r = nullptr, *d_z = nullptr, *d_p = nullptr, *d_q = nullptr, *d_xs = nullptr, *d_part = nullptr;
  double *d_full = nullptr, *d_full2 = nullptr;
  double* h_scal = nullptr;
  ~DistSolve();
};
}  // namespace hs

struct hs_handle_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // factor work off the critical path (apply operators T_s)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool own_stream = false;
  int world = 1, rank = 0;
  hs::Comm* comm = nullptr;     // world > 1: NCCL or loopback transport
  std::string err;
  hs::VmmPool vmm;              // physical chunks of the block stores (destroyed after the cache)
  hs::DevCache cache;           // declared before the staging buffers (destroyed after them)
  hs::Upload upA, upB, upC;     // descriptor staging, reused across factors
  hs::HostStage dirstage;       // pinned staging of the level directories (one upload per level)
  // per-factor host buffers kept across factors (pinned / mapped allocations cost milliseconds)
  int32_t* h_rank = nullptr;    // pinned, pub_cap entries
  void* pub = nullptr;          // mapped RankPub + pub_cap ranks
  int pub_cap = 0;
};

struct hs_factor_s {
  hs_handle_s* h = nullptr;
  const hs::Analysis* an = nullptr;
  hs_factor_opts opt{};
  // CSR in the original ordering (SpMV)
  int64_t* d_rowptr = nullptr;
  int32_t* d_colind = nullptr;
  double* d_vals = nullptr;
  int64_t* d_perm = nullptr;
  std::vector<hs::LevelRT> lv;
  double* d_top = nullptr;
  int64_t ntop = 0;
  std::vector<int32_t> top_sizes;
  hs::ApplyPlan ap;
  std::unique_ptr<hs::DistSolve> ds;     // world > 1: the distributed solve (records stay at their owners)
  bool keep_records = false;             // HS_KEEP_RECORDS: per-cluster G, V, tau, B stay exportable
  hs::RecSpace rec;                      // large factors: T_s / C_s records, spillable during the factorization
  hs_factor_stats_t stats{};
  // PCG work vectors
  double *d_r = nullptr, *d_z = nullptr, *d_p = nullptr, *d_q = nullptr, *d_x = nullptr, *d_b = nullptr;
  double* d_red = nullptr;     // reduction scratch
  double* h_red = nullptr;     // pinned
  ~hs_factor_s();
};

namespace hs {
hs_factor_s* factor_create(hs_handle_s* h, const Analysis* an, const double* values, const hs_factor_opts& opt);
void apply(hs_factor_s* f, const double* d_b, double* d_x);         // device pointers
void pcg(hs_factor_s* f, const double* d_b, double* d_x, double tol, int maxit, hs_pcg_report* rep);
void gmres(hs_factor_s* f, const double* d_b, double* d_x, double tol, int restart, int maxit, hs_pcg_report* rep);
void spmv(hs_factor_s* f, const double* d_x, double* d_y);
struct DistPlan;
void dist_solve_build(hs_factor_s* f, const DistPlan& DP);
void dist_apply(hs_factor_s* f, const double* d_b, double* d_x);         // collective, global vectors
void dist_pcg(hs_factor_s* f, const double* d_b, double* d_x, double tol, int maxit, hs_pcg_report* rep);
void dist_spmv_global(hs_factor_s* f, const double* d_x, double* d_y);
}  // namespace hs
