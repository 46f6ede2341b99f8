// Host runtime structures of libhsolve (handle, factor, apply plan).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

#include "device.h"
#include "internal.h"


struct hs_analysis_s {
  hs::Analysis* an = nullptr;
};

namespace hs {

// device buffer that grows on demand (used for per-launch descriptor uploads)
struct DevScratch {
  char* d = nullptr;
  size_t cap = 0;
  cudaStream_t st = nullptr;   // stream-ordered pool allocation
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

// Uploads a set of host vectors into one device scratch region with one memcpy.
struct Upload {
  HostStage stage;
  DevScratch dev;
  std::vector<std::pair<size_t, size_t>> parts;   // (offset, bytes)
  size_t total = 0;
  void reset() {
    parts.clear();
    total = 0;
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
  std::vector<int64_t> voff;            // apply-vector offsets (prefix sums of cap)
  int64_t vlen = 0;
  double* arena = nullptr;              // G, V, tau, nu, B of every cluster
  int32_t* iarena = nullptr;            // pivots
  std::vector<double*> G, V, tau, B, nu;
  std::vector<int32_t*> piv;
  size_t arena_bytes = 0;
};

struct ApplyBatch {
  int32_t local_begin, local_end;       // into fwd_local / bwd_local item arrays
  int32_t tgt_begin, tgt_end;           // forward scatter targets
  int64_t cap_fwd = 0;                  // dynamic smem (doubles) of the forward local kernel
  int32_t kn_bwd = 0;                   // x_n staging size of the backward kernel
  int64_t cap_bwd = 0;                  // total dynamic smem (doubles) of the backward kernel
  int32_t chunk_begin = 0, chunk_end = 0;   // backward matvec chunks
  int32_t max_m = 0;                        // largest cluster of the batch (kernel variant)
};

struct ApplyPlan {
  std::vector<ApplyLocal> local;        // shared by forward (nb range unused) and backward
  std::vector<ApplyNb> nb;
  std::vector<ApplyTarget> tgt;
  std::vector<ApplyContrib> con;
  std::vector<std::vector<ApplyBatch>> batches;   // per level
  std::vector<int32_t> lvl_local, lvl_nb, lvl_con, lvl_tgt;   // per-level start indices (address patching)
  std::vector<ApplyBatchDev*> d_lvl_batches;   // per level: the batches' item ranges (device)
  std::vector<int32_t> lvl_max_m;
  std::vector<int64_t> lvl_cap;
  std::vector<ApplyChunk> chunks;        // backward matvec column chunks
  ApplyChunk* d_chunks = nullptr;
  int64_t max_parts = 0;                 // partial sums of the largest batch
  double* d_parts = nullptr;
  std::vector<std::vector<int64_t>> trans_src, trans_dst;   // level l -> l+1 vector transition
  // device copies
  ApplyLocal* d_local = nullptr;
  ApplyNb* d_nb = nullptr;
  ApplyTarget* d_tgt = nullptr;
  ApplyContrib* d_con = nullptr;
  std::vector<int64_t*> d_tsrc, d_tdst;
  std::vector<int64_t> vbase;            // per level + top
  int64_t vtotal = 0;
  double* d_y = nullptr;                 // the apply vector (all levels + top)
  cudaGraphExec_t graph = nullptr;
  int64_t graph_kernels = 0;
  int32_t max_kn = 0;                    // largest n-part of a cluster with fine DOFs (apply smem)
  const double* graph_in = nullptr;
  double* graph_out = nullptr;
};

}  // namespace hs

struct hs_handle_s {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int world = 1, rank = 0;
  std::string err;
  hs::Upload upA, upB;          // descriptor staging, reused across factors
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
void spmv(hs_factor_s* f, const double* d_x, double* d_y);
}  // namespace hs
