// Device-side structures shared by the host drivers and the kernels (sm_100a).
// All work items carry absolute device addresses; they are built on the host per
// batch and uploaded with one cudaMemcpyAsync per launch group.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "internal.h"

#define HS_CUDA(call)                                                                       \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess)                                                                  \
      ::hs::fail(e_ == cudaErrorMemoryAllocation ? HS_E_OOM : HS_E_CUDA,                    \
                 std::string(#call) + ": " + cudaGetErrorString(e_));                       \
  } while (0)

namespace hs {

// Batched 2-D copy with optional transpose:
//   dst[i*dld + j] = trans ? src[j*sld + i] : src[i*sld + j]   (i < rows, j < cols)
// Used by pack (a0), write-back (a6), level assembly (A_c) and the top.
struct CopyItem {
  const double* src;
  double* dst;
  int32_t sld, dld, rows, cols, trans, pad;
};

// One cluster of a batch (a1-a4).
struct CluItem {
  double* G;        // m x m, row-major ld m: holds A_ss on entry, the lower factor G_s on exit
  double* V;        // m x m, column j = Householder vector v_j (col-major, ld m)
  double* tau;      // m
  double* B;        // B_s = [A_sw | A_sn], m x ldB row-major, w columns first
  int32_t* piv;     // m canonical pivot columns
  double* nu;       // kw scratch column norms
  int32_t m, kw, kn, ldB;
  int32_t level, cluster, pad0, pad1;
};

struct TrsmItem {   // one column tile of one cluster's B_s
  int32_t ci, c0, nc, pad;
};

// Schur target tile (a5):
//   dst[i*ld + j] -= sum_{contrib} sum_{k<K} C[k*ldC + colP + i0 + i] * C[k*ldC + colQ + j0 + j]
struct SchurTile {
  double* dst;               // tile origin
  int32_t ld, rows, cols;    // tile extent (<= 64 x 64)
  int32_t c_begin, c_end;    // contributions [c_begin, c_end), source cluster ascending
  int32_t i0, j0, pad;
};
struct SchurContrib {
  const double* C;           // C_s row 0 (= B_s + r*ldB + kw), ld ldC
  int32_t ldC, K, colP, colQ;
};

// Schur update v2 (a5), one source cluster per tile, device-side target lookup:
// the tile (i0, j0) of X = C^T C (C = K x kn, the n-part of the fine rows) is computed
// densely and each element subtracted from its target block A(q_a, q_b) (q_a >= q_b).
// Diagonal blocks keep LOWER-triangle semantics (only li >= lj is maintained).
// Sources of one launch ("wave") never share a neighbour, so no two tiles of a launch
// touch the same target element (deterministic, no atomics).
struct SchurSrc {
  const double* C;           // fine rows of the n-part, ld ldC
  int32_t ldC, K, kn, nb_off, nnb, pad;
};
struct SchurTile2 {
  int32_t src, i0, j0, pad;
};
struct NbCol {               // neighbour q occupies columns [col, col+len) of the n-part
  int32_t q, col, len, pad;
};
struct BlockDir {            // the level's block store: row p has blocks (p, q<=p) sorted by q
  double* blk;
  const int64_t* ptr;
  const int32_t* q;
  const int64_t* off;
  const int32_t* cap;
};

// Apply (Algorithm 2) items.
struct ApplyLocal {          // forward: y_s <- U^T G^{-1} y_s
                             // backward: x_f = y_f - sum C x_q, x_s <- G^{-T} U x_s
  const double* G;
  const double* V;
  const double* tau;
  double* y;                 // the cluster's segment (m entries)
  const double* C;           // C_s (fine rows), n-part column 0, ld ldC
  int32_t m, r, nb_begin, nb_end, ldC, part_off, kn, pad;
};
constexpr int BWD_CHUNK = 256;   // columns of C per backward matvec CTA
struct ApplyChunk {          // backward matvec: columns [c0, c0+BWD_CHUNK) of cluster `li` of the batch
  int32_t li, c0, part, pad;    // partial sums of the K rows go to parts[part .. part+K)
};
struct ApplyNb {             // backward: C_s[:, col:col+len] x_q
  const double* xq;
  int32_t col, len;
};
struct ApplyTarget {         // forward: y_q[0:len] -= sum_s C_s[:, col:col+len]^T y_f,s
  double* yq;
  int32_t len, c_begin, c_end, pad;
};
struct ApplyContrib {
  const double* C;           // C_s (fine rows), n-part column 0
  const double* yf;          // y_f,s
  int32_t ldC, K, col, pad;
};
struct ApplyBatchDev {       // a batch's item ranges in the apply arrays
  int32_t local_begin, local_end, tgt_begin, tgt_end, chunk_begin, chunk_end;
};
struct ApplyLevelArgs {      // one level of the apply, swept by one cooperative kernel
  const ApplyBatchDev* batches;
  int32_t nbatch, pad;
  const ApplyLocal* local;
  const ApplyTarget* tgt;
  const ApplyContrib* con;
  const ApplyNb* nb;
  const ApplyChunk* chunks;
  double* parts;
  int64_t cap;               // dynamic shared memory (doubles) for factor staging
};

// First error raised on the device (POTRF breakdown).
struct DevStatus {
  int32_t flag, level, cluster, pivot;
  double value;
};

// ---- launch accounting (every launcher counts its kernels; graphs count their nodes) -----
void count_launch(int64_t n);
int64_t launch_count();

// ---- kernel launchers (kernels.cu / solve_kernels.cu) -------------------------------------
// values symmetry: *flag = 1 if |v[k] - v[tmap[k]]| > 1e-12 max(|v[k]|, |v[tmap[k]]|) for some k
void launch_symcheck(const double* vals, const int64_t* tmap, int64_t nnz, int32_t* flag, cudaStream_t st);
void launch_copy2d(const CopyItem* d_items, int n, cudaStream_t st);
void launch_identity(double* const* d_ptr, const int32_t* d_ld, const int32_t* d_r, int n, cudaStream_t st);
void launch_scatter(const double* vals, const int64_t* map, int64_t nnz, double* blk, cudaStream_t st);
void launch_potrf(const CluItem* d_items, int n, int max_m, DevStatus* status, cudaStream_t st);
void launch_trsm(const CluItem* d_clu, const TrsmItem* d_items, int n, int max_m, cudaStream_t st);
void launch_cpqr(const CluItem* d_items, int n, double eps, int relative, int32_t* d_rank, cudaStream_t st);
// thread-block-cluster CPQR; picks the cluster size from the batch shape, returns it
int launch_cpqr2(const CluItem* d_items, const std::vector<CluItem>& h_items, double eps, int relative,
                 int32_t* d_rank, cudaStream_t st);
void launch_schur(const SchurTile* d_tiles, const SchurContrib* d_con, int n, cudaStream_t st);
void launch_schur2(const SchurTile2* d_tiles, int n, const SchurSrc* d_src, const NbCol* d_nb, const BlockDir& dir,
                   cudaStream_t st);
// Dense blocked Cholesky of the top matrix (row-major, ld).  On return the
// diagonal NB x NB blocks hold G_kk (lower) and the block rows right of them hold
// U_kj = G_kk^{-1} A_kj (i.e. L^T); the strictly lower off-diagonal blocks are stale.
void dense_potrf(double* A, int N, int ld, DevStatus* status, int level, double* scratch_items,
                 cudaStream_t st);
constexpr int TOP_NB = 64;

void launch_apply_fwd_local(const ApplyLocal* d, int n, int64_t cap, int max_m, cudaStream_t st);
void launch_apply_fwd_scatter(const ApplyTarget* d, const ApplyContrib* c, int n, cudaStream_t st);
// backward, stage 1: partial sums of C x_n over column chunks (many CTAs per cluster)
void launch_apply_bwd_partial(const ApplyLocal* d_local_batch, const ApplyNb* nb, const ApplyChunk* ch, int n,
                              double* parts, cudaStream_t st);
// backward, stage 2: x_f = y_f - sum of the partials (fixed order), x_s <- G^{-T} U [x_c; x_f]
void launch_apply_bwd(const ApplyLocal* d, const double* parts, int n, int64_t cap, int max_m, cudaStream_t st);
// one cooperative launch per level and direction (grid-wide barriers between batches)
void launch_apply_level(const ApplyLevelArgs& a, int max_m, int backward, cudaStream_t st);
void launch_top_solve(double* y, const double* A, int N, int ld, cudaStream_t st);
void launch_permute(const double* src, double* dst, const int64_t* idx, int64_t n, int scatter, cudaStream_t st);
void launch_spmv(const int64_t* rowptr, const int32_t* colind, const double* vals, const double* x, double* y,
                 int64_t n, cudaStream_t st);

constexpr int MAX_M = 512;   // largest cluster the kernels handle (HS_E_UNSUPPORTED beyond)
constexpr int SMEM_M = 128;  // POTRF/TRSM stage the whole G in shared memory up to this size

}  // namespace hs
