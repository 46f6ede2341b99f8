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

// ---- programmatic dependent launch (sm_90+) ------------------------------------------
// The per-batch kernels are launched with programmatic stream serialization: a kernel may be
// scheduled while its stream predecessor drains; it calls pdl_wait() (griddepcontrol.wait:
// the predecessor grid has completed and its writes are visible) before touching anything
// the predecessor produced, and pdl_trigger() to let its own successor launch early.
bool pdl_enabled();   // HS_NO_PDL=1 turns the attribute off (A/B)
#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <typename... KArgs, typename... Args>
void launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  HS_CUDA(cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...));
}
#endif

struct FusedSeg;

// One cluster of a batch (a1-a4).
struct CluItem {
  double* G;        // m x m, row-major ld m: holds A_ss on entry, the lower factor G_s on exit
  double* V;        // m x m, column j = Householder vector v_j (col-major, ld m)
  double* tau;      // m
  double* B;        // B_s = [A_sw | A_sn], m x ldB row-major, w columns first
  int32_t* piv;     // m canonical pivot columns
  double* nu;       // kw scratch column norms
  unsigned long long* nmax;   // max n-column norm of B_n (double bits; zeroed by the upload, set by TRSM)
  int32_t m, kw, kn, ldB;
  int32_t level, cluster, pad0, pad1;
  // direct write-back (dwb = 1, DC path with device patching): CPQR writes the coarse-w rows
  // and I_r, k_rotate_n the coarse-n rows, straight into the store blocks of row s (seg:
  // the cluster's store segments in column order), and C = rows [r, m) of the rotated B_n
  // into its persistent slab Cout (ld kn)
  const FusedSeg* seg;
  double* Dss;      // the diagonal store block (s, s), ld ldss
  double* Cout;
  int32_t nseg, ldss, dwb, keepB;   // keepB: also write the coarse rows / rotated B_n back to B (records)
  // CPQR global-memory mode (a w-block too large for a 16-CTA cluster's shared memory): the
  // slices live column-major in this scratch ((kw + 16) x (m + 16) doubles, coalesced group
  // loads) instead of shared memory; null = shared-memory mode
  double* Wt;
  // the apply operator formed by k_rotate_n: T_s = Qᵀ G_s^{-1} from k_chol's G^{-1} (fused path)
  const double* Ginv;
  double* Tout;
  // support-restricted level 0 (support.cpp): B_s holds only the structurally
  // nonzero columns of its blocks (the segments' idx lists); kwd = the dense w-width (-1: B_s
  // is dense).  Cout = C_s on the same (compressed) n-columns, ld ldC = kn: the apply's record.
  int32_t ldC, kwd;
};

struct FormTItem {  // T_s = U^T G^{-1} of one eliminated cluster (apply operator, m x m row-major)
  const double* G;
  const double* Ginv;  // G^{-1} when k_chol formed it (then no substitution here), else null
  const double* V;
  const double* tau;
  double* T;
  int32_t m, r;
};

// a0 + a1 + a2 for the DC path (fused.cu): per cluster (k_chol_inv) or per 64-column tile
// (k_scale_tile) of a cluster
struct FusedItem {
  const double* Ass;          // diagonal block in the store (lower, row-major, ld lda)
  double* G;                  // workspace G_s
  double* Ginv;               // workspace G_s^{-1} (lower, row-major ld m): k_chol writes it, the
                              // scaling (DMMA product) and the apply operator T_s read it
  double* B;                  // workspace B_s (m x ldB)
  unsigned long long* nmax;   // R-floor slot
  int32_t m, lda, ldB, kw;
  int32_t c0, nc, seg_begin, seg_end;
  int32_t level, cluster, bi, pad;
};
struct FusedSeg {             // block (s, q) of the store: B_s columns [col, col + len)
  const double* src;
  const int32_t* idx;         // column col + c of B_s = local column idx[c] of the block (null: c)
  int32_t sld, trans, col, len;
  int32_t dcol, pad;          // the block's first column in the dense B_s (canonical pivot index)
};
struct ScaleTile {            // k_scale_mma: columns [c0, c0 + nc) of cluster item ci's B_s
  int32_t ci, c0, nc, seg_begin, seg_end, pad;   // the segments overlapping the tile
};
constexpr int CI_MAX_M = 112;   // k_scale_tile: G (ld m + 1) and a 64-column tile in shared memory, <= 28 rows per lane

struct TrsmItem {   // one column tile of one cluster's B_s
  int32_t ci, c0, nc, pad;   // k_rotate_n: pad = 1 for a tile of T_s = Qᵀ G_s^{-1} (columns of Ginv)
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
  double** pairs;            // [nnb (nnb+1) / 2] target block of neighbour pair (a >= b), or null
};
// Device-side patch of a batch's pre-planned second half with the kept ranks r_s read from
// d_rank (no host round trip between CPQR and the Schur update): one thread per item.
enum PatchKind : int32_t { PK_SRC = 0, PK_ROWS, PK_COLS, PK_I32, PK_FT, PK_CCOPY, PK_K };
struct PatchItem {
  void* target;          // SchurSrc* / CopyItem* / int32_t* / FormTItem*
  const double* base;    // B_s
  int32_t bi, kind, m, ldB;
  int32_t kw, i0, step, pad;
};


// A batch's kept ranks and the status published to mapped pinned host memory by one small
// kernel (no D2H copies or events in the stream); the host spins on seq.
struct RankPub {
  volatile int32_t seq;
  int32_t flag, level, cluster, pivot, pad;
  double value;
  int32_t rank[1];   // [max batch]
};


struct SchurTile2 {
  int32_t src, i0, j0, pad;
};
struct NbCol {               // neighbour q occupies columns [col, col+len) of the (compressed) n-part
  int32_t q, col, len, idx;  // idx: position of q in the full n(s) list (pair table index)
  const int32_t* sup;        // column col + c = local column sup[c] of q (null: c; support.cpp)
};
struct BlockDir {            // the level's block store: row p has blocks (p, q<=p) sorted by q
  double* blk;
  int64_t total;             // doubles in the store (bounds checks)
  const int64_t* ptr;
  const int32_t* q;
  const int64_t* off;
  const int32_t* cap;
};

// Apply (Algorithm 2) as a dependency-driven task list per level.
// The local transform of cluster s is the explicit m x m matrix T_s = U_s^T G_s^{-1}
// (E_s S_s of W_s), formed once by the factor (k_form_T), so the forward step
// [y_c; y_f] = T_s y_s and the backward step x_s = T_s^T [x_c; x_f] are parallel matvecs.
// Coarse outputs are written straight to the parent level's vector (the level
// transition of P:636), the fine part y_f to a per-level buffer for the backward sweep.
struct ApplySrc {
  const double* T;           // m x m row-major
  const double* C;           // C_s (fine rows), n-part column 0, ld ldC
  const double* y;           // live segment at elimination (level vector), m entries
  double* yc;                // coarse destination (parent level vector), r entries
  double* yf;                // fine buffer, K = m - r entries
  double* x;                 // backward output (the x vector's level segment)
  const double* xc;          // x_c: s's coarse rows in the parent's x segment (final before this level)
  int32_t m, r, ldC, kn;
  int32_t pre;               // forward events on s before its elimination
  int32_t nchunk;            // backward tasks of s (>= 1)
  int32_t nb_begin, nb_end;  // neighbour list (backward gather)
  int64_t part;              // partial sums of the backward chunks: nchunk x K
  int32_t pre_begin, pre_end;    // forward contributions to y_s from sources eliminated before s
  int32_t post_begin, post_end;  // contributions to s's coarse part from sources eliminated after s
  int32_t tg_begin, tg_end;      // the contributions s produces (Contrib list)
};
struct PullSrc {             // y[0:len] -= contrib[slot : slot+len], produced by source t
  int64_t slot;
  int32_t t, pad;
};
struct Contrib {             // contrib[slot : slot+dlen] = C_s[:, cols(q)]^T y_f,s (source s)
  int64_t slot;
  int32_t col, len;          // q's columns [col, col+len) of C_s
  int32_t q, pre;            // target; pre: q is eliminated later (counts toward arr[q])
  int32_t dlen, pad;         // entries of the contribution (q's live size)
  // a support-restricted record (level 0): entry i is C_s column col + inv[i], or 0 when
  // inv[i] < 0; null: entry i is column col + i (dlen == len)
  const int32_t* inv;
};
struct FwdTgt {              // y_q[0:len] -= C_s[:, col:col+len]^T y_f,s
  double* y;                 // q's live segment (level or parent vector)
  int32_t q, col, len, seq;  // seq: forward event number of this update on q
  int32_t proc, pad;         // proc: q already eliminated (its live segment is coarse)
};
struct FwdTask {             // a group of targets of source s; `first` also emits s's outputs
  int32_t s, t_begin, t_end, first;
};
struct BwdNb {               // neighbour q: columns [col, col+len) of C_s read x from `x`
  const double* x;
  int32_t q, col, len, later;   // later: q eliminated after s at this level (wait for it)
  int32_t off, pad;             // position of q's columns inside its backward chunk
  const int32_t* sup;           // support-restricted record: column col + i reads x[sup[i]] (null: x[i])
};
struct BwdTask {             // neighbours bnb[b0, b1) of s (nc columns in all) -> partial sums
  int32_t s, b0, b1, nc, chunk, pad;
};
constexpr int APPLY_THREADS = 256;
constexpr int BWD_COLS = 512;        // columns of C per backward task
constexpr int BWD_CRIT = 2;          // later neighbours with a backward chunk of their own
constexpr int FWD_COLS = 256;        // target columns per forward task
struct ApplyLevelArgs {
  const ApplySrc* src;
  const PullSrc* pull;       // pre / post contribution lists (pull-mode forward sweep)
  const Contrib* ctb;        // contributions produced per source
  double* contrib;           // their values
  const int32_t* post_cl;    // clusters with post contributions
  int32_t npost, pad0;
  const FwdTask* ftask;
  const FwdTgt* ftgt;
  const BwdTask* btask;
  const BwdNb* bnb;
  double* parts;
  int32_t* cnt;              // forward event counters (nclus)
  int32_t* bcnt;             // backward chunk arrivals (nclus)
  int32_t* done;             // backward completion flags (nclus)
  int32_t* arr;              // forward: contributions arrived per target (nclus)
  int32_t* ticket;           // [0] forward, [1] backward
  int32_t nftask, nbtask;
  int32_t spare0, spare1;
  long long* trace;          // HS_APPLY_TRACE: 8 globaltimer stamps per task (profiling only)
};

// First error raised on the device (POTRF breakdown).
struct DevStatus {
  int32_t flag, level, cluster, pivot;
  double value;
};
// A level of small clusters eliminated wave by wave on the device (small.cu)
constexpr int SMALL_M = 32;    // largest cluster of such a level
constexpr int SMALL_K = 512;   // largest k_n + k_w (level-start sizes)
struct SmallArgs {
  BlockDir dir;
  const int32_t *nptr, *nidx, *wptr, *widx;   // n(s), w(s) of the level (CSR)
  int32_t *live, *rank, *kn, *kw;             // per cluster (live: updated as clusters are eliminated)
  double* T;                                  // apply-operator arena, T_s at toff[s]
  const int64_t* toff;
  int32_t* piv;
  const int64_t* poff;
  double* C;                                  // C_s at coff[s] (room for m x k_n at level-start sizes)
  const int64_t* coff;
  const int32_t* items;                       // the waves' clusters, concatenated
  DevStatus* status;
  double eps;
  int32_t relative, level, m_max, k_max, nseg_max, npair_max;
};
size_t small_smem_bytes(int m_max, int k_max, int nseg_max, int npair_max);
void launch_elim_small(const SmallArgs& a, int first, int n, cudaStream_t st);
// the patch items (the batch's ranks are published by launch_publish right after the CPQR)
void launch_patch(const PatchItem* d_items, int n, const int32_t* d_rank, cudaStream_t st);
void launch_publish(const int32_t* d_rank, int n, const DevStatus* d_status, RankPub* pub, int32_t seq,
                    cudaStream_t st);
void launch_chol(const FusedItem* d_items, int n, int max_m, DevStatus* status, cudaStream_t st);
void launch_scale_tiles(const FusedItem* d_clus, const ScaleTile* d_tiles, int n, const FusedSeg* d_segs, int max_m,
                        cudaStream_t st);

// ---- launch accounting (every launcher counts its kernels; graphs count their nodes) -----
void count_launch(int64_t n);
int64_t launch_count();

// ---- kernel launchers (kernels.cu / solve_kernels.cu) -------------------------------------
// values symmetry: *flag = 1 if |v[k] - v[tmap[k]]| > 1e-12 max(|v[k]|, |v[tmap[k]]|) for some k
// NEXT f1 (nodc.cu): the original LoRaSp step without deferred compression
void set_smem_attr(const void* f, size_t bytes);   // opt-in dynamic smem (only ever grows)
void launch_nmax(const CluItem* d_clu, const TrsmItem* d_items, int n, cudaStream_t st);
void launch_rot2(const CluItem* d_clu, int n, int max_m, const int32_t* d_rank, cudaStream_t st);
void launch_coarse_update(const CluItem* d_clu, const TrsmItem* d_items, int n, const int32_t* d_rank,
                          cudaStream_t st);
void launch_form_T_nodc(const FormTItem* d_items, int n, int max_m, cudaStream_t st);
void launch_symcheck(const double* vals, const int64_t* tmap, int64_t nnz, int32_t* flag, cudaStream_t st);
void launch_copy2d(const CopyItem* d_items, int n, cudaStream_t st);
// splits items larger than ~16K elements into row ranges (one CTA each) in place
void split_copies(std::vector<CopyItem>& items);
void launch_identity(double* const* d_ptr, const int32_t* d_ld, const int32_t* d_r, int n, cudaStream_t st);
void launch_scatter(const double* vals, const int64_t* map, int64_t nnz, double* blk, cudaStream_t st);
void launch_potrf(const CluItem* d_items, int n, int max_m, DevStatus* status, cudaStream_t st);
void launch_trsm(const CluItem* d_clu, const TrsmItem* d_items, int n, int max_m, cudaStream_t st);
// a2 on the FP64 tensor cores for the non-fused DC path (trsm_mma.cu): strips of trsm_mma_tile_cols()
void launch_trsm_mma(const CluItem* d_clu, const TrsmItem* d_items, int n, int max_m, cudaStream_t st);
int trsm_mma_tile_cols();
// thread-block-cluster CPQR; picks the cluster size from the batch shape, returns it
// a3+a4 v3 (cpqr.cu): thread-block cluster per graph cluster, column groups of G lanes,
// one DSMEM exchange per step, n-columns rotated after the pivoting loop; returns CS
// words of global scratch a cluster's CPQR needs (0: it runs from shared memory); max_m is
// the largest cluster of the batch (it fixes the kernels' rows-per-lane)
size_t cpqr_global_words(int m, int kw, int max_m);
int launch_cpqr3(const CluItem* d_items, const std::vector<CluItem>& h_items, double eps, int relative,
                 int32_t* d_rank, cudaStream_t st);
// a4 for the n-columns: B_n <- Q^T B_n with Q = H_0...H_{r-1} from the CPQR (rank from d_rank).
// items: (cluster, first column within the n-part, count) tiles of rot_tile_cols(m) columns.
int rot_tile_cols(int m, int max_m);   // columns per rotation tile (max_m: of the launch)
void launch_rotate_n(const CluItem* d_clu, const TrsmItem* d_items, int n, int max_m, const int32_t* d_rank,
                     cudaStream_t st);
void launch_schur(const SchurTile* d_tiles, const SchurContrib* d_con, int n, cudaStream_t st);
void launch_schur2(const SchurTile2* d_tiles, int n, const SchurSrc* d_src, const NbCol* d_nb, const BlockDir& dir,
                   cudaStream_t st);
// per-source column owners (nb index per n-column), once per batch before the waves
// per level: target block of every neighbour pair (a >= b) of every cluster's n(s) list
// (hptr/hq: n(s) as CSR; poff: offsets of each cluster's triangular table in pairs)
void launch_level_pairs(const int64_t* hptr, const int32_t* hq, const int64_t* poff, int nclus, int64_t nrows,
                        const int64_t* row_cl, double** pairs, const BlockDir& dir, cudaStream_t st);
// Dense blocked Cholesky of the top matrix (row-major, ld).  On return the
// diagonal NB x NB blocks hold G_kk (lower) and the block rows right of them hold
// U_kj = G_kk^{-1} A_kj (i.e. L^T); the strictly lower off-diagonal blocks are stale.
void dense_potrf(double* A, int N, int ld, DevStatus* status, int level, double* scratch_items,
                 cudaStream_t st);
constexpr int TOP_NB = 64;

// T_s = U^T G^{-1} for the clusters of a batch (after CPQR; the rank comes from d_rank)
void launch_form_T(const FormTItem* d_items, int n, int max_m, cudaStream_t st);
void launch_apply_fwd_level(const ApplyLevelArgs& a, cudaStream_t st);
void launch_apply_post_level(const ApplyLevelArgs& a, cudaStream_t st);
void launch_apply_bwd_level(const ApplyLevelArgs& a, cudaStream_t st);
// batch-synchronous sweeps: the clusters d_cl[0, n) of one batch (levels of large batches)
constexpr int BS_MAXG = 128;       // contributions per source
constexpr int BS_MAXCOLS = 4096;   // k_n per source
void launch_apply_fwd_batch(const ApplyLevelArgs& a, const int32_t* d_cl, int n, cudaStream_t st);
void launch_apply_bwd_batch(const ApplyLevelArgs& a, const int32_t* d_cl, int n, cudaStream_t st);
void launch_top_solve(double* y, const double* A, int N, int ld, cudaStream_t st);
void launch_permute(const double* src, double* dst, const int64_t* idx, int64_t n, int scatter, cudaStream_t st);
void launch_spmv(const int64_t* rowptr, const int32_t* colind, const double* vals, const double* x, double* y,
                 int64_t n, cudaStream_t st);

constexpr int MAX_M = 512;   // largest cluster the kernels handle (HS_E_UNSUPPORTED beyond)
constexpr int SMEM_M = 128;  // POTRF/TRSM stage the whole G in shared memory up to this size

}  // namespace hs
