/*
 * hsolve.h — C ABI of the B200-native deferred-compression LoRaSp hot path.
 *
 * Chen, Cambier, Boman, Rajamanickam, Tuminaro, Darve, "A Robust Hierarchical
 * Solver for Ill-conditioned Systems with Applications to Ice Sheet Modeling"
 * (arXiv 1811.11248).  "P:n" below is line n of /root/reference/PAPER.md.
 *
 * The library solves an (ill-conditioned) SPD system A x = b (P:478-481,
 * Eq. ax=b).  Four calls follow the paper's statement of the problem:
 *   hs_analyze  clustering of the graph of A, computed algebraically
 *               (extruded columns P:786-798), the cluster tree and
 *               the per-level elimination schedule (Alg. 1 loop);
 *   hs_factor   Algorithm 1 with the scaled low-rank elimination of
 *               §3.1: POTRF of A_ss, deferred-compression TRSM
 *               G_s^{-1}A_sw, column-pivoted QR to eps,
 *               sparsification, fine-DOF Schur update (Eq. CC:eqn:elim), top
 *               dense Cholesky;  eps is "the (only) other
 *               parameter";
 *   hs_apply    Algorithm 2: x = M^{-1} b by forward/backward
 *               substitution with the factor;
 *   hs_pcg      preconditioned CG with the factor as M (north_star; the paper
 *               uses right-preconditioned GMRES).
 *
 * Conventions (all calls):
 *   - Every call returns hs_status; no C++ exception crosses the ABI.  The
 *     detail of the last error (level, cluster, pivot index/value, CUDA string)
 *     is available from hs_last_error(h).
 *   - Ownership: the caller owns every input array; the library copies what it
 *     needs before returning and keeps no caller pointer.  Output arrays are
 *     caller-allocated.  Handles are created and destroyed only by the library.
 *   - Vectors b, x are in the ORIGINAL ordering; the library applies its
 *     permutation internally.  on_device = 0: host pointers; 1: device pointers
 *     on the handle's device (e.g. torch CUDA tensors).
 *   - Matrices are CSR with BOTH triangles stored: int64 rowptr[n+1], int32
 *     colind[nnz] (sorted per row), double values[nnz].
 *   - A handle is used by one host thread at a time.  A factor is immutable
 *     after hs_factor; hs_apply / hs_pcg only read it.
 *   - There is no CPU fallback: factor/apply/pcg fail with HS_E_NO_DEVICE when
 *     no CUDA device is present.  hs_analyze is host integer code and may be
 *     called with h == NULL.
 */
#ifndef HSOLVE_H
#define HSOLVE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HS_OK = 0,
  HS_E_INVALID_ARG = 1,        /* NULL pointer, bad option value                       */
  HS_E_DIM = 2,                /* size mismatch (pattern vs analysis, vector length)  */
  HS_E_NOT_SYMMETRIC = 3,      /* pattern (analyze) or values (factor) not symmetric   */
  HS_E_NOT_SPD = 4,            /* a Cholesky pivot <= 0; factor not created    */
  HS_E_COLUMN_SPLIT = 5,       /* a single extruded column exceeds the leaf size       */
  HS_E_PRECOND_NOT_POSITIVE = 6,/* PCG: <r, M^{-1} r> <= 0                             */
  HS_E_NOT_CONVERGED = 7,      /* PCG hit maxit; x and the report are still filled     */
  HS_E_OOM = 8,                /* device allocation failed                             */
  HS_E_CUDA = 9,               /* CUDA runtime error                                   */
  HS_E_NCCL = 10,              /* NCCL error                                           */
  HS_E_NO_DEVICE = 11,         /* no CUDA device: there is no CPU fallback             */
  HS_E_UNSUPPORTED = 12,       /* a size outside what the kernels support              */
  HS_E_INTERNAL = 13
} hs_status;

typedef struct hs_handle_s*   hs_handle;    /* device, stream, (NCCL comm)             */
typedef struct hs_analysis_s* hs_analysis;  /* host, integer: perm, tree, schedule     */
typedef struct hs_factor_s*   hs_factor;    /* device-resident factor                  */

typedef struct {
  int32_t leaf_size;     /* DOFs per leaf when column_id == NULL (C1: 16, C2: 64)             */
  int32_t leaf_columns;  /* columns per leaf when column_id != NULL (C3: 8, C4: 2, C5: 4)      */
  int32_t top_log2;      /* base case at the first level with <= 2^top_log2 clusters (3 -> 8) */
  int32_t nsub_log2;     /* fixed subdomain depth (3 -> 8 subdomains); must be <= top_log2    */
  int32_t coarse_fill;   /* neighbours n(s) at the coarse levels l >= 1:
                            0 (default): reading R-coarse -- the merged structural
                              neighbours (H_{l+1} = merge-quotient of H_l), so that "the number of
                              neighbor clusters is bounded by a constant" (Thm 1) and the
                              per-level cost falls proportionally; blocks created by fill
                              stay well-separated (w) and are compressed again at every level;
                            1: SURVEY O2.9 literally (P:494 applied to A_c): every nonzero block of
                              A_c is a neighbour -- the neighbour sets double per level on 2-D/3-D
                              grids and the coarse levels become a dense block Cholesky.
                            Both readings start each level from the whole block pattern of A_c. */
} hs_analyze_opts;

typedef struct {
  double  eps;           /* truncation tolerance, >= 0                 */
  int32_t eps_relative;  /* 1: tau_s = eps * max column norm of G^{-1}A_sw (reading Q1); 0: absolute */
  int32_t dc;            /* 1: deferred compression (the paper's method); 0: the original
                            LoRaSp step without it (NEXT f1)                     */
  int32_t values_on_device; /* 1: `values` is a device pointer on the handle's device          */
  int32_t reserved;
} hs_factor_opts;

typedef struct {
  int64_t n;             /* number of DOFs                                   */
  int32_t depth;         /* D: the tree has 2^D leaves                       */
  int32_t L_top;         /* number of hierarchical levels (top = level L_top) */
  int32_t nsub_log2;     /* effective subdomain depth                        */
  int32_t top_log2;
} hs_analysis_info;

/* keys for hs_analysis_export (all integer arrays, exported as int64) */
enum {
  HS_EXP_PERM = 0,       /* [n]      perm[new] = old                                    */
  HS_EXP_LEAF_OFF = 1,   /* [2^D+1]  DOF offsets of the leaves in the permuted order     */
  HS_EXP_H_PTR = 2,      /* level l: CSR of H_l (structural block pattern; n(s) = H_l-adj(s)) */
  HS_EXP_H_IDX = 3,
  HS_EXP_W_PTR = 4,      /* level l: w(s) at elimination time (ascending)               */
  HS_EXP_W_IDX = 5,
  HS_EXP_BATCH_PTR = 6,  /* level l: batches (independent sets), in elimination order   */
  HS_EXP_BATCH_IDX = 7,
  HS_EXP_INTERIOR = 8,   /* level l: 1 if the cluster's whole starting pattern shares its subdomain */
  HS_EXP_F_PTR = 9,      /* level l: fill graph after the level                          */
  HS_EXP_F_IDX = 10,
  HS_EXP_NPHASE1 = 11,   /* level l: [1] number of phase-I (interior) batches            */
  HS_EXP_HTOP_PTR = 12,  /* block pattern of the top level                               */
  HS_EXP_HTOP_IDX = 13,
  HS_EXP_FS_PTR = 14,    /* level l: block pattern at the level start (merge of F_final(l-1)) */
  HS_EXP_FS_IDX = 15
};

/* keys for hs_dist_plan_export (multi-GPU decomposition plan) */
enum {
  HS_DEXP_OWNER = 0,     /* level l (0..L_top): int64[nclus] owning rank of each cluster       */
  HS_DEXP_RECV_PTR = 1,  /* level l < L_top: int64[nclus+1] offsets into RECV                  */
  HS_DEXP_RECV = 2,      /* ranks (other than the owner) receiving cluster s's elimination     */
                         /* record (r, C_s, coarse rows) -- phase-II clusters only             */
  HS_DEXP_HELD_PTR = 3,  /* level l < L_top: int64[nclus+1] offsets into HELD                  */
  HS_DEXP_HELD = 4       /* for each p: the q <= p of the level's final fill graph whose block */
                         /* (p, q) rank `rank` stores (it owns p or q)                        */
};

/* keys for hs_factor_export */
enum {
  HS_FEXP_RANKS = 0,     /* level l: int64[nclus] kept rank r_s                          */
  HS_FEXP_LIVE0 = 1,     /* level l: int64[nclus] live size at the start of the level    */
  HS_FEXP_PIV_PTR = 2,   /* level l: int64[nclus+1] offsets into PIV                      */
  HS_FEXP_PIV = 3,       /* level l: canonical pivot columns of every cluster, pivot order */
  HS_FEXP_TOP = 4,       /* [ntop] live sizes at the top level                            */
  HS_FEXP_KN = 5,        /* level l: int64[nclus] k_n, live columns of n(s) at elimination */
  HS_FEXP_KW = 6         /* level l: int64[nclus] k_w, live columns of w(s) at elimination        */
};

typedef struct {
  double  t_factor_s;    /* device time of hs_factor (CUDA events)                      */
  double  flops;         /* algorithmic factor flops     */
  double  factor_bytes;  /* bytes of the stored factor (G, V, tau, C, top L)            */
  int64_t n_top;         /* DOFs at the top level                                       */
  int32_t n_levels;
  int32_t n_batches;
  int32_t max_m;         /* largest cluster size eliminated                             */
  int32_t max_rank;
  double  t_phase_s[8];  /* per-kernel-class device time: 0 gather 1 potrf 2 trsm 3 cpqr
                            (and the fused elimination of small-cluster levels, all of whose
                            flops are counted in flops_phase[3]) 4 schur 5 writeback/assemble
                            6 top 7 host planning (wall).
                            Entries 0-6 are measured with CUDA events between the kernels
                            only when HS_PHASE_EVENTS=all (or =cpqr: entry 3 only) is set
                            at factor time — the events cost stream time per batch; they
                            are 0 otherwise                                              */
  double  flops_phase[8];
  double  t_level_s[32]; /* device time of each level l < n_levels (its batches and the A_c
                            assembly, CUDA events at the level boundaries)   */
  double  flops_level[32];
} hs_factor_stats_t;

typedef struct {
  int32_t iters;         /* number of SpMVs                                             */
  int32_t converged;
  double  relres;        /* recurrence ||r_k|| / ||b||                                   */
  double  relres_true;   /* ||b - A x|| / ||b|| computed on the device at the end        */
  double  t_pcg_s;       /* device time                                                  */
  double  t_apply_s;     /* device time spent in the preconditioner                      */
  double  t_spmv_s;      /* device time spent in the CSR SpMV (CUDA events)              */
  double* history;       /* in: caller buffer for ||r_k|| / ||b||, k = 0..iters (or NULL) */
  int32_t history_cap;   /* in: its capacity                                             */
  int32_t history_len;   /* out: entries written (min(iters + 1, history_cap))           */
} hs_pcg_report;

/* ---- handle --------------------------------------------------------------------- */
/* device: CUDA ordinal.  world_size/rank/nccl_unique_id: multi-GPU (world_size 1 and
 * NULL id for one GPU).  Fails with HS_E_NO_DEVICE when CUDA is unavailable. */
hs_status hs_create(hs_handle* h, int device, int world_size, int rank, const void* nccl_unique_id);
/* Rank 0 of a multi-GPU job creates the 128-byte NCCL id, broadcasts it over the job's own
 * process group (e.g. torch.distributed) and every rank passes it to hs_create.  NCCL is
 * loaded on first use (dlopen of libnccl.so.2, HS_NCCL_LIB overrides); HS_E_NCCL if absent. */
hs_status hs_nccl_unique_id(void* out128);
/* Test harness for the multi-GPU factor on ONE device: world_size ranks run as host threads
 * of one process, each with its own handle (hs_create_loopback); their exchanges become
 * device-to-device copies ordered by CUDA events between the ranks' streams and host
 * barriers (no kernel waits on another rank).  The world object outlives its handles. */
hs_status hs_loopback_world_create(int32_t world_size, void** world);
void      hs_loopback_world_destroy(void* world);
hs_status hs_create_loopback(hs_handle* h, int device, void* world, int32_t rank);
/* stream: a cudaStream_t on the handle's device (e.g. torch.cuda.current_stream()),
 * or NULL for the library's own stream.  All device work of the handle runs on it. */
hs_status hs_set_stream(hs_handle h, void* stream);
void      hs_destroy(hs_handle h);
const char* hs_last_error(hs_handle h);     /* never NULL; h may be NULL (global last error) */
const char* hs_status_string(hs_status s);

/* ---- analyze (host, integer; bit-exact with the oracle) --------------------------- */
/* coords: n*coord_dim row-major (recursive coordinate bisection), or NULL:
 * coordinate-free recursive BFS bisection of the matrix graph (NEXT f4; the
 * paper's "algebraic" clustering): at every tree node a BFS of the induced
 * subgraph from its smallest unit finds a pseudo-peripheral unit g, the BFS order from g
 * is split into its first ceil(|I|/2) units (left) and the rest.  column_id: n entries or
 * NULL (with column_id, coordinates are required: HS_E_UNSUPPORTED otherwise). */
hs_status hs_analyze(hs_handle h, int64_t n, const int64_t* rowptr, const int32_t* colind,
                     const double* coords, int32_t coord_dim, const int32_t* column_id,
                     const hs_analyze_opts* opt, hs_analysis* out);
hs_status hs_analysis_get_info(hs_analysis a, hs_analysis_info* info);
/* Writes min(cap, len) entries of the array `key` of level `level` into out and the full
 * length into *len (call with out == NULL to query the length). */
hs_status hs_analysis_export(hs_analysis a, int32_t key, int32_t level, int64_t* out,
                             int64_t cap, int64_t* len);
void      hs_analysis_destroy(hs_analysis a);
/* The decomposition plan of rank `rank` of `world` GPUs (host, integer; no device needed).
 * world must divide the number of fixed subdomains (8 by default).  Same length-query
 * convention as hs_analysis_export.  HS_E_INVALID_ARG on a bad key/level/world/rank. */
hs_status hs_dist_plan_export(hs_analysis a, int32_t world, int32_t rank, int32_t key, int32_t level,
                              int64_t* out, int64_t cap, int64_t* len);

/* ---- factor (device) -------------------------------------------------------------- */
/* values: CSR values on the pattern given to hs_analyze (host pointer, or device pointer
 * when opt->values_on_device).  The analysis must outlive every factor made from it: the
 * first factor caches the pattern and its level-0 scatter map on the device inside the
 * analysis, so re-factoring new values on the same pattern (Newton / continuation
 * sequences) uploads only the values.  On HS_E_NOT_SPD no factor is created and
 * hs_last_error names (level, cluster, pivot, value).
 * Memory: the handle owns a caching allocator; large factors (a level-0 block store of
 * >= 24 GB, e.g. C4) keep their records in a virtual range whose completed levels are
 * copied to pinned HOST memory when a later level's block store needs the device memory,
 * and mapped back at the same addresses before the call returns (the apply reads device
 * memory only).  HS_E_OOM if the store of one level plus the running level's records do
 * not fit the device, or the records of the whole factor exceed it. */
hs_status hs_factor_create(hs_handle h, hs_analysis a, const double* values,
                           const hs_factor_opts* opt, hs_factor* out);
hs_status hs_factor_get_stats(hs_factor f, hs_factor_stats_t* st);
hs_status hs_factor_export(hs_factor f, int32_t key, int32_t level, int64_t* out,
                           int64_t cap, int64_t* len);
/* Debug/parity aid: the elimination record of one cluster (doubles, row-major):
 *   HS_CEXP_SHAPE [5]        m, r, kw, kn, ldB
 *   HS_CEXP_G     [m*m]      G_s (lower)
 *   HS_CEXP_V     [r*m]      Householder vectors v_0..v_{r-1} (each m long, zeros above j)
 *   HS_CEXP_TAU   [r]
 *   HS_CEXP_B     [m*ldB]    B_s after the elimination: columns [0,kw) = w part, [kw,kw+kn) =
 *                            n part; rows [0,r) = coarse rows, rows [r,m) of the n part = C.
 * Copies from the device; same length-query convention as hs_analysis_export.  G, V,
 * TAU and B live in per-batch workspace that is recycled unless the factor was created
 * with HS_KEEP_RECORDS=1 in the environment (HS_E_UNSUPPORTED otherwise). */
enum { HS_CEXP_SHAPE = 0, HS_CEXP_G = 1, HS_CEXP_V = 2, HS_CEXP_TAU = 3, HS_CEXP_B = 4 };
hs_status hs_factor_export_cluster(hs_factor f, int32_t key, int32_t level, int32_t cluster,
                                   double* out, int64_t cap, int64_t* len);
void      hs_factor_destroy(hs_factor f);

/* ---- solve (device) --------------------------------------------------------------- */
/* x = M^{-1} b (Algorithm 2).  b and x may alias. */
hs_status hs_apply(hs_factor f, const double* b, double* x, int32_t on_device);
/* PCG on A (the CSR given to hs_factor) with M = the factor; x0 = 0; stops when
 * ||r_k|| / ||b|| <= tol (iteration count = SpMVs).  HS_E_NOT_CONVERGED still fills
 * x and rep. */
hs_status hs_pcg(hs_factor f, const double* b, double* x, double tol, int32_t maxit,
                 int32_t on_device, hs_pcg_report* rep);
/* Right-preconditioned restarted GMRES(restart) with M = the factor -- the paper's Krylov
 * protocol (GMRES(200), tol 1e-12, maxit 1000; NEXT f3).  x0 = 0; stops when the
 * recurrence residual |g_{j+1}| / ||b|| <= tol; rep->iters = Arnoldi steps, t_pcg_s = the
 * solve's device time.  HS_E_NOT_CONVERGED still fills x and rep. */
hs_status hs_gmres(hs_factor f, const double* b, double* x, double tol, int32_t restart, int32_t maxit,
                   int32_t on_device, hs_pcg_report* rep);
/* y = A x with the factor's CSR (device SpMV); helper for tests and the bench. */
hs_status hs_spmv(hs_factor f, const double* x, double* y, int32_t on_device);

/* Number of kernels this process has launched through the library so far (every node
 * of a replayed CUDA graph counts).  Evidence for the bench's gpu_launches. */
int64_t hs_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HSOLVE_H */
