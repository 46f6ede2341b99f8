// a3 + a4: rank-revealing compression of the deferred-compression block B_w = G_s^{-1} A_sw
// (Eq. offdiag_new) by Businger-Golub column-pivoted QR, and the
// sparsification rotation U^T of the neighbour columns B_n = G_s^{-1} A_sn
// (Eq. CC:eqn:sparse).  Decisions follow SURVEY §8(c) O3.4 / DESIGN.md §2:
//   * exact column norms nu_i = ||W[j:m, i]|| recomputed from the current entries each step;
//   * tau_s = eps * nu_max(0) (relative, with the R-floor 1e-12 * max(nu_max(B_w), nu_max(B_n)));
//   * stop with r = j as soon as nu_max <= tau_s (keep iff nu_max > tau_s);
//   * pivot = lowest canonical column among nu_i >= (1 - 1e-10) nu_max;
//   * LAPACK dlarfg Householder convention.
//
// Design (sm_100a).  One thread-block cluster of CS CTAs per graph cluster s.  The w-columns
// are split in contiguous slices over the CTAs and live in shared memory for all r steps
// (global-memory mode when they do not fit even at CS = 16).  Inside a CTA a column is
// owned by a group of G lanes (G = rows / MR, rows interleaved), so the dot product and the
// norm of a column are G-lane shuffle reductions instead of one thread's serial chain.
// Per step the cluster exchanges one triple per CTA through distributed shared memory:
// (local max norm M_c, its lowest local candidate i_c, nu(i_c)).  That resolves the pivot
// with ONE cluster barrier whenever the lowest-ranked CTA holding a global candidate has
// nu(i_c) >= (1 - 1e-10) max_c M_c (always, unless near-ties straddle the local and global
// windows); otherwise a second exchange of the exact lowest candidates decides.
// The neighbour columns are not touched during the pivoting loop: k_rotate_n applies
// Q^T = H_{r-1}...H_0 to B_n afterwards, a column per lane group held in registers and the
// reflectors staged in shared memory (rows [0, r) -> coarse-n, rows [r, m) -> C = U_2^T G^{-1} A_sn).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cfloat>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "device.h"

namespace hs {

namespace {

constexpr int CQ_THREADS = 512;
constexpr int CQ_WARPS = CQ_THREADS / 32;
constexpr double CQ_WINDOW = 1.0 - 1e-10;   // pivot tie window

// lanes per column: the smallest power of two G with G * MR >= m (G <= 32)
__host__ __device__ __forceinline__ int cq_group(int m, int MR) {
  int G = 1;
  while (G < 32 && G * MR < m) G <<= 1;
  return G;
}
// Shared-memory layout of the w-slice: COLUMN-major, column stride ldm >= m with
// ldm == G (mod 16) for G < 16, so that a half-warp (16/G columns x G consecutive rows)
// touches 16 distinct 8-byte bank pairs, and a lane's rows l = t + i G sit at compile-time
// offsets i G from its column base.
__host__ __device__ __forceinline__ int cq_ldm(int m, int G) {
  int l = m < 1 ? 1 : m;
  // G >= 16: a half-warp reads 16 consecutive rows of one column (conflict-free for any
  // stride); an odd stride also keeps the staging transpose's column-strided stores apart
  if (G >= 16) return l | 1;
  const int rem = ((l - G) % 16 + 16) % 16;
  return l + (rem ? 16 - rem : 0);
}
__host__ __device__ __forceinline__ int cq_msg_words(int m);
// dynamic shared memory words: W slice (SM mode) + norms + message staging and slots
__host__ __device__ __forceinline__ size_t cq_smem_words(int m, int kw, int CS, int MR, bool sm, bool light = false) {
  const int wchunk = (kw + CS - 1) / CS;
  const size_t w = sm ? (((size_t)wchunk * cq_ldm(m, cq_group(m, MR)) + 1) & ~(size_t)1) : 0;
  return w + (size_t)((wchunk + 1) & ~1) + (light ? (size_t)2 * cq_msg_words(m) + (size_t)2 * CS * 8
                                                  : (size_t)(2 + 2 * CS) * cq_msg_words(m));
}
// direct write-back: the store element (row l of s, column j of B_s), j in the segment list
__device__ __forceinline__ int seg_find(const FusedSeg* seg, int nseg, int j) {
  int lo = 0, hi = nseg - 1;
  while (lo < hi) {   // last segment with col <= j
    const int mid = (lo + hi + 1) >> 1;
    if (seg[mid].col <= j) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}
// (g.idx: the supported columns of a support-restricted level-0 block, see FusedSeg)
__device__ __forceinline__ double* dwb_addr(const FusedSeg* seg, int nseg, int j, int l) {
  const FusedSeg g = seg[seg_find(seg, nseg, j)];
  if (j < g.col || j >= g.col + g.len) return nullptr;   // a column of an empty neighbour: none
  const int lc = g.idx ? g.idx[j - g.col] : j - g.col;
  double* p = const_cast<double*>(g.src);
  return g.trans ? p + (int64_t)lc * g.sld + l : p + (int64_t)l * g.sld + lc;
}
// the canonical (dense) index of B_s column j: the pivot order of the dense B_s
__device__ __forceinline__ int dense_col(const CluItem& it, int j) {
  if (it.kwd < 0) return j;
  const FusedSeg g = it.seg[seg_find(it.seg, it.nseg, j)];
  return g.dcol + (g.idx ? g.idx[j - g.col] : j - g.col);
}

template <int G>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = 1; o < G; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int wmin_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- cluster messaging primitives (mbarrier + st.shared::cluster) ----------------------
__device__ __forceinline__ uint32_t sm_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t remote(uint32_t local, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void bar_init(uint32_t bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(ok)
        : "r"(bar), "r"(parity), "r"(1000000u)   // suspend (not spin) up to 1 ms per try
        : "memory");
}

__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// bulk copy (async proxy) of `bytes` from this CTA's shared memory into another CTA's,
// signalling complete_tx on the destination's mbarrier
__device__ __forceinline__ void bulk_push(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src_cta), "r"(bytes), "r"(bar_cluster)
               : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct __align__(16) CqFb {     // fallback message: exact lowest candidate w.r.t. the global window
  int F, pad[3];
};
struct CqShared {
  unsigned long long bar1[2], bar2, bar3[2];   // step messages / fallback vector / fallback candidates
  CqFb mine3[2], slot3[2][16];
  double wred[CQ_WARPS];                        // per-warp max norm
  double wcnu[CQ_WARPS];                        // nu of the warp's candidate
  int wcand[CQ_WARPS];                          // per-warp lowest local candidate (INT_MAX: none)
  __align__(16) double vstage[MAX_M + 8];      // fallback: owner's (tau, beta, v) staging
  __align__(16) double vbuf[MAX_M + 8];        // fallback: received (tau, beta, v)
};
// Step message of one CTA (doubles): [0] M_c, [1] nu(i_c), [2] i_c (canonical, -1: none),
// [3] tau, [4] beta of the Householder reflector of column i_c, [5..8) pad, [8, 8+m) v
__host__ __device__ __forceinline__ int cq_msg_words(int m) { return (8 + m + 1) & ~1; }

// dlarfg (LAPACK convention) of column col, rows j..m-1, by one warp: the column in registers
// once (m <= 32 MR), x_norm from them, dst[8 + l] = v_l (zero above j, one at j, x_l / (alpha -
// beta) below); tau and beta in every lane.
template <int MR>
__device__ __forceinline__ void form_reflector(const double* col, int j, int m, int lane, double* dst, double& tau,
                                               double& beta) {
  double xr[MR];
  double xs = 0.0;
  const double alpha = col[j];
#pragma unroll
  for (int i = 0; i < MR; ++i) {
    const int l = lane + 32 * i;
    xr[i] = l < m ? col[l] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < MR; ++i)
    if (lane + 32 * i > j) xs += xr[i] * xr[i];
  xs = wsum(xs);
  const double xnorm = sqrt(xs);
  double rden;
  if (xnorm == 0.0) {
    tau = 0.0;
    beta = alpha;
    rden = 0.0;
  } else {
    const double h = sqrt(alpha * alpha + xnorm * xnorm);
    beta = alpha >= 0.0 ? -h : h;
    tau = (beta - alpha) / beta;
    rden = 1.0 / (alpha - beta);   // dlarfg scales x by 1/(alpha - beta)
  }
#pragma unroll
  for (int i = 0; i < MR; ++i) {
    const int l = lane + 32 * i;
    if (l < m) dst[8 + l] = (l < j) ? 0.0 : (l == j) ? 1.0 : xr[i] * rden;
  }
}

// The pivoting loop for a fixed group size G (lanes per column).
//
// Step j, every CTA c of the cluster (messages double-buffered by j & 1):
//   (1) local max M_c of its column norms, its lowest local candidate i_c w.r.t. the local
//       window, and -- speculatively -- the Householder reflector of column i_c; warp 0
//       bulk-copies the message (M_c, nu(i_c), i_c, tau, beta, v) into slot c of every CTA
//       (cp.async.bulk shared::cta -> shared::cluster, complete_tx on the receiver's bar1);
//   (2) wait on the local bar1 and decide (stop, p) from the CS messages -- the same
//       arithmetic in every CTA, so the decision is uniform.  The pivot is i_c of the
//       lowest CTA c holding a global candidate, whose reflector arrived with it; only a
//       near-tie straddling the local and global windows takes a second exchange (bar3)
//       and an owner push of the reflector (bar2);
//   (3) apply H_j to the local active columns and recompute their norms; the owner writes
//       the pivot column as (beta, 0, ..., 0) and the reflector to V / tau / piv.
// One mbarrier wait per step, no cluster-wide barrier inside the loop.
template <int MR, int G, bool SM, int NT, int U>
__device__ __forceinline__ void cpqr_body(const CluItem& it, double eps, int relative, int32_t* rank_slot,
                                          double* dsm, CqShared& sh, long long* trace, bool light) {
  // HS_CQ_TRACE debug aid: clock64 timeline of cluster 0 / CTA 0 / thread 0
#define CQ_TR(k)                                                            \
  do {                                                                      \
    if (trace && (long long)blockIdx.x == trace[254] && threadIdx.x == 0) trace[k] = clock64(); \
  } while (0)
  const bool trace_split = trace && trace[255] != 0;   // HS_CQ_TRACE_SPLIT: stamp 4 at the push
  const bool trace_fine = trace && trace[253] != 0;    // HS_CQ_TRACE_FINE: warp 0's dlarfg / push sub-steps
#define CQ_TF(j, k)                                 \
  do {                                              \
    if (trace_fine && (j) < 12) CQ_TR(100 + 8 * (j) + (k)); \
  } while (0)
  CQ_TR(0);
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const int m = it.m, kw = it.kw, ld = it.ldB;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int t = tid % G, grp = tid / G;
  constexpr int NGRP = NT / G;
  const int wchunk = (kw + CS - 1) / CS;
  const int w_lo = crank * wchunk;
  const int nw = max(0, min(kw - w_lo, wchunk));
  const int ldm = cq_ldm(m, G);
  // light messages (header only; the owner of the chosen pivot pushes its reflector after the
  // decision): the slots shrink from (2 + 2 CS)(8 + m) to (2 + 2 CS) 8 words, so wide blocks
  // keep their whole slice in shared memory
  // light: the own message buffers hold the header AND the speculatively formed reflector of
  // the local candidate (formed while the headers travel; pushed only if it wins)
  const int msgw = light ? 8 : cq_msg_words(m);             // slot stride
  const int msgo = light ? cq_msg_words(m) : msgw;          // own buffer stride
  const uint32_t msgb = (uint32_t)(msgw * 8);
  // element (l, c) of the slice, column-major with column stride ldm: in shared memory (SM)
  // or in the cluster's global scratch (global mode: coalesced group loads through L2)
  const int sr = 1;
  // dynamic shared memory (16-byte aligned regions, the bulk copies require it):
  // [W (SM mode): wchunk x ldm] [nu: wchunk] [mine: 2 x msgw] [slots: 2 x CS x msgw]
  // global mode (hybrid): [nu] [mine] [slots] [the first nsmc columns of the slice]; columns
  // [nsmc, nw) live in the global scratch (same column-major layout), so only the part of
  // the slice that exceeds the CTA's shared memory streams through L2 every step
  double* nu = SM ? dsm + (((size_t)wchunk * ldm + 1) & ~(size_t)1) : dsm;
  double* mine = nu + ((wchunk + 1) & ~1);
  double* slots = mine + 2 * msgo;
  double* const Wsm = SM ? dsm : slots + (((size_t)2 * CS * msgw + 1) & ~(size_t)1);
  double* const Wg = SM ? dsm : it.Wt + (size_t)w_lo * ldm;
  int nsmc = nw;
  if (!SM) {
    uint32_t dyn;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    const long long room = (long long)(dyn / 8) - (long long)(Wsm - dsm);
    nsmc = (int)max(0LL, min((long long)nw, room / ldm));
  }
  auto Wc = [&](int c) -> double* { return (SM || c < nsmc ? Wsm : Wg) + (size_t)c * ldm; };
  const int kiters = (nw + NGRP - 1) / NGRP;
  const int nr = (m - t + G - 1) / G;   // rows l = t + i G < m of this lane: i < nr

  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      bar_init(sm_addr(&sh.bar1[b]), 1);   // the local expect_tx; CS bulk copies complete it
      bar_init(sm_addr(&sh.bar3[b]), 1);
    }
    bar_init(sm_addr(&sh.bar2), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // ---- stage the w-slice (transpose to column-major; coalesced global reads) ----------
  if (nw > 0) {   // thread (row rr + k rpp, column cc): coalesced row segments, no division per element
    const double* __restrict__ src = it.B + w_lo;
    const int rpp = nw <= NT ? NT / nw : 1;   // rows per pass
    const int cc0 = nw <= NT ? tid % nw : tid, rr = nw <= NT ? tid / nw : 0;
    if (rr < rpp)
      for (int cc = cc0; cc < nw; cc += NT)
        for (int l0 = rr; l0 < m; l0 += 4 * rpp) {
          double v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int l = l0 + u * rpp;
            v[u] = l < m ? src[(size_t)l * ld + cc] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int l = l0 + u * rpp;
            if (l < m) Wc(cc)[l] = v[u];
          }
        }
  }
  __syncthreads();
  CQ_TR(1);
  // ---- initial column norms of the slice ------------------------------------------------
  double lm = -1.0;
  for (int k = 0; k < kiters; ++k) {
    const int c = grp + k * NGRP;
    const double* colp = Wc(c < nw ? c : 0) + (size_t)t * sr;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < MR; ++i)
      if (c < nw && i < nr) {
        const double x = colp[(size_t)i * G * sr];
        s += x * x;
      }
    s = group_sum<G>(s);
    if (c < nw) {
      const double v = sqrt(s);
      if (t == 0) nu[c] = v;
      lm = fmax(lm, v);
    }
  }
  // max n-column norm of B_n from the TRSM: the same value in every CTA (R-floor)
  const double Rn = __longlong_as_double((long long)*it.nmax);
  cl.sync();   // barriers initialised cluster-wide before any remote complete_tx
  CQ_TR(2);

  const int kmax = min(m, kw);
  int spec_li = INT_MAX;               // light: warp 0's local candidate of this step
  double spec_tau = 0.0, spec_beta = 0.0;
  double tau_s = 0.0;
  int r = kmax;
  int use3[2] = {0, 0}, use2 = 0;
  for (int j = 0; j < kmax; ++j) {
    const int buf = j & 1;
    const uint32_t par = (uint32_t)((j >> 1) & 1);
    double* mymsg = mine + buf * msgo;
    double* slot = slots + (size_t)buf * CS * msgw;
    // (1) local max, local candidate and its reflector -> every CTA
    lm = wmax(lm);
    {   // every warp, over the columns its own groups updated (their norms are the warp's own
        // writes): its max M_w and its lowest column with nu >= (1 - 1e-10) M_w
      __syncwarp();
      const double thr_w = CQ_WINDOW * lm;
      int lw = INT_MAX;
      if (lm >= 0.0)
        for (int k = t; k < kiters; k += G) {
          const int c = grp + k * NGRP;
          if (c < nw && nu[c] >= thr_w) {
            lw = c;
            break;
          }
        }
      lw = wmin_i(lw);
      if (lane == 0) {
        sh.wred[wid] = lm;
        sh.wcand[wid] = lw;
        sh.wcnu[wid] = lw != INT_MAX ? nu[lw] : -1.0;
      }
    }
    if (tid == 0) bar_expect(sm_addr(&sh.bar1[buf]), (uint32_t)CS * msgb);
    __syncthreads();
    if (j < (trace_fine ? 24 : 60)) CQ_TR(3 + 4 * j);
    if (wid == 0) {
      CQ_TF(j, 0);
      double Mc = lane < (NT / 32) ? sh.wred[lane] : -1.0;
      Mc = wmax(Mc);
      // the CTA's lowest column over the CTA window: the lowest warp candidate inside it; a warp
      // that reaches the window with its own candidate below it (a near-tie straddling the warp
      // and CTA windows) makes warp 0 rescan every column
      const double thr_c = CQ_WINDOW * Mc;
      const bool reach = Mc >= 0.0 && lane < (NT / 32) && sh.wred[lane] >= thr_c;
      const bool okc = reach && sh.wcnu[lane] >= thr_c;
      int li = okc ? sh.wcand[lane] : INT_MAX;
      li = wmin_i(li);
      if (__any_sync(0xffffffffu, reach && !okc)) {
        li = INT_MAX;
        for (int c = lane; c < nw; c += 32)
          if (nu[c] >= thr_c) {
            li = c;
            break;
          }
        li = wmin_i(li);
      }
      spec_li = light ? li : INT_MAX;
      if (li != INT_MAX && light) {
        if (lane == 0) {
          mymsg[1] = nu[li];
          mymsg[2] = (double)(w_lo + li);
        }
      } else if (li != INT_MAX) {   // dlarfg of column li, rows j..m-1
        double tau, beta;
        form_reflector<MR>(Wc(li), j, m, lane, mymsg, tau, beta);
        CQ_TF(j, 3);
        if (lane == 0) {
          mymsg[1] = nu[li];
          mymsg[2] = (double)(w_lo + li);
          mymsg[3] = tau;
          mymsg[4] = beta;
        }
      } else if (lane == 0) {
        mymsg[1] = -1.0;
        mymsg[2] = -1.0;
      }
      if (lane == 0) mymsg[0] = Mc;
      fence_proxy_async();
      CQ_TF(j, 4);
      __syncwarp();
      if (lane < CS)
        bulk_push(remote(sm_addr(slot + (size_t)crank * msgw), lane), sm_addr(mymsg), msgb,
                  remote(sm_addr(&sh.bar1[buf]), lane));
      CQ_TF(j, 5);
      if (spec_li != INT_MAX)   // light: the candidate's reflector while the headers travel
        form_reflector<MR>(Wc(spec_li), j, m, lane, mymsg, spec_tau, spec_beta);
      if (trace_split && j < (trace_fine ? 24 : 60)) CQ_TR(4 + 4 * j);   // local work done, message sent
    }
    // (2) decision from the CS messages (identical in every thread of every CTA)
    bar_wait(sm_addr(&sh.bar1[buf]), par);
    if (!trace_split && j < (trace_fine ? 24 : 60)) CQ_TR(4 + 4 * j);
    // the CS local maxima: lane k of every warp reads CTA k's (CS <= 16), warp max and a
    // ballot for the lowest CTA over the window (the same values in every warp)
    const double sv = lane < CS ? slot[(size_t)lane * msgw] : -1.0;
    double M = sv;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (j == 0) {
      tau_s = relative ? eps * M : eps;
      if (relative && eps > 0.0) tau_s = fmax(tau_s, 1e-12 * fmax(M, Rn));
    }
    if (!(M > tau_s)) {
      r = j;
      break;
    }
    const double thr = CQ_WINDOW * M;
    const unsigned over = __ballot_sync(0xffffffffu, lane < CS && sv >= thr);
    const int k0 = over ? __ffs(over) - 1 : 0;           // lowest CTA holding a global candidate
    const double* vmsg = slot + (size_t)k0 * msgw;     // its reflector
    int p = (int)vmsg[2];
    bool push = light;   // light: the owner forms and pushes the reflector of p
    if (!(vmsg[1] >= thr)) {
      // near-tie straddling the local and global windows: exchange the exact candidates,
      // then the owner forms and pushes the reflector of the true pivot
      push = true;
      const uint32_t par3 = (uint32_t)(use3[buf]++ & 1);
      if (tid == 0) bar_expect(sm_addr(&sh.bar3[buf]), (uint32_t)(CS * sizeof(CqFb)));
      if (wid == 0) {
        int li = INT_MAX;
        for (int c = lane; c < nw; c += 32)
          if (nu[c] >= thr) {
            li = c;
            break;
          }
        li = wmin_i(li);
        if (lane == 0) {
          sh.mine3[buf].F = li == INT_MAX ? INT_MAX : w_lo + li;
          fence_proxy_async();
        }
        __syncwarp();
        if (lane < CS)
          bulk_push(remote(sm_addr(&sh.slot3[buf][crank]), lane), sm_addr(&sh.mine3[buf]), (uint32_t)sizeof(CqFb),
                    remote(sm_addr(&sh.bar3[buf]), lane));
      }
      bar_wait(sm_addr(&sh.bar3[buf]), par3);
      p = INT_MAX;
      for (int k = 0; k < CS; ++k) p = min(p, sh.slot3[buf][k].F);
    }
    if (push) {
      const int ow = p / wchunk;
      const uint32_t vbytes = (uint32_t)(((8 + m) * 8 + 15) & ~15);
      const uint32_t par2 = (uint32_t)(use2++ & 1);
      if (tid == 0) bar_expect(sm_addr(&sh.bar2), vbytes);
      if (crank == ow && wid == 0) {
        double* src = sh.vstage;
        if (spec_li != INT_MAX && p == w_lo + spec_li) {   // the speculative reflector won
          src = mymsg;
          if (lane == 0) {
            src[3] = spec_tau;
            src[4] = spec_beta;
          }
        } else {
          double tau, beta;
          form_reflector<MR>(Wc(p - ow * wchunk), j, m, lane, sh.vstage, tau, beta);
          if (lane == 0) {
            sh.vstage[2] = (double)p;
            sh.vstage[3] = tau;
            sh.vstage[4] = beta;
          }
        }
        fence_proxy_async();
        __syncwarp();
        if (lane < CS)
          bulk_push(remote(sm_addr(sh.vbuf), lane), sm_addr(src), vbytes, remote(sm_addr(&sh.bar2), lane));
      }
      bar_wait(sm_addr(&sh.bar2), par2);
      vmsg = sh.vbuf;
    }
    const int owner = p / wchunk, ploc = p - owner * wchunk;
    const double tau = vmsg[3], beta = vmsg[4];
    if (crank == owner && wid == 0) {   // the reflector for the apply operators / rotation
      for (int l = lane; l < m; l += 32) it.V[(size_t)j * m + l] = vmsg[8 + l];
      if (lane == 0) {
        it.tau[j] = tau;
        it.piv[j] = dense_col(it, p);
        nu[ploc] = -1.0;   // visible to the other warps after the next step's barrier
      }
    }
    if (j < (trace_fine ? 24 : 60)) CQ_TR(5 + 4 * j);
    // (3) apply H_j to the active columns (two per group in flight), norms over rows > j.
    // v is zero above row j, so rows < j pass through unchanged: every row of the lane is
    // loaded, updated and stored without a row predicate; only the norm is masked (l > j).
    double vr[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) vr[i] = (i < nr) ? vmsg[8 + t + i * G] : 0.0;
    const int gi = (j >= t) ? (j - t) / G + 1 : 0;   // rows l > j of this lane: i >= gi
    lm = -1.0;
    // U columns in flight per group: two up to 8 rows a lane; one at MR = 16 (two need 64
    // registers of column values and spill ~1 KB a thread under the 128-register bound)
    for (int k = 0; k < kiters; k += U) {
      double* cp[U];
      int cxs[U];
      bool act[U], piv[U];
      double x[U][MR], d[U], ss[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int c = grp + (k + u) * NGRP;
        const bool in = (k + u) < kiters && c < nw;
        const int cx = in ? c : 0;
        cxs[u] = cx;
        cp[u] = Wc(cx) + (size_t)t * sr;
        piv[u] = in && crank == owner && c == ploc;
        act[u] = in && !piv[u] && nu[cx] >= 0.0;
        d[u] = 0.0;
#pragma unroll
        for (int i = 0; i < MR; ++i) {
          x[u][i] = (i < nr) ? cp[u][(size_t)i * G * sr] : 0.0;
          d[u] += vr[i] * x[u][i];
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) d[u] = group_sum<G>(d[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double td = tau * d[u];
        ss[u] = 0.0;
        if (act[u]) {
#pragma unroll
          for (int i = 0; i < MR; ++i) {
            const double y = x[u][i] - td * vr[i];
            if (i < nr) cp[u][(size_t)i * G * sr] = y;
            if (i >= gi) ss[u] += y * y;
          }
        } else if (piv[u]) {   // the pivot column: (beta, 0, ..., 0) from row j; out of the search
          if (t == 0) nu[cxs[u]] = -1.0;
#pragma unroll
          for (int i = 0; i < MR; ++i)
            if (i < nr && t + i * G >= j) cp[u][(size_t)i * G * sr] = (t + i * G == j) ? beta : 0.0;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) ss[u] = group_sum<G>(ss[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (act[u]) {
          const double v = sqrt(ss[u]);
          if (t == 0) nu[cxs[u]] = v;
          lm = fmax(lm, v);
        }
    }
    if (j < (trace_fine ? 24 : 60)) CQ_TR(6 + 4 * j);
  }
  CQ_TR(250);
  __syncthreads();
  // ---- coarse-w rows back to global memory (rows [0, r) of the slice) -----------------
  if (!it.dwb || it.keepB)   // (direct write-back: only the debug records need B)
    for (int e = tid; e < r * nw; e += NT) {
      const int l = e / nw, c = e % nw;
      it.B[(size_t)l * ld + w_lo + c] = Wc(c)[l];
    }
  if (it.dwb) {   // ... and straight into the store blocks (s, q), q in w(s); I_r on (s, s)
    for (int c = tid; c < nw; c += NT) {
      const double* src = Wc(c);
      const size_t sst = 1;
      for (int l = 0; l < r; ++l) {
        double* d = dwb_addr(it.seg, it.nseg, w_lo + c, l);
        if (d) *d = src[(size_t)l * sst];
      }
    }
    if (crank == 0)
      for (int e = tid; e < r * r; e += NT) {
        const int i = e / r, j = e % r;
        it.Dss[(size_t)i * it.ldss + j] = (i == j) ? 1.0 : 0.0;
      }
  }
  cl.sync();   // no CTA leaves while another may still copy into its shared memory
  CQ_TR(251);
  if (trace && (long long)blockIdx.x == trace[254] && threadIdx.x == 0) trace[252] = r;
#undef CQ_TR
  if (crank == 0 && tid == 0) *rank_slot = r;
}

// NT threads per CTA, 512 / NT CTAs per SM (<= 128 registers a thread either way): smaller CTAs
// let several clusters' latency-bound step chains share an SM when their slices fit
template <int MR, bool SM, int NT, int U>
__global__ void __launch_bounds__(NT, 512 / NT) k_cpqr3(const CluItem* __restrict__ items, double eps, int relative,
                                                          int32_t* __restrict__ rank_out, long long* trace,
                                                          int light) {
  pdl_trigger();
  pdl_wait();
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int item = blockIdx.x / (int)cl.num_blocks();
  const CluItem it = items[item];
  if ((it.Wt == nullptr) != SM) return;   // the other mode's launch eliminates this cluster
  if (it.m == 0 || it.kw == 0) {   // uniform over the cluster: nobody reaches a cluster barrier
    if (cl.block_rank() == 0 && threadIdx.x == 0) rank_out[item] = 0;
    return;
  }
  extern __shared__ double dsm[];
  __shared__ CqShared sh;
  switch (cq_group(it.m, MR)) {
    case 1: cpqr_body<MR, 1, SM, NT, U>(it, eps, relative, rank_out + item, dsm, sh, trace, light != 0); break;
    case 2: cpqr_body<MR, 2, SM, NT, U>(it, eps, relative, rank_out + item, dsm, sh, trace, light != 0); break;
    case 4: cpqr_body<MR, 4, SM, NT, U>(it, eps, relative, rank_out + item, dsm, sh, trace, light != 0); break;
    case 8: cpqr_body<MR, 8, SM, NT, U>(it, eps, relative, rank_out + item, dsm, sh, trace, light != 0); break;
    case 16: cpqr_body<MR, 16, SM, NT, U>(it, eps, relative, rank_out + item, dsm, sh, trace, light != 0); break;
    default: cpqr_body<MR, 32, SM, NT, U>(it, eps, relative, rank_out + item, dsm, sh, trace, light != 0); break;
  }
}

// a4 on the n-columns: one CTA per tile of NGRP = CQ_THREADS / G columns of one cluster.
template <int MR, int G>
__device__ __forceinline__ void rotate_body(const CluItem& it, int c0, int nc, int r, const double* Vs,
                                            const double* ts, bool tcols) {
  const int m = it.m, ld = tcols ? m : it.ldB;
  const int tid = threadIdx.x, t = tid % G, grp = tid / G;
  const bool act = grp < nc;
  const double* col = tcols ? it.Ginv + c0 + grp : it.B + it.kw + c0 + grp;
  double x[MR];
#pragma unroll
  for (int i = 0; i < MR; ++i) {
    const int l = t + i * G;
    x[i] = (act && l < m) ? col[(size_t)l * ld] : 0.0;
  }
  for (int j = 0; j < r; ++j) {
    const double* v = Vs + (size_t)j * m;
    double vv[MR];
    double d = 0.0;
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int l = t + i * G;
      vv[i] = (l < m) ? v[l] : 0.0;
      d += vv[i] * x[i];
    }
    d = group_sum<G>(d);
    const double td = ts[j] * d;
#pragma unroll
    for (int i = 0; i < MR; ++i) x[i] -= td * vv[i];
  }
  if (tcols) {   // T_s[:, c0 + grp] (row-major m x m)
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int l = t + i * G;
      if (act && l < m) it.Tout[(size_t)l * m + c0 + grp] = x[i];
    }
    return;
  }
  double* colw = const_cast<double*>(col);
  if (!it.dwb || it.keepB)
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int l = t + i * G;
      if (act && l < m) colw[(size_t)l * ld] = x[i];
    }
  if (it.dwb && act) {   // coarse-n rows into the store blocks (s, q), C rows into the slab
    const int jn = c0 + grp;
#pragma unroll
    for (int i = 0; i < MR; ++i) {
      const int l = t + i * G;
      if (l >= m) continue;
      if (l < r) {
        double* d = dwb_addr(it.seg, it.nseg, it.kw + jn, l);
        if (d) *d = x[i];
      } else {
        it.Cout[(size_t)(l - r) * it.ldC + jn] = x[i];
      }
    }
  }
}

template <int MR>
__global__ void __launch_bounds__(CQ_THREADS) k_rotate_n(const CluItem* __restrict__ clu,
                                                         const TrsmItem* __restrict__ items,
                                                         const int32_t* __restrict__ rank, int cap_words) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double rsm[];
  const TrsmItem ti = items[blockIdx.x];
  const CluItem it = clu[ti.ci];
  const int r = rank[ti.ci];
  const bool tcols = ti.pad == 1;   // a tile of T_s = Qᵀ G^{-1}
  if (it.m == 0 || (r == 0 && !it.dwb && !tcols)) return;   // dwb with r = 0: C = B_n still goes to its slab
  // reflectors staged in shared memory when they fit, else read through L1
  const bool staged = (size_t)it.m * r + r <= (size_t)cap_words;
  const double* Vs = it.V;
  const double* ts = it.tau;
  if (staged) {
    for (int e = threadIdx.x; e < it.m * r; e += CQ_THREADS) rsm[e] = it.V[e];
    for (int e = threadIdx.x; e < r; e += CQ_THREADS) rsm[(size_t)it.m * r + e] = it.tau[e];
    __syncthreads();
    Vs = rsm;
    ts = rsm + (size_t)it.m * r;
  }
  switch (cq_group(it.m, MR)) {
    case 1: rotate_body<MR, 1>(it, ti.c0, ti.nc, r, Vs, ts, tcols); break;
    case 2: rotate_body<MR, 2>(it, ti.c0, ti.nc, r, Vs, ts, tcols); break;
    case 4: rotate_body<MR, 4>(it, ti.c0, ti.nc, r, Vs, ts, tcols); break;
    case 8: rotate_body<MR, 8>(it, ti.c0, ti.nc, r, Vs, ts, tcols); break;
    case 16: rotate_body<MR, 16>(it, ti.c0, ti.nc, r, Vs, ts, tcols); break;
    default: rotate_body<MR, 32>(it, ti.c0, ti.nc, r, Vs, ts, tcols); break;
  }
}

// a4 (and T_s = Qᵀ G_s^{-1}) on the FP64 tensor cores: Qᵀ X = H_{r-1} ... H_0 X in panels of
// RW_B reflectors in compact-WY form, H_{j0+b-1} ... H_{j0} = I - V_p T_pᵀ V_pᵀ (T_p upper
// triangular, LAPACK dlarft forward/columnwise), per panel
//     Y = V_pᵀ X (b x NC, K = m: DMMA),   Z = T_pᵀ Y,   X <- X - V_p Z (m x NC, K = b: DMMA).
// One CTA of 8 warps per (cluster, 32-column tile); X stays in shared memory for all panels,
// T_p is formed per tile from the panel's Gram matrix (the panel's reflectors are read once
// per tile from L2).  Same quantity as the reflector-by-reflector rotation, other rounding
// order (DESIGN.md §2 "Rounding order").  m <= 256.
constexpr int RW_NC = 32;        // tile columns
constexpr int RW_B = 16;         // reflectors per panel
constexpr int RW_LDX = RW_NC + 4;   // X row stride (== 4 mod 16 doubles: conflict-free fragments)
constexpr int RW_LDV = RW_B + 4;    // V_p row stride

__device__ __forceinline__ void rw_dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) k_rotate_wy(const CluItem* __restrict__ clu, const TrsmItem* __restrict__ items,
                                                    const int32_t* __restrict__ rank) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double rws[];
  const TrsmItem ti = items[blockIdx.x];
  const CluItem it = clu[ti.ci];
  const int r = rank[ti.ci];
  const bool tcols = ti.pad == 1;   // a tile of T_s = Qᵀ G_s^{-1}
  const int m = it.m;
  if (m == 0 || (r == 0 && !it.dwb && !tcols)) return;
  const int c0 = ti.c0, nc = ti.nc;
  const int mp = (m + 7) & ~7;                    // rows padded to the 8-row DMMA tiles
  double* X = rws;                                // mp x RW_LDX
  double* Vp = X + (size_t)mp * RW_LDX;           // mp x RW_LDV  (V_p, row l, column i)
  double* Tp = Vp + (size_t)mp * RW_LDV;          // RW_B x RW_B  (T_p, upper)
  double* Gm = Tp + RW_B * RW_B;                  // RW_B x RW_B  (Gram V_pᵀ V_p)
  double* Y = Gm + RW_B * RW_B;                   // RW_B x RW_LDX (Y, then Z)
  double* tauv = Y + RW_B * RW_LDX;               // RW_B
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  const double* src = tcols ? it.Ginv + c0 : it.B + it.kw + c0;
  const int lds = tcols ? m : it.ldB;
  for (int e = tid; e < mp * RW_NC; e += 256) {   // X <- the tile (zero-padded)
    const int l = e / RW_NC, c = e % RW_NC;
    X[l * RW_LDX + c] = (l < m && c < nc) ? src[(size_t)l * lds + c] : 0.0;
  }
  for (int j0 = 0; j0 < r; j0 += RW_B) {
    const int b = min(RW_B, r - j0);
    __syncthreads();   // the previous panel's users of Vp / Y are done
    for (int e = tid; e < mp * RW_B; e += 256) {   // V_p: column i = v_{j0+i} (zeros beyond b / m)
      const int i = e / mp, l = e % mp;
      Vp[l * RW_LDV + i] = (i < b && l < m) ? it.V[(size_t)(j0 + i) * m + l] : 0.0;
    }
    if (tid < RW_B) tauv[tid] = tid < b ? it.tau[j0 + tid] : 0.0;
    __syncthreads();
    if (w < 4) {   // Gram matrix V_pᵀ V_p: 2 x 2 tiles of 8 x 8 on warps 0-3 (K = mp, from row j0)
      const int ti8 = w >> 1, tj8 = w & 1;
      double c[2] = {0.0, 0.0};
      for (int k = j0 & ~3; k < mp; k += 4) {
        const double a = Vp[(k + fc) * RW_LDV + 8 * ti8 + fr];
        const double bb = Vp[(k + fc) * RW_LDV + 8 * tj8 + fr];
        rw_dmma(c, a, bb);
      }
      Gm[(8 * ti8 + fr) * RW_B + 8 * tj8 + 2 * fc] = c[0];
      Gm[(8 * ti8 + fr) * RW_B + 8 * tj8 + 2 * fc + 1] = c[1];
    }
    __syncthreads();
    if (w == 0) {   // dlarft: T[i][i] = tau_i, T[0:i, i] = -tau_i T[0:i, 0:i] (V_pᵀ v_i)[0:i]
      for (int i = 0; i < RW_B; ++i) {
        double t = 0.0;
        if (lane < i) {
          for (int q = lane; q < i; ++q) t = fma(Tp[lane * RW_B + q], Gm[q * RW_B + i], t);
          t *= -tauv[i];
        }
        if (lane < RW_B) {
          if (lane < i) Tp[lane * RW_B + i] = t;
          else if (lane == i) Tp[i * RW_B + i] = tauv[i];
          else Tp[lane * RW_B + i] = 0.0;
        }
        __syncwarp();
      }
    }
    // Y = V_pᵀ X: 2 x 4 output tiles of 8 x 8, one per warp, K = mp
    {
      const int ti8 = w >> 2, tn = w & 3;
      double c[2] = {0.0, 0.0};
      for (int k = 0; k < mp; k += 4) {
        const double a = Vp[(k + fc) * RW_LDV + 8 * ti8 + fr];   // A = V_pᵀ: (row i, col k)
        const double bb = X[(k + fc) * RW_LDX + 8 * tn + fr];    // B = X: (k, n)
        rw_dmma(c, a, bb);
      }
      Y[(8 * ti8 + fr) * RW_LDX + 8 * tn + 2 * fc] = c[0];
      Y[(8 * ti8 + fr) * RW_LDX + 8 * tn + 2 * fc + 1] = c[1];
    }
    __syncthreads();
    {   // Z = T_pᵀ Y (in place, by column): Z[i][n] = sum_{k <= i} T[k][i] Y[k][n]
      const int n = tid % RW_NC, i0 = tid / RW_NC;   // 8 row pairs x 32 columns
      double z[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int i = 2 * i0 + h;
        double acc = 0.0;
        for (int k = 0; k <= i; ++k) acc = fma(Tp[k * RW_B + i], Y[k * RW_LDX + n], acc);
        z[h] = acc;
      }
      __syncthreads();
      Y[(2 * i0) * RW_LDX + n] = z[0];
      Y[(2 * i0 + 1) * RW_LDX + n] = z[1];
    }
    __syncthreads();
    // X <- X - V_p Z: (mp / 8) x 4 tiles over the warps, K = RW_B
    for (int t8 = w; t8 < (mp >> 3) * 4; t8 += 8) {
      const int tr = t8 >> 2, tn = t8 & 3;
      double* xp = X + (8 * tr + fr) * RW_LDX + 8 * tn + 2 * fc;
      double c[2] = {xp[0], xp[1]};
#pragma unroll
      for (int k = 0; k < RW_B; k += 4) {
        const double a = -Vp[(8 * tr + fr) * RW_LDV + k + fc];
        const double bb = Y[(k + fc) * RW_LDX + 8 * tn + fr];
        rw_dmma(c, a, bb);
      }
      xp[0] = c[0];
      xp[1] = c[1];
    }
  }
  __syncthreads();
  // epilogue (as rotate_body): T_s tile, or B_n write-back / coarse-n rows to the store / C_s
  for (int e = tid; e < m * nc; e += 256) {
    const int l = e / nc, c = e % nc;
    const double x = X[l * RW_LDX + c];
    if (tcols) {
      it.Tout[(size_t)l * m + c0 + c] = x;
      continue;
    }
    if (!it.dwb || it.keepB) const_cast<double*>(src)[(size_t)l * lds + c] = x;
    if (it.dwb) {
      const int jn = c0 + c;
      if (l < r) {
        double* d = dwb_addr(it.seg, it.nseg, it.kw + jn, l);
        if (d) *d = x;
      } else {
        it.Cout[(size_t)(l - r) * it.ldC + jn] = x;
      }
    }
  }
}

template <int MR, bool SM, int NT, int U = (MR >= 16 ? 1 : 2)>
void launch_one(const CluItem* d_items, int n, int CS, size_t smem, double eps, int relative, int32_t* d_rank,
                cudaStream_t st, long long* trace, bool light) {
  auto kern = k_cpqr3<MR, SM, NT, U>;
  static std::once_flag once;
  std::call_once(once, [&] {
    HS_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    HS_CUDA(cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  });
  cudaLaunchConfig_t cfg{};
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.gridDim = dim3(n * CS);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;   // programmatic dependent launch (pdl_wait precedes every read)
  static const bool cq_log = std::getenv("HS_CQ_LOG") != nullptr;
  if (cq_log) {   // co-resident clusters of this shape (GPC packing)
    int ncl = -1;
    cudaLaunchConfig_t oc = cfg;
    oc.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&ncl, (const void*)kern, &oc) != cudaSuccess) cudaGetLastError();
    std::fprintf(stderr, "[cq log]   max active clusters %d (CS %d, NT %d, smem %zu)\n", ncl, CS, NT, smem);
  }
  HS_CUDA(cudaLaunchKernelEx(&cfg, kern, d_items, eps, relative ? 1 : 0, d_rank, trace, light ? 1 : 0));
  count_launch(1);
}

}  // namespace

// Host side: pick the cluster size CS (smallest power of two whose per-CTA w-slice fits the
// shared-memory target; HS_CPQR_SMEM_KB overrides the 192 KB default), the rows-per-lane
// template (MR = 8 up to m = 256, else 16) and shared vs global mode.
static int cq_mr(int max_m) { return max_m <= 256 ? 8 : 16; }
static constexpr size_t CQ_CAP_BYTES = 200 * 1024 - sizeof(CqShared);

size_t cpqr_global_words(int m, int kw, int max_m) {
  if (m <= 0 || kw <= 0) return 0;
  if (std::getenv("HS_CPQR_GLOBAL") == nullptr &&
      cq_smem_words(m, kw, 16, cq_mr(max_m), true, std::getenv("HS_CPQR_LIGHT") == nullptr ||
                                                      std::atoi(std::getenv("HS_CPQR_LIGHT")) != 0) *
              sizeof(double) <= CQ_CAP_BYTES)
    return 0;
  return (size_t)(kw + 16) * (m + 16);
}

// Host side: two launches per batch, one per mode (a cluster whose w-block does not fit a
// 16-CTA cluster's shared memory runs from its global scratch; the others keep theirs in
// shared memory, so one large cluster no longer moves its whole batch to the slow mode).
// Per launch: the cluster size CS = the smallest power of two whose per-CTA slice fits the
// shared-memory target (HS_CPQR_SMEM_KB overrides the 192 KB default), widened for batches of
// few clusters; the rows-per-lane template MR = 8 up to m = 256, else 16.
int launch_cpqr3(const CluItem* d_items, const std::vector<CluItem>& h_items, double eps, int relative,
                 int32_t* d_rank, cudaStream_t st) {
  const int n = (int)h_items.size();
  if (n <= 0) return 0;
  // read per launch (tests force the modes): HS_CPQR_SMEM_KB = per-CTA slice target
  const size_t target = [] {
    const char* e = std::getenv("HS_CPQR_SMEM_KB");
    return (size_t)(e ? std::atoi(e) : 192) * 1024;
  }();
  int max_m = 0;
  for (const auto& it : h_items) max_m = std::max(max_m, it.m);
  const int MR = cq_mr(max_m);
  static const int nsm = [] {
    int dev = 0, v = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  // HS_CQ_TRACE=k: clock64 timeline of the k-th launch (cluster 0, CTA 0) on stderr
  static const int trace_at = [] {
    const char* e = std::getenv("HS_CQ_TRACE");
    return e ? std::atoi(e) : -1;
  }();
  static std::atomic<int> launches{0};
  int CS_ret = 0;
  for (int mode = 0; mode < 2; ++mode) {   // 0: shared-memory clusters, 1: global-scratch clusters
    const bool sm = mode == 0;
    // light messages (HS_CPQR_LIGHT=1 forces them, =0 forbids them): the global-mode launch
    // always (its slices keep more columns in shared memory), the shared-mode launch when its
    // widest slice does not fit a 16-CTA cluster with the speculative reflector messages
    static const int light_env = [] {
      const char* e = std::getenv("HS_CPQR_LIGHT");
      return e ? std::atoi(e) : -1;
    }();
    bool light = light_env == 1 || (!sm && light_env != 0);
    auto need = [&](int cs) {
      size_t w = 2;
      for (const auto& it : h_items)
        if (it.m > 0 && it.kw > 0 && (it.Wt == nullptr) == sm)
          w = std::max(w, cq_smem_words(it.m, it.kw, cs, MR, sm, light));
      return w * sizeof(double);
    };
    int n_act = 0, max_kw = 0;
    for (const auto& it : h_items)
      if (it.m > 0 && it.kw > 0 && (it.Wt == nullptr) == sm) {
        ++n_act;
        max_kw = std::max(max_kw, it.kw);
      }
    int n_mode = 0;   // the shared-memory launch also writes r = 0 for the empty clusters
    for (const auto& it : h_items) n_mode += (it.Wt == nullptr) == sm;
    if (n_mode == 0) continue;
    int CS = 1;
    while (CS < 16 && need(CS) > std::min(target, CQ_CAP_BYTES)) CS *= 2;
    if (sm && !light && light_env != 0 && need(CS) > std::min(target, CQ_CAP_BYTES)) {
      light = true;
      CS = 1;
      while (CS < 16 && need(CS) > std::min(target, CQ_CAP_BYTES)) CS *= 2;
    }
    // shared mode: smaller CTAs (NT = 256 / 128 threads, 2 / 4 CTAs per SM) when every slice
    // still fits their share of the SM's shared memory at CS <= 16 and the batch fills the
    // GPU: several clusters' step chains then interleave on an SM (HS_CQ_NT forces 128/256/512)
    static const int nt_env = [] {
      const char* e = std::getenv("HS_CQ_NT");
      return e ? std::atoi(e) : 0;
    }();
    int NT = 512;
    if (sm && nt_env != 512) {
      for (int nt : {128, 256}) {
        if (nt_env && nt != nt_env) continue;
        const int B = 512 / nt;
        const size_t lim = (228 * 1024) / B - sizeof(CqShared) - 1024;
        const bool light0 = light;
        int cs = 1;
        while (cs < 16 && need(cs) > lim) cs *= 2;
        if (need(cs) > lim && !light && light_env != 0) {   // light messages may make it fit
          light = true;
          cs = 1;
          while (cs < 16 && need(cs) > lim) cs *= 2;
        }
        if (need(cs) > lim || (!nt_env && (size_t)n_act * std::max(cs, CS) < (size_t)nsm * B)) {
          light = light0;   // does not fit, or a partial wave: keep 512
          continue;
        }
        NT = nt;
        CS = std::max(CS, cs);
        break;
      }
    }
    // a batch of few clusters leaves most SMs idle: split the columns over more CTAs (a
    // shorter update per step for a costlier exchange) while the clusters still fill at most
    // a quarter of the GPU and every CTA keeps >= 128 columns (C2 level 3: CPQR 38 -> 29 ms)
    while (CS < 16 && n_act * CS * 4 <= nsm && max_kw / (2 * CS) >= 128) CS *= 2;
    // global mode is bound by each SM's L2 bandwidth (the slice streams through L2 every
    // step): spread its clusters over as many SMs as the batch leaves free
    // global mode keeps as many columns of each slice in shared memory as fit (hybrid): the
    // widest cluster and all the shared memory, the rest streams through L2 every step
    if (!sm && std::getenv("HS_CPQR_GLOBAL") == nullptr) CS = 16;
    if (!sm)
      while (CS < 16 && n_act * CS * 2 <= nsm && max_kw / (2 * CS) >= 32) CS *= 2;
    size_t smem = sm ? need(CS) : std::max(need(CS), std::min(target, CQ_CAP_BYTES));
    if (!sm && std::getenv("HS_CPQR_GLOBAL")) {   // forced (tests): about half of each slice in shared memory
      size_t half = 0;
      for (const auto& it : h_items)
        if (it.m > 0 && it.kw > 0)
          half = std::max(half, (size_t)cq_ldm(it.m, cq_group(it.m, MR)) * (((it.kw + CS - 1) / CS + 1) / 2));
      smem = std::min(CQ_CAP_BYTES, need(CS) + 8 * half + 16);
    }
    if (smem > CQ_CAP_BYTES) fail(HS_E_UNSUPPORTED, "cpqr: cluster block too large for the shared-memory messages");
    static const bool cq_log = std::getenv("HS_CQ_LOG") != nullptr;
    if (cq_log) {
      int mm = 0;
      double work = 0.0;
      for (const auto& it : h_items)
        if (it.m > 0 && it.kw > 0 && (it.Wt == nullptr) == sm) {
          mm = std::max(mm, it.m);
          work += (double)it.m * it.kw;
        }
      std::fprintf(stderr, "[cq log] launch %d %s%s: items %d active %d CS %d NT %d smem %zu max m %d max kw %d sum m*kw %.3g\n",
                   launches.load(), sm ? "shared" : "global", light ? " light" : "", n, n_act, CS, NT, smem, mm, max_kw, work);
    }
    long long* trace = nullptr;
    if (launches++ == trace_at) {
      HS_CUDA(cudaMalloc(&trace, 256 * sizeof(long long)));
      HS_CUDA(cudaMemsetAsync(trace, 0, 256 * sizeof(long long), st));
      long long tb = 0;   // the first CTA of the first cluster of this launch's mode
      for (int i = 0; i < n; ++i)
        if (h_items[i].m > 0 && h_items[i].kw > 0 && (h_items[i].Wt == nullptr) == sm) {
          tb = (long long)i * CS;
          break;
        }
      HS_CUDA(cudaMemcpyAsync(trace + 254, &tb, sizeof tb, cudaMemcpyHostToDevice, st));
      HS_CUDA(cudaStreamSynchronize(st));
      if (std::getenv("HS_CQ_TRACE_FINE")) {
        static const long long one = 1;
        HS_CUDA(cudaMemcpyAsync(trace + 253, &one, sizeof one, cudaMemcpyHostToDevice, st));
      }
      if (std::getenv("HS_CQ_TRACE_SPLIT")) {
        static const long long one = 1;
        HS_CUDA(cudaMemcpyAsync(trace + 255, &one, sizeof one, cudaMemcpyHostToDevice, st));
      }
    }
    if (MR == 8) {
      if (!sm) launch_one<8, false, 512>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else if (NT == 128) launch_one<8, true, 128>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else if (NT == 256) launch_one<8, true, 256>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else launch_one<8, true, 512>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
    } else if (std::getenv("HS_CQ_U2")) {   // A/B: two columns in flight at MR = 16 (spills)
      if (!sm) launch_one<16, false, 512, 2>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else if (NT == 128) launch_one<16, true, 128, 2>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else if (NT == 256) launch_one<16, true, 256, 2>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else launch_one<16, true, 512, 2>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
    } else {
      if (!sm) launch_one<16, false, 512>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else if (NT == 128) launch_one<16, true, 128>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else if (NT == 256) launch_one<16, true, 256>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
      else launch_one<16, true, 512>(d_items, n, CS, smem, eps, relative, d_rank, st, trace, light);
    }
    CS_ret = std::max(CS_ret, CS);
    if (trace) {
      long long h[256];
      HS_CUDA(cudaMemcpyAsync(h, trace, sizeof h, cudaMemcpyDeviceToHost, st));
      HS_CUDA(cudaStreamSynchronize(st));
      cudaFree(trace);
      const long long t0 = h[0];
      std::fprintf(stderr, "[cq trace] launch %d (%s mode): n=%d active=%d CS=%d smem=%zu max kw %d r=%lld | stage %lld norms %lld cyc\n",
                   trace_at, sm ? "shared" : "global", n, n_act, CS, smem, max_kw, h[252], h[1] - t0, h[2] - h[1]);
      for (int j = 0; j < 60 && h[3 + 4 * j]; ++j)
        std::fprintf(stderr, "[cq trace]  step %2d: B1 %6lld  C1 %6lld  B3 %6lld  upd %6lld\n", j,
                     h[3 + 4 * j] - (j ? h[6 + 4 * (j - 1)] : h[2]), h[4 + 4 * j] - h[3 + 4 * j],
                     h[5 + 4 * j] - h[4 + 4 * j], h[6 + 4 * j] - h[5 + 4 * j]);
      std::fprintf(stderr, "[cq trace]  loop end %lld, exit %lld, total %lld cyc\n", h[250] - t0, h[251] - h[250],
                   h[251] - t0);
      if (std::getenv("HS_CQ_TRACE_FINE"))
        for (int j = 0; j < 12 && h[100 + 8 * j]; ++j)
          std::fprintf(stderr, "[cq fine]  step %2d: sync->w0 %6lld  xnorm %6lld  scalars %6lld  msg %6lld  fence %6lld  push %6lld\n",
                       j, h[100 + 8 * j] - h[3 + 4 * j], h[101 + 8 * j] - h[100 + 8 * j], h[102 + 8 * j] - h[101 + 8 * j],
                       h[103 + 8 * j] - h[102 + 8 * j], h[104 + 8 * j] - h[103 + 8 * j], h[105 + 8 * j] - h[104 + 8 * j]);
    }
  }
  return CS_ret;
}

// rows per lane: 8 up to m = 256 (the kernels' group size G <= 32), else 16
static int rot_mr(int max_m) { return max_m <= 256 ? 8 : 16; }
static bool rot_wy(int max_m) {   // the compact-WY DMMA rotation (HS_ROTATE_LEGACY=1: reflector by reflector)
  static const bool legacy = std::getenv("HS_ROTATE_LEGACY") != nullptr;
  return !legacy && max_m <= 256;
}
int rot_tile_cols(int m, int max_m) {
  return rot_wy(max_m) ? RW_NC : CQ_THREADS / cq_group(std::max(m, 1), rot_mr(max_m));
}

void launch_rotate_n(const CluItem* d_clu, const TrsmItem* d_items, int n, int max_m, const int32_t* d_rank,
                     cudaStream_t st) {
  if (n <= 0) return;
  if (rot_wy(max_m)) {
    const int mp = (max_m + 7) & ~7;
    const size_t smem = sizeof(double) * ((size_t)mp * (RW_LDX + RW_LDV) + 2 * RW_B * RW_B + RW_B * RW_LDX + RW_B);
    static std::once_flag once;
    std::call_once(once, [] {
      HS_CUDA(cudaFuncSetAttribute((const void*)k_rotate_wy, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    launch_pdl(k_rotate_wy, dim3(n), dim3(256), smem, st, d_clu, d_items, (const int32_t*)d_rank);
    count_launch(1);
    return;
  }
  const size_t words = std::min<size_t>((size_t)max_m * max_m + max_m, 24 * 1024);
  const size_t smem = sizeof(double) * words;
  if (max_m <= 256) {
    static std::once_flag once;
    std::call_once(once, [] {
      HS_CUDA(cudaFuncSetAttribute((const void*)k_rotate_n<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    launch_pdl(k_rotate_n<8>, dim3(n), dim3(CQ_THREADS), smem, st, d_clu, d_items, (const int32_t*)d_rank, (int)words);
  } else {
    static std::once_flag once;
    std::call_once(once, [] {
      HS_CUDA(cudaFuncSetAttribute((const void*)k_rotate_n<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    });
    launch_pdl(k_rotate_n<16>, dim3(n), dim3(CQ_THREADS), smem, st, d_clu, d_items, (const int32_t*)d_rank, (int)words);
  }
  count_launch(1);
}

}  // namespace hs
