// Solve-phase kernels (sm_100a): Algorithm 2 `Hierarchical_Solve` and the
// CSR SpMV / vector helpers of PCG.  HBM/latency bound: every factor byte is read once
// per sweep.  A cluster's local solve runs in one warp with lane-owned vector entries
// (entry l lives in lane l % 32, slot l / 32), so no block barrier is needed.
#include <cuda_runtime.h>

#include "device.h"

namespace hs {

namespace {


__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---- dependency-driven level sweeps -------------------------------------------------------
// Tasks are claimed in list order through an atomic ticket, so a claimed task only ever
// waits on tasks with smaller tickets, which are held by running CTAs (no co-residency
// assumption, no deadlock).  Producers: write, __threadfence, barrier, one atomic.
// Consumers: acquire-load spin, barrier, then L2 (__ldcg) reads of the vector data.
__device__ __forceinline__ int32_t ld_acquire(const int32_t* p) {
  int32_t v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_ge(const int32_t* p, int32_t v) {
  while (ld_acquire(p) < v) __nanosleep(32);
}
// Forward contribution slots are reset to an all-ones NaN before every apply: no FP64
// arithmetic result has that bit pattern (results are canonical NaNs), so a slot holding
// anything else holds its final value, and a consumer can poll the values themselves
// instead of a counter (no fence or atomic on the producer's path).
constexpr unsigned long long CONTRIB_EMPTY = 0xFFFFFFFFFFFFFFFFull;
__device__ __forceinline__ double ld_poll(const double* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  while (v == CONTRIB_EMPTY) {
    __nanosleep(32);
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  }
  return __longlong_as_double((long long)v);
}
// A NaN produced by the arithmetic (or carried in from a NaN input) is stored as the
// canonical quiet NaN, so no polled value can ever take the all-ones "empty" pattern and a
// consumer never spins on a produced value.
__device__ __forceinline__ double canon(double v) { return isnan(v) ? __longlong_as_double(0x7ff8000000000000LL) : v; }
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

// Forward sweep of one level (Algorithm 2 lines 3-6 for every cluster of the level, in the
// batch order of the factor), produce-then-pull.  Two task kinds, ticketed in elimination
// order (a task only waits on tasks with smaller tickets, held by running CTAs):
//   T(s): wait until every contribution to y_s from sources eliminated before s has
//         arrived (arr[s]), y_s -= those contributions in elimination order, z = T_s y_s,
//         coarse part z[0:r] -> parent vector, y_f = z[r:m] -> fine buffer, publish cnt[s];
//   P(s, group): wait for cnt[s], then contrib(s -> q) = C_s[:, cols(q)]^T y_f for the
//         group's targets (a warp per target), count them into arr[q].
// The contributions to clusters eliminated before their source (their coarse parts) are
// subtracted by k_apply_post after the level.  Every entry is accumulated in the factor's
// event order, so the sweep is deterministic and equal to the sequential Algorithm 2 loop;
// no target waits on another target's update.
__device__ __forceinline__ long long gtime() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define AP_TR(t, k)                                            \
  do {                                                         \
    if (a.trace && threadIdx.x == 0) a.trace[(int64_t)(t) * 8 + (k)] = gtime(); \
  } while (0)
constexpr int PRE_SMEM = 1024;   // pre-contribution slots staged in shared memory

// contrib(s -> q) = C_s[:, cols(q)]^T y_f for the group's targets (a warp per target); the
// first nst targets read C from shared memory (sC + soff[j], ld = the target's width)
__device__ __forceinline__ void produce(const ApplyLevelArgs& a, const ApplySrc& S, int K, const double* zf, int g0,
                                        int g1, const double* sC = nullptr, const int* soff = nullptr, int nst = 0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = APPLY_THREADS / 32;
  for (int g = g0 + warp; g < g1; g += nw) {
    const Contrib c = a.ctb[g];
    const bool st = g - g0 < nst;
    for (int i = lane; i < c.dlen; i += 32) {
      double acc = 0.0;
      const int cc = c.inv ? c.inv[i] : i;   // the entry's column among q's columns of C_s (< 0: zero)
      if (cc < 0) {
      } else if (st) {
        const double* Ci = sC + soff[g - g0] + cc;
        for (int k = 0; k < K; ++k) acc += Ci[k * c.len] * zf[k];
      } else {
        const double* Ci = S.C + c.col + cc;
        int k = 0;
        for (; k + 8 <= K; k += 8) {   // 8 loads in flight, accumulated in k order
          double cv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) cv[u] = Ci[(int64_t)(k + u) * S.ldC];
#pragma unroll
          for (int u = 0; u < 8; ++u) acc += cv[u] * zf[k + u];
        }
        for (; k < K; ++k) acc += Ci[(int64_t)k * S.ldC] * zf[k];
      }
      asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(a.contrib + c.slot + i), "d"(canon(acc)) : "memory");
    }
  }
}

// the L2 lines of a contribution group's columns of C_s (targets in any column order)
__device__ __forceinline__ void prefetch_group(const ApplyLevelArgs& a, const ApplySrc& S, int K, int g0, int g1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = APPLY_THREADS / 32;
  for (int g = g0; g < g1; ++g) {
    const Contrib c = a.ctb[g];
    for (int k = warp; k < K; k += nw)
      for (int cc = lane * 16; cc < c.len; cc += 32 * 16) prefetch_l2(S.C + (int64_t)k * S.ldC + c.col + cc);
  }
}

constexpr int PRE_BUF = 1024;   // pre-contribution values staged per round (doubles)
static_assert(MAX_M < PRE_BUF, "a round holds at least one contribution");
constexpr int PSUM = 512;       // partial sums of a round (np x m)
constexpr int FWD_STAGE = 3072; // T_s and the first targets' C columns, loaded while T(s) waits (doubles)

__global__ void __launch_bounds__(APPLY_THREADS) k_apply_fwd(ApplyLevelArgs a) {
  __shared__ double ys[MAX_M];
  __shared__ double z[MAX_M];
  __shared__ int64_t pslot[PRE_SMEM];
  __shared__ double pbuf[PRE_BUF];
  __shared__ double psum[PSUM];
  __shared__ int s_task;
  __shared__ int soff[16];
  extern __shared__ double stg[];   // FWD_STAGE doubles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = APPLY_THREADS / 32;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= a.nftask) return;
    AP_TR(t, 0);
    const FwdTask tk = a.ftask[t];
    const int s = tk.s;
    const ApplySrc S = a.src[s];
    const int m = S.m, r = S.r, K = m - r;
    if (tk.first) {   // ---- T(s) and s's first contribution group
      // while the contributions to y_s are outstanding: T_s and the C columns of the first
      // targets (the next hops of the chain) into shared memory, the rest into L2
      const bool tst = m * m <= FWD_STAGE;
      int used = tst ? m * m : 0, nst = 0;
      for (int g = tk.t_begin; g < tk.t_end && nst < 16; ++g) {
        const int len = a.ctb[g].len;
        if (used + K * len > FWD_STAGE) break;
        if (tid == 0) soff[nst] = used;
        used += K * len;
        ++nst;
      }
      if (tst)
        for (int e = tid; e < m * m; e += APPLY_THREADS) stg[e] = S.T[e];
      else
        for (int e = tid * 16; e < m * m; e += APPLY_THREADS * 16) prefetch_l2(S.T + e);
      {
        int off = tst ? m * m : 0;
        for (int j = 0; j < nst; ++j) {
          const Contrib c = a.ctb[tk.t_begin + j];
          for (int e = tid; e < K * c.len; e += APPLY_THREADS) {
            const int k = e / c.len, i = e - k * c.len;
            stg[off + e] = S.C[(int64_t)k * S.ldC + c.col + i];
          }
          off += K * c.len;
        }
      }
      prefetch_group(a, S, K, tk.t_begin + nst, tk.t_end);
      const int npre = S.pre_end - S.pre_begin;
      const bool staged = npre <= PRE_SMEM;
      if (staged)
        for (int e = tid; e < npre; e += APPLY_THREADS) pslot[e] = a.pull[S.pre_begin + e].slot;
      __syncthreads();
      AP_TR(t, 1);
      // y_s minus its pre-contributions in elimination order: rounds of up to PRE_BUF values
      // loaded by the whole CTA at once, then summed per entry from shared memory
      const int per = PRE_BUF / max(m, 1);   // m <= MAX_M < PRE_BUF
      // entry i's values of a round are summed by np threads (interleaved subsets, each in
      // order), then combined in subset order: a fixed order for a given m (deterministic)
      const int np = max(1, min(APPLY_THREADS / max(m, 1), (int)(PSUM / max(m, 1))));
      {
        for (int i = tid; i < m; i += APPLY_THREADS) ys[i] = __ldcg(S.y + i);
        for (int e0 = 0; e0 < npre; e0 += per) {
          const int ne = min(per, npre - e0);
          for (int x = tid; x < ne * m; x += APPLY_THREADS) {
            const int e = e0 + x / m, i = x % m;
            const double* src = a.contrib + (staged ? pslot[e] : a.pull[S.pre_begin + e].slot) + i;
            pbuf[x] = ld_poll(src);
          }
          __syncthreads();
          if (np > 1) {
            if (tid < np * m) {
              const int i = tid % m, pp = tid / m;
              double v = 0.0;
              for (int e = pp; e < ne; e += np) v += pbuf[e * m + i];
              psum[pp * m + i] = v;
            }
            __syncthreads();
            for (int i = tid; i < m; i += APPLY_THREADS) {
              double v = ys[i];
              for (int pp = 0; pp < np; ++pp) v -= psum[pp * m + i];
              ys[i] = v;
            }
          } else {
            for (int i = tid; i < m; i += APPLY_THREADS) {
              double v = ys[i];
              for (int e = 0; e < ne; ++e) v -= pbuf[e * m + i];
              ys[i] = v;
            }
          }
          __syncthreads();
        }
      }
      __syncthreads();
      AP_TR(t, 2);
      for (int i = warp; i < m; i += nw) {
        const double* Ti = tst ? stg + i * m : S.T + (int64_t)i * m;
        double acc = 0.0;
        for (int j = lane; j < m; j += 32) acc += Ti[j] * ys[j];
        acc = wsum(acc);
        if (lane == 0) z[i] = acc;
      }
      __syncthreads();
      // the first group (the targets eliminated soonest: the next hop of the chain) before
      // the outputs that only the other groups and the parent level read
      AP_TR(t, 3);
      produce(a, S, K, z + r, tk.t_begin, tk.t_end, stg, soff, nst);
      AP_TR(t, 4);
      for (int i = tid; i < r; i += APPLY_THREADS) S.yc[i] = z[i];
      for (int k = tid; k < K; k += APPLY_THREADS) S.yf[k] = z[r + k];
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicExch(a.cnt + s, 1);
      AP_TR(t, 5);
    } else {          // ---- P(s, group)
      prefetch_group(a, S, K, tk.t_begin, tk.t_end);
      if (tid == 0) wait_ge(a.cnt + s, 1);
      __syncthreads();
      AP_TR(t, 1);
      for (int k = tid; k < K; k += APPLY_THREADS) z[k] = __ldcg(S.yf + k);
      __syncthreads();
      produce(a, S, K, z, tk.t_begin, tk.t_end);
      AP_TR(t, 5);
    }
    __syncthreads();   // s_task, ys, z reusable
  }
}

// Contributions to the coarse parts of clusters eliminated before their sources
// (Algorithm 2: y_q -= C^T y_f for processed q), every one of the level being final.
__global__ void __launch_bounds__(APPLY_THREADS) k_apply_post(ApplyLevelArgs a) {
  const int q = a.post_cl[blockIdx.x];
  const ApplySrc Q = a.src[q];
  for (int i = threadIdx.x; i < Q.r; i += APPLY_THREADS) {
    double v = Q.yc[i];
    for (int e = Q.post_begin; e < Q.post_end; ++e) v -= a.contrib[a.pull[e].slot + i];
    Q.yc[i] = v;
  }
}

constexpr int BWD_STAGE = 4096;    // C columns of a chunk, then T_s + partials for the finish (doubles)

// Backward sweep of one level (Algorithm 2 backward substitution, reverse batch order).
// Task (s, neighbours bnb[b0, b1) of s): the chunk's columns of C_s go to shared memory
// while the later neighbours finish; once their x values appear (polled: x starts empty),
// partial sums p[k] = sum over the chunk's columns c of C_s[k][c] x_n[c].  The chunks
// follow the neighbours' readiness (host plan) and the LAST chunk of s — the one waiting
// for the neighbour that finishes last — finishes s: it polls the other chunks' partials
// (they start empty too), x_f = y_f - sum of the partials (chunk order),
// x_s = T_s^T [x_c; x_f].  No fences, counters or flags on the chain: every value a task
// waits for is polled directly.  A chunk only waits on tasks with smaller tickets.
__global__ void __launch_bounds__(APPLY_THREADS) k_apply_bwd(ApplyLevelArgs a) {
  __shared__ double xn[BWD_COLS];
  __shared__ int ccol[BWD_COLS];
  __shared__ double u[MAX_M];
  __shared__ double pown[MAX_M];   // the finisher's own partial
  __shared__ int s_task;
  extern __shared__ double bst[];  // BWD_STAGE doubles
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = APPLY_THREADS / 32;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(a.ticket + 1, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= a.nbtask) return;
    const int tt = a.nftask + t;
    AP_TR(tt, 0);
    const BwdTask tk = a.btask[t];
    const ApplySrc S = a.src[tk.s];
    const int m = S.m, r = S.r, K = m - r;
    const bool fin = tk.chunk == S.nchunk - 1;
    const bool has_parts = tk.nc > 0;
    const bool cst = has_parts && K * tk.nc <= BWD_STAGE;
    // shared-memory stage: [the chunk's C columns | T_s | the other chunks' partials]
    const int coff = cst ? K * tk.nc : 0;
    const bool tst = coff + m * m <= BWD_STAGE;
    double* tS = bst + coff;
    const int np = has_parts ? (S.nchunk - 1) * K : 0;
    double* pS = bst + coff + (tst ? m * m : 0);
    const bool pst = coff + (tst ? m * m : 0) + np <= BWD_STAGE;
    if (fin) {   // the finisher's inputs that are final already: x_c, y_f, T_s (before any wait)
      for (int i = tid; i < r; i += APPLY_THREADS) u[i] = __ldcg(S.xc + i);
      for (int k = tid; k < K; k += APPLY_THREADS) u[r + k] = __ldcg(S.yf + k);
      if (tst)
        for (int e = tid; e < m * m; e += APPLY_THREADS) tS[e] = S.T[e];
    }
    if (has_parts) {
      const int nnb = tk.b1 - tk.b0;
      for (int b = warp; b < nnb; b += nw) {   // column map (+ the chunk's C columns)
        const BwdNb nb = a.bnb[tk.b0 + b];
        for (int i = lane; i < nb.len; i += 32) ccol[nb.off + i] = nb.col + i;
      }
      __syncthreads();
      if (cst) {
        for (int e = tid; e < K * tk.nc; e += APPLY_THREADS) {
          const int k = e / tk.nc, c = e - k * tk.nc;
          bst[e] = S.C[(int64_t)k * S.ldC + ccol[c]];
        }
      } else {
        for (int b = 0; b < nnb; ++b) {
          const BwdNb nb = a.bnb[tk.b0 + b];
          for (int k = warp; k < K; k += nw)
            for (int c = lane * 16; c < nb.len; c += 32 * 16) prefetch_l2(S.C + (int64_t)k * S.ldC + nb.col + c);
        }
      }
      for (int b = tid; b < nnb; b += APPLY_THREADS) {   // one waiter per later neighbour
        const BwdNb nb = a.bnb[tk.b0 + b];
        if (nb.later) ld_poll(nb.x);
      }
      __syncthreads();
      AP_TR(tt, 1);
      for (int b = warp; b < nnb; b += nw) {   // gather x_n (final once not empty)
        const BwdNb nb = a.bnb[tk.b0 + b];
        for (int i = lane; i < nb.len; i += 32) xn[nb.off + i] = ld_poll(nb.x + (nb.sup ? nb.sup[i] : i));
      }
      __syncthreads();
      double* part = a.parts + S.part + (int64_t)tk.chunk * K;
      for (int k = warp; k < K; k += nw) {
        double acc = 0.0;
        if (cst) {
          const double* Ck = bst + k * tk.nc;
          for (int c = lane; c < tk.nc; c += 32) acc += Ck[c] * xn[c];
        } else {
          const double* Ck = S.C + (int64_t)k * S.ldC;
          int c = lane;
          for (; c + 32 * 7 < tk.nc; c += 32 * 8) {   // 8 loads in flight, accumulated in c order
            double cv[8];
#pragma unroll
            for (int w = 0; w < 8; ++w) cv[w] = Ck[ccol[c + 32 * w]];
#pragma unroll
            for (int w = 0; w < 8; ++w) acc += cv[w] * xn[c + 32 * w];
          }
          for (; c < tk.nc; c += 32) acc += Ck[ccol[c]] * xn[c];
        }
        acc = wsum(acc);
        if (lane == 0) {
          if (fin) pown[k] = acc;
          else asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(part + k), "d"(canon(acc)) : "memory");
        }
      }
      AP_TR(tt, 2);
      if (!fin) {
        __syncthreads();   // bst, ccol, xn reusable
        continue;
      }
    }
    // ---- finish s: the other chunks' partials (polled), x_f = y_f - their sum (chunk
    // order), x_s = T_s^T [x_c; x_f]
    if (pst)
      for (int e = tid; e < np; e += APPLY_THREADS) pS[e] = ld_poll(a.parts + S.part + e);
    __syncthreads();
    if (has_parts)
      for (int k = tid; k < K; k += APPLY_THREADS) {
        double s = 0.0;
        for (int q = 0; q < S.nchunk - 1; ++q) s += pst ? pS[q * K + k] : ld_poll(a.parts + S.part + (int64_t)q * K + k);
        s += pown[k];
        u[r + k] -= s;
      }
    __syncthreads();
    const double* Tm = tst ? tS : S.T;
    for (int i = tid; i < m; i += APPLY_THREADS) {
      double acc = 0.0;
      int j = 0;
      for (; j + 8 <= m; j += 8) {   // 8 loads in flight, accumulated in j order
        double tv[8];
#pragma unroll
        for (int w = 0; w < 8; ++w) tv[w] = Tm[(int64_t)(j + w) * m + i];
#pragma unroll
        for (int w = 0; w < 8; ++w) acc += tv[w] * u[j + w];
      }
      for (; j < m; ++j) acc += Tm[(int64_t)j * m + i] * u[j];
      asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(S.x + i), "d"(canon(acc)) : "memory");
    }
    AP_TR(tt, 3);
    __syncthreads();   // u, bst reusable
  }
}

// top: y <- L^{-T} L^{-1} y with the storage of dense_potrf (diagonal NB-blocks lower G_kk,
// off-diagonal U = L^T in the block rows to the right).  One CTA, column-oriented sweeps.
__device__ __forceinline__ double Lval(const double* A, int ld, int i, int l) {  // L[i][l], i >= l
  return (i / TOP_NB == l / TOP_NB) ? A[(int64_t)i * ld + l] : A[(int64_t)l * ld + i];
}
__global__ void k_top_solve(double* y, const double* A, int N, int ld) {
  for (int l = 0; l < N; ++l) {
    __syncthreads();
    const double yl = y[l] / A[(int64_t)l * ld + l];
    __syncthreads();
    if (threadIdx.x == 0) y[l] = yl;
    for (int i = l + 1 + threadIdx.x; i < N; i += blockDim.x) y[i] -= Lval(A, ld, i, l) * yl;
  }
  for (int l = N - 1; l >= 0; --l) {
    __syncthreads();
    const double xl = y[l] / A[(int64_t)l * ld + l];
    __syncthreads();
    if (threadIdx.x == 0) y[l] = xl;
    for (int i = threadIdx.x; i < l; i += blockDim.x) y[i] -= Lval(A, ld, l, i) * xl;
  }
}

__global__ void k_permute(const double* __restrict__ src, double* __restrict__ dst, const int64_t* __restrict__ idx,
                          int64_t n, int scatter) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (scatter) dst[idx[i]] = src[i];
    else dst[i] = src[idx[i]];
  }
}

// CSR SpMV, 8 lanes per row (rows have <= 54 entries on the configs)
__global__ void k_spmv(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ colind,
                       const double* __restrict__ vals, const double* __restrict__ x, double* __restrict__ y,
                       int64_t n) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t row = g >> 3;
  const int sub = threadIdx.x & 7;
  double acc = 0.0;
  if (row < n) {
    const int64_t b = rowptr[row], e = rowptr[row + 1];
    for (int64_t k = b + sub; k < e; k += 8) acc += vals[k] * __ldg(x + colind[k]);
  }
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (row < n && sub == 0) y[row] = acc;
}

// ---- batch-synchronous sweeps (levels of large batches) -----------------------------------
// One launch per batch of the factor's schedule, a CTA per cluster of the batch, no waiting:
// every value a cluster reads (its pre-contributions forward, its neighbours' x backward) was
// written by an earlier launch.  The factor records stream from HBM with the loads of the
// whole CTA in flight: T_s row by row (a warp per 4 rows, coalesced), C_s column-parallel
// (a thread per contribution entry, the K rows unrolled by 8) forward and row-parallel (a warp
// per 4 rows) backward.  Same sums in a fixed order (deterministic).
constexpr int BSF_PRE = 4096;   // pre-contribution values staged per round (doubles)

__global__ void __launch_bounds__(APPLY_THREADS) k_apply_fwd_b(ApplyLevelArgs a, const int32_t* __restrict__ cl) {
  __shared__ double ys[MAX_M], yf[MAX_M];
  __shared__ double pv[BSF_PRE];
  __shared__ int gpre[BS_MAXG + 1];
  const int s = cl[blockIdx.x];
  const ApplySrc S = a.src[s];
  const int m = S.m, r = S.r, K = m - r;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (m == 0) return;
  for (int i = tid; i < m; i += APPLY_THREADS) ys[i] = __ldcg(S.y + i);
  // y_s minus its pre-contributions in elimination order (staged round by round)
  const int npre = S.pre_end - S.pre_begin, per = max(1, BSF_PRE / m);
  for (int e0 = 0; e0 < npre; e0 += per) {
    const int ne = min(per, npre - e0);
    __syncthreads();
    for (int x = tid; x < ne * m; x += APPLY_THREADS) {
      const int e = e0 + x / m, i = x % m;
      pv[x] = __ldcg(a.contrib + a.pull[S.pre_begin + e].slot + i);
    }
    __syncthreads();
    for (int i = tid; i < m; i += APPLY_THREADS) {
      double v = ys[i];
      for (int e = 0; e < ne; ++e) v -= pv[e * m + i];
      ys[i] = v;
    }
  }
  const int ng = S.tg_end - S.tg_begin;
  if (tid == 0) {   // flattened (contribution, entry) index of the producing phase
    int acc = 0;
    for (int g = 0; g < ng; ++g) {
      gpre[g] = acc;
      acc += a.ctb[S.tg_begin + g].dlen;
    }
    gpre[ng] = acc;
  }
  __syncthreads();
  // z = T_s y_s: a warp per 4 rows
  for (int i0 = 4 * warp; i0 < m; i0 += 4 * (APPLY_THREADS / 32)) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = lane; j < m; j += 32) {
      const double yj = ys[j];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u < m) acc[u] += S.T[(int64_t)(i0 + u) * m + j] * yj;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double v = wsum(acc[u]);
      const int i = i0 + u;
      if (lane == 0 && i < m) {
        if (i < r) S.yc[i] = v;
        else {
          yf[i - r] = v;
          S.yf[i - r] = v;
        }
      }
    }
  }
  __syncthreads();
  // contributions C_s[:, cols(q)]ᵀ y_f: a thread per entry
  const int tot = gpre[ng];
  for (int t = tid; t < tot; t += APPLY_THREADS) {
    int lo = 0, hi = ng - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (gpre[mid] <= t) lo = mid;
      else hi = mid - 1;
    }
    const Contrib c = a.ctb[S.tg_begin + lo];
    const int i = t - gpre[lo];
    const int cc = c.inv ? c.inv[i] : i;   // (< 0: an unsupported entry, zero)
    const double* Ci = S.C + c.col + max(cc, 0);
    double acc = 0.0;
    int k = cc < 0 ? K : 0;
    for (; k + 8 <= K; k += 8) {
      double cv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cv[u] = Ci[(int64_t)(k + u) * S.ldC];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc += cv[u] * yf[k + u];
    }
    for (; k < K; ++k) acc += Ci[(int64_t)k * S.ldC] * yf[k];
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(a.contrib + c.slot + i), "d"(canon(acc)) : "memory");
  }
}

__global__ void __launch_bounds__(APPLY_THREADS) k_apply_bwd_b(ApplyLevelArgs a, const int32_t* __restrict__ cl) {
  __shared__ double u[MAX_M];
  __shared__ double xn[BS_MAXCOLS];
  const int s = cl[blockIdx.x];
  const ApplySrc S = a.src[s];
  const int m = S.m, r = S.r, K = m - r;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = APPLY_THREADS / 32;
  if (m == 0) return;
  for (int i = tid; i < r; i += APPLY_THREADS) u[i] = __ldcg(S.xc + i);
  for (int k = tid; k < K; k += APPLY_THREADS) u[r + k] = __ldcg(S.yf + k);
  int kn = 0;
  for (int b = S.nb_begin; b < S.nb_end; ++b) kn = max(kn, a.bnb[b].col + a.bnb[b].len);
  for (int b = S.nb_begin + warp; b < S.nb_end; b += nw) {   // x of the neighbours' columns
    const BwdNb nb = a.bnb[b];
    for (int i = lane; i < nb.len; i += 32) xn[nb.col + i] = __ldcg(nb.x + (nb.sup ? nb.sup[i] : i));
  }
  __syncthreads();
  // x_f = y_f - C_s x_n: a warp per 4 rows of C_s
  for (int k0 = 4 * warp; k0 < K && kn > 0; k0 += 4 * nw) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int c = lane; c < kn; c += 32) {
      const double xc = xn[c];
#pragma unroll
      for (int v = 0; v < 4; ++v)
        if (k0 + v < K) acc[v] += S.C[(int64_t)(k0 + v) * S.ldC + c] * xc;
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double w = wsum(acc[v]);
      if (lane == 0 && k0 + v < K) u[r + k0 + v] -= w;
    }
  }
  __syncthreads();
  // x_s = T_sᵀ [x_c; x_f]: a thread per entry, T_s rows coalesced
  for (int i = tid; i < m; i += APPLY_THREADS) {
    double acc = 0.0;
    int j = 0;
    for (; j + 8 <= m; j += 8) {
      double tv[8];
#pragma unroll
      for (int w = 0; w < 8; ++w) tv[w] = S.T[(int64_t)(j + w) * m + i];
#pragma unroll
      for (int w = 0; w < 8; ++w) acc += tv[w] * u[j + w];
    }
    for (; j < m; ++j) acc += S.T[(int64_t)j * m + i] * u[j];
    asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(S.x + i), "d"(canon(acc)) : "memory");
  }
}

}  // namespace

static int apply_grid(const void* fn, int ntask) {
  static int per_sm[2] = {0, 0}, nsm = 0;
  const int k = fn == (const void*)k_apply_fwd ? 0 : 1;
  if (!per_sm[k]) {
    const size_t dyn = sizeof(double) * (k == 0 ? FWD_STAGE : BWD_STAGE);
    if (dyn) set_smem_attr(fn, dyn);
    HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[k], fn, APPLY_THREADS, dyn));
    int dev = 0;
    HS_CUDA(cudaGetDevice(&dev));
    HS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm[k] <= 0) fail(HS_E_INTERNAL, "apply level kernel does not fit on an SM");
  }
  return std::max(1, std::min(ntask, nsm * per_sm[k]));
}
void launch_apply_fwd_level(const ApplyLevelArgs& a, cudaStream_t st) {
  if (a.nftask <= 0) return;
  k_apply_fwd<<<apply_grid((const void*)k_apply_fwd, a.nftask), APPLY_THREADS, sizeof(double) * FWD_STAGE, st>>>(a);
  count_launch(1);
}
void launch_apply_post_level(const ApplyLevelArgs& a, cudaStream_t st) {
  if (a.npost <= 0) return;
  k_apply_post<<<a.npost, APPLY_THREADS, 0, st>>>(a);
  count_launch(1);
}
void launch_apply_bwd_level(const ApplyLevelArgs& a, cudaStream_t st) {
  if (a.nbtask <= 0) return;
  k_apply_bwd<<<apply_grid((const void*)k_apply_bwd, a.nbtask), APPLY_THREADS,
                sizeof(double) * BWD_STAGE, st>>>(a);
  count_launch(1);
}

void launch_apply_fwd_batch(const ApplyLevelArgs& a, const int32_t* d_cl, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_apply_fwd_b<<<n, APPLY_THREADS, 0, st>>>(a, d_cl);
  count_launch(1);
}
void launch_apply_bwd_batch(const ApplyLevelArgs& a, const int32_t* d_cl, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_apply_bwd_b<<<n, APPLY_THREADS, 0, st>>>(a, d_cl);
  count_launch(1);
}

void launch_top_solve(double* y, const double* A, int N, int ld, cudaStream_t st) {
  if (N <= 0) return;
  k_top_solve<<<1, 1024, 0, st>>>(y, A, N, ld);
  count_launch(1);
}
void launch_permute(const double* src, double* dst, const int64_t* idx, int64_t n, int scatter, cudaStream_t st) {
  if (n <= 0) return;
  k_permute<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 8), 256, 0, st>>>(src, dst, idx, n, scatter);
  count_launch(1);
}
void launch_spmv(const int64_t* rowptr, const int32_t* colind, const double* vals, const double* x, double* y,
                 int64_t n, cudaStream_t st) {
  if (n <= 0) return;
  k_spmv<<<(int)((n * 8 + 255) / 256), 256, 0, st>>>(rowptr, colind, vals, x, y, n);
  count_launch(1);
}

}  // namespace hs
