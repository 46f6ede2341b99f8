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
__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
constexpr int NB_SMEM = 512;   // neighbour tables up to this size are staged in shared memory

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
constexpr int PRE_SMEM = 1024;   // pre-contribution slots staged in shared memory

__device__ __forceinline__ void produce(const ApplyLevelArgs& a, const ApplySrc& S, int K, const double* zf, int g0,
                                        int g1) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = APPLY_THREADS / 32;
  for (int g = g0 + warp; g < g1; g += nw) {
    const Contrib c = a.ctb[g];
    for (int i = lane; i < c.len; i += 32) {
      const double* Ci = S.C + c.col + i;
      double acc = 0.0;
#pragma unroll 4
      for (int k = 0; k < K; ++k) acc += Ci[(int64_t)k * S.ldC] * zf[k];
      a.contrib[c.slot + i] = acc;
    }
    __threadfence();
    __syncwarp();
    if (lane == 0 && c.pre) atomicAdd(a.arr + c.q, 1);
  }
}

__global__ void __launch_bounds__(APPLY_THREADS) k_apply_fwd(ApplyLevelArgs a) {
  __shared__ double ys[MAX_M];
  __shared__ double z[MAX_M];
  __shared__ int64_t pslot[PRE_SMEM];
  __shared__ int s_task;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = APPLY_THREADS / 32;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(a.ticket, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= a.nftask) return;
    const FwdTask tk = a.ftask[t];
    const int s = tk.s;
    const ApplySrc S = a.src[s];
    const int m = S.m, r = S.r, K = m - r;
    if (tk.first) {   // ---- T(s) and s's first contribution group
      for (int e = tid * 16; e < m * m; e += APPLY_THREADS * 16) prefetch_l2(S.T + e);
      if (tk.t_end > tk.t_begin) {
        const Contrib c0 = a.ctb[tk.t_begin], c1 = a.ctb[tk.t_end - 1];
        for (int k = warp; k < K; k += nw)
          for (int c = c0.col + lane * 16; c < c1.col + c1.len; c += 32 * 16) prefetch_l2(S.C + (int64_t)k * S.ldC + c);
      }
      const int npre = S.pre_end - S.pre_begin;
      const bool staged = npre <= PRE_SMEM;
      if (staged)
        for (int e = tid; e < npre; e += APPLY_THREADS) pslot[e] = a.pull[S.pre_begin + e].slot;
      if (tid == 0) wait_ge(a.arr + s, npre);
      __syncthreads();
      for (int i = tid; i < m; i += APPLY_THREADS) {
        double v = __ldcg(S.y + i);
        int e = 0;
        for (; e + 8 <= npre; e += 8) {   // 8 loads in flight, subtracted in order
          double c[8];
#pragma unroll
          for (int u = 0; u < 8; ++u)
            c[u] = __ldcg(a.contrib + (staged ? pslot[e + u] : a.pull[S.pre_begin + e + u].slot) + i);
#pragma unroll
          for (int u = 0; u < 8; ++u) v -= c[u];
        }
        for (; e < npre; ++e) v -= __ldcg(a.contrib + (staged ? pslot[e] : a.pull[S.pre_begin + e].slot) + i);
        ys[i] = v;
      }
      __syncthreads();
      for (int i = warp; i < m; i += nw) {
        const double* Ti = S.T + (int64_t)i * m;
        double acc = 0.0;
        for (int j = lane; j < m; j += 32) acc += Ti[j] * ys[j];
        acc = wsum(acc);
        if (lane == 0) z[i] = acc;
      }
      __syncthreads();
      for (int i = tid; i < r; i += APPLY_THREADS) S.yc[i] = z[i];
      for (int k = tid; k < K; k += APPLY_THREADS) S.yf[k] = z[r + k];
      __threadfence();
      __syncthreads();
      if (tid == 0) atomicExch(a.cnt + s, 1);
      produce(a, S, K, z + r, tk.t_begin, tk.t_end);
    } else {          // ---- P(s, group)
      const Contrib c0 = a.ctb[tk.t_begin], c1 = a.ctb[tk.t_end - 1];
      for (int k = warp; k < K; k += nw)
        for (int c = c0.col + lane * 16; c < c1.col + c1.len; c += 32 * 16) prefetch_l2(S.C + (int64_t)k * S.ldC + c);
      if (tid == 0) wait_ge(a.cnt + s, 1);
      __syncthreads();
      for (int k = tid; k < K; k += APPLY_THREADS) z[k] = __ldcg(S.yf + k);
      __syncthreads();
      produce(a, S, K, z, tk.t_begin, tk.t_end);
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

// Backward sweep of one level (Algorithm 2 backward substitution, reverse batch order).
// Task (s, columns [c0, c0+nc) of C_s): wait for the neighbours eliminated after s whose
// columns overlap the chunk, then partial sums p[k] = sum_c C_s[k][c] x_n[c].  The last
// chunk of s to arrive finishes s: x_f = y_f - sum of the partials (chunk order),
// x_s = T_s^T [x_c; x_f], and publishes done[s].
__global__ void __launch_bounds__(APPLY_THREADS) k_apply_bwd(ApplyLevelArgs a) {
  __shared__ double xn[BWD_COLS];
  __shared__ double u[MAX_M];
  __shared__ int ncol[NB_SMEM];
  __shared__ const double* nx[NB_SMEM];
  __shared__ int s_task, s_last;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = APPLY_THREADS / 32;
  for (;;) {
    if (tid == 0) s_task = atomicAdd(a.ticket + 1, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= a.nbtask) return;
    const BwdTask tk = a.btask[t];
    const ApplySrc S = a.src[tk.s];
    const int m = S.m, r = S.r, K = m - r;
    if (tk.nc > 0) {
      const int c1 = tk.c0 + tk.nc;
      const int nnb = S.nb_end - S.nb_begin;
      const bool staged = nnb <= NB_SMEM;
      for (int b = tid; b < nnb; b += APPLY_THREADS) {   // neighbour table -> smem; wait for later ones
        const BwdNb nb = a.bnb[S.nb_begin + b];
        if (staged) {
          ncol[b] = nb.col;
          nx[b] = nb.x;
        }
        if (nb.later && nb.col < c1 && nb.col + nb.len > tk.c0) wait_ge(a.done + nb.q, 1);
      }
      // prefetch the chunk's rows of C while the neighbours finish
      for (int k = warp; k < K; k += nw)
        for (int c = lane * 16; c < tk.nc; c += 32 * 16) prefetch_l2(S.C + (int64_t)k * S.ldC + tk.c0 + c);
      __syncthreads();
      for (int c = tid; c < tk.nc; c += APPLY_THREADS) {   // gather x_n: owner by binary search
        const int cc = tk.c0 + c;
        int lo = 0, hi = nnb - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          const int col = staged ? ncol[mid] : a.bnb[S.nb_begin + mid].col;
          if (col <= cc) lo = mid;
          else hi = mid - 1;
        }
        const int col = staged ? ncol[lo] : a.bnb[S.nb_begin + lo].col;
        const double* x = staged ? nx[lo] : a.bnb[S.nb_begin + lo].x;
        xn[c] = __ldcg(x + (cc - col));
      }
      __syncthreads();
      double* part = a.parts + S.part + (int64_t)tk.chunk * K;
      for (int k = warp; k < K; k += nw) {
        const double* Ck = S.C + (int64_t)k * S.ldC + tk.c0;
        double acc = 0.0;
        for (int c = lane; c < tk.nc; c += 32) acc += Ck[c] * xn[c];
        acc = wsum(acc);
        if (lane == 0) part[k] = acc;
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) s_last = (atomicAdd(a.bcnt + tk.s, 1) == S.nchunk - 1);
      __syncthreads();
      if (!s_last) continue;
      __threadfence();
    }
    const bool has_parts = tk.nc > 0;
    for (int i = tid; i < r; i += APPLY_THREADS) u[i] = __ldcg(S.yc + i);
    for (int k = tid; k < K; k += APPLY_THREADS) {
      double s = 0.0;
      if (has_parts)
        for (int q = 0; q < S.nchunk; ++q) s += __ldcg(a.parts + S.part + (int64_t)q * K + k);
      u[r + k] = __ldcg(S.yf + k) - s;
    }
    __syncthreads();
    for (int i = tid; i < m; i += APPLY_THREADS) {
      double acc = 0.0;
      for (int j = 0; j < m; ++j) acc += S.T[(int64_t)j * m + i] * u[j];
      S.x[i] = acc;
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) atomicExch(a.done + tk.s, 1);
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

}  // namespace

static int apply_grid(const void* fn, int ntask) {
  static int per_sm[2] = {0, 0}, nsm = 0;
  const int k = fn == (const void*)k_apply_fwd ? 0 : 1;
  if (!per_sm[k]) {
    HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm[k], fn, APPLY_THREADS, 0));
    int dev = 0;
    HS_CUDA(cudaGetDevice(&dev));
    HS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (per_sm[k] <= 0) fail(HS_E_INTERNAL, "apply level kernel does not fit on an SM");
  }
  return std::max(1, std::min(ntask, nsm * per_sm[k]));
}
void launch_apply_fwd_level(const ApplyLevelArgs& a, cudaStream_t st) {
  if (a.nftask <= 0) return;
  k_apply_fwd<<<apply_grid((const void*)k_apply_fwd, a.nftask), APPLY_THREADS, 0, st>>>(a);
  count_launch(1);
}
void launch_apply_post_level(const ApplyLevelArgs& a, cudaStream_t st) {
  if (a.npost <= 0) return;
  k_apply_post<<<a.npost, APPLY_THREADS, 0, st>>>(a);
  count_launch(1);
}
void launch_apply_bwd_level(const ApplyLevelArgs& a, cudaStream_t st) {
  if (a.nbtask <= 0) return;
  k_apply_bwd<<<apply_grid((const void*)k_apply_bwd, a.nbtask), APPLY_THREADS, 0, st>>>(a);
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
