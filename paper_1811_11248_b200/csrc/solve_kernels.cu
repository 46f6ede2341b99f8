// Solve-phase kernels (sm_100a): Algorithm 2 `Hierarchical_Solve` and the
// CSR SpMV / vector helpers of PCG.  HBM/latency bound: every factor byte is read once
// per sweep.  A cluster's local solve runs in one warp with lane-owned vector entries
// (entry l lives in lane l % 32, slot l / 32), so no block barrier is needed.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include "device.h"

namespace hs {

namespace {


__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// y <- G^{-1} y (G lower, row-major ld m): row-oriented, coalesced row reads
template <int SLOTS>
__device__ __forceinline__ void warp_trsv_lower(const double* G, int m, double (&y)[SLOTS], int lane) {
  for (int i = 0; i < m; ++i) {
    double p = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int l = lane + 32 * s;
      if (l < i) p += G[(int64_t)i * m + l] * y[s];
    }
    p = wsum(p);
    if ((i & 31) == lane) {
      const double gi = G[(int64_t)i * m + i];
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
        if (s == (i >> 5)) y[s] = (y[s] - p) / gi;
    }
  }
}

// y <- G^{-T} y : column-oriented backward substitution, rows of G read contiguously
template <int SLOTS>
__device__ __forceinline__ void warp_trsv_upper_t(const double* G, int m, double (&y)[SLOTS], int lane) {
  for (int i = m - 1; i >= 0; --i) {
    double xi = 0.0;
#pragma unroll
    for (int s = 0; s < SLOTS; ++s)
      if (s == (i >> 5)) xi = y[s];
    xi = __shfl_sync(0xffffffffu, xi, i & 31);
    xi /= G[(int64_t)i * m + i];
    if ((i & 31) == lane) {
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
        if (s == (i >> 5)) y[s] = xi;
    }
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int l = lane + 32 * s;
      if (l < i) y[s] -= G[(int64_t)i * m + l] * xi;
    }
  }
}

// apply H_j (j = 0..r-1 forward, r-1..0 backward): y[j:] -= tau_j v_j (v_j . y[j:])
template <int SLOTS>
__device__ __forceinline__ void warp_reflect(const double* V, const double* tau, int m, int j, double (&y)[SLOTS],
                                             int lane) {
  const double t = tau[j];
  if (t == 0.0) return;
  double d = 0.0;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int l = lane + 32 * s;
    if (l >= j && l < m) d += V[(int64_t)j * m + l] * y[s];
  }
  d = wsum(d) * t;
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    const int l = lane + 32 * s;
    if (l >= j && l < m) y[s] -= d * V[(int64_t)j * m + l];
  }
}

// Stage G (m x m), V (m x r) and tau (r) of a cluster in shared memory at `sm` when they
// fit in `cap` doubles (one coalesced pass by the whole CTA instead of a latency-bound
// chain of dependent global loads in the warp solve); returns the pointers to use.
__device__ __forceinline__ void stage_local(const ApplyLocal& it, double* sm, int64_t cap, const double*& G,
                                            const double*& V, const double*& tau) {
  const int64_t mm = (int64_t)it.m * it.m, mr = (int64_t)it.m * it.r;
  G = it.G;
  V = it.V;
  tau = it.tau;
  if (mm + mr + it.r > cap) return;
  for (int64_t e = threadIdx.x; e < mm; e += blockDim.x) sm[e] = it.G[e];
  for (int64_t e = threadIdx.x; e < mr; e += blockDim.x) sm[mm + e] = it.V[e];
  for (int e = threadIdx.x; e < it.r; e += blockDim.x) sm[mm + mr + e] = it.tau[e];
  G = sm;
  V = sm + mm;
  tau = sm + mm + mr;
}

// The vector y (and the backward partial sums) change inside a level kernel, so they are
// read with __ldcg (L2, bypassing the non-coherent L1); factor data are read normally.
// forward: y_s <- U^T G^{-1} y_s (S_s then E_s of W_s = P_s G_s E_s S_s).
// CTA-level device function (every thread of the CTA calls it): the CTA stages the
// factors, warp 0 solves.  `sm` is the CTA's dynamic shared memory (cap doubles).
template <int SLOTS>
__device__ void dev_fwd_local(const ApplyLocal& it, double* sm, int64_t cap) {
  if (it.m == 0) return;
  const int lane = threadIdx.x & 31;
  const double *G, *V, *tau;
  stage_local(it, sm, cap, G, V, tau);
  __syncthreads();
  if (threadIdx.x < 32) {
    double y[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int l = lane + 32 * s;
      y[s] = l < it.m ? __ldcg(it.y + l) : 0.0;
    }
    warp_trsv_lower(G, it.m, y, lane);
    for (int j = 0; j < it.r; ++j) warp_reflect(V, tau, it.m, j, y, lane);
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int l = lane + 32 * s;
      if (l < it.m) it.y[l] = y[s];
    }
  }
  __syncthreads();   // smem reusable by the CTA's next item
}

// forward: y_q -= C_s[:, col:col+len]^T y_f,s summed over the batch members s with q in n(s)
// (G_s of Eq. CC:eqn:elim); warp-level, contributions in source order, the K loads of an
// entry issued back to back.
__device__ __forceinline__ void dev_fwd_scatter(const ApplyTarget& t, const ApplyContrib* __restrict__ con, int lane) {
  for (int i0 = 0; i0 < t.len; i0 += 32) {
    const int i = i0 + lane;
    double acc = 0.0;
    for (int c = t.c_begin; c < t.c_end; ++c) {
      const ApplyContrib a = con[c];
      if (i < t.len) {
        const double* Ci = a.C + a.col + i;
#pragma unroll 8
        for (int k = 0; k < a.K; ++k) acc += Ci[(int64_t)k * a.ldC] * __ldcg(a.yf + k);
      }
    }
    if (i < t.len) t.yq[i] = __ldcg(t.yq + i) - acc;
  }
}

// backward stage 1 (CTA-level, blockDim == BWD_CHUNK): for BWD_CHUNK columns c of C_s,
// parts[k] = sum_c C_s[k][c] x_n[c] (x_n[c] read straight from the neighbour's segment); a
// thread per column, the K rows in groups of 8 independent loads, fixed-order reduction.
constexpr int NB_SMEM = 512;
__device__ void dev_bwd_partial(const ApplyLocal* __restrict__ items, const ApplyNb* __restrict__ nbs,
                                const ApplyChunk& ch, double* __restrict__ parts) {
  const ApplyLocal it = items[ch.li];
  __shared__ ApplyNb snb[NB_SMEM];
  __shared__ double wred[BWD_CHUNK / 32][8];
  const int nnb = it.nb_end - it.nb_begin;
  const ApplyNb* nbl = nbs + it.nb_begin;
  if (nnb <= NB_SMEM) {
    for (int b = threadIdx.x; b < nnb; b += blockDim.x) snb[b] = nbl[b];
    __syncthreads();
    nbl = snb;
  }
  const int K = it.m - it.r;
  const int c = ch.c0 + threadIdx.x;
  double x = 0.0;
  if (c < it.kn) {
    int lo = 0, hi = nnb - 1;   // last neighbour with col <= c
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (nbl[mid].col <= c) lo = mid;
      else hi = mid - 1;
    }
    x = __ldcg(nbl[lo].xq + (c - nbl[lo].col));
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double* Cc = it.C + c;
  for (int k0 = 0; k0 < K; k0 += 8) {
    double p[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = (c < it.kn && k0 + q < K) ? Cc[(int64_t)(k0 + q) * it.ldC] * x : 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) p[q] = wsum(p[q]);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 8; ++q) wred[wid][q] = p[q];
    __syncthreads();
    if (threadIdx.x < 8 && k0 + threadIdx.x < K) {
      double s = 0.0;
      for (int w = 0; w < nw; ++w) s += wred[w][threadIdx.x];
      parts[ch.part + k0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
  __syncthreads();   // snb reusable
}

// backward stage 2 (CTA-level): x_f = y_f - sum_chunks parts (fixed order) ;
// x_s <- G^{-T} U [x_c; x_f] (S_s^T E_s^T G_s^T of W_s^T, Alg. 2 backward substitution).
template <int SLOTS>
__device__ void dev_bwd_local(const ApplyLocal& it, const double* __restrict__ parts, double* sm, int64_t cap) {
  if (it.m == 0) return;
  __shared__ double xf[MAX_M];
  const double *G, *V, *tau;
  stage_local(it, sm, cap, G, V, tau);
  const int K = it.m - it.r;
  const int lane = threadIdx.x & 31;
  const int nch = (it.nb_end > it.nb_begin && K > 0) ? (it.kn + BWD_CHUNK - 1) / BWD_CHUNK : 0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < nch; ++q) s += __ldcg(parts + it.part_off + (int64_t)q * K + k);
    xf[k] = __ldcg(it.y + it.r + k) - s;
  }
  __syncthreads();   // staged G/V and x_f visible
  if (threadIdx.x < 32) {
    double y[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int l = lane + 32 * s;
      y[s] = l < it.r ? __ldcg(it.y + l) : (l < it.m ? xf[l - it.r] : 0.0);
    }
    for (int j = it.r - 1; j >= 0; --j) warp_reflect(V, tau, it.m, j, y, lane);
    warp_trsv_upper_t(G, it.m, y, lane);
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const int l = lane + 32 * s;
      if (l < it.m) it.y[l] = y[s];
    }
  }
  __syncthreads();
}

// ---- per-batch kernels (eager path, HS_APPLY_PER_BATCH=1) ---------------------------------
template <int SLOTS>
__global__ void k_apply_fwd_local(const ApplyLocal* __restrict__ items, int n, int64_t cap) {
  extern __shared__ double sm[];
  dev_fwd_local<SLOTS>(items[blockIdx.x], sm, cap);
}
__global__ void k_apply_fwd_scatter(const ApplyTarget* __restrict__ tg, const ApplyContrib* __restrict__ con, int n) {
  const int w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (w < n) dev_fwd_scatter(tg[w], con, threadIdx.x & 31);
}
__global__ void __launch_bounds__(BWD_CHUNK) k_apply_bwd_partial(const ApplyLocal* __restrict__ items,
                                                                 const ApplyNb* __restrict__ nbs,
                                                                 const ApplyChunk* __restrict__ chunks,
                                                                 double* __restrict__ parts) {
  dev_bwd_partial(items, nbs, chunks[blockIdx.x], parts);
}
template <int SLOTS>
__global__ void k_apply_bwd(const ApplyLocal* __restrict__ items, const double* __restrict__ parts, int64_t cap) {
  extern __shared__ double sm[];
  dev_bwd_local<SLOTS>(items[blockIdx.x], parts, sm, cap);
}

// ---- one cooperative kernel per level and direction: the level's batches in order, a
// grid-wide barrier between dependent phases (local -> scatter -> next batch) ---------------
template <int SLOTS>
__global__ void __launch_bounds__(BWD_CHUNK) k_apply_fwd_level(ApplyLevelArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group g = cg::this_grid();
  extern __shared__ double sm[];
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
  for (int b = 0; b < a.nbatch; ++b) {
    const ApplyBatchDev B = a.batches[b];
    for (int i = B.local_begin + blockIdx.x; i < B.local_end; i += gridDim.x) dev_fwd_local<SLOTS>(a.local[i], sm, a.cap);
    g.sync();
    for (int t = B.tgt_begin + gw; t < B.tgt_end; t += nwarps) dev_fwd_scatter(a.tgt[t], a.con, threadIdx.x & 31);
    g.sync();
  }
}
template <int SLOTS>
__global__ void __launch_bounds__(BWD_CHUNK) k_apply_bwd_level(ApplyLevelArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group g = cg::this_grid();
  extern __shared__ double sm[];
  for (int b = a.nbatch - 1; b >= 0; --b) {
    const ApplyBatchDev B = a.batches[b];
    for (int c = B.chunk_begin + blockIdx.x; c < B.chunk_end; c += gridDim.x)
      dev_bwd_partial(a.local + B.local_begin, a.nb, a.chunks[c], a.parts);
    g.sync();
    for (int i = B.local_begin + blockIdx.x; i < B.local_end; i += gridDim.x)
      dev_bwd_local<SLOTS>(a.local[i], a.parts, sm, a.cap);
    g.sync();
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

static void set_dyn_smem(const void* f, size_t bytes, size_t& configured) {
  if (bytes > configured) {
    HS_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
    configured = bytes;
  }
}

template <int S>
void fwd_local_s(const ApplyLocal* d, int n, int64_t cap, cudaStream_t st) {
  static size_t configured = 0;
  const size_t sm = sizeof(double) * (size_t)std::max<int64_t>(cap, 1);
  set_dyn_smem((const void*)k_apply_fwd_local<S>, sm, configured);
  k_apply_fwd_local<S><<<n, 128, sm, st>>>(d, n, cap);
}
void launch_apply_fwd_local(const ApplyLocal* d, int n, int64_t cap, int max_m, cudaStream_t st) {
  if (n <= 0) return;
  if (max_m <= 128) fwd_local_s<4>(d, n, cap, st);
  else if (max_m <= 256) fwd_local_s<8>(d, n, cap, st);
  else fwd_local_s<16>(d, n, cap, st);
  count_launch(1);
}
void launch_apply_fwd_scatter(const ApplyTarget* d, const ApplyContrib* c, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_apply_fwd_scatter<<<(n + 3) / 4, 128, 0, st>>>(d, c, n);
  count_launch(1);
}
void launch_apply_bwd_partial(const ApplyLocal* d_local_batch, const ApplyNb* nb, const ApplyChunk* ch, int n,
                              double* parts, cudaStream_t st) {
  if (n <= 0) return;
  k_apply_bwd_partial<<<n, BWD_CHUNK, 0, st>>>(d_local_batch, nb, ch, parts);
  count_launch(1);
}
template <int S>
void bwd_s(const ApplyLocal* d, const double* parts, int n, int64_t cap, cudaStream_t st) {
  static size_t configured = 0;
  const size_t sm = sizeof(double) * (size_t)std::max<int64_t>(cap, 1);
  set_dyn_smem((const void*)k_apply_bwd<S>, sm, configured);
  k_apply_bwd<S><<<n, 128, sm, st>>>(d, parts, cap);
}
void launch_apply_bwd(const ApplyLocal* d, const double* parts, int n, int64_t cap, int max_m, cudaStream_t st) {
  if (n <= 0) return;
  if (max_m <= 128) bwd_s<4>(d, parts, n, cap, st);
  else if (max_m <= 256) bwd_s<8>(d, parts, n, cap, st);
  else bwd_s<16>(d, parts, n, cap, st);
  count_launch(1);
}
template <int S>
void level_s(const ApplyLevelArgs& a, int backward, cudaStream_t st) {
  const void* fn = backward ? (const void*)k_apply_bwd_level<S> : (const void*)k_apply_fwd_level<S>;
  const size_t sm = sizeof(double) * (size_t)std::max<int64_t>(a.cap, 1);
  static size_t configured[2] = {0, 0};
  set_dyn_smem(fn, sm, configured[backward ? 1 : 0]);
  int per_sm = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, BWD_CHUNK, sm));
  if (per_sm <= 0) fail(HS_E_INTERNAL, "apply level kernel: no co-resident CTA fits");
  int dev = 0, nsm = 0;
  HS_CUDA(cudaGetDevice(&dev));
  HS_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  const int grid = nsm * std::min(per_sm, 4);
  ApplyLevelArgs args = a;
  void* params[] = {&args};
  HS_CUDA(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(BWD_CHUNK), params, sm, st));
}
void launch_apply_level(const ApplyLevelArgs& a, int max_m, int backward, cudaStream_t st) {
  if (a.nbatch <= 0) return;
  if (max_m <= 128) level_s<4>(a, backward, st);
  else if (max_m <= 256) level_s<8>(a, backward, st);
  else level_s<16>(a, backward, st);
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
