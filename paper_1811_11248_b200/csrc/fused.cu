// a0 + a1 + a2 for the DC path (clusters up to CI_MAX_M): the deferred-compression scaling
// B_s = G_s^{-1} [A_sw | A_sn] with A_ss = G_s G_s^T (Eq. CC:eqn:scaling)
// as two kernels, no gather pass and no CTA-wide barrier inside the triangular solve:
//   k_chol       one CTA per cluster: A_ss read straight from the level's block store into
//                shared memory (as its upper triangle), right-looking Cholesky with one
//                barrier per pivot (the trailing update uses the unscaled row, the scaling
//                by sqrt(d_j) happens once at the end), G_s stored to the workspace;
//   k_scale_tile one CTA per (cluster, 64-column tile): the tile of [A_sw | A_sn] gathered
//                from the store segments, forward substitution with G_s where each warp owns
//                8 columns held in registers (4 row groups x 8 columns per warp, pivots
//                broadcast by shuffle: warp-synchronous, no __syncthreads in the chain), B
//                stored and the largest n-column norm (R-floor) reduced.
// Replaces the gather / POTRF / TRSM triple.
#include <cuda_runtime.h>

#include <cstdlib>

#include "device.h"

namespace hs {

namespace {

constexpr int ST_TW = 64;   // columns per k_scale_tile CTA

__global__ void __launch_bounds__(256) k_chol(const FusedItem* __restrict__ items, DevStatus* status) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double sm[];
  const FusedItem it = items[blockIdx.x];
  const int m = it.m;
  if (m == 0) return;
  const int ldu = m + 1;
  double* U = sm;   // U = the upper triangle (A_ss^T), ld m + 1
  __shared__ double rd[CI_MAX_M];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int i = e / m, k = e % m;   // A[i][k], k <= i  ->  U[k][i]
    if (k <= i) U[k * ldu + i] = it.Ass[(int64_t)i * it.lda + k];
  }
  __syncthreads();
  // step j subtracts U[j][i] U[j][k] / d_j from the trailing U[i][k] (j < i <= k); row j is
  // final after step j and never written again
  for (int j = 0; j < m; ++j) {
    const double* uj = U + j * ldu;
    const double d = uj[j];
    if (!(d > 0.0)) {   // every thread reads the same d: uniform exit
      if (tid == 0 && atomicCAS(&status->flag, 0, 1) == 0) {
        status->level = it.level;
        status->cluster = it.cluster;
        status->pivot = j;
        status->value = d;
      }
      return;
    }
    const double inv = 1.0 / d;
    double ujr[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int k = lane + 32 * t;
      ujr[t] = (k > j && k < m) ? uj[k] : 0.0;
    }
    int i = j + 1 + wid;
    for (; i + nw < m; i += 2 * nw) {   // two rows at a time: independent loads before stores
      const int i2 = i + nw;
      const double f1 = uj[i] * inv, f2 = uj[i2] * inv;
      double* u1 = U + i * ldu;
      double* u2 = U + i2 * ldu;
      double a1[4], a2[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int k = lane + 32 * t;
        a1[t] = (k >= i && k < m) ? u1[k] : 0.0;
        a2[t] = (k >= i2 && k < m) ? u2[k] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int k = lane + 32 * t;
        if (k >= i && k < m) u1[k] = a1[t] - f1 * ujr[t];
        if (k >= i2 && k < m) u2[k] = a2[t] - f2 * ujr[t];
      }
    }
    if (i < m) {
      const double f1 = uj[i] * inv;
      double* u1 = U + i * ldu;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int k = lane + 32 * t;
        if (k >= i && k < m) u1[k] -= f1 * ujr[t];
      }
    }
    __syncthreads();
  }
  if (tid < m) rd[tid] = 1.0 / sqrt(U[tid * ldu + tid]);
  __syncthreads();
  // U <- G^T in place: G[i][j] = U[j][i] / sqrt(d_j) (i > j), G[j][j] = sqrt(d_j)
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int j = e / m, i = e % m;
    if (i > j) U[j * ldu + i] *= rd[j];
    else if (i == j) U[j * ldu + j] = sqrt(U[j * ldu + j]);
  }
  __syncthreads();
  for (int e = tid; e < m * m; e += blockDim.x) {   // G_s (lower, zeros above)
    const int i = e / m, j = e % m;
    it.G[e] = j <= i ? U[j * ldu + i] : 0.0;
  }
}

// B[:, c0:c0+nc] = G^{-1} A[:, c0:c0+nc].  Warp w owns columns 8w + (lane & 7); lane group
// g = lane >> 3 owns rows g + 4t (t < R4) in registers.  Row i = 4 ti + gi is final once
// the steps before it are applied: its owner lane divides by G_ii and the value is
// broadcast to the 4 row groups of the same column by shuffle.
template <int R4>
__global__ void __launch_bounds__(256) k_scale_tile(const FusedItem* __restrict__ items,
                                                    const FusedSeg* __restrict__ segs) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double sm[];
  const FusedItem it = items[blockIdx.x];
  const int m = it.m;
  if (m == 0 || it.nc <= 0) return;
  const int ldg = m + 1;
  double* g = sm;               // m x m, ld m + 1
  double* x = sm + m * ldg;     // m x ST_TW
  const int tid = threadIdx.x;
  for (int e = tid; e < m * m; e += blockDim.x) {
    const int i = e / m, k = e % m;
    if (k <= i) g[i * ldg + k] = it.G[e];
  }
  // 1 / G_ii in the unused last slot of row i: the substitution chain multiplies instead of
  // dividing (a long FP64 instruction sequence on the critical path of every step)
  if (tid < m) g[tid * ldg + m] = 1.0 / it.G[(int64_t)tid * m + tid];
  for (int e = tid; e < m * ST_TW; e += blockDim.x) x[e] = 0.0;
  __syncthreads();
  for (int sg = it.seg_begin; sg < it.seg_end; ++sg) {   // the tile's columns from the store
    const FusedSeg sgm = segs[sg];
    const int j0 = max(it.c0, sgm.col), j1 = min(it.c0 + it.nc, sgm.col + sgm.len);
    const int w = j1 - j0;
    if (sgm.trans) {
      for (int e = tid; e < m * w; e += blockDim.x) {   // consecutive threads: consecutive rows i
        const int j = j0 + e / m, i = e % m;
        x[i * ST_TW + (j - it.c0)] = sgm.src[(int64_t)(j - sgm.col) * sgm.sld + i];
      }
    } else {
      for (int e = tid; e < m * w; e += blockDim.x) {
        const int i = e / w, j = j0 + e % w;
        x[i * ST_TW + (j - it.c0)] = sgm.src[(int64_t)i * sgm.sld + (j - sgm.col)];
      }
    }
  }
  __syncthreads();
  const int lane = tid & 31, col = (tid >> 5) * 8 + (lane & 7), gr = lane >> 3;
  double r[R4];
#pragma unroll
  for (int t = 0; t < R4; ++t) {
    const int l = gr + 4 * t;
    r[t] = l < m ? x[l * ST_TW + col] : 0.0;
  }
#pragma unroll
  for (int ti = 0; ti < R4; ++ti) {
#pragma unroll
    for (int gi = 0; gi < 4; ++gi) {
      const int i = 4 * ti + gi;
      if (i < m) {   // uniform over the CTA
        if (gr == gi) r[ti] = r[ti] * g[i * ldg + m];
        const double xi = __shfl_sync(0xffffffffu, r[ti], (lane & 7) + 8 * gi);
#pragma unroll
        for (int t = ti; t < R4; ++t) {
          const int l = gr + 4 * t;
          if (l > i && l < m) r[t] = fma(-g[l * ldg + i], xi, r[t]);
        }
      }
    }
  }
  __syncthreads();
#pragma unroll
  for (int t = 0; t < R4; ++t) {
    const int l = gr + 4 * t;
    if (l < m) x[l * ST_TW + col] = r[t];
  }
  __syncthreads();
  for (int e = tid; e < m * ST_TW; e += blockDim.x) {
    const int i = e / ST_TW, cc = e % ST_TW;
    if (cc < it.nc) it.B[(int64_t)i * it.ldB + it.c0 + cc] = x[e];
  }
  if (it.nmax && it.c0 + it.nc > it.kw) {   // largest n-column norm (R-floor of tau_s)
    double s = -1.0;
    const int n0 = max(0, it.kw - it.c0);
    if (tid < ST_TW && tid >= n0 && tid < it.nc) {
      s = 0.0;
      for (int i = 0; i < m; ++i) s += x[i * ST_TW + tid] * x[i * ST_TW + tid];
      s = sqrt(s);
    }
    for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
    if ((tid & 31) == 0 && s >= 0.0) atomicMax(it.nmax, (unsigned long long)__double_as_longlong(s));
  }
}

}  // namespace

void launch_chol(const FusedItem* d_items, int n, int max_m, DevStatus* status, cudaStream_t st) {
  if (n <= 0) return;
  const size_t sm = sizeof(double) * (size_t)max_m * (max_m + 1);
  set_smem_attr((const void*)k_chol, sm);
  launch_pdl(k_chol, dim3(n), dim3(256), sm, st, d_items, status);
  count_launch(1);
}

void launch_scale_tiles(const FusedItem* d_items, int n, const FusedSeg* d_segs, int max_m, cudaStream_t st) {
  if (n <= 0) return;
  const size_t sm = sizeof(double) * ((size_t)max_m * (max_m + 1) + (size_t)max_m * ST_TW);
  const int R = (max_m + 15) / 16;   // R4 = 4 R rows per lane group
#define HS_ST(RR)                                                     \
  case RR:                                                            \
    set_smem_attr((const void*)k_scale_tile<4 * RR>, sm);             \
    launch_pdl(k_scale_tile<4 * RR>, dim3(n), dim3(256), sm, st, d_items, d_segs); \
    break;
  switch (R) {
    HS_ST(1) HS_ST(2) HS_ST(3) HS_ST(4) HS_ST(5) HS_ST(6) HS_ST(7)
    default: fail(HS_E_INTERNAL, "launch_scale_tiles: m above CI_MAX_M");
  }
#undef HS_ST
  count_launch(1);
}

}  // namespace hs
