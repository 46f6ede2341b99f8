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

template <int R4, bool INV>
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
  if (!INV || !it.Ginv) return;
  // G_s^{-1} (lower) by forward substitution on I, warp-synchronously: warp w owns columns
  // cb + 8w + (lane & 7), lane group gr = lane >> 3 owns rows gr + 4t in registers; the
  // pivot of row i is broadcast by shuffle (no CTA barrier in the m-step chain)
  const int gr = lane >> 3;
  for (int cb = 0; cb < m; cb += 64) {
    const int col = cb + wid * 8 + (lane & 7);
    double r[R4];
#pragma unroll
    for (int t = 0; t < R4; ++t) r[t] = (gr + 4 * t == col) ? 1.0 : 0.0;
#pragma unroll
    for (int ti = 0; ti < R4; ++ti) {
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        const int i = 4 * ti + gi;
        if (i < m) {   // uniform over the CTA
          const double* gc = U + i * ldu;   // column i of G: gc[l] = G[l][i], l >= i
          if (gr == gi) r[ti] = r[ti] / gc[i];
          const double xi = __shfl_sync(0xffffffffu, r[ti], (lane & 7) + 8 * gi);
#pragma unroll
          for (int t = ti; t < R4; ++t) {
            const int l = gr + 4 * t;
            if (l > i && l < m) r[t] = fma(-gc[l], xi, r[t]);
          }
        }
      }
    }
    if (col < m)
#pragma unroll
      for (int t = 0; t < R4; ++t) {
        const int l = gr + 4 * t;
        if (l < m) it.Ginv[(int64_t)l * m + col] = r[t];
      }
  }
}

// B[:, c0:c0+nc] = G^{-1} A[:, c0:c0+nc] as a product with the explicit inverse (register-
// tiled FFMA, lower triangle only): thread (rg, cg) owns rows rg + 16 r, columns cg + 16 j.
template <int R>
__global__ void __launch_bounds__(256) k_scale_gemm(const FusedItem* __restrict__ items,
                                                    const FusedSeg* __restrict__ segs) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double sm[];
  const FusedItem it = items[blockIdx.x];
  const int m = it.m;
  if (m == 0 || it.nc <= 0) return;
  double* gi = sm;              // m x m
  double* x = sm + m * m;       // m x ST_TW
  const int tid = threadIdx.x;
  for (int e = tid; e < m * m; e += blockDim.x) gi[e] = it.Ginv[e];
  for (int e = tid; e < m * ST_TW; e += blockDim.x) x[e] = 0.0;
  __syncthreads();
  for (int sg = it.seg_begin; sg < it.seg_end; ++sg) {   // the tile's columns from the store
    const FusedSeg g = segs[sg];
    const int j0 = max(it.c0, g.col), j1 = min(it.c0 + it.nc, g.col + g.len);
    const int w = j1 - j0;
    if (g.trans) {
      for (int e = tid; e < m * w; e += blockDim.x) {   // consecutive threads: consecutive rows i
        const int j = j0 + e / m, i = e % m;
        x[i * ST_TW + (j - it.c0)] = g.src[(int64_t)(j - g.col) * g.sld + i];
      }
    } else {
      for (int e = tid; e < m * w; e += blockDim.x) {
        const int i = e / w, j = j0 + e % w;
        x[i * ST_TW + (j - it.c0)] = g.src[(int64_t)i * g.sld + (j - g.col)];
      }
    }
  }
  __syncthreads();
  const int cg = tid & 15, rg = tid >> 4;
  double acc[R][4];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[r][j] = 0.0;
  const int kend = min(m, rg + 16 * (R - 1) + 1);   // G^{-1} is lower triangular
  for (int k = 0; k < kend; ++k) {
    double b[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) b[j] = x[k * ST_TW + cg + 16 * j];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = rg + 16 * r;
      const double a = (i < m) ? gi[i * m + k] : 0.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[r][j] = fma(a, b[j], acc[r][j]);
    }
  }
  __syncthreads();   // x is reused for the result
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = rg + 16 * r;
    if (i < m)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int cc = cg + 16 * j;
        x[i * ST_TW + cc] = acc[r][j];
        if (cc < it.nc) it.B[(int64_t)i * it.ldB + it.c0 + cc] = acc[r][j];
      }
  }
  if (it.nmax && it.c0 + it.nc > it.kw) {   // largest n-column norm (R-floor of tau_s)
    __syncthreads();
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
  const int R = (max_m + 15) / 16;   // R4 = 4 R rows per lane group (the inverse)
  if (!scale_by_inverse()) {   // no inverse: one lean instantiation for every m
    set_smem_attr((const void*)k_chol<4, false>, sm);
    launch_pdl(k_chol<4, false>, dim3(n), dim3(256), sm, st, d_items, status);
    count_launch(1);
    return;
  }
#define HS_CH(RR)                                               \
  case RR:                                                      \
    set_smem_attr((const void*)k_chol<4 * RR, true>, sm);       \
    launch_pdl(k_chol<4 * RR, true>, dim3(n), dim3(256), sm, st, d_items, status); \
    break;
  switch (R) {
    HS_CH(1) HS_CH(2) HS_CH(3) HS_CH(4) HS_CH(5) HS_CH(6) HS_CH(7)
    default: fail(HS_E_INTERNAL, "launch_chol: m above CI_MAX_M");
  }
#undef HS_CH
  count_launch(1);
}

// HS_SCALE_INVERSE=1: k_chol also forms G^{-1} and the tiles multiply by it (k_scale_gemm)
// instead of the warp-synchronous forward substitution.  Measured on C2: the same total —
// the inverse's m-step chain moves into k_chol (which then needs up to 255 registers, one
// CTA per SM) and the tiles get cheaper by as much; the substitution is the default.
bool scale_by_inverse() {
  static const bool v = std::getenv("HS_SCALE_INVERSE") != nullptr;
  return v;
}

void launch_scale_tiles(const FusedItem* d_items, int n, const FusedSeg* d_segs, int max_m, cudaStream_t st) {
  if (n <= 0) return;
  if (scale_by_inverse()) {
    const size_t sm = sizeof(double) * ((size_t)max_m * max_m + (size_t)max_m * ST_TW);
#define HS_SG(RR)                                                     \
  case RR:                                                            \
    set_smem_attr((const void*)k_scale_gemm<RR>, sm);                 \
    launch_pdl(k_scale_gemm<RR>, dim3(n), dim3(256), sm, st, d_items, d_segs); \
    break;
    switch ((max_m + 15) / 16) {
      HS_SG(1) HS_SG(2) HS_SG(3) HS_SG(4) HS_SG(5) HS_SG(6) HS_SG(7)
      default: fail(HS_E_INTERNAL, "launch_scale_tiles: m above CI_MAX_M");
    }
#undef HS_SG
    count_launch(1);
    return;
  }
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
