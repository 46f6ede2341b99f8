// a0 + a1 + a2 for the DC path (clusters up to CI_MAX_M): the deferred-compression scaling
// B_s = G_s^{-1} [A_sw | A_sn] with A_ss = G_s G_s^T (Eq. CC:eqn:scaling)
// as two kernels, no gather pass and no CTA-wide barrier inside the triangular solve:
//   k_chol       one CTA per cluster: A_ss read straight from the level's block store into
//                shared memory (as its upper triangle), right-looking Cholesky with one
//                barrier per pivot (the trailing update uses the unscaled row, the scaling
//                by sqrt(d_j) happens once at the end), G_s stored to the workspace;
//                It also forms G_s^{-1} (warp-synchronous forward substitution on I);
//   k_scale_mma  one CTA per (cluster, 64-column tile): the tile of [A_sw | A_sn] gathered
//                from the store segments, B = G_s^{-1} A as an m x m by m x 64 product on the
//                FP64 tensor cores (DMMA), B stored and the largest n-column norm (R-floor)
//                reduced.
// Replaces the gather / POTRF / TRSM triple.
#include <cuda_runtime.h>

#include <cstdlib>

#include "device.h"

namespace hs {

namespace {

constexpr int ST_TW = 64;   // columns per k_scale_mma CTA

template <int R4>
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
  // G_s^{-1} (lower) by forward substitution on I, warp-synchronously: warp w owns columns
  // cb + 8w + (lane & 7), lane group gr = lane >> 3 owns rows gr + 4t in registers; the
  // pivot of row i is broadcast by shuffle (no CTA barrier in the m-step chain).  Both the
  // deferred-compression scaling (a DMMA product, k_scale_mma) and the apply operator
  // T_s = U^T G_s^{-1} (k_form_T) consume it.
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
        if (i < m && i >= cb) {   // uniform over the CTA; rows above the block stay zero
          const double* gc = U + i * ldu;   // column i of G: gc[l] = G[l][i], l >= i
          if (gr == gi) r[ti] = r[ti] * rd[i];   // 1 / G_ii (rd holds 1/sqrt(d_i) = 1/G_ii)
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

// B[:, c0:c0+nc] = G^{-1} A[:, c0:c0+nc] on the FP64 tensor cores: the tile of [A_sw | A_sn]
// is gathered from the store segments into shared memory, G_s^{-1} (lower) staged beside it,
// and the m x 64 product formed with DMMA (mma.sync.m8n8k4.f64): warp w owns output columns
// 8w..8w+7 and every 8-row block, the k loop skips the zero upper triangle of G^{-1}.
// Row strides == 4 (mod 16) make the fragment loads conflict-free.  The result goes back to
// B_s through shared memory (coalesced rows) and the largest n-column norm (R-floor) is
// reduced from it.
constexpr int SM_LDX = 68;   // tile row stride (doubles)
__host__ __device__ __forceinline__ int mma_ldg(int m) { return ((m + 11) / 16) * 16 + 4; }   // >= m, == 4 mod 16
template <int NRB>
__global__ void __launch_bounds__(256) k_scale_mma(const FusedItem* __restrict__ items,
                                                   const FusedSeg* __restrict__ segs) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double sm[];
  const FusedItem it = items[blockIdx.x];
  const int m = it.m;
  if (m == 0 || it.nc <= 0) return;
  const int ldg = mma_ldg(m), mp = 8 * NRB;   // rows padded to the 8-row blocks
  double* gi = sm;                  // mp x ldg, G^{-1} (zeros above the diagonal and below m)
  double* x = sm + (size_t)mp * ldg;   // mp x SM_LDX
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // staging: every thread issues 4 independent global loads before its shared stores (the
  // kernel is bound by the latency of these loads at a few CTAs per SM)
  for (int e0 = tid; e0 < mp * ldg; e0 += 4 * 256) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + 256 * u, i = e / ldg, k = e % ldg;
      v[u] = (e < mp * ldg && i < m && k <= i) ? it.Ginv[(int64_t)i * m + k] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (e0 + 256 * u < mp * ldg) gi[e0 + 256 * u] = v[u];
  }
  for (int e = tid; e < mp * SM_LDX; e += blockDim.x) x[e] = 0.0;
  __syncthreads();
  for (int sg = it.seg_begin; sg < it.seg_end; ++sg) {   // the tile's columns from the store
    const FusedSeg sgm = segs[sg];
    const int j0 = max(it.c0, sgm.col), j1 = min(it.c0 + it.nc, sgm.col + sgm.len);
    const int wd = j1 - j0, tot = m * wd;
    for (int e0 = tid; e0 < tot; e0 += 4 * 256) {
      double v[4];
      int dst[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + 256 * u;
        int i, j;
        if (sgm.trans) {   // consecutive threads: consecutive rows i
          j = j0 + e / m;
          i = e % m;
        } else {
          i = e / wd;
          j = j0 + e % wd;
        }
        dst[u] = e < tot ? i * SM_LDX + (j - it.c0) : -1;
        const int lc = e >= tot ? 0 : (it.colmap ? it.colmap[j] : j - sgm.col);   // column inside the block
        v[u] = e < tot ? (sgm.trans ? sgm.src[(int64_t)lc * sgm.sld + i] : sgm.src[(int64_t)i * sgm.sld + lc])
                       : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (dst[u] >= 0) x[dst[u]] = v[u];
    }
  }
  __syncthreads();
  // acc[rb] = rows 8 rb + (lane >> 2), columns 8 w + 2 (lane & 3) + {0, 1}
  double acc[NRB][2];
#pragma unroll
  for (int rb = 0; rb < NRB; ++rb) acc[rb][0] = acc[rb][1] = 0.0;
  const int fr = lane >> 2, fc = lane & 3;
  for (int k0 = 0; k0 < mp; k0 += 4) {
    const double b = x[(k0 + fc) * SM_LDX + 8 * w + fr];   // B = X[k0:k0+4, 8w:8w+8], col-major 4 x 8
#pragma unroll
    for (int rb = 0; rb < NRB; ++rb) {
      if (8 * rb + 8 > k0) {   // G^{-1} rows 8rb..8rb+7 vanish for columns k > 8 rb + 7
        const double a = gi[(8 * rb + fr) * ldg + k0 + fc];   // A = G^{-1}[8rb:8rb+8, k0:k0+4], row-major 8 x 4
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[rb][0]), "+d"(acc[rb][1])
                     : "d"(a), "d"(b));
      }
    }
  }
  __syncthreads();   // every warp has read x: overwrite it with the result
#pragma unroll
  for (int rb = 0; rb < NRB; ++rb) {
    const int i = 8 * rb + fr;
    x[i * SM_LDX + 8 * w + 2 * fc] = acc[rb][0];
    x[i * SM_LDX + 8 * w + 2 * fc + 1] = acc[rb][1];
  }
  __syncthreads();
  for (int e = tid; e < m * ST_TW; e += blockDim.x) {
    const int i = e / ST_TW, cc = e % ST_TW;
    if (cc < it.nc) it.B[(int64_t)i * it.ldB + it.c0 + cc] = x[i * SM_LDX + cc];
  }
  if (it.nmax && it.c0 + it.nc > it.kw) {   // largest n-column norm (R-floor of tau_s)
    double s = -1.0;
    const int n0 = max(0, it.kw - it.c0);
    if (tid < ST_TW && tid >= n0 && tid < it.nc) {
      s = 0.0;
      for (int i = 0; i < m; ++i) s += x[i * SM_LDX + tid] * x[i * SM_LDX + tid];
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
#define HS_CH(RR)                                               \
  case RR:                                                      \
    set_smem_attr((const void*)k_chol<4 * RR>, sm);             \
    launch_pdl(k_chol<4 * RR>, dim3(n), dim3(256), sm, st, d_items, status); \
    break;
  switch (R) {
    HS_CH(1) HS_CH(2) HS_CH(3) HS_CH(4) HS_CH(5) HS_CH(6) HS_CH(7)
    default: fail(HS_E_INTERNAL, "launch_chol: m above CI_MAX_M");
  }
#undef HS_CH
  count_launch(1);
}

void launch_scale_tiles(const FusedItem* d_items, int n, const FusedSeg* d_segs, int max_m, cudaStream_t st) {
  if (n <= 0) return;
  const int nrb = (max_m + 7) / 8;
  const size_t sm = sizeof(double) * ((size_t)8 * nrb * mma_ldg(max_m) + (size_t)8 * nrb * SM_LDX);
#define HS_SM(NB)                                                     \
  case NB:                                                            \
    set_smem_attr((const void*)k_scale_mma<NB>, sm);                  \
    launch_pdl(k_scale_mma<NB>, dim3(n), dim3(256), sm, st, d_items, d_segs); \
    break;
  switch (nrb) {
    HS_SM(1) HS_SM(2) HS_SM(3) HS_SM(4) HS_SM(5) HS_SM(6) HS_SM(7)
    HS_SM(8) HS_SM(9) HS_SM(10) HS_SM(11) HS_SM(12) HS_SM(13) HS_SM(14)
    default: fail(HS_E_INTERNAL, "launch_scale_tiles: m above CI_MAX_M");
  }
#undef HS_SM
  count_launch(1);
}

}  // namespace hs
