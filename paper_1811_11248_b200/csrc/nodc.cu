// NEXT f1: the original LoRaSp elimination WITHOUT deferred compression (P:153-203,
// Eq. offdiag; oracle/factor.py eliminate_nodc), on the same kernels as the DC path plus:
//   k_nmax          largest column norm of the unscaled A_sn (the R-floor of tau_s)
//   k_rot2          A_ss <- U^T A_ss U in place (the rotation of row AND column s)
//   (k_potrf / k_trsm on sub-blocks: L_f L_f^T = (U^T A_ss U)_ff, C_c, C_n = L_f^{-1} [...])
//   k_coarse_update [A_cc | A_cn] -= C_c^T [C_c | C_n]  (the coarse block of s)
//   k_form_T_nodc   T_s = [[I, -C_c^T], [0, I]] diag(I, L_f^{-1}) U^T  (the apply operator:
//                   forward [y_c; y_f] = T_s y_s, backward x_s = T_s^T [x_c; x_f])
#include <cuda_runtime.h>

#include "device.h"

namespace hs {

namespace {

// max over the n-columns of ||B[:, c]|| for a tile of columns (R-floor)
__global__ void k_nmax(const CluItem* __restrict__ clu, const TrsmItem* __restrict__ items) {
  const TrsmItem t = items[blockIdx.x];
  const CluItem it = clu[t.ci];
  const int c = t.c0 + (int)threadIdx.x;
  double s = -1.0;
  if ((int)threadIdx.x < t.nc && c >= it.kw && it.m > 0) {
    s = 0.0;
    for (int i = 0; i < it.m; ++i) {
      const double x = it.B[(int64_t)i * it.ldB + c];
      s += x * x;
    }
    s = sqrt(s);
  }
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0 && s >= 0.0) atomicMax(it.nmax, (unsigned long long)__double_as_longlong(s));
}

// A <- Q^T A Q for the symmetric m x m A (row-major, ld m) with Q = H_0 ... H_{r-1}:
// left application (H_0 first) on every column, then right application on every row.
// One CTA per cluster; A staged in shared memory up to SMEM_M, else in place.
__global__ void __launch_bounds__(256) k_rot2(const CluItem* __restrict__ clu, const int32_t* __restrict__ rank,
                                              int use_smem) {
  extern __shared__ double sm[];
  const CluItem it = clu[blockIdx.x];
  const int m = it.m, r = rank[blockIdx.x];
  if (m == 0 || r == 0) return;
  const bool staged = use_smem && m <= SMEM_M;
  double* A = staged ? sm : it.G;
  if (staged)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) A[e] = it.G[e];
  __syncthreads();
  for (int side = 0; side < 2; ++side)
    for (int j = 0; j < r; ++j) {
      const double* v = it.V + (int64_t)j * m;   // zeros above row j, v[j] = 1
      const double t = it.tau[j];
      if (t != 0.0)
        for (int c = threadIdx.x; c < m; c += blockDim.x) {
          // side 0: column c of A; side 1: row c of A
          const int64_t st = side == 0 ? m : 1, base = side == 0 ? c : (int64_t)c * m;
          double d = 0.0;
          for (int i = j; i < m; ++i) d += v[i] * A[base + i * st];
          const double td = t * d;
          for (int i = j; i < m; ++i) A[base + i * st] -= td * v[i];
        }
      __syncthreads();
    }
  if (staged)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) it.G[e] = A[e];
}

// [A_cc | A_cn] -= C_c^T [C_c | C_n]: output column j of the r x (r + kn) update, one thread
// per column; C_c = G[r:m, 0:r] (ld m), C_n = B[r:m, kw:kw+kn] (ld ldB).
__global__ void k_coarse_update(const CluItem* __restrict__ clu, const TrsmItem* __restrict__ items,
                                const int32_t* __restrict__ rank) {
  const TrsmItem t = items[blockIdx.x];
  const CluItem it = clu[t.ci];
  const int m = it.m, r = rank[t.ci], K = m - r;
  const int j = t.c0 + (int)threadIdx.x;
  if ((int)threadIdx.x >= t.nc || r == 0 || K == 0 || j >= r + it.kn) return;
  const double* Cc = it.G + (int64_t)r * m;
  const bool coarse = j < r;
  const double* X = coarse ? Cc + j : it.B + (int64_t)r * it.ldB + it.kw + (j - r);
  const int64_t ldx = coarse ? m : it.ldB;
  double* out = coarse ? it.G + j : it.B + it.kw + (j - r);
  const int64_t ldo = coarse ? m : it.ldB;
  for (int i = 0; i < r; ++i) {
    double acc = 0.0;
    for (int k = 0; k < K; ++k) acc += Cc[(int64_t)k * m + i] * X[(int64_t)k * ldx];
    out[(int64_t)i * ldo] -= acc;
  }
}

// T_s = [[I, -C_c^T], [0, I]] diag(I, L_f^{-1}) Q^T, one CTA per (cluster, 64-column tile):
// X = I tile; X <- H_j X (j = 0..r-1); rows f: forward substitution with L_f = G[r:, r:];
// rows c: X_c -= C_c^T X_f.  G holds (U^T A_ss U) after the coarse update: C_c in G[r:, :r],
// L_f in the lower part of G[r:, r:].
__global__ void __launch_bounds__(256) k_form_T_nodc(const FormTItem* __restrict__ items, int tiles_per, int TW) {
  extern __shared__ double x[];   // m x TW
  const int ci = blockIdx.x / tiles_per, tile = blockIdx.x % tiles_per;
  const FormTItem it = items[ci];
  const int m = it.m, r = it.r;
  const int c0 = tile * TW;
  if (m == 0 || c0 >= m) return;
  const int nc = min(TW, m - c0);
  const int c = threadIdx.x % TW, grp = threadIdx.x / TW;
  for (int e = threadIdx.x; e < m * TW; e += blockDim.x) {
    const int i = e / TW, cc = e % TW;
    x[e] = (cc < nc && i == c0 + cc) ? 1.0 : 0.0;
  }
  __syncthreads();
  if (grp == 0 && c < nc) {   // a column per thread: Q^T, then the fine solve, then the coarse rows
    for (int j = 0; j < r; ++j) {
      const double t = it.tau[j];
      if (t == 0.0) continue;
      const double* v = it.V + (int64_t)j * m;
      double d = 0.0;
      for (int i = j; i < m; ++i) d += v[i] * x[i * TW + c];
      const double td = t * d;
      for (int i = j; i < m; ++i) x[i * TW + c] -= td * v[i];
    }
    const double* G = it.G;
    for (int i = r; i < m; ++i) {   // x_f <- L_f^{-1} x_f
      double acc = x[i * TW + c];
      for (int k = r; k < i; ++k) acc -= G[(int64_t)i * m + k] * x[k * TW + c];
      x[i * TW + c] = acc / G[(int64_t)i * m + i];
    }
    for (int i = 0; i < r; ++i) {   // x_c -= C_c^T x_f
      double acc = 0.0;
      for (int k = r; k < m; ++k) acc += G[(int64_t)k * m + i] * x[k * TW + c];
      x[i * TW + c] -= acc;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < m * TW; e += blockDim.x) {
    const int i = e / TW, cc = e % TW;
    if (cc < nc) it.T[(int64_t)i * m + c0 + cc] = x[e];
  }
}

}  // namespace

void launch_nmax(const CluItem* d_clu, const TrsmItem* d_items, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_nmax<<<n, 64, 0, st>>>(d_clu, d_items);
  count_launch(1);
}
void launch_rot2(const CluItem* d_clu, int n, int max_m, const int32_t* d_rank, cudaStream_t st) {
  if (n <= 0) return;
  const size_t sm = max_m <= SMEM_M ? sizeof(double) * max_m * max_m : 0;
  set_smem_attr((const void*)k_rot2, sm);
  k_rot2<<<n, 256, sm, st>>>(d_clu, d_rank, max_m <= SMEM_M ? 1 : 0);
  count_launch(1);
}
void launch_coarse_update(const CluItem* d_clu, const TrsmItem* d_items, int n, const int32_t* d_rank, cudaStream_t st) {
  if (n <= 0) return;
  k_coarse_update<<<n, 256, 0, st>>>(d_clu, d_items, d_rank);
  count_launch(1);
}
void launch_form_T_nodc(const FormTItem* d_items, int n, int max_m, cudaStream_t st) {
  if (n <= 0 || max_m <= 0) return;
  const int TW = max_m <= 256 ? 64 : 32;   // m x TW staged: <= 128 KB
  const size_t sm = sizeof(double) * max_m * TW;
  set_smem_attr((const void*)k_form_T_nodc, sm);
  const int tiles = (max_m + TW - 1) / TW;
  k_form_T_nodc<<<n * tiles, 256, sm, st>>>(d_items, tiles, TW);
  count_launch(1);
}

}  // namespace hs
