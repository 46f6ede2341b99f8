// Factor kernels (sm_100a), one per row of SURVEY §8(a):
//   a0 pack / a6 write-back / A_c assembly : k_copy2d (batched 2-D copy, smem-tiled transpose)
//   a1 POTRF  A_ss = G_s G_s^T                 : k_potrf
//   a2 TRSM   B = G_s^{-1}[A_sw | A_sn] (deferred compression) : k_trsm
//   a3+a4 CPQR of G_s^{-1}A_sw to eps with the rotation U^T fused onto the
//        n-columns (Eq. offdiag_new, Eq. CC:eqn:sparse P:537-565) : k_cpqr
//   a5 Schur  A_pq -= C_p^T C_q (Eq. CC:eqn:elim)    : k_schur
//   a7 top dense Cholesky                             : dense_potrf
// No kernel shares code with the oracle; see DESIGN.md for each kernel's roofline.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cfloat>
#include <cstdlib>
#include <atomic>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "device.h"

namespace hs {

namespace {

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ int warp_min_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide reductions; red must hold >= 32 entries; all threads get the result
__device__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double r = lane < nw ? red[lane] : -DBL_MAX;
  r = warp_max(r);
  return r;
}
__device__ int block_min_int(int v, int* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_min_int(v);
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  int r = lane < nw ? red[lane] : INT_MAX;
  return warp_min_int(r);
}

// ---------------------------------------------------------------------------------------
// a0/a6: batched 2-D copy.  Non-transposed: coalesced row copy.  Transposed: 32x32 smem tiles
// so that both the read and the write are coalesced.
__global__ void k_copy2d(const CopyItem* __restrict__ items) {
  const CopyItem it = items[blockIdx.x];
  if (it.rows <= 0 || it.cols <= 0) return;
  if (it.trans == 2) {   // square block with lower-triangle semantics -> full symmetric copy
    const int64_t tot = (int64_t)it.rows * it.cols;
    for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
      const int i = (int)(e / it.cols), j = (int)(e % it.cols);
      it.dst[(int64_t)i * it.dld + j] = i >= j ? it.src[(int64_t)i * it.sld + j] : it.src[(int64_t)j * it.sld + i];
    }
    return;
  }
  if (!it.trans) {   // a warp per row (no integer division), rows strided over the warps
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = w; i < it.rows; i += nw) {
      const double* __restrict__ s = it.src + (int64_t)i * it.sld;
      double* __restrict__ d = it.dst + (int64_t)i * it.dld;
      for (int j = lane; j < it.cols; j += 32) d[j] = s[j];
    }
    return;
  }
  __shared__ double tile[32][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5, ny = blockDim.x >> 5;
  for (int ti = 0; ti < it.rows; ti += 32)
    for (int tj = 0; tj < it.cols; tj += 32) {
      // src element (row j, col i) for dst (i, j): read along i (contiguous in src row j)
      for (int jj = ty; jj < 32; jj += ny) {
        const int j = tj + jj, i = ti + tx;
        tile[jj][tx] = (j < it.cols && i < it.rows) ? it.src[(int64_t)j * it.sld + i] : 0.0;
      }
      __syncthreads();
      for (int ii = ty; ii < 32; ii += ny) {
        const int i = ti + ii, j = tj + tx;
        if (i < it.rows && j < it.cols) it.dst[(int64_t)i * it.dld + j] = tile[tx][ii];
      }
      __syncthreads();
    }
}

__global__ void k_identity(double* const* ptr, const int32_t* ld, const int32_t* r) {
  double* p = ptr[blockIdx.x];
  const int n = r[blockIdx.x], l = ld[blockIdx.x];
  for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
    const int i = e / n, j = e % n;
    p[(int64_t)i * l + j] = (i == j) ? 1.0 : 0.0;
  }
}

__global__ void k_scatter(const double* __restrict__ vals, const int64_t* __restrict__ map, int64_t nnz,
                          double* __restrict__ blk) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = map[k];
    if (d >= 0) blk[d] = vals[k];
  }
}

// ---------------------------------------------------------------------------------------
// a1: right-looking Cholesky of an m x m block held in shared memory (m <= MAX_M).
// A pivot <= 0 (or NaN) records the first failure in *status (no shift, no jitter).
__device__ void potrf_core(double* g, int ld, int m, double* a, DevStatus* status, int level, int cluster) {
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) a[e] = g[(int64_t)(e / m) * ld + (e % m)];
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (threadIdx.x == 0) {
      const double d = a[j * m + j];
      if (!(d > 0.0)) {
        bad = 1;
        if (atomicCAS(&status->flag, 0, 1) == 0) {
          status->level = level;
          status->cluster = cluster;
          status->pivot = j;
          status->value = d;
        }
      } else {
        a[j * m + j] = sqrt(d);
      }
    }
    __syncthreads();
    if (bad) return;
    const double piv = a[j * m + j];
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) a[i * m + j] /= piv;
    __syncthreads();
    // trailing update of the lower triangle: a[i][k] -= a[i][j] * a[k][j], j < k <= i
    const int t = m - j - 1;
    const int tot = t * (t + 1) / 2;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) {
      // map e -> (i, k) with 0 <= k <= i < t
      int i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      while (i * (i + 1) / 2 > e) --i;
      const int k = e - i * (i + 1) / 2;
      const int ii = j + 1 + i, kk = j + 1 + k;
      a[ii * m + kk] -= a[ii * m + j] * a[kk * m + j];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
    const int i = e / m, k = e % m;
    g[(int64_t)i * ld + k] = (k <= i) ? a[e] : 0.0;
  }
}

__global__ void k_potrf(const CluItem* __restrict__ items, DevStatus* status) {
  extern __shared__ double smem[];
  const CluItem it = items[blockIdx.x];
  if (it.m == 0 || it.m > SMEM_M) return;
  potrf_core(it.G, it.pad0 ? it.pad0 : it.m, it.m, smem, status, it.level, it.cluster);   // pad0: ld of G
}

// a1 for m > SMEM_M: the same right-looking Cholesky in place in global memory (L1/L2
// resident: <= 2 MB per cluster), 1024 threads.  Coarse clusters only.
__global__ void __launch_bounds__(1024) k_potrf_gl(const CluItem* __restrict__ items, DevStatus* status) {
  const CluItem it = items[blockIdx.x];
  const int m = it.m;
  if (m <= SMEM_M) return;
  double* a = it.G;
  const int64_t ld = it.pad0 ? it.pad0 : m;   // pad0: ld of G (sub-block factorizations)
  __shared__ int bad;
  __shared__ double piv;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < m; ++j) {
    if (threadIdx.x == 0) {
      const double d = a[(int64_t)j * ld + j];
      if (!(d > 0.0)) {
        bad = 1;
        if (atomicCAS(&status->flag, 0, 1) == 0) {
          status->level = it.level;
          status->cluster = it.cluster;
          status->pivot = j;
          status->value = d;
        }
      } else {
        piv = sqrt(d);
        a[(int64_t)j * ld + j] = piv;
      }
    }
    __syncthreads();
    if (bad) return;
    for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) a[(int64_t)i * ld + j] /= piv;
    __syncthreads();
    const int t = m - j - 1;
    // rows i of the trailing lower triangle: a warp per row, lanes over k <= i
    for (int i = (threadIdx.x >> 5); i < t; i += (blockDim.x >> 5)) {
      const int ii = j + 1 + i;
      const double aij = a[(int64_t)ii * ld + j];
      for (int k = (threadIdx.x & 31); k <= i; k += 32) {
        const int kk = j + 1 + k;
        a[(int64_t)ii * ld + kk] -= aij * a[(int64_t)kk * ld + j];
      }
    }
    __syncthreads();
  }
  for (int64_t e = threadIdx.x; e < (int64_t)m * m; e += blockDim.x)
    if ((e % m) > (e / m)) a[(e / m) * ld + (e % m)] = 0.0;
}

__global__ void k_potrf_raw(double* g, int ld, int m, DevStatus* status, int level) {
  extern __shared__ double smem[];
  potrf_core(g, ld, m, smem, status, level, -1);
}

// ---------------------------------------------------------------------------------------
// a2: X = G^{-1} B for a column tile (<= 64 columns) of B (m x ncols, row-major ld ldB),
// G lower m x m (ld ldG).  G and the tile live in shared memory; 256 threads =
// 64 columns x 4 row groups, right-looking forward substitution.
// Tile width TW = 64 with G staged in smem for m <= SMEM_M; TW = 32 with G read through
// L1/L2 for larger m (the tile alone then fits: 32 x 512 doubles = 128 KB).
__device__ void trsm_core(const double* G, int ldG, int m, double* B, int ldB, int c0, int nc, double* sm) {
  const bool gs = m <= SMEM_M;
  const int TW = gs ? 64 : 32;
  const double* g;
  int ldg;
  double* x;
  if (gs) {
    double* gg = sm;              // m*m
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
      const int i = e / m, k = e % m;
      gg[e] = (k <= i) ? G[(int64_t)i * ldG + k] : 0.0;
    }
    g = gg;
    ldg = m;
    x = sm + m * m;               // m*TW
  } else {
    g = G;
    ldg = ldG;
    x = sm;
  }
  for (int e = threadIdx.x; e < m * TW; e += blockDim.x) {
    const int i = e / TW, c = e % TW;
    x[e] = c < nc ? B[(int64_t)i * ldB + c0 + c] : 0.0;
  }
  __syncthreads();
  const int c = threadIdx.x % TW, grp = threadIdx.x / TW, ngrp = blockDim.x / TW;
  for (int i = 0; i < m; ++i) {
    if (grp == 0) x[i * TW + c] /= g[(int64_t)i * ldg + i];
    __syncthreads();
    const double xi = x[i * TW + c];
    for (int l = i + 1 + grp; l < m; l += ngrp) x[l * TW + c] -= g[(int64_t)l * ldg + i] * xi;
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * TW; e += blockDim.x) {
    const int i = e / TW, cc = e % TW;
    if (cc < nc) B[(int64_t)i * ldB + c0 + cc] = x[e];
  }
}

// largest column norm of the n-columns [n0, nc) of the solved tile (R-floor of tau_s)
__device__ void trsm_nmax(const double* x, int m, int TW, int n0, int nc, unsigned long long* nmax) {
  const int c = threadIdx.x;
  double s = -1.0;
  if (c < TW && c >= n0 && c < nc) {
    s = 0.0;
    for (int i = 0; i < m; ++i) s += x[i * TW + c] * x[i * TW + c];
    s = sqrt(s);
  }
  for (int o = 16; o > 0; o >>= 1) s = fmax(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0 && s >= 0.0) atomicMax(nmax, (unsigned long long)__double_as_longlong(s));
}

__global__ void k_trsm(const CluItem* __restrict__ clu, const TrsmItem* __restrict__ items) {
  extern __shared__ double smem[];
  const TrsmItem t = items[blockIdx.x];
  const CluItem it = clu[t.ci];
  if (it.m == 0) return;
  trsm_core(it.G, it.pad0 ? it.pad0 : it.m, it.m, it.B, it.ldB, t.c0, t.nc, smem);   // pad0: ld of G
  if (it.nmax && t.c0 + t.nc > it.kw) {
    __syncthreads();
    const int TW = it.m <= SMEM_M ? 64 : 32;
    const double* x = it.m <= SMEM_M ? smem + it.m * it.m : smem;
    trsm_nmax(x, it.m, TW, max(0, it.kw - t.c0), t.nc, it.nmax);
  }
}

__global__ void k_trsm_raw(const double* G, int ldG, int m, double* B, int ldB, int ncols) {
  extern __shared__ double smem[];
  const int c0 = blockIdx.x * 64;
  trsm_core(G, ldG, m, B, ldB, c0, min(64, ncols - c0), smem);
}

// ---------------------------------------------------------------------------------------
// Apply operator of a cluster: T_s = U_s^T G_s^{-1} = H_{r-1} ... H_0 G_s^{-1} (the E_s S_s
// of W_s = P_s G_s E_s S_s), m x m row-major, formed once after CPQR so that the
// apply's local steps (Algorithm 2) are parallel matvecs instead of a serial
// triangular solve.  One CTA per (cluster, column tile): the tile of the identity is
// forward-substituted with G (smem-staged for m <= SMEM_M, else read through L1/L2),
// then the r reflectors are applied, H_0 first.  Launched once per level, after its last
// batch, on a side stream: T_s is only read by the apply, so it overlaps the next level.
__global__ void __launch_bounds__(256) k_form_T(const FormTItem* __restrict__ items, int tiles_per) {
  extern __shared__ double sm[];
  const int ci = blockIdx.x / tiles_per, tile = blockIdx.x % tiles_per;
  const FormTItem it = items[ci];
  const int m = it.m;
  const bool gs = m <= SMEM_M;
  const int TW = gs ? 64 : 32;
  const int c0 = tile * TW;
  if (m == 0 || c0 >= m) return;
  const int nc = min(TW, m - c0);
  const int r = it.r;
  const double* g;
  int ldg;
  double* x;
  if (gs) {
    double* gg = sm;
    if (!it.Ginv)   // G^{-1} given: no substitution, G is not needed
      for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int i = e / m, k = e % m;
        gg[e] = (k <= i) ? it.G[(int64_t)i * m + k] : 0.0;
      }
    g = gg;
    ldg = m;
    x = sm + m * m;
  } else {
    g = it.G;
    ldg = m;
    x = sm;
  }
  __shared__ double red[8][64];
  const int c = threadIdx.x % TW, grp = threadIdx.x / TW, ngrp = blockDim.x / TW;
  if (it.Ginv) {   // G^{-1} formed by k_chol: X = its columns [c0, c0 + nc)
    for (int e = threadIdx.x; e < m * TW; e += blockDim.x) {
      const int i = e / TW, cc = e % TW;
      x[e] = cc < nc ? it.Ginv[(int64_t)i * m + c0 + cc] : 0.0;
    }
    __syncthreads();
  } else {
    for (int e = threadIdx.x; e < m * TW; e += blockDim.x) {
      const int i = e / TW, cc = e % TW;
      x[e] = (cc < nc && i == c0 + cc) ? 1.0 : 0.0;
    }
    __syncthreads();
  }
  // X <- G^{-1} X  (rows above c0 stay zero: start the substitution at row c0)
  for (int i = it.Ginv ? m : c0; i < m; ++i) {
    if (grp == 0) x[i * TW + c] /= g[(int64_t)i * ldg + i];
    __syncthreads();
    const double xi = x[i * TW + c];
    for (int l = i + 1 + grp; l < m; l += ngrp) x[l * TW + c] -= g[(int64_t)l * ldg + i] * xi;
    __syncthreads();
  }
  // X <- H_j X for j = 0 .. r-1, H_j = I - tau_j v_j v_j^T (v_j = column j of V, zeros above j)
  for (int j = 0; j < r; ++j) {
    const double t = it.tau[j];
    const double* v = it.V + (int64_t)j * m;
    double d = 0.0;
    for (int l = j + grp; l < m; l += ngrp) d += v[l] * x[l * TW + c];
    red[grp][c] = d;
    __syncthreads();
    double s = 0.0;
    for (int q = 0; q < ngrp; ++q) s += red[q][c];
    const double td = t * s;
    for (int l = j + grp; l < m; l += ngrp) x[l * TW + c] -= td * v[l];
    __syncthreads();
  }
  for (int e = threadIdx.x; e < m * TW; e += blockDim.x) {
    const int i = e / TW, cc = e % TW;
    if (cc < nc) it.T[(int64_t)i * m + c0 + cc] = x[e];
  }
}

// ---------------------------------------------------------------------------------------

// ---------------------------------------------------------------------------------------
// a5: Schur update tiles, FP64 FMA (64 x 64 tile, 256 threads, 4 x 4 per thread),
// K staged through shared memory 16 rows at a time.  Contributions of a tile are summed
// in source-cluster order before the single read-modify-write of the target.
__global__ void __launch_bounds__(256) k_schur(const SchurTile* __restrict__ tiles,
                                               const SchurContrib* __restrict__ con) {
  const SchurTile t = tiles[blockIdx.x];
  __shared__ double ap[16][64];
  __shared__ double aq[16][64];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int c = t.c_begin; c < t.c_end; ++c) {
    const SchurContrib s = con[c];
    const double* Cp = s.C + s.colP + t.i0;
    const double* Cq = s.C + s.colQ + t.j0;
    for (int k0 = 0; k0 < s.K; k0 += 16) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = threadIdx.x + 256 * q;
        const int kk = e >> 6, ii = e & 63;
        const bool kin = k0 + kk < s.K;
        ap[kk][ii] = (kin && ii < t.rows) ? Cp[(int64_t)(k0 + kk) * s.ldC + ii] : 0.0;
        aq[kk][ii] = (kin && ii < t.cols) ? Cq[(int64_t)(k0 + kk) * s.ldC + ii] : 0.0;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < 16; ++kk) {
        double x[4], y[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) x[a] = ap[kk][ty + 16 * a];
#pragma unroll
        for (int b = 0; b < 4; ++b) y[b] = aq[kk][tx + 16 * b];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = fma(x[a], y[b], acc[a][b]);
      }
      __syncthreads();
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = ty + 16 * a, j = tx + 16 * b;
      if (i < t.rows && j < t.cols) t.dst[(int64_t)i * t.ld + j] -= acc[a][b];
    }
}

// ---------------------------------------------------------------------------------------
// a5: Schur update X_nn -= C^T C (Eq. CC:eqn:elim) for one source cluster per 64 x 64 tile
// of C^T C.  Target blocks are found on the device: row/column owners by binary search in
// the source's neighbour-column table, block pointers from the level's neighbour-pair
// tables (k_level_pairs, one directory search per pair per level).
constexpr int SCH_MAXO = 32;   // distinct owners per tile side held in the pointer table
constexpr int SCH_NBS = 512;   // neighbour column starts staged for the owner searches (k_schur3)

__device__ __forceinline__ int64_t dir_find(const BlockDir& d, int p, int q) {   // p >= q; -1 if absent
  int64_t lo = d.ptr[p], hi = d.ptr[p + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (d.q[mid] < q) lo = mid + 1;
    else hi = mid;
  }
  return (lo < d.ptr[p + 1] && d.q[lo] == q) ? d.off[lo] : -1;
}

// The C tile loads, the owner loads and the owner dedupe (warp ballots) overlap; the 64 x 64
// tile forms on the FP64 tensor cores (DMMA m8n8k4); the target addresses are resolved after
// the product and the subtraction is a fire-and-forget FP64 reduction in L2
// (red.global.add.f64): one update per target element per launch (the waves of a batch
// never share a target), so the result is the same as load-subtract-store.
__global__ void __launch_bounds__(256, 4) k_schur3(const SchurTile2* __restrict__ tiles, const SchurSrc* __restrict__ srcs,
                                                const NbCol* __restrict__ nbc, BlockDir dir) {
  pdl_trigger();
  pdl_wait();
  const SchurTile2 t = tiles[blockIdx.x];
  const SchurSrc s = srcs[t.src];
  if (s.K <= 0) return;   // planned before its rank was known and kept everything (uniform)
  const NbCol* nb = nbc + s.nb_off;
  __shared__ double ap[16][68];   // row stride == 4 (mod 16): conflict-free m8n8k4 fragments
  __shared__ double aq[16][68];
  __shared__ int r_own[64], r_loc[64], c_own[64], c_loc[64];
  __shared__ int r_slot[64], c_slot[64];
  __shared__ int r_list[64], c_list[64];
  __shared__ int nr, nc;
  __shared__ double* ptab[SCH_MAXO][SCH_MAXO];
  __shared__ int ldtab[SCH_MAXO];
  __shared__ int nbcol[SCH_NBS];
  const int rows = min(64, s.kn - t.i0), cols = min(64, s.kn - t.j0);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // (1) the neighbours' column starts into shared memory (the owner searches) + the first
  // K-chunk of C (this thread's columns i0 + ii / j0 + ii, ii = tid & 63 in every chunk)
  const bool nst = s.nnb <= SCH_NBS;
  if (nst)
    for (int a = tid; a < s.nnb; a += blockDim.x) nbcol[a] = nb[a].col;
  const int ii0 = tid & 63;
  const double* Cp = s.C + t.i0 + (ii0 < rows ? ii0 : 0);
  const double* Cq = s.C + t.j0 + (ii0 < cols ? ii0 : 0);
  auto load_chunk = [&](int k0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;
      const int kk = e >> 6, ii = e & 63;
      const bool kin = k0 + kk < s.K;
      ap[kk][ii] = (kin && ii < rows) ? Cp[(int64_t)(k0 + kk) * s.ldC] : 0.0;
      aq[kk][ii] = (kin && ii < cols) ? Cq[(int64_t)(k0 + kk) * s.ldC] : 0.0;
    }
  };
  load_chunk(0);
  __syncthreads();
  if (w < 2) {   // (2) owners of the tile's rows (warp 0) / columns (warp 1) by binary search,
                 // distinct owners in order (rows/cols are sorted by owner): ballots
    const int lim = w == 0 ? rows : cols, base = w == 0 ? t.i0 : t.j0;
    auto owner = [&](int c) {   // last a with col(a) <= c
      int lo = 0, hi = s.nnb - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((nst ? nbcol[mid] : nb[mid].col) <= c) lo = mid;
        else hi = mid - 1;
      }
      return lo;
    };
    const int o0 = lane < lim ? owner(base + lane) : -1;
    const int o1 = lane + 32 < lim ? owner(base + lane + 32) : -1;
    const int prev0 = __shfl_up_sync(0xffffffffu, o0, 1);
    const int last0 = __shfl_sync(0xffffffffu, o0, 31);
    const int prev1 = __shfl_up_sync(0xffffffffu, o1, 1);
    const bool f0 = lane < lim && (lane == 0 || o0 != prev0);
    const bool f1 = lane + 32 < lim && (lane == 0 ? o1 != last0 : o1 != prev1);
    const unsigned m0 = __ballot_sync(0xffffffffu, f0), m1 = __ballot_sync(0xffffffffu, f1);
    const unsigned le = 0xffffffffu >> (31 - lane);
    const int s0 = __popc(m0 & le) - 1, s1 = __popc(m0) + __popc(m1 & le) - 1;
    int* own = w == 0 ? r_own : c_own;
    int* loc = w == 0 ? r_loc : c_loc;
    int* slot = w == 0 ? r_slot : c_slot;
    int* list = w == 0 ? r_list : c_list;
    if (lane < lim) {
      own[lane] = o0;
      const NbCol g = nb[o0];
      const int c = base + lane - g.col;
      loc[lane] = g.sup ? g.sup[c] : c;
      slot[lane] = s0;
      if (f0) list[s0] = o0;
    }
    if (lane + 32 < lim) {
      own[lane + 32] = o1;
      const NbCol g = nb[o1];
      const int c = base + lane + 32 - g.col;
      loc[lane + 32] = g.sup ? g.sup[c] : c;
      slot[lane + 32] = s1;
      if (f1) list[s1] = o1;
    }
    if (lane == 0) (w == 0 ? nr : nc) = __popc(m0) + __popc(m1);
  }
  __syncthreads();
  // (3) target block pointers of the distinct owner pairs
  const bool table = nr <= SCH_MAXO && nc <= SCH_MAXO;
  if (table) {
    for (int e = tid; e < nr * nc; e += blockDim.x) {
      const int ra = e / nc, cb = e % nc;
      const int a = nb[r_list[ra]].idx, b = nb[c_list[cb]].idx;
      ptab[ra][cb] = a >= b ? s.pairs[(int64_t)a * (a + 1) / 2 + b] : nullptr;
    }
    for (int cb = tid; cb < nc; cb += blockDim.x) ldtab[cb] = dir.cap[nb[c_list[cb]].q];
  }
  __syncthreads();
  // (4) target addresses (nullptr = none)
  auto target = [&](int tc, int e) -> double* {
    const int i = 8 * w + (lane >> 2), j = 8 * tc + 2 * (lane & 3) + e;
    if (i >= rows || j >= cols) return nullptr;
    const int oa = r_own[i], ob = c_own[j];
    if (oa < ob) return nullptr;                          // upper: the transposed block
    const int li = r_loc[i], lj = c_loc[j];
    if (oa == ob && li < lj) return nullptr;              // diagonal block: lower triangle only
    double* p;
    int ld;
    if (table) {
      p = ptab[r_slot[i]][c_slot[j]];
      ld = ldtab[c_slot[j]];
    } else {
      const int fa = nb[oa].idx, fb = nb[ob].idx;
      p = s.pairs[(int64_t)fa * (fa + 1) / 2 + fb];
      ld = dir.cap[nb[ob].q];
    }
    return p ? p + (int64_t)li * ld + lj : nullptr;
  };
  // (5) the 64 x 64 tile of C^T C forms on the FP64 tensor cores (DMMA m8n8k4):
  // warp w owns output rows 8w..8w+7; lane l holds rows 8w + l/4, columns 8 tc + 2 (l % 4) + {0, 1}
  double acc[8][2];
#pragma unroll
  for (int tc = 0; tc < 8; ++tc) acc[tc][0] = acc[tc][1] = 0.0;
  for (int k0 = 0; k0 < s.K; k0 += 16) {
    if (k0 > 0) {
      __syncthreads();
      load_chunk(k0);
      __syncthreads();
    }
#pragma unroll
    for (int kk = 0; kk < 16; kk += 4) {
      const double a = ap[kk + (lane & 3)][8 * w + (lane >> 2)];   // A = C_p^T, row-major 8 x 4
#pragma unroll
      for (int tc = 0; tc < 8; ++tc) {
        const double b = aq[kk + (lane & 3)][8 * tc + (lane >> 2)];   // B = C_q, col-major 4 x 8
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(acc[tc][0]), "+d"(acc[tc][1])
                     : "d"(a), "d"(b));
      }
    }
  }
#pragma unroll
  for (int tc = 0; tc < 8; ++tc)
#pragma unroll
    for (int e = 0; e < 2; ++e) {   // addresses resolved after the product: nothing but acc live across it
      double* o = target(tc, e);
      if (o) atomicAdd(o, -acc[tc][e]);
    }
}

__global__ void k_symcheck(const double* __restrict__ v, const int64_t* __restrict__ tmap, int64_t nnz,
                           int32_t* flag) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const double a = v[k], t = v[tmap[k]];
    if (!(fabs(a - t) <= 1e-12 * fmax(fabs(a), fabs(t)))) *flag = 1;
  }
}

// The opt-in dynamic shared memory of a kernel only ever grows: handles on other host
// threads (multi-rank loopback, several solvers in one process) launch the same kernels, so
// lowering it could make a concurrent launch fail.
void set_smem(const void* f, size_t bytes) {
  static std::mutex mu;
  static std::unordered_map<const void*, size_t> cur;
  std::lock_guard<std::mutex> lk(mu);
  size_t& c = cur[f];
  if (bytes <= c) return;
  HS_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  c = bytes;
}

std::atomic<int64_t> g_launches{0};

}  // namespace

bool pdl_enabled() {
  static const bool on = std::getenv("HS_NO_PDL") == nullptr;
  return on;
}

void set_smem_attr(const void* f, size_t bytes) { set_smem(f, bytes); }

namespace {

}  // namespace

void count_launch(int64_t n) {
  g_launches += n;
  // a launch that could not start (configuration error) must not pass silently
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(HS_E_CUDA, std::string("kernel launch: ") + cudaGetErrorString(e));
  }
}
int64_t launch_count() { return g_launches.load(); }

// ---- launchers -----------------------------------------------------------------------------
void launch_symcheck(const double* vals, const int64_t* tmap, int64_t nnz, int32_t* flag, cudaStream_t st) {
  if (nnz <= 0) return;
  k_symcheck<<<(int)std::min<int64_t>((nnz + 255) / 256, 148 * 16), 256, 0, st>>>(vals, tmap, nnz, flag);
  count_launch(1);
}
namespace {
__device__ void publish_body(const int32_t* __restrict__ rank, int n, const DevStatus* __restrict__ status,
                             RankPub* pub, int32_t seq) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) pub->rank[i] = rank[i];
  if (threadIdx.x == 0) {
    pub->flag = status->flag;
    pub->level = status->level;
    pub->cluster = status->cluster;
    pub->pivot = status->pivot;
    pub->value = status->value;
  }
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    pub->seq = seq;
  }
}

// the patch items: one thread each
__global__ void k_patch(const PatchItem* __restrict__ items, int n, const int32_t* __restrict__ rank) {
  pdl_trigger();
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const PatchItem p = items[i];
  const int r = p.m == 0 ? 0 : rank[p.bi], K = p.m - r;
  switch (p.kind) {
    case PK_SRC: {   // C_s = B_s[r:, kw:], K fine rows (a full rank leaves a phantom source)
      SchurSrc* t = (SchurSrc*)p.target;
      t->C = p.base + (int64_t)r * p.ldB + p.kw;
      t->K = K;
      break;
    }
    case PK_K: ((SchurSrc*)p.target)->K = K; break;   // C already in its slab
    case PK_ROWS: ((CopyItem*)p.target)->rows = r; break;
    case PK_COLS: ((CopyItem*)p.target)->cols = r; break;
    case PK_I32: *(int32_t*)p.target = r; break;
    case PK_FT: ((FormTItem*)p.target)->r = r; break;
    case PK_CCOPY: {   // rows [i0, i0 + step) of C_s into its slab
      CopyItem* t = (CopyItem*)p.target;
      t->src = p.base + (int64_t)(r + p.i0) * p.ldB + p.kw;
      t->rows = max(0, min(p.step, K - p.i0));
      break;
    }
  }
}
}  // namespace

namespace {
__device__ void publish_body(const int32_t* __restrict__ rank, int n, const DevStatus* __restrict__ status,
                             RankPub* pub, int32_t seq);
__global__ void k_publish(const int32_t* __restrict__ rank, int n, const DevStatus* __restrict__ status, RankPub* pub,
                          int32_t seq) {
  pdl_trigger();
  pdl_wait();
  publish_body(rank, n, status, pub, seq);
}
}  // namespace

void launch_publish(const int32_t* d_rank, int n, const DevStatus* d_status, RankPub* pub, int32_t seq,
                    cudaStream_t st) {
  launch_pdl(k_publish, dim3(1), dim3(256), 0, st, d_rank, n, d_status, pub, seq);
  count_launch(1);
}

void launch_patch(const PatchItem* d_items, int n, const int32_t* d_rank, cudaStream_t st) {
  const int blocks = (n + 127) / 128;
  if (blocks <= 0) return;
  launch_pdl(k_patch, dim3(blocks), dim3(128), 0, st, d_items, n, d_rank);
  count_launch(1);
}

void split_copies(std::vector<CopyItem>& items) {
  constexpr int64_t PIECE = 16384;
  bool big = false;
  for (const auto& it : items) big |= (int64_t)it.rows * it.cols > PIECE && it.trans != 2;
  if (!big) return;
  std::vector<CopyItem> out;
  out.reserve(items.size() * 2);
  for (const auto& it : items) {
    if ((int64_t)it.rows * it.cols <= PIECE || it.trans == 2) {
      out.push_back(it);
      continue;
    }
    const int step = std::max(1, (int)(PIECE / std::max(it.cols, 1)));
    for (int i0 = 0; i0 < it.rows; i0 += step) {
      CopyItem p = it;
      p.rows = std::min(step, it.rows - i0);
      // dst rows [i0, i0+rows); source rows (trans 0) or source columns (trans 1)
      p.dst = it.dst + (int64_t)i0 * it.dld;
      p.src = it.trans ? it.src + i0 : it.src + (int64_t)i0 * it.sld;
      out.push_back(p);
    }
  }
  items.swap(out);
}
void launch_copy2d(const CopyItem* d_items, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_copy2d<<<n, 256, 0, st>>>(d_items);
  count_launch(1);
}
void launch_identity(double* const* d_ptr, const int32_t* d_ld, const int32_t* d_r, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_identity<<<n, 128, 0, st>>>(d_ptr, d_ld, d_r);
  count_launch(1);
}
void launch_scatter(const double* vals, const int64_t* map, int64_t nnz, double* blk, cudaStream_t st) {
  if (nnz <= 0) return;
  k_scatter<<<(int)std::min<int64_t>((nnz + 255) / 256, 148 * 16), 256, 0, st>>>(vals, map, nnz, blk);
  count_launch(1);
}
void launch_potrf(const CluItem* d_items, int n, int max_m, DevStatus* status, cudaStream_t st) {
  if (n <= 0) return;
  const int ms = std::min(max_m, SMEM_M);
  const size_t sm = (size_t)ms * ms * sizeof(double);
  set_smem((const void*)k_potrf, sm);
  k_potrf<<<n, 256, sm, st>>>(d_items, status);
  count_launch(1);
  if (max_m > SMEM_M) {
    k_potrf_gl<<<n, 1024, 0, st>>>(d_items, status);
    count_launch(1);
  }
}
void launch_trsm(const CluItem* d_clu, const TrsmItem* d_items, int n, int max_m, cudaStream_t st) {
  if (n <= 0) return;
  const int ms = std::min(max_m, SMEM_M);
  size_t words = (size_t)ms * ms + (size_t)ms * 64;
  if (max_m > SMEM_M) words = std::max(words, (size_t)max_m * 32);
  const size_t sm = words * sizeof(double);
  set_smem((const void*)k_trsm, sm);
  k_trsm<<<n, 256, sm, st>>>(d_clu, d_items);
  count_launch(1);
}
void launch_form_T(const FormTItem* d_items, int n, int max_m, cudaStream_t st) {
  if (n <= 0 || max_m <= 0) return;
  const bool gs = max_m <= SMEM_M;
  const int TW = gs ? 64 : 32;
  const int ms = std::min(max_m, SMEM_M);
  size_t words = (size_t)ms * ms + (size_t)ms * 64;
  if (!gs) words = std::max(words, (size_t)max_m * 32);
  const size_t sm = words * sizeof(double);
  set_smem((const void*)k_form_T, sm);
  const int tiles = (max_m + TW - 1) / TW;
  k_form_T<<<n * tiles, 256, sm, st>>>(d_items, tiles);
  count_launch(1);
}
void launch_schur(const SchurTile* d_tiles, const SchurContrib* d_con, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_schur<<<n, 256, 0, st>>>(d_tiles, d_con);
  count_launch(1);
}
// Level pair tables: a warp per (cluster s, neighbour a); lanes over b <= a look the block
// (q_a, q_b) up in the level's directory.  Pattern-only, once per level.
__global__ void __launch_bounds__(256) k_level_pairs(const int64_t* __restrict__ hptr, const int32_t* __restrict__ hq,
                                                     const int64_t* __restrict__ poff, const int64_t* __restrict__ row_cl,
                                                     int64_t nrows, double** __restrict__ pairs, BlockDir dir) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nrows) return;
  const int64_t s = row_cl[w];
  const int a = (int)(w - hptr[s]);
  const int32_t* q = hq + hptr[s];
  double** out = pairs + poff[s] + (int64_t)a * (a + 1) / 2;
  for (int b = lane; b <= a; b += 32) {
    const int64_t o = dir_find(dir, q[a], q[b]);
    out[b] = o >= 0 ? dir.blk + o : nullptr;
  }
}
void launch_level_pairs(const int64_t* hptr, const int32_t* hq, const int64_t* poff, int nclus, int64_t nrows,
                        const int64_t* row_cl, double** pairs, const BlockDir& dir, cudaStream_t st) {
  if (nrows <= 0) return;
  k_level_pairs<<<(unsigned)((nrows * 32 + 255) / 256), 256, 0, st>>>(hptr, hq, poff, row_cl, nrows, pairs, dir);
  count_launch(1);
}
void launch_schur2(const SchurTile2* d_tiles, int n, const SchurSrc* d_src, const NbCol* d_nb, const BlockDir& dir,
                   cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_schur3, dim3(n), dim3(256), 0, st, d_tiles, d_src, d_nb, dir);
  count_launch(1);
}

// a7: blocked right-looking Cholesky of the dense top matrix.
void dense_potrf(double* A, int N, int ld, DevStatus* status, int level, double* /*unused*/, cudaStream_t st) {
  const int NB = TOP_NB;
  set_smem((const void*)k_potrf_raw, (size_t)NB * NB * sizeof(double));
  set_smem((const void*)k_trsm_raw, ((size_t)NB * NB + (size_t)NB * 64) * sizeof(double));
  std::vector<SchurTile> tiles;
  SchurContrib* d_con = nullptr;
  SchurTile* d_tiles = nullptr;
  const int nblk = (N + NB - 1) / NB;
  const size_t max_tiles = (size_t)nblk * (nblk + 1) / 2 + 1;
  HS_CUDA(cudaMalloc(&d_con, sizeof(SchurContrib) * nblk));
  HS_CUDA(cudaMalloc(&d_tiles, sizeof(SchurTile) * max_tiles));
  std::vector<SchurContrib> cons(nblk);
  for (int k = 0; k < N; k += NB) {
    const int nb = std::min(NB, N - k);
    k_potrf_raw<<<1, 256, (size_t)nb * nb * sizeof(double), st>>>(A + (int64_t)k * ld + k, ld, nb, status, level);
    const int rest = N - k - nb;
    if (rest <= 0) {
      count_launch(1);
      break;
    }
    k_trsm_raw<<<(rest + 63) / 64, 256, ((size_t)nb * nb + (size_t)nb * 64) * sizeof(double), st>>>(
        A + (int64_t)k * ld + k, ld, nb, A + (int64_t)k * ld + k + nb, ld, rest);
    const int kb = k / NB;
    cons[kb] = SchurContrib{A + (int64_t)k * ld + k + nb, ld, nb, 0, 0};
    tiles.clear();
    for (int i0 = 0; i0 < rest; i0 += 64)
      for (int j0 = i0; j0 < rest; j0 += 64) {
        SchurTile t{};
        t.dst = A + (int64_t)(k + nb + i0) * ld + (k + nb + j0);
        t.ld = ld;
        t.rows = std::min(64, rest - i0);
        t.cols = std::min(64, rest - j0);
        t.c_begin = kb;
        t.c_end = kb + 1;
        t.i0 = i0;
        t.j0 = j0;
        tiles.push_back(t);
      }
    HS_CUDA(cudaMemcpyAsync(d_con + kb, &cons[kb], sizeof(SchurContrib), cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(d_tiles, tiles.data(), sizeof(SchurTile) * tiles.size(),
                            cudaMemcpyHostToDevice, st));
    k_schur<<<(int)tiles.size(), 256, 0, st>>>(d_tiles, d_con);
    count_launch(3);
    HS_CUDA(cudaStreamSynchronize(st));   // host vectors are reused; the top runs once per factor
  }
  HS_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_con);
  cudaFree(d_tiles);
}

}  // namespace hs
