// a0 + a1 + a2 for the DC path (clusters up to CI_MAX_M): the deferred-compression scaling
// B_s = G_s^{-1} [A_sw | A_sn] with A_ss = G_s G_s^T (Eq. CC:eqn:scaling)
// as two kernels, no gather pass and no CTA-wide barrier inside the triangular solve:
//   k_chol_mma   one CTA per cluster: A_ss read straight from the level's block store into
//                shared memory, blocked (8 x 8 tiles) Cholesky and G_s^{-1} with the panel,
//                trailing and inverse products on the FP64 tensor cores; G_s and G_s^{-1}
//                stored to the workspace;
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

// B[:, c0:c0+nc] = G^{-1} A[:, c0:c0+nc] on the FP64 tensor cores: the tile of [A_sw | A_sn]
// is gathered from the store segments into shared memory, G_s^{-1} (lower) staged beside it,
// and the m x 64 product formed with DMMA (mma.sync.m8n8k4.f64): warp w owns output columns
// 8w..8w+7 and every 8-row block, the k loop skips the zero upper triangle of G^{-1}.
// Row strides == 4 (mod 16) make the fragment loads conflict-free.  The result goes back to
// B_s through shared memory (coalesced rows) and the largest n-column norm (R-floor) is
// reduced from it.
constexpr int SM_LDX = 68;   // tile row stride (doubles)
__host__ __device__ __forceinline__ int mma_ldg(int m) { return ((m + 11) / 16) * 16 + 4; }   // >= m, == 4 mod 16
// A_ss = G_s G_s^T and G_s^{-1}, blocked by 8 x 8 tiles on the FP64 tensor cores
// (DMMA m8n8k4).  One CTA per cluster, the matrix in shared memory (rows padded to 8 NB8
// with an identity tail, row stride == 4 mod 16: conflict-free fragments).  Per diagonal
// tile kb: warp 0 factors the 8 x 8 tile and inverts it (8 warp-synchronous steps each);
// the panel L[ib][kb] = A[ib][kb] L_kk^{-T} and the trailing update A[ib][jb] -= L[ib][kb]
// L[jb][kb]^T are 8 x 8 x 8 DMMA products spread over the warps (3 barriers per tile
// column instead of one per pivot).  G^{-1} follows by blocked forward substitution,
// X[ib][jb] = -X[ib][ib] sum_{jb <= t < ib} L[ib][t] X[t][jb], one tile row at a time.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}
// One warp: the 8 x 8 lower tile T = G_kk G_kk^T factored in place (G_kk) and its inverse
// written to Y, in registers: lane c (and its copies c + 8, c + 16, c + 24) holds column c of
// T and of Y; step j broadcasts column j (shuffles), every lane updates its column (the
// loop over j is unrolled, so every register index is static).  false: pivot j not positive.
__device__ __forceinline__ bool diag8(double* T, double* Y, int ld, int lane, double& dbad, int& jbad) {
  const int c = lane & 7;
  double t[8], y[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    t[r] = T[r * ld + c];
    y[r] = r == c ? 1.0 : 0.0;
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const double d = __shfl_sync(0xffffffffu, t[j], j);
    if (!(d > 0.0)) {   // the same d on every lane
      dbad = d;
      jbad = j;
      return false;
    }
    const double g = sqrt(d), rg = 1.0 / g;
    if (c == j) {
      t[j] = g;
#pragma unroll
      for (int r = j + 1; r < 8; ++r) t[r] *= rg;
    }
    double v[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) v[r] = __shfl_sync(0xffffffffu, t[r], j);   // column j of G
    double vc = v[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) vc = c == q ? v[q] : vc;   // G[c][j]
#pragma unroll
    for (int r = j + 1; r < 8; ++r)
      if (c > j && r >= c) t[r] = fma(-v[r], vc, t[r]);   // T[r][c] -= G[r][j] G[c][j]
    y[j] *= rg;                                             // Y[j][c] final
#pragma unroll
    for (int r = j + 1; r < 8; ++r) y[r] = fma(-v[r], y[j], y[r]);
  }
  if (lane < 8)
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r >= c) T[r * ld + c] = t[r];
      Y[r * ld + c] = r >= c ? y[r] : 0.0;
    }
  __syncwarp();
  return true;
}
template <int NB8>
__global__ void __launch_bounds__(256) k_chol_mma(const FusedItem* __restrict__ items, DevStatus* status) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double sm[];
  constexpr int MP = 8 * NB8;
  const int ld = mma_ldg(MP);
  double* L = sm;              // MP x ld: A (lower), overwritten by G
  double* X = sm + MP * ld;    // MP x ld: G^{-1} (lower)
  __shared__ int bad;
  const FusedItem it = items[blockIdx.x];
  const int m = it.m;
  if (m == 0) return;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;
  for (int e0 = tid; e0 < MP * MP; e0 += 8 * 256) {   // 8 loads in flight per thread
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + 256 * u, i = e / MP, k = e % MP;
      v[u] = (e < MP * MP && i < m && k <= i) ? it.Ass[(int64_t)i * it.lda + k] : (i == k ? 1.0 : 0.0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e = e0 + 256 * u, i = e / MP, k = e % MP;
      if (e < MP * MP) {
        L[i * ld + k] = v[u];
        X[i * ld + k] = 0.0;
      }
    }
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int kb = 0; kb < NB8; ++kb) {
    const int o = 8 * kb;
    if (w == 0) {   // factor the diagonal tile T = L[o:o+8, o:o+8] and invert it into X
      double d;
      int jbad;
      if (!diag8(L + o * ld + o, X + o * ld + o, ld, lane, d, jbad) && lane == 0) {
        bad = 1;
        if (atomicCAS(&status->flag, 0, 1) == 0) {
          status->level = it.level;
          status->cluster = it.cluster;
          status->pivot = o + jbad;
          status->value = d;
        }
      }
    }
    __syncthreads();
    if (bad) return;
    // panel: L[ib][kb] = A[ib][kb] Y^T (Y = L_kk^{-1}), a tile per warp
    for (int ib = kb + 1 + w; ib < NB8; ib += 8) {
      double* P = L + 8 * ib * ld + o;
      const double* Y = X + o * ld + o;
      double c[2] = {0.0, 0.0};
      const double a0 = P[fr * ld + fc], a1 = P[fr * ld + 4 + fc];
      const double b0 = Y[fr * ld + fc], b1 = Y[fr * ld + 4 + fc];   // B[k][n] = Y[n][k]
      dmma(c, a0, b0);
      dmma(c, a1, b1);
      P[fr * ld + 2 * fc] = c[0];
      P[fr * ld + 2 * fc + 1] = c[1];
    }
    __syncthreads();
    // trailing: A[ib][jb] -= L[ib][kb] L[jb][kb]^T, kb < jb <= ib
    const int Tn = NB8 - kb - 1;
    for (int t = w; t < Tn * (Tn + 1) / 2; t += 8) {
      int ib = 0;
      while ((ib + 1) * (ib + 2) / 2 <= t) ++ib;
      const int jb = t - ib * (ib + 1) / 2;
      const int I = 8 * (kb + 1 + ib), J = 8 * (kb + 1 + jb);
      double* C = L + I * ld + J;
      double c[2] = {C[fr * ld + 2 * fc], C[fr * ld + 2 * fc + 1]};
      const double* Pi = L + I * ld + o;
      const double* Pj = L + J * ld + o;
      dmma(c, -Pi[fr * ld + fc], Pj[fr * ld + fc]);
      dmma(c, -Pi[fr * ld + 4 + fc], Pj[fr * ld + 4 + fc]);
      C[fr * ld + 2 * fc] = c[0];
      C[fr * ld + 2 * fc + 1] = c[1];
    }
    __syncthreads();
  }
  // G^{-1}: tile row ib, every jb < ib on its own warp
  for (int ib = 1; ib < NB8; ++ib) {
    for (int jb = w; jb < ib; jb += 8) {
      double s[2] = {0.0, 0.0};
      for (int t = jb; t < ib; ++t) {   // S = sum_t L[ib][t] X[t][jb]
        const double* Lt = L + 8 * ib * ld + 8 * t;
        const double* Xt = X + 8 * t * ld + 8 * jb;
        dmma(s, Lt[fr * ld + fc], Xt[fc * ld + fr]);
        dmma(s, Lt[fr * ld + 4 + fc], Xt[(4 + fc) * ld + fr]);
      }
      double* D = X + 8 * ib * ld + 8 * jb;   // S staged in its destination, then X = -Y_ib S
      D[fr * ld + 2 * fc] = s[0];
      D[fr * ld + 2 * fc + 1] = s[1];
      __syncwarp();
      const double* Y = X + 8 * ib * ld + 8 * ib;
      const double a0 = -Y[fr * ld + fc], a1 = -Y[fr * ld + 4 + fc];
      const double b0 = D[fc * ld + fr], b1 = D[(4 + fc) * ld + fr];
      double x[2] = {0.0, 0.0};
      dmma(x, a0, b0);
      dmma(x, a1, b1);
      __syncwarp();
      D[fr * ld + 2 * fc] = x[0];
      D[fr * ld + 2 * fc + 1] = x[1];
    }
    __syncthreads();
  }
  for (int e = tid; e < m * m; e += 256) {   // G and G^{-1}: lower, zeros above
    const int i = e / m, k = e % m;
    it.G[e] = k <= i ? L[i * ld + k] : 0.0;
    it.Ginv[e] = k <= i ? X[i * ld + k] : 0.0;
  }
}

template <int NRB>
__global__ void __launch_bounds__(256) k_scale_mma(const FusedItem* __restrict__ clus,
                                                   const ScaleTile* __restrict__ tiles,
                                                   const FusedSeg* __restrict__ segs) {
  pdl_trigger();
  pdl_wait();
  extern __shared__ double sm[];
  const ScaleTile tl = tiles[blockIdx.x];
  const FusedItem it = clus[tl.ci];
  const int m = it.m;
  if (m == 0 || tl.nc <= 0) return;
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
  for (int sg = tl.seg_begin; sg < tl.seg_end; ++sg) {   // the tile's columns from the store
    const FusedSeg sgm = segs[sg];
    const int j0 = max(tl.c0, sgm.col), j1 = min(tl.c0 + tl.nc, sgm.col + sgm.len);
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
        dst[u] = e < tot ? i * SM_LDX + (j - tl.c0) : -1;
        const int lc = e >= tot ? 0 : (sgm.idx ? sgm.idx[j - sgm.col] : j - sgm.col);   // column inside the block
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
    if (cc < tl.nc) it.B[(int64_t)i * it.ldB + tl.c0 + cc] = x[i * SM_LDX + cc];
  }
  if (it.nmax && tl.c0 + tl.nc > it.kw) {   // largest n-column norm (R-floor of tau_s)
    double s = -1.0;
    const int n0 = max(0, it.kw - tl.c0);
    if (tid < ST_TW && tid >= n0 && tid < tl.nc) {
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
  const int NB8 = (max_m + 7) / 8;
#define HS_CH(B)                                                                   \
  case B: {                                                                        \
    const size_t sm = sizeof(double) * 2 * (size_t)(8 * B) * mma_ldg(8 * B);        \
    set_smem_attr((const void*)k_chol_mma<B>, sm);                                 \
    launch_pdl(k_chol_mma<B>, dim3(n), dim3(256), sm, st, d_items, status);        \
    break;                                                                         \
  }
  switch (NB8) {
    HS_CH(1) HS_CH(2) HS_CH(3) HS_CH(4) HS_CH(5) HS_CH(6) HS_CH(7)
    HS_CH(8) HS_CH(9) HS_CH(10) HS_CH(11) HS_CH(12) HS_CH(13) HS_CH(14)
    default: fail(HS_E_INTERNAL, "launch_chol: m above CI_MAX_M");
  }
#undef HS_CH
  count_launch(1);
}

void launch_scale_tiles(const FusedItem* d_clus, const ScaleTile* d_tiles, int n, const FusedSeg* d_segs, int max_m,
                        cudaStream_t st) {
  if (n <= 0) return;
  const int nrb = (max_m + 7) / 8;
  const size_t sm = sizeof(double) * ((size_t)8 * nrb * mma_ldg(max_m) + (size_t)8 * nrb * SM_LDX);
#define HS_SM(NB)                                                     \
  case NB:                                                            \
    set_smem_attr((const void*)k_scale_mma<NB>, sm);                  \
    launch_pdl(k_scale_mma<NB>, dim3(n), dim3(256), sm, st, d_clus, d_tiles, d_segs); \
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
