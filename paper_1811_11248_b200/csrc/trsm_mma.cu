// a2 for clusters above the fused path's CI_MAX_M (coarse levels, m <= MAX_M): the deferred-
// compression scaling B_s <- G_s^{-1} [A_sw | A_sn] as a blocked forward
// substitution on the FP64 tensor cores, in place in the gathered B_s.
//
// One CTA per (cluster, 32-column strip) of B_s.  The strip's rows are split in 8-row blocks
// and the blocks are dealt round-robin to the warps (warp w owns blocks w, w + NWARP, ...),
// each warp keeping its blocks of the strip in DMMA accumulator registers for the whole
// solve.  With Y_b = G_bb^{-1} (the 8 x 8 diagonal inverses, formed up front in shared
// memory) the right-looking block step b is
//     X_b <- Y_b X_b                        (owner warp of block b, 8 x 8 x 32 DMMA)
//     X_i <- X_i - G_ib X_b   for i > b     (every warp on its blocks, 8 x 8 x 32 DMMA each)
// with X_b handed over through a double-buffered shared-memory tile: one CTA barrier per
// 8 rows instead of two per row (trsm_core), and the rank-8 trailing updates on DMMA
// (mma.sync.m8n8k4.f64).  The G_ib fragments of step b + 1 are loaded while step b computes.
// Same quantity as trsm_core, other rounding order (DESIGN.md §2 "Rounding order").
#include <cuda_runtime.h>

#include "device.h"

namespace hs {

namespace {

constexpr int TM_TW = 32;        // strip width (columns)
constexpr int TM_LDS = 36;       // hand-over tile row stride (== 4 mod 16: conflict-free fragments)

__device__ __forceinline__ void dmma8(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

template <int NWARP, int NW>
__global__ void __launch_bounds__(NWARP * 32) k_trsm_mma(const CluItem* __restrict__ clu,
                                                          const TrsmItem* __restrict__ items) {
  extern __shared__ double sm[];
  const TrsmItem t = items[blockIdx.x];
  const CluItem it = clu[t.ci];
  const int m = it.m;
  if (m == 0) return;
  const int nb = (m + 7) >> 3;
  const int ldG = it.pad0 ? it.pad0 : m;
  const double* __restrict__ G = it.G;
  double* Yd = sm;                          // nb x 64: Y_b row-major 8 x 8
  double* buf = sm + (size_t)nb * 64;       // 2 x 8 x TM_LDS hand-over tiles
  double* red = buf + 2 * 8 * TM_LDS;       // NWARP x 32 column sums (R-floor)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int fr = lane >> 2, fc = lane & 3;

  // ---- the diagonal inverses: lane c < 8 of a warp solves G_bb y = e_c (column c of Y_b) ---
  for (int b = w; b < nb; b += NWARP) {
    if (lane < 8) {
      const int c = lane;
      double y[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int gj = 8 * b + j;
        double s = (j == c) ? 1.0 : 0.0;
        if (gj < m) {
#pragma unroll
          for (int k = 0; k < j; ++k) s = fma(-G[(int64_t)gj * ldG + 8 * b + k], y[k], s);
          y[j] = (j >= c) ? s / G[(int64_t)gj * ldG + gj] : 0.0;
        } else {
          y[j] = (j == c) ? 1.0 : 0.0;   // padded rows: identity
        }
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) Yd[b * 64 + j * 8 + c] = y[j];
    }
  }

  // ---- the strip in registers: acc[j][cb] = rows 8 (j NWARP + w) + fr, cols 8 cb + 2 fc + {0,1}
  // t.pad == 2: the strip is columns [c0, c0 + nc) of the identity and the result goes to
  // G_s^{-1} (m x m row-major, it.Ginv) -- the input of T_s = Qᵀ G_s^{-1} (k_rotate_n);
  // its rows above c0 stay zero, so the substitution starts at block c0 / 8
  double acc[NW][4][2];
  const int c0 = t.c0, nc = t.nc;
  const bool ident = t.pad == 2;
  const int bstart = ident ? (c0 >> 3) : 0;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    const int row = 8 * (j * NWARP + w) + fr;
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * cb + 2 * fc + h;
        acc[j][cb][h] = (row < m && col < nc) ? (ident ? (row == c0 + col ? 1.0 : 0.0)
                                                       : it.B[(int64_t)row * it.ldB + c0 + col])
                                              : 0.0;
      }
  }
  // G_ib fragments of the coming step (negated: the DMMA accumulates X_i += (-G_ib) X_b)
  double an[NW][2];
  auto load_g = [&](int b) {
#pragma unroll
    for (int j = 0; j < NW; ++j) {
      const int i = j * NWARP + w, row = 8 * i + fr;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int col = 8 * b + 4 * k + fc;
        an[j][k] = (i > b && row < m && col < m) ? -G[(int64_t)row * ldG + col] : 0.0;
      }
    }
  };
  __syncthreads();   // Yd
  if (bstart + 1 < nb) load_g(bstart);

#pragma unroll
  for (int bb = 0; bb < NW; ++bb) {
    for (int wo = 0; wo < NWARP; ++wo) {
      const int b = bb * NWARP + wo;
      if (b >= nb) break;   // uniform across the CTA
      if (b < bstart) continue;
      double* hb = buf + (b & 1) * 8 * TM_LDS;
      if (w == wo) {   // owner: X_b <- Y_b X_b, published in the hand-over tile
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          hb[fr * TM_LDS + 8 * cb + 2 * fc] = acc[bb][cb][0];
          hb[fr * TM_LDS + 8 * cb + 2 * fc + 1] = acc[bb][cb][1];
        }
        __syncwarp();
        double bf[2][4];
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) bf[k][cb] = hb[(4 * k + fc) * TM_LDS + 8 * cb + fr];
        __syncwarp();
        const double y0 = Yd[b * 64 + fr * 8 + fc], y1 = Yd[b * 64 + fr * 8 + 4 + fc];
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
          double c[2] = {0.0, 0.0};
          dmma8(c, y0, bf[0][cb]);
          dmma8(c, y1, bf[1][cb]);
          acc[bb][cb][0] = c[0];
          acc[bb][cb][1] = c[1];
          hb[fr * TM_LDS + 8 * cb + 2 * fc] = c[0];
          hb[fr * TM_LDS + 8 * cb + 2 * fc + 1] = c[1];
        }
      }
      __syncthreads();
      if (b + 1 < nb) {
        double ac[NW][2];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          ac[j][0] = an[j][0];
          ac[j][1] = an[j][1];
        }
        if (b + 2 < nb) load_g(b + 1);   // in flight during this step's products
        double bf[2][4];
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
          for (int cb = 0; cb < 4; ++cb) bf[k][cb] = hb[(4 * k + fc) * TM_LDS + 8 * cb + fr];
#pragma unroll
        for (int j = 0; j < NW; ++j) {
          if (j * NWARP + w > b && j * NWARP + w < nb) {
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
              dmma8(acc[j][cb], ac[j][0], bf[0][cb]);
              dmma8(acc[j][cb], ac[j][1], bf[1][cb]);
            }
          }
        }
      }
    }
  }

  // ---- store the solved strip; the largest n-column norm (R-floor of tau_s) ---------------
  double cs[4][2];
#pragma unroll
  for (int cb = 0; cb < 4; ++cb) cs[cb][0] = cs[cb][1] = 0.0;
#pragma unroll
  for (int j = 0; j < NW; ++j) {
    const int row = 8 * (j * NWARP + w) + fr;
    if (row < m) {
#pragma unroll
      for (int cb = 0; cb < 4; ++cb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * cb + 2 * fc + h;
          if (col < nc) {
            if (ident) const_cast<double*>(it.Ginv)[(int64_t)row * m + c0 + col] = acc[j][cb][h];
            else it.B[(int64_t)row * it.ldB + c0 + col] = acc[j][cb][h];
          }
          cs[cb][h] = fma(acc[j][cb][h], acc[j][cb][h], cs[cb][h]);
        }
    }
  }
  if (it.nmax && c0 + nc > it.kw && !ident) {
#pragma unroll
    for (int cb = 0; cb < 4; ++cb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double v = cs[cb][h];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        if (fr == 0) red[w * 32 + 8 * cb + 2 * fc + h] = v;
      }
    __syncthreads();
    if (w == 0) {
      double s = 0.0;
      for (int q = 0; q < NWARP; ++q) s += red[q * 32 + lane];
      const int n0 = max(0, it.kw - c0);
      double v = (lane >= n0 && lane < nc) ? sqrt(s) : -1.0;
      for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
      if (lane == 0 && v >= 0.0) atomicMax(it.nmax, (unsigned long long)__double_as_longlong(v));
    }
  }
}

template <int NWARP, int NW>
void launch_tm(const CluItem* d_clu, const TrsmItem* d_items, int n, int nb, cudaStream_t st) {
  const size_t sm = sizeof(double) * ((size_t)nb * 64 + 2 * 8 * TM_LDS + NWARP * 32);
  set_smem_attr((const void*)k_trsm_mma<NWARP, NW>, sm);
  k_trsm_mma<NWARP, NW><<<n, NWARP * 32, sm, st>>>(d_clu, d_items);
}

}  // namespace

int trsm_mma_tile_cols() { return TM_TW; }

void launch_trsm_mma(const CluItem* d_clu, const TrsmItem* d_items, int n, int max_m, cudaStream_t st) {
  if (n <= 0) return;
  const int nb = (max_m + 7) / 8;
  if (nb <= 8) launch_tm<8, 1>(d_clu, d_items, n, nb, st);
  else if (nb <= 16) launch_tm<8, 2>(d_clu, d_items, n, nb, st);
  else if (nb <= 24) launch_tm<8, 3>(d_clu, d_items, n, nb, st);
  else if (nb <= 32) launch_tm<8, 4>(d_clu, d_items, n, nb, st);
  else if (nb <= 48) launch_tm<16, 3>(d_clu, d_items, n, nb, st);
  else if (nb <= 64) launch_tm<16, 4>(d_clu, d_items, n, nb, st);
  else fail(HS_E_INTERNAL, "launch_trsm_mma: m above MAX_M");
  count_launch(1);
}

}  // namespace hs
