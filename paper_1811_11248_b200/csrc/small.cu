// The elimination of a level of small clusters in ONE kernel per wave, planned on the device
// (verdict r01 item 7: the sequential batch chains of the coarse levels were host-bound —
// every batch of the regular pipeline needs the previous batch's ranks on the host before
// its shapes can be planned, ~0.1 ms of host work per batch for a few microseconds of GPU
// work when the clusters hold a handful of DOFs).
//
// For a level whose clusters all have m <= SMALL_M DOFs (and k_n + k_w <= SMALL_K live
// columns at their level-start sizes), each batch (independent set, Alg. 1 loop P:633) is
// split into waves of clusters without a common neighbour (pattern only, planned once per
// level), and each wave is one launch, one CTA per cluster, doing the whole scaled low-rank
// elimination of §3.1 in shared memory:
//   its shapes from the device array of live sizes (the ranks of the clusters eliminated
//   before it), its blocks found in the level's block directory,
//   A_ss = G_s G_sᵀ, B = G_s⁻¹[A_sw | A_sn] (the deferred compression),
//   CPQR of B_w to eps with exact norms and the readings Q1-Q5 + R-floor,
//   the rotation of B_n by Qᵀ (E_s), the write-back of row s [I_r | coarse],
//   the Schur update A_pq -= C_pᵀC_q on n(s)² (Eq. CC:eqn:elim) by plain
//   load-subtract-store (no other cluster of the wave touches these blocks: no common
//   neighbour), the apply operator T_s = Qᵀ G_s⁻¹ and C_s into the factor record.
// The host launches the level's waves back to back and reads the ranks once, at the level's
// end.  Same decisions as the batch pipeline and the oracle (parity tests); other rounding
// order (sequential per-thread dot products).
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "device.h"

namespace hs {

namespace {


__device__ __forceinline__ int64_t sdir_find(const BlockDir& d, int p, int q) {   // p >= q; -1 if absent
  int64_t lo = d.ptr[p], hi = d.ptr[p + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (d.q[mid] < q) lo = mid + 1;
    else hi = mid;
  }
  return (lo < d.ptr[p + 1] && d.q[lo] == q) ? d.off[lo] : -1;
}

template <int ST>
__device__ double block_max(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = red[0];
  for (int k = 1; k < ST / 32; ++k) r = fmax(r, red[k]);
  return r;
}
template <int ST>
__device__ int block_min_i(int v, int* red) {
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  int r = red[0];
  for (int k = 1; k < ST / 32; ++k) r = min(r, red[k]);
  return r;
}

template <int ST>
__global__ void __launch_bounds__(ST) k_elim_small(SmallArgs a, int first) {
  extern __shared__ double sm[];
  const int s = a.items[first + blockIdx.x];
  const int tid = threadIdx.x;
  const int MX = a.m_max, KX = a.k_max, NX = a.nseg_max, PX = a.npair_max;
  // shared memory carve-up (the host sizes it from the same formula: small_smem_bytes)
  double* G = sm;                            // MX x (MX + 1): A_ss, then its lower factor
  double* B = G + MX * (MX + 1);             // MX x (KX + MX) row-major (ld kb): [B_w | B_n | G^{-1}]
  double* V = B + (size_t)MX * (KX + MX);    // MX x MX: reflector j in row j
  double* tau = V + MX * MX;                 // MX
  double* nu = tau + MX;                     // KX column norms (-1: pivoted)
  double* red = nu + KX;                     // 8 (+ 8 ints)
  int* redi = (int*)(red + 8);
  double** sptr = (double**)(red + 16);      // NX segment pointers
  int* scol = (int*)(sptr + NX);             // NX column offsets in B
  int* slen = scol + NX;
  int* sld = slen + NX;
  int* strn = sld + NX;
  int* sq = strn + NX;
  double** pptr = (double**)(sq + NX + (NX & 1));   // PX target blocks of the Schur pairs
  int* poff = (int*)(pptr + PX);             // PX + 1 element prefix
  int* pa = poff + PX + 1;                   // PX: n-segment index of the row side
  int* pb = pa + PX;                         // PX: n-segment index of the column side
  __shared__ int nseg, nw_seg, kw, kn, failed, rr, npair;
  __shared__ double* Dss;
  __shared__ int ldss;
  const int m = a.live[s];
  // segment table: the directory lookups and live-size reads run in parallel (a serial chain
  // of dependent global loads in one thread would dominate a cluster of a few DOFs)
  const int nw0 = a.wptr[s + 1] - a.wptr[s], nn0 = a.nptr[s + 1] - a.nptr[s], nall = nw0 + nn0;
  if (tid == 0) failed = (nall > NX) ? 2 : 0;
  __syncthreads();
  if (!failed) {
    for (int t = tid; t < nall; t += ST) {   // raw (uncompacted) entries in slots [0, nall)
      const int q = t < nw0 ? a.widx[a.wptr[s] + t] : a.nidx[a.nptr[s] + t - nw0];
      const int L = a.live[q];
      slen[t] = L;
      sq[t] = q;
      const int p0 = max(s, q), q0 = min(s, q);
      const int64_t o = L > 0 ? sdir_find(a.dir, p0, q0) : 0;
      if (o < 0) failed = 2;
      sptr[t] = L > 0 ? a.dir.blk + o : nullptr;
      sld[t] = a.dir.cap[q0];
      strn[t] = q > s ? 1 : 0;
    }
    if (tid == 32) {
      const int64_t od = sdir_find(a.dir, s, s);
      Dss = od >= 0 ? a.dir.blk + od : nullptr;
      ldss = a.dir.cap[s];
      if (!Dss && m > 0) failed = 2;
    }
  }
  __syncthreads();
  if (tid == 0 && !failed) {   // compact the empty neighbours away, column offsets (shared memory only)
    int col = 0, ns = 0;
    for (int t = 0; t < nall; ++t) {
      if (t == nw0) {
        kw = col;
        nw_seg = ns;
      }
      if (slen[t] == 0) continue;
      sptr[ns] = sptr[t];
      slen[ns] = slen[t];
      sld[ns] = sld[t];
      strn[ns] = strn[t];
      sq[ns] = sq[t];
      scol[ns] = col;
      col += slen[ns];
      ++ns;
    }
    if (nw0 == nall) {
      kw = col;
      nw_seg = ns;
    }
    nseg = ns;
    kn = col - kw;
    int np = 0, e = 0;   // Schur pairs (x >= y over the non-empty n-segments, ascending cluster id)
    for (int x = nw_seg; x < ns; ++x)
      for (int y = nw_seg; y <= x; ++y) {
        if (np >= PX) {
          failed = 2;
          break;
        }
        pa[np] = x;
        pb[np] = y;
        poff[np] = e;
        e += (x == y) ? slen[x] * (slen[x] + 1) / 2 : slen[x] * slen[y];
        ++np;
      }
    poff[np] = e;
    npair = np;
  }
  __syncthreads();
  if (!failed)
    for (int t = tid; t < npair; t += ST) {   // the target blocks of the pairs, in parallel
      const int64_t o = sdir_find(a.dir, sq[pa[t]], sq[pb[t]]);
      if (o < 0) failed = 2;
      pptr[t] = o >= 0 ? a.dir.blk + o : nullptr;
    }
  __syncthreads();
  if (tid == 0 && failed == 2 && atomicCAS(&a.status->flag, 0, 2) == 0) {
    a.status->level = a.level;
    a.status->cluster = s;
    a.status->pivot = -1;
    a.status->value = 0.0;
  }
  __syncthreads();
  if (failed) return;
  const int k = kw + kn;
  const int kb = k + m;   // B = [A_sw | A_sn | I_m]: the substitution also forms G^{-1}, the rotation Qᵀ G^{-1} = T_s
  if (m == 0) {
    if (tid == 0) {
      a.rank[s] = 0;
      a.kn[s] = kn;
      a.kw[s] = kw;
    }
    return;
  }
  // ---- load A_ss (lower triangle of the stored diagonal block) and [A_sw | A_sn | I] --------
  for (int e = tid; e < m * m; e += ST) {
    const int i = e / m, j = e % m;
    G[i * (MX + 1) + j] = j <= i ? Dss[(int64_t)i * ldss + j] : 0.0;
    B[i * kb + k + j] = (i == j) ? 1.0 : 0.0;
  }
  {   // every element of [A_sw | A_sn]: 4 independent global loads in flight per thread
    const int tot = m * k;
    for (int e0 = tid; e0 < tot; e0 += 4 * ST) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * ST;
        v[u] = 0.0;
        if (e < tot) {
          const int i = e / k, c = e % k;
          int lo = 0, hi = nseg - 1;   // the segment holding column c
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (scol[mid] <= c) lo = mid;
            else hi = mid - 1;
          }
          const int j = c - scol[lo];
          v[u] = strn[lo] ? sptr[lo][(int64_t)j * sld[lo] + i] : sptr[lo][(int64_t)i * sld[lo] + j];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * ST;
        if (e < tot) B[(e / k) * kb + (e % k)] = v[u];
      }
    }
  }
  __syncthreads();
  // ---- A_ss = G Gᵀ (right-looking) --------------------------------------------------
  for (int j = 0; j < m; ++j) {
    const double d = G[j * (MX + 1) + j];
    if (!(d > 0.0)) {   // uniform: every thread reads the same d
      if (tid == 0 && atomicCAS(&a.status->flag, 0, 1) == 0) {
        a.status->level = a.level;
        a.status->cluster = s;
        a.status->pivot = j;
        a.status->value = d;
      }
      return;
    }
    const double g = sqrt(d);
    __syncthreads();
    if (tid == 0) G[j * (MX + 1) + j] = g;
    for (int i = j + 1 + tid; i < m; i += ST) G[i * (MX + 1) + j] /= g;
    __syncthreads();
    const int t = m - j - 1;
    for (int e = tid; e < t * t; e += ST) {
      const int i = j + 1 + e / t, l = j + 1 + e % t;
      if (l <= i) G[i * (MX + 1) + l] -= G[i * (MX + 1) + j] * G[l * (MX + 1) + j];
    }
    __syncthreads();
  }
  // ---- B = G⁻¹ [A_sw | A_sn | I]: forward substitution, a thread per column ------------------
  for (int c = tid; c < kb; c += ST) {
    for (int i = 0; i < m; ++i) {
      double b = B[i * kb + c];
      for (int l = 0; l < i; ++l) b -= G[i * (MX + 1) + l] * B[l * kb + c];
      B[i * kb + c] = b / G[i * (MX + 1) + i];
    }
  }
  __syncthreads();
  // R-floor: the largest n-column norm of B_n
  double rn = 0.0;
  for (int c = kw + tid; c < k; c += ST) {
    double s2 = 0.0;
    for (int i = 0; i < m; ++i) s2 += B[i * kb + c] * B[i * kb + c];
    rn = fmax(rn, sqrt(s2));
  }
  const double Rn = block_max<ST>(rn, red);
  // ---- CPQR of B_w to eps (Q1-Q5): exact norms, strict keep rule, lowest-index tie window -
  for (int c = tid; c < kw; c += ST) nu[c] = 0.0;
  if (tid == 0) rr = min(m, kw);
  __syncthreads();
  double tau_s = 0.0;
  const int jmax = min(m, kw);
  for (int j = 0; j < jmax; ++j) {
    double lmax = -1.0;
    for (int c = tid; c < kw; c += ST) {
      if (nu[c] < 0.0) continue;
      double s2 = 0.0;
      for (int i = j; i < m; ++i) s2 += B[i * kb + c] * B[i * kb + c];
      nu[c] = sqrt(s2);
      lmax = fmax(lmax, nu[c]);
    }
    const double numax = block_max<ST>(lmax, red);
    if (j == 0) {
      tau_s = a.relative ? a.eps * numax : a.eps;
      if (a.relative && a.eps > 0.0) tau_s = fmax(tau_s, 1e-12 * fmax(numax, Rn));
    }
    if (!(numax > tau_s)) {
      if (tid == 0) rr = j;
      break;
    }
    const double thr = (1.0 - 1e-10) * numax;
    int lo = INT_MAX;
    for (int c = tid; c < kw; c += ST)
      if (nu[c] >= thr) {
        lo = c;
        break;
      }
    const int p = block_min_i<ST>(lo, redi);
    // dlarfg of column p, rows j..m-1 (one warp)
    if (tid < 32) {
      double xs = 0.0;
      for (int l = j + 1 + tid; l < m; l += 32) xs += B[l * kb + p] * B[l * kb + p];
      for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
      const double alpha = B[j * kb + p], xnorm = sqrt(xs);
      double t, beta, rden;
      if (xnorm == 0.0) {
        t = 0.0;
        beta = alpha;
        rden = 0.0;
      } else {
        const double h = sqrt(alpha * alpha + xnorm * xnorm);
        beta = alpha >= 0.0 ? -h : h;
        t = (beta - alpha) / beta;
        rden = 1.0 / (alpha - beta);
      }
      for (int l = tid; l < m; l += 32) V[j * MX + l] = (l < j) ? 0.0 : (l == j) ? 1.0 : B[l * kb + p] * rden;
      if (tid == 0) {
        tau[j] = t;
        red[7] = beta;
        a.piv[a.poff[s] + j] = p;
      }
    }
    __syncthreads();
    const double t = tau[j], beta = red[7];
    for (int c = tid; c < kw; c += ST) {
      if (c == p || nu[c] < 0.0 || t == 0.0) continue;
      double w = 0.0;
      for (int l = j; l < m; ++l) w += V[j * MX + l] * B[l * kb + c];
      const double tw = t * w;
      for (int l = j; l < m; ++l) B[l * kb + c] -= tw * V[j * MX + l];
    }
    __syncthreads();
    if (tid == 0) {
      B[j * kb + p] = beta;
      for (int l = j + 1; l < m; ++l) B[l * kb + p] = 0.0;
      nu[p] = -1.0;
    }
    __syncthreads();
  }
  __syncthreads();
  const int r = kw > 0 ? rr : 0, K = m - r;
  // ---- E_s on the n-columns and on G⁻¹: Qᵀ B_n and T_s = Qᵀ G⁻¹ (H_0 first) ---------------------
  for (int c = kw + tid; c < kb; c += ST)
    for (int j = 0; j < r; ++j) {
      if (tau[j] == 0.0) continue;
      double w = 0.0;
      for (int l = j; l < m; ++l) w += V[j * MX + l] * B[l * kb + c];
      const double tw = tau[j] * w;
      for (int l = j; l < m; ++l) B[l * kb + c] -= tw * V[j * MX + l];
    }
  __syncthreads();
  double* T = a.T + a.toff[s];
  for (int e = tid; e < m * m; e += ST) T[e] = B[(e / m) * kb + k + (e % m)];   // T_s row-major
  // ---- C_s = rows [r, m) of the rotated B_n into the factor record (ld kn) -----------------
  if (kn > 0 && K > 0) {
    double* C = a.C + a.coff[s];
    for (int e = tid; e < K * kn; e += ST) C[e] = B[(r + e / kn) * kb + kw + e % kn];
  }
  // ---- write-back of row s: I_r on (s, s), the coarse rows into the blocks (s, q) -----------
  for (int e = tid; e < r * r; e += ST) {
    const int i = e / r, j = e % r;
    if (j <= i) Dss[(int64_t)i * ldss + j] = (i == j) ? 1.0 : 0.0;
  }
  for (int g = 0; g < nseg; ++g) {
    double* p = sptr[g];
    const int L = slen[g], ld = sld[g], c0 = scol[g];
    if (strn[g]) {
      for (int e = tid; e < r * L; e += ST) {
        const int j = e / r, i = e % r;
        p[(int64_t)j * ld + i] = B[i * kb + c0 + j];
      }
    } else {
      for (int e = tid; e < r * L; e += ST) {
        const int i = e / L, j = e % L;
        p[(int64_t)i * ld + j] = B[i * kb + c0 + j];
      }
    }
  }
  // ---- Schur update on n(s)²: A_pq -= C_pᵀ C_q (the wave has no other writer of these) -----
  if (K > 0) {
    const int tot = poff[npair];
    for (int e = tid; e < tot; e += ST) {
      int lo = 0, hi = npair - 1;   // the pair holding element e
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (poff[mid] <= e) lo = mid;
        else hi = mid - 1;
      }
      const int x = pa[lo], y = pb[lo], o = e - poff[lo];
      int i, j;
      if (x == y) {   // lower triangle: row i holds i + 1 entries
        i = (int)((sqrt(8.0 * o + 1.0) - 1.0) * 0.5);
        while ((i + 1) * (i + 2) / 2 <= o) ++i;
        while (i * (i + 1) / 2 > o) --i;
        j = o - i * (i + 1) / 2;
      } else {
        i = o / slen[y];
        j = o % slen[y];
      }
      const int cp = scol[x] - kw + i, cq = scol[y] - kw + j;
      double acc = 0.0;
      for (int kk = 0; kk < K; ++kk) acc += B[(r + kk) * kb + kw + cp] * B[(r + kk) * kb + kw + cq];
      double* tgt = pptr[lo] + (int64_t)i * a.dir.cap[sq[y]] + j;   // block (p, q): row-major, ld cap[q]
      *tgt -= acc;
    }
  }
  if (tid == 0) {
    a.rank[s] = r;
    a.kn[s] = kn;
    a.kw[s] = kw;
    a.live[s] = r;   // no other cluster of this batch reads it (independent set)
  }
}

}  // namespace

size_t small_smem_bytes(int m_max, int k_max, int nseg_max, int npair_max) {
  const size_t d = (size_t)m_max * (m_max + 1) + (size_t)m_max * (k_max + m_max) + (size_t)m_max * m_max + m_max +
                   k_max + 16;
  const size_t pbytes = sizeof(double*) * (size_t)(nseg_max + npair_max);
  const size_t ibytes = sizeof(int) * (size_t)(5 * nseg_max + 1 + (nseg_max & 1) + 3 * npair_max + 1);
  return d * sizeof(double) + pbytes + ibytes + 64;
}

void launch_elim_small(const SmallArgs& a, int first, int n, cudaStream_t st) {
  if (n <= 0) return;
  const size_t smem = small_smem_bytes(a.m_max, a.k_max, a.nseg_max, a.npair_max);
  // threads per CTA (HS_SMALL_THREADS: 64 / 128 / 256): the column loops use at most
  // k_w threads, so fewer threads mostly shorten the CTA barriers of the step chains
  static const int nt = [] {
    const char* e = std::getenv("HS_SMALL_THREADS");
    const int v = e ? std::atoi(e) : 128;
    return (v == 64 || v == 256) ? v : 128;
  }();
  if (nt == 64) {
    set_smem_attr((const void*)k_elim_small<64>, smem);
    k_elim_small<64><<<n, 64, smem, st>>>(a, first);
  } else if (nt == 256) {
    set_smem_attr((const void*)k_elim_small<256>, smem);
    k_elim_small<256><<<n, 256, smem, st>>>(a, first);
  } else {
    set_smem_attr((const void*)k_elim_small<128>, smem);
    k_elim_small<128><<<n, 128, smem, st>>>(a, first);
  }
  count_launch(1);
}

}  // namespace hs
