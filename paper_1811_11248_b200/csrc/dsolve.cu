// Distributed solve (SURVEY §8(e) "Apply" and "PCG"; the reconstruction of the parallel
// algorithm the paper defers to parallel LoRaSp, Thm 2).
//
// Owner computes, nothing gathered: every rank keeps the elimination records (T_s, C_s) of
// the clusters it eliminated and applies only those; the vectors of Algorithm 2
// are laid out as on one GPU (per level, every cluster's segment at its level-start size),
// each rank filling the segments it owns.
//   forward, per batch: k_dfwd forms z = T_s y_s of the owned clusters (coarse part into the
//     parent's segment, fine part kept) and the contributions C_sᵀ y_f to all neighbours;
//     after a phase-II batch the contributions travel to the owners of their targets (grouped
//     send/recv); k_dacc subtracts every owned target's contributions in source order (no
//     batch member is another's target, so this is the sequential order of Alg. 2);
//   top: the top segments are gathered to rank 0, which solves with its dense L L^T and
//     scatters the result back;
//   backward, per batch in reverse: before a phase-II batch the owners of the remote
//     neighbours send their current x segments; k_dbwd forms x_f = y_f - sum_q C[:, q] x_q
//     and x_s = T_sᵀ [x_c; x_f].
// Phase-I batches never communicate (interior clusters touch only their subdomain, O2.8).
// PCG: each rank owns the contiguous permuted DOF range of its subdomains; the SpMV of the
// owned rows reads the ghost entries of other ranks from a halo exchanged once per
// iteration (one message per peer, packed by k_dgather), dot products are per-rank partial
// sums all-reduced over the ranks.
#include <algorithm>
#include <cstring>

#include "runtime.h"

namespace hs {

namespace {

constexpr int DT = 256;   // threads per CTA of the distributed-solve kernels

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// z = T_s y_s (a warp per row, lanes along the row of T), coarse / fine parts out, then the
// contributions slot[j] = sum_k C[k][j] z_f[k] (a thread per column of C, coalesced rows)
__global__ void __launch_bounds__(DT) k_dfwd(const DFwdItem* __restrict__ items) {
  extern __shared__ double sm[];
  const DFwdItem it = items[blockIdx.x];
  const int m = it.m, r = it.r, K = m - r;
  double* y = sm;
  double* z = sm + m;
  for (int i = threadIdx.x; i < m; i += DT) y[i] = it.y[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = w; i < m; i += DT / 32) {
    const double* Ti = it.T + (int64_t)i * m;
    double acc = 0.0;
    for (int k = lane; k < m; k += 32) acc += Ti[k] * y[k];
    acc = warp_sum(acc);
    if (lane == 0) z[i] = acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += DT) {
    if (i < r) it.yc[i] = z[i];
    else it.yf[i - r] = z[i];
  }
  if (it.slot)
    for (int j = threadIdx.x; j < it.kn; j += DT) {
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc += it.C[(int64_t)k * it.kn + j] * z[r + k];
      it.slot[j] = acc;
    }
}

// y_q -= sum of its contributions of the batch, in source order
__global__ void __launch_bounds__(DT) k_dacc(const DAccItem* __restrict__ items, const double* const* __restrict__ src) {
  const DAccItem it = items[blockIdx.x];
  for (int i = threadIdx.x; i < it.len; i += DT) {
    double acc = it.y[i];
    for (int k = 0; k < it.ns; ++k) acc -= src[it.s0 + k][i];
    it.y[i] = acc;
  }
}

// x_f = y_f - C [x_q]_q (a warp per row of C), then x_s = T_sᵀ [x_c; x_f] (a thread per entry)
__global__ void __launch_bounds__(DT) k_dbwd(const DBwdItem* __restrict__ items, const DNb* __restrict__ nbs) {
  extern __shared__ double sm[];
  const DBwdItem it = items[blockIdx.x];
  const int m = it.m, r = it.r, K = m - r;
  double* v = sm;          // [x_c; x_f], m
  double* xn = sm + m;     // neighbour segments, kn
  for (int a = 0, off = 0; a < it.nnb; ++a) {
    const DNb nb = nbs[it.nb0 + a];
    for (int i = threadIdx.x; i < nb.len; i += DT) xn[off + i] = nb.x[i];
    off += nb.len;
  }
  for (int i = threadIdx.x; i < r; i += DT) v[i] = it.xc[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = w; k < K; k += DT / 32) {
    const double* Ck = it.C + (int64_t)k * it.kn;
    double acc = 0.0;
    for (int j = lane; j < it.kn; j += 32) acc += Ck[j] * xn[j];
    acc = warp_sum(acc);
    if (lane == 0) v[r + k] = it.yf[k] - acc;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < m; i += DT) {
    double acc = 0.0;
    for (int k = 0; k < m; ++k) acc += it.T[(int64_t)k * m + i] * v[k];
    it.x[i] = acc;
  }
}

__global__ void k_dgather(const double* __restrict__ src, const int32_t* __restrict__ idx, double* __restrict__ dst,
                          int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[idx[i]];
}
__global__ void k_dperm(const double* __restrict__ src, double* __restrict__ dst, const int64_t* __restrict__ idx,
                        int64_t n, int scatter) {   // scatter: dst[idx[i]] = src[i]; else dst[i] = src[idx[i]]
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (scatter) dst[idx[i]] = src[i];
    else dst[i] = src[idx[i]];
  }
}
// deterministic dot: per-block partial sums in a fixed order, then one block adds them
constexpr int DDOT_BLOCKS = 296;
__global__ void __launch_bounds__(DT) k_ddot(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                             double* __restrict__ part) {
  __shared__ double red[DT / 32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)DT + threadIdx.x; i < n; i += (int64_t)gridDim.x * DT) acc += a[i] * b[i];
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < DT / 32; ++k) s += red[k];
    part[blockIdx.x] = s;
  }
}
__global__ void k_ddot_fin(const double* __restrict__ part, int n, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += part[k];
    *out = s;
  }
}
__global__ void k_daxpy(double* __restrict__ y, const double* __restrict__ x, double a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] += a * x[i];
}
__global__ void k_dxpby(double* __restrict__ p, const double* __restrict__ z, double b, int64_t n) {   // p = z + b p
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + b * p[i];
}

int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + DT - 1) / DT, 148 * 8)); }

template <class T>
T* upload(DevCache& dc, const std::vector<T>& v, cudaStream_t st, std::vector<void*>& owned) {
  if (v.empty()) return nullptr;
  T* d = (T*)dc.alloc(sizeof(T) * v.size());
  HS_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st));
  owned.push_back(d);
  return d;
}

}  // namespace

DistSolve::~DistSolve() {
  if (h_scal) cudaFreeHost(h_scal);
  if (!dc) return;
  for (void* p : owned) dc->free(p);
}

// ---- plan (host, at the end of a distributed factor) ----------------------------------------
void dist_solve_build(hs_factor_s* f, const DistPlan& DP) {
  const Analysis& an = *f->an;
  hs_handle_s* h = f->h;
  cudaStream_t st = h->stream;
  auto* D = new DistSolve();
  f->ds.reset(D);
  D->dc = &h->cache;
  D->rank = h->rank;
  D->world = h->world;
  const int Lt = an.L_top;
  // vector layout: per level every cluster's segment at its level-start size, top last
  D->vbase.assign(Lt + 2, 0);
  std::vector<std::vector<int64_t>> voff(Lt + 1);
  for (int l = 0; l <= Lt; ++l) {
    const std::vector<int32_t>& cap = l < Lt ? f->lv[l].cap : f->top_sizes;
    voff[l].assign(cap.size() + 1, 0);
    for (size_t c = 0; c < cap.size(); ++c) voff[l][c + 1] = voff[l][c] + cap[c];
    D->vbase[l + 1] = D->vbase[l] + voff[l].back();
  }
  D->vtotal = D->vbase[Lt + 1];
  D->d_y = (double*)D->dc->alloc(sizeof(double) * std::max<int64_t>(D->vtotal, 1));
  D->d_x = (double*)D->dc->alloc(sizeof(double) * std::max<int64_t>(D->vtotal, 1));
  D->owned.push_back(D->d_y);
  D->owned.push_back(D->d_x);
  HS_CUDA(cudaMemsetAsync(D->d_y, 0, sizeof(double) * std::max<int64_t>(D->vtotal, 1), st));
  HS_CUDA(cudaMemsetAsync(D->d_x, 0, sizeof(double) * std::max<int64_t>(D->vtotal, 1), st));
  int64_t ftot = 0;
  std::vector<std::vector<int64_t>> foff(Lt), soff(Lt);
  for (int l = 0; l < Lt; ++l) {
    const LevelRT& L = f->lv[l];
    foff[l].assign(L.nclus, -1);
    for (int s = 0; s < L.nclus; ++s)
      if (DP.own(l, s)) {
        foff[l][s] = ftot;
        ftot += L.cap[s] - L.rank[s];
      }
  }
  D->d_f = (double*)D->dc->alloc(sizeof(double) * std::max<int64_t>(ftot, 1));
  D->owned.push_back(D->d_f);
  int64_t stot = 0;
  for (int l = 0; l < Lt; ++l) {
    const LevelRT& L = f->lv[l];
    soff[l].assign(L.nclus, 0);
    for (int s = 0; s < L.nclus; ++s) {
      soff[l][s] = stot;
      stot += L.kn[s];
    }
  }
  D->d_slot = (double*)D->dc->alloc(sizeof(double) * std::max<int64_t>(stot, 1));
  D->owned.push_back(D->d_slot);
  std::vector<DFwdItem> fwd;
  std::vector<DAccItem> acc;
  std::vector<const double*> accsrc;
  std::vector<DBwdItem> bwd;
  std::vector<DNb> nbv;
  auto Y = [&](int l, int c) { return D->d_y + D->vbase[l] + voff[l][c]; };
  auto X = [&](int l, int c) { return D->d_x + D->vbase[l] + voff[l][c]; };
  for (int l = 0; l < Lt; ++l) {
    const Level& lev = an.levels[l];
    const LevelRT& L = f->lv[l];
    std::vector<int32_t> bpos(lev.nclus, 0);
    for (size_t b = 0; b < lev.batches.size(); ++b)
      for (int32_t c : lev.batches[b]) bpos[c] = (int32_t)b;
    // the coarse part of c inside its parent's segment
    auto pofs = [&](int c) { return (int64_t)((c & 1) ? L.rank[c - 1] : 0); };
    auto ppos_y = [&](int c) { return Y(l + 1, c >> 1) + pofs(c); };
    auto ppos_x = [&](int c) { return X(l + 1, c >> 1) + pofs(c); };
    for (size_t b = 0; b < lev.batches.size(); ++b) {
      DistBatch B;
      B.level = l;
      B.phase2 = (int)b >= lev.nphase1;
      B.fwd0 = (int32_t)fwd.size();
      B.bwd0 = (int32_t)bwd.size();
      std::vector<std::vector<std::pair<const double*, int32_t>>> tin(lev.nclus);   // target -> (slot col ptr, source)
      for (int32_t s : lev.batches[b]) {
        const int32_t m = L.cap[s], r = L.rank[s], kn = L.kn[s];
        if (m == 0) continue;
        const bool mine = DP.own(l, s);
        if (mine) {
          DFwdItem it{L.T[s], L.C[s], Y(l, s), ppos_y(s), D->d_f + foff[l][s], (kn > 0 && m > r) ? D->d_slot + soff[l][s] : nullptr,
                      m, r, kn, 0};
          fwd.push_back(it);
          DBwdItem bi{L.T[s], L.C[s], ppos_x(s), D->d_f + foff[l][s], X(l, s), m, r, kn, (int32_t)nbv.size(), 0, 0};
          int32_t col = 0;
          for (int32_t q : lev.H[s]) {
            const bool proc = bpos[q] < (int32_t)b;
            const int32_t lq = proc ? L.rank[q] : L.cap[q];
            if (lq == 0) continue;
            nbv.push_back(DNb{proc ? ppos_x(q) : X(l, q), lq, 0});
            col += lq;
          }
          bi.nnb = (int32_t)nbv.size() - bi.nb0;
          if (m > r) bwd.push_back(bi);
          else bwd.push_back(bi);   // r = m: x_s = T_sᵀ x_c (no fine part)
        }
        // contributions of s to its neighbours (a source with K = 0 contributes nothing)
        if (m > r && kn > 0) {
          int32_t col = 0;
          for (int32_t q : lev.H[s]) {
            const bool proc = bpos[q] < (int32_t)b;
            const int32_t lq = proc ? L.rank[q] : L.cap[q];
            if (lq == 0) continue;
            if (DP.own(l, q)) tin[q].push_back({D->d_slot + soff[l][s] + col, s});
            col += lq;
          }
        }
        // exchange plan: forward slots to the owners of remote targets, backward x of
        // remote neighbours from their owners
        if (B.phase2) {
          std::vector<int32_t> dests;
          for (int32_t q : lev.H[s]) {
            const int g = DP.owner[l][q];
            if (g != DP.owner[l][s]) dests.push_back(g);
          }
          std::sort(dests.begin(), dests.end());
          dests.erase(std::unique(dests.begin(), dests.end()), dests.end());
          const bool has_slot = m > L.rank[s] && kn > 0;
          for (int32_t g : dests) {
            if (!has_slot) continue;
            if (mine) B.fsend.push_back(DMsg{D->d_slot + soff[l][s], kn, g});
            else if (g == DP.rank) B.frecv.push_back(DMsg{D->d_slot + soff[l][s], kn, DP.owner[l][s]});
          }
        }
      }
      if (B.phase2) {   // backward halo of the batch (dedupe per (q, dest) / q, s ascending)
        std::vector<std::pair<int32_t, int32_t>> sent;   // (q, dest)
        std::vector<int32_t> got;
        for (int32_t s : lev.batches[b]) {
          if (L.cap[s] == 0) continue;
          const int gs = DP.owner[l][s];
          for (int32_t q : lev.H[s]) {
            const int gq = DP.owner[l][q];
            if (gq == gs) continue;
            const bool proc = bpos[q] < (int32_t)b;
            const int32_t lq = proc ? L.rank[q] : L.cap[q];
            if (lq == 0) continue;
            double* loc = proc ? ppos_x(q) : X(l, q);
            if (gq == DP.rank && std::find(sent.begin(), sent.end(), std::make_pair(q, (int32_t)gs)) == sent.end()) {
              sent.push_back({q, gs});
              B.bsend.push_back(DMsg{loc, lq, gs});
            }
            if (gs == DP.rank && std::find(got.begin(), got.end(), q) == got.end()) {
              got.push_back(q);
              B.brecv.push_back(DMsg{loc, lq, gq});
            }
          }
        }
      }
      B.acc0 = (int32_t)acc.size();
      for (int32_t q = 0; q < lev.nclus; ++q) {
        if (tin[q].empty()) continue;
        auto& v = tin[q];
        std::stable_sort(v.begin(), v.end(), [](const auto& x, const auto& y) { return x.second < y.second; });
        const bool proc = bpos[q] < (int32_t)b;
        DAccItem ai{proc ? ppos_y(q) : Y(l, q), proc ? L.rank[q] : L.cap[q], (int32_t)accsrc.size(), (int32_t)v.size(), 0};
        for (auto& e : v) accsrc.push_back(e.first);
        acc.push_back(ai);
      }
      B.nfwd = (int32_t)fwd.size() - B.fwd0;
      B.nbwd = (int32_t)bwd.size() - B.bwd0;
      B.nacc = (int32_t)acc.size() - B.acc0;
      D->batches.push_back(std::move(B));
    }
  }
  for (const auto& it : fwd) D->max_m = std::max(D->max_m, it.m);
  for (const auto& it : bwd) D->max_kn = std::max(D->max_kn, it.kn);
  D->d_fwd = upload(*D->dc, fwd, st, D->owned);
  D->d_acc = upload(*D->dc, acc, st, D->owned);
  D->d_accsrc = upload(*D->dc, accsrc, st, D->owned);
  D->d_bwd = upload(*D->dc, bwd, st, D->owned);
  D->d_nb = upload(*D->dc, nbv, st, D->owned);
  // top: every top cluster's segment to / from rank 0
  const int ntc = (int)f->top_sizes.size();
  for (int c = 0; c < ntc; ++c) {
    const int g = Lt > 0 ? DP.owner[Lt][c] : 0;
    D->top.push_back(DMsg{nullptr, f->top_sizes[c], g});
    D->top_off.push_back(D->vbase[Lt] + voff[Lt][c]);
  }
  // ---- PCG: owned permuted range, local CSR, halo ----------------------------------------
  const int nleaf = (int)an.leaf_off.size() - 1;
  int c_lo = nleaf, c_hi = -1;
  for (int c = 0; c < nleaf; ++c)
    if (DP.own(0, c)) {
      c_lo = std::min(c_lo, c);
      c_hi = std::max(c_hi, c);
    }
  D->r0 = c_hi >= 0 ? an.leaf_off[c_lo] : 0;
  D->r1 = c_hi >= 0 ? an.leaf_off[c_hi + 1] : 0;
  for (int c = c_lo; c <= c_hi; ++c)
    if (!DP.own(0, c)) fail(HS_E_INTERNAL, "dist solve: owned leaves not contiguous");
  const int64_t n = an.n, nl = D->r1 - D->r0;
  D->nloc = nl;
  // owner of a permuted index (its leaf's level-0 owner)
  std::vector<int32_t> leaf_owner(nleaf);
  for (int c = 0; c < nleaf; ++c) leaf_owner[c] = DP.owner[0].empty() ? 0 : DP.owner[0][c];
  auto owner_of = [&](int64_t p) {
    const int c = (int)(std::upper_bound(an.leaf_off.begin(), an.leaf_off.end(), p) - an.leaf_off.begin()) - 1;
    return leaf_owner[c];
  };
  std::vector<int64_t> lrow(nl + 1, 0), vidx;
  std::vector<int64_t> gcol;   // permuted column of each entry (ghosts resolved below)
  for (int64_t i = 0; i < nl; ++i) {
    const int64_t o = an.perm[D->r0 + i];
    for (int64_t k = an.rowptr[o]; k < an.rowptr[o + 1]; ++k) {
      vidx.push_back(k);
      gcol.push_back(an.iperm[an.colind[k]]);
    }
    lrow[i + 1] = (int64_t)vidx.size();
  }
  std::vector<int64_t> ghosts;
  for (int64_t pj : gcol)
    if (pj < D->r0 || pj >= D->r1) ghosts.push_back(pj);
  std::sort(ghosts.begin(), ghosts.end());
  ghosts.erase(std::unique(ghosts.begin(), ghosts.end()), ghosts.end());
  std::vector<int32_t> lcol(gcol.size());
  for (size_t e = 0; e < gcol.size(); ++e) {
    const int64_t pj = gcol[e];
    lcol[e] = (pj >= D->r0 && pj < D->r1) ? (int32_t)(pj - D->r0)
                                          : (int32_t)(nl + (std::lower_bound(ghosts.begin(), ghosts.end(), pj) - ghosts.begin()));
  }
  D->nghost = (int64_t)ghosts.size();
  // halo receives: the ghosts of peer g form one contiguous run (peers own contiguous ranges)
  for (int64_t k = 0; k < (int64_t)ghosts.size();) {
    const int g = owner_of(ghosts[k]);
    int64_t k1 = k;
    while (k1 < (int64_t)ghosts.size() && owner_of(ghosts[k1]) == g) ++k1;
    D->hrecv.push_back(DMsg{nullptr, (int32_t)(k1 - k), g});
    D->hrecv_off.push_back(nl + k);
    k = k1;
  }
  // halo sends: my rows that reference peer g's range (symmetric pattern), ascending
  std::vector<std::vector<int32_t>> need(h->world);
  for (int64_t i = 0; i < nl; ++i) {
    std::vector<int> gs;
    for (int64_t e = lrow[i]; e < lrow[i + 1]; ++e)
      if (lcol[e] >= nl) gs.push_back(owner_of(gcol[e]));
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
    for (int g : gs) need[g].push_back((int32_t)i);
  }
  std::vector<int32_t> sidx;
  for (int g = 0; g < h->world; ++g) {
    if (need[g].empty()) continue;
    D->hsend.push_back(DMsg{nullptr, (int32_t)need[g].size(), g});
    D->hsend_off.push_back((int64_t)sidx.size());
    sidx.insert(sidx.end(), need[g].begin(), need[g].end());
  }
  D->d_lrow = upload(*D->dc, lrow, st, D->owned);
  D->d_lcol = upload(*D->dc, lcol, st, D->owned);
  std::vector<int64_t> vidx64(vidx.begin(), vidx.end());
  D->d_vidx = upload(*D->dc, vidx64, st, D->owned);
  D->d_sidx = upload(*D->dc, sidx, st, D->owned);
  D->nnz_loc = (int64_t)vidx.size();
  D->d_lval = (double*)D->dc->alloc(sizeof(double) * std::max<int64_t>(D->nnz_loc, 1));
  D->owned.push_back(D->d_lval);
  if (D->nnz_loc)
    k_dperm<<<grid_for(D->nnz_loc), DT, 0, st>>>(f->d_vals, D->d_lval, D->d_vidx, D->nnz_loc, 0);
  count_launch(1);
  auto vec = [&](int64_t len) {
    double* p = (double*)D->dc->alloc(sizeof(double) * std::max<int64_t>(len, 1));
    D->owned.push_back(p);
    return p;
  };
  D->d_xext = vec(nl + D->nghost);
  D->d_sbuf = vec((int64_t)sidx.size());
  D->d_r = vec(nl); D->d_z = vec(nl); D->d_p = vec(nl); D->d_q = vec(nl); D->d_xs = vec(nl);
  D->d_part = vec(DDOT_BLOCKS + 8);
  D->d_full = vec(n);
  D->d_full2 = vec(n);
  HS_CUDA(cudaMallocHost(&D->h_scal, sizeof(double) * 8));
  HS_CUDA(cudaStreamSynchronize(st));
  (void)ftot;
}

// ---- apply: b (permuted, owned range at d_y level 0) -> x (owned range at d_x level 0) ------
static void dist_sweeps(hs_factor_s* f) {
  DistSolve* D = f->ds.get();
  Comm* cm = f->h->comm;
  cudaStream_t st = f->h->stream;
  const size_t smf = sizeof(double) * 2 * std::max(D->max_m, 1);
  const size_t smb = sizeof(double) * (std::max(D->max_m, 1) + std::max(D->max_kn, 1));
  set_smem_attr((const void*)k_dfwd, smf);
  set_smem_attr((const void*)k_dbwd, smb);
  for (const auto& B : D->batches) {
    if (B.nfwd) k_dfwd<<<B.nfwd, DT, smf, st>>>(D->d_fwd + B.fwd0);
    if (B.phase2) {   // every rank takes part in every phase-II exchange (the same group sequence)
      comm_group_start(cm);
      for (const auto& m : B.fsend) comm_send_f64(cm, m.ptr, (size_t)m.len, m.peer, st);
      for (const auto& m : B.frecv) comm_recv_f64(cm, m.ptr, (size_t)m.len, m.peer, st);
      comm_group_end(cm, st);
    }
    if (B.nacc) k_dacc<<<B.nacc, DT, 0, st>>>(D->d_acc + B.acc0, D->d_accsrc);
    count_launch((B.nfwd ? 1 : 0) + (B.nacc ? 1 : 0));
  }
  // top on rank 0
  const int ntc = (int)D->top.size();
  comm_group_start(cm);
  for (int c = 0; c < ntc; ++c) {
    const auto& t = D->top[c];
    if (t.peer == 0 || !t.len) continue;
    if (D->rank == t.peer) comm_send_f64(cm, D->d_y + D->top_off[c], (size_t)t.len, 0, st);
    else if (D->rank == 0) comm_recv_f64(cm, D->d_y + D->top_off[c], (size_t)t.len, t.peer, st);
  }
  comm_group_end(cm, st);
  if (D->rank == 0 && f->ntop > 0) {
    double* yt = D->d_y + D->top_off[0];
    HS_CUDA(cudaMemcpyAsync(D->d_x + D->top_off[0], yt, sizeof(double) * f->ntop, cudaMemcpyDeviceToDevice, st));
    launch_top_solve(D->d_x + D->top_off[0], f->d_top, (int)f->ntop, (int)f->ntop, st);
  }
  comm_group_start(cm);
  for (int c = 0; c < ntc; ++c) {
    const auto& t = D->top[c];
    if (t.peer == 0 || !t.len) continue;
    if (D->rank == 0) comm_send_f64(cm, D->d_x + D->top_off[c], (size_t)t.len, t.peer, st);
    else if (D->rank == t.peer) comm_recv_f64(cm, D->d_x + D->top_off[c], (size_t)t.len, 0, st);
  }
  comm_group_end(cm, st);
  for (auto it = D->batches.rbegin(); it != D->batches.rend(); ++it) {
    const auto& B = *it;
    if (B.phase2) {
      comm_group_start(cm);
      for (const auto& m : B.bsend) comm_send_f64(cm, m.ptr, (size_t)m.len, m.peer, st);
      for (const auto& m : B.brecv) comm_recv_f64(cm, m.ptr, (size_t)m.len, m.peer, st);
      comm_group_end(cm, st);
    }
    if (B.nbwd) {
      k_dbwd<<<B.nbwd, DT, smb, st>>>(D->d_bwd + B.bwd0, D->d_nb);
      count_launch(1);
    }
  }
}

// x_loc = M^{-1} r_loc on the owned permuted range
static void dist_apply_local(hs_factor_s* f, const double* r_loc, double* x_loc) {
  DistSolve* D = f->ds.get();
  cudaStream_t st = f->h->stream;
  if (D->nloc)
    HS_CUDA(cudaMemcpyAsync(D->d_y + D->r0, r_loc, sizeof(double) * D->nloc, cudaMemcpyDeviceToDevice, st));
  dist_sweeps(f);
  if (D->nloc)
    HS_CUDA(cudaMemcpyAsync(x_loc, D->d_x + D->r0, sizeof(double) * D->nloc, cudaMemcpyDeviceToDevice, st));
}

// the owned range of every rank into d_full (permuted order) on every rank
static void dist_allgather(hs_factor_s* f, const double* loc, double* full) {
  DistSolve* D = f->ds.get();
  Comm* cm = f->h->comm;
  cudaStream_t st = f->h->stream;
  if (D->nloc) HS_CUDA(cudaMemcpyAsync(full + D->r0, loc, sizeof(double) * D->nloc, cudaMemcpyDeviceToDevice, st));
  comm_group_start(cm);
  for (int g = 0; g < D->world; ++g) {
    if (g == D->rank) continue;
    comm_send_f64(cm, full + D->r0, (size_t)D->nloc, g, st);
    const int64_t a = D->range_lo[g], b = D->range_hi[g];
    comm_recv_f64(cm, full + a, (size_t)(b - a), g, st);
  }
  comm_group_end(cm, st);
}

static void ensure_ranges(hs_factor_s* f) {
  DistSolve* D = f->ds.get();
  if (!D->range_lo.empty()) return;
  std::vector<int32_t> v(2 * D->world, 0);
  v[2 * D->rank] = (int32_t)D->r0;
  v[2 * D->rank + 1] = (int32_t)D->r1;
  int32_t* d = (int32_t*)D->dc->alloc(sizeof(int32_t) * v.size());
  HS_CUDA(cudaMemcpyAsync(d, v.data(), sizeof(int32_t) * v.size(), cudaMemcpyHostToDevice, f->h->stream));
  comm_allreduce_sum_i32(f->h->comm, d, v.size(), f->h->stream);
  HS_CUDA(cudaMemcpyAsync(v.data(), d, sizeof(int32_t) * v.size(), cudaMemcpyDeviceToHost, f->h->stream));
  HS_CUDA(cudaStreamSynchronize(f->h->stream));
  D->dc->free(d);
  for (int g = 0; g < D->world; ++g) {
    D->range_lo.push_back(v[2 * g]);
    D->range_hi.push_back(v[2 * g + 1]);
  }
}

void dist_apply(hs_factor_s* f, const double* d_b, double* d_x) {   // global vectors, original order
  DistSolve* D = f->ds.get();
  cudaStream_t st = f->h->stream;
  ensure_ranges(f);
  const int64_t n = f->an->n;
  k_dperm<<<grid_for(n), DT, 0, st>>>(d_b, D->d_full, f->d_perm, n, 0);   // permuted b
  count_launch(1);
  dist_apply_local(f, D->d_full + D->r0, D->d_xs);
  dist_allgather(f, D->d_xs, D->d_full2);
  k_dperm<<<grid_for(n), DT, 0, st>>>(D->d_full2, d_x, f->d_perm, n, 1);
  count_launch(1);
}

static double dist_dot(hs_factor_s* f, const double* a, const double* b) {
  DistSolve* D = f->ds.get();
  cudaStream_t st = f->h->stream;
  k_ddot<<<DDOT_BLOCKS, DT, 0, st>>>(a, b, D->nloc, D->d_part);
  k_ddot_fin<<<1, 32, 0, st>>>(D->d_part, DDOT_BLOCKS, D->d_part + DDOT_BLOCKS);
  count_launch(2);
  comm_allreduce_sum_f64(f->h->comm, D->d_part + DDOT_BLOCKS, 1, st);
  HS_CUDA(cudaMemcpyAsync(D->h_scal, D->d_part + DDOT_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, st));
  HS_CUDA(cudaStreamSynchronize(st));
  return D->h_scal[0];
}

static void dist_spmv(hs_factor_s* f, const double* x_loc, double* y_loc) {
  DistSolve* D = f->ds.get();
  Comm* cm = f->h->comm;
  cudaStream_t st = f->h->stream;
  if (D->nloc) HS_CUDA(cudaMemcpyAsync(D->d_xext, x_loc, sizeof(double) * D->nloc, cudaMemcpyDeviceToDevice, st));
  const int64_t ns = D->hsend.empty() ? 0 : D->hsend_off.back() + D->hsend.back().len;
  if (ns) {
    k_dgather<<<grid_for(ns), DT, 0, st>>>(x_loc, D->d_sidx, D->d_sbuf, ns);
    count_launch(1);
  }
  comm_group_start(cm);
  for (size_t k = 0; k < D->hsend.size(); ++k)
    comm_send_f64(cm, D->d_sbuf + D->hsend_off[k], (size_t)D->hsend[k].len, D->hsend[k].peer, st);
  for (size_t k = 0; k < D->hrecv.size(); ++k)
    comm_recv_f64(cm, D->d_xext + D->hrecv_off[k], (size_t)D->hrecv[k].len, D->hrecv[k].peer, st);
  comm_group_end(cm, st);
  if (D->nloc) launch_spmv(D->d_lrow, D->d_lcol, D->d_lval, D->d_xext, y_loc, D->nloc, st);
}

void dist_spmv_global(hs_factor_s* f, const double* d_x, double* d_y) {   // original order, global
  DistSolve* D = f->ds.get();
  cudaStream_t st = f->h->stream;
  ensure_ranges(f);
  const int64_t n = f->an->n;
  k_dperm<<<grid_for(n), DT, 0, st>>>(d_x, D->d_full, f->d_perm, n, 0);
  count_launch(1);
  dist_spmv(f, D->d_full + D->r0, D->d_xs);
  dist_allgather(f, D->d_xs, D->d_full2);
  k_dperm<<<grid_for(n), DT, 0, st>>>(D->d_full2, d_y, f->d_perm, n, 1);
  count_launch(1);
}

void dist_pcg(hs_factor_s* f, const double* d_b, double* d_xout, double tol, int maxit, hs_pcg_report* rep) {
  DistSolve* D = f->ds.get();
  cudaStream_t st = f->h->stream;
  ensure_ranges(f);
  const int64_t n = f->an->n, nl = D->nloc;
  cudaEvent_t e0, e1;
  HS_CUDA(cudaEventCreate(&e0));
  HS_CUDA(cudaEventCreate(&e1));
  HS_CUDA(cudaEventRecord(e0, st));
  k_dperm<<<grid_for(n), DT, 0, st>>>(d_b, D->d_full, f->d_perm, n, 0);
  count_launch(1);
  double* r = D->d_r;
  double* z = D->d_z;
  double* p = D->d_p;
  double* q = D->d_q;
  double* x = D->d_xs;
  if (nl) {
    HS_CUDA(cudaMemcpyAsync(r, D->d_full + D->r0, sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    HS_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * nl, st));
  }
  rep->history_len = 0;
  auto hist = [&](double v) {
    if (rep->history && rep->history_len < rep->history_cap) rep->history[rep->history_len++] = v;
  };
  const double bb = dist_dot(f, r, r);
  rep->iters = 0;
  rep->converged = 0;
  rep->relres = 1.0;
  hist(bb == 0.0 ? 0.0 : 1.0);
  hs_status err = HS_OK;
  if (bb == 0.0) {
    rep->converged = 1;
    rep->relres = 0.0;
  } else {
    const double nb = std::sqrt(bb);
    dist_apply_local(f, r, z);
    if (nl) HS_CUDA(cudaMemcpyAsync(p, z, sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    double rho = dist_dot(f, r, z);
    if (!(rho > 0.0)) err = HS_E_PRECOND_NOT_POSITIVE;
    for (int k = 1; k <= maxit && err == HS_OK; ++k) {
      dist_spmv(f, p, q);
      const double alpha = rho / dist_dot(f, p, q);
      if (nl) {
        k_daxpy<<<grid_for(nl), DT, 0, st>>>(x, p, alpha, nl);
        k_daxpy<<<grid_for(nl), DT, 0, st>>>(r, q, -alpha, nl);
        count_launch(2);
      }
      const double rel = std::sqrt(std::max(dist_dot(f, r, r), 0.0)) / nb;
      rep->iters = k;
      rep->relres = rel;
      hist(rel);
      if (rel <= tol) {
        rep->converged = 1;
        break;
      }
      dist_apply_local(f, r, z);
      const double rho2 = dist_dot(f, r, z);
      if (!(rho2 > 0.0)) {
        err = HS_E_PRECOND_NOT_POSITIVE;
        break;
      }
      if (nl) {
        k_dxpby<<<grid_for(nl), DT, 0, st>>>(p, z, rho2 / rho, nl);
        count_launch(1);
      }
      rho = rho2;
    }
  }
  HS_CUDA(cudaEventRecord(e1, st));
  HS_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  HS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  rep->t_pcg_s = ms * 1e-3;
  rep->t_apply_s = 0.0;
  rep->t_spmv_s = 0.0;
  // true residual ||b - A x|| / ||b|| (every rank: its rows, all-reduced)
  dist_spmv(f, x, q);
  if (nl) {
    HS_CUDA(cudaMemcpyAsync(z, D->d_full + D->r0, sizeof(double) * nl, cudaMemcpyDeviceToDevice, st));
    k_daxpy<<<grid_for(nl), DT, 0, st>>>(z, q, -1.0, nl);
    count_launch(1);
  }
  const double rr = dist_dot(f, z, z);
  rep->relres_true = bb > 0 ? std::sqrt(rr / bb) : 0.0;
  dist_allgather(f, x, D->d_full2);
  k_dperm<<<grid_for(n), DT, 0, st>>>(D->d_full2, d_xout, f->d_perm, n, 1);
  count_launch(1);
  HS_CUDA(cudaStreamSynchronize(st));
  if (err != HS_OK) fail(err, "pcg: <r, M^{-1} r> <= 0 (preconditioner not positive)");
  if (!rep->converged) fail(HS_E_NOT_CONVERGED, "pcg: maxit reached");
}

}  // namespace hs
