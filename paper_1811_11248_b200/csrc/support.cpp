// Structural column supports of the level-0 blocks (SURVEY §8(d) "k-hat", O2.10).
//
// At level 0 every block A_pq of the store is a cap_p x cap_q dense array, but only the
// columns of q that touch p -- the interface DOFs -- are nonzero: the columns of A_pq that are
// structurally zero stay exactly zero through every step of an elimination:
//   * the scaling G_s^{-1} [A_sw | A_sn] and the rotation Qᵀ act on the left, column by column;
//   * a zero column has norm 0 and is never a CPQR pivot (the pivot rule and its 1e-10 tie
//     window only ever admit columns with norm >= (1 - 1e-10) max > 0), and a
//     Householder reflector maps it to zero;
//   * the Schur update A_pq -= C_pᵀ C_q only reaches the columns in the support of C_q, which
//     is the support of A_sq.
// So a cluster's B_s restricted to the supported columns gives the same ranks, pivots and
// values on those columns as the dense B_s, with k-hat instead of k columns in the scaling,
// the CPQR, the rotation and the Schur products.  The supports only depend on the pattern and
// the schedule, so they are computed once per analysis by the symbolic simulation below:
//   supp(p, q) = { local j of q : A_pq[:, j] != 0 } initially (the CSR pattern), then for every
//   eliminated s (in batch order) and every pair p != q of n(s) not yet eliminated:
//   supp(p, q) |= supp(s, q).
// A block whose column cluster q was eliminated earlier on the level has q's r_q coarse
// columns, all of them potentially nonzero (dense).
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "internal.h"

namespace hs {

namespace {
std::mutex g_mu;
}

const int32_t* l0_support_device(Analysis& an, int device) {
  std::lock_guard<std::mutex> lk(g_mu);
  L0Support& o = an.l0s;
  if (!o.built) fail(HS_E_INTERNAL, "support: not built");
  if (o.d_idx && o.dev == device) return o.d_idx;
  if (o.d_idx) {   // cached on another device
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(o.dev);
    cudaFree(o.d_idx);
    cudaSetDevice(cur);
    o.d_idx = nullptr;
  }
  const size_t bytes = sizeof(int32_t) * std::max<size_t>(o.idx.size(), 1);
  if (cudaMalloc(&o.d_idx, bytes) != cudaSuccess) fail(HS_E_OOM, "support: device copy");
  if (!o.idx.empty() &&
      cudaMemcpy(o.d_idx, o.idx.data(), sizeof(int32_t) * o.idx.size(), cudaMemcpyHostToDevice) != cudaSuccess)
    fail(HS_E_CUDA, "support: device copy");
  o.dev = device;
  return o.d_idx;
}

void build_l0_support(Analysis& an) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (an.l0s.built) return;
  const Level& lev = an.levels.at(0);
  const int32_t nc = lev.nclus;
  const Adj& F = lev.Ffinal;   // every block the level-0 store holds
  auto size_of = [&](int32_t c) { return (int32_t)(an.leaf_off[c + 1] - an.leaf_off[c]); };
  auto nwords = [&](int32_t c) { return (size_t)(size_of(c) + 63) / 64; };
  // one bitset per stored off-diagonal block (p, q), q in F[p]
  std::vector<size_t> boff(1, 0);
  std::vector<int64_t> rptr(nc + 1, 0);
  for (int32_t p = 0; p < nc; ++p) {
    rptr[p + 1] = rptr[p] + (int64_t)F[p].size();
    for (int32_t q : F[p]) boff.push_back(boff.back() + nwords(q));
  }
  std::vector<uint64_t> bits(boff.back(), 0);
  auto slot = [&](int32_t p, int32_t q) -> int64_t {
    const auto& r = F[p];
    const auto it = std::lower_bound(r.begin(), r.end(), q);
    return (it != r.end() && *it == q) ? rptr[p] + (it - r.begin()) : -1;
  };
  std::vector<int32_t> leaf_of(an.n);
  for (int32_t c = 0; c < nc; ++c)
    for (int64_t k = an.leaf_off[c]; k < an.leaf_off[c + 1]; ++k) leaf_of[k] = c;
  for (int64_t i = 0; i < an.n; ++i) {   // the pattern, in the permuted numbering
    const int32_t x = leaf_of[i];
    const int64_t old = an.perm[i];
    for (int64_t k = an.rowptr[old]; k < an.rowptr[old + 1]; ++k) {
      const int64_t j = an.iperm[an.colind[k]];
      const int32_t y = leaf_of[j];
      if (y == x) continue;
      const int64_t b = slot(x, y);
      if (b < 0) fail(HS_E_INTERNAL, "support: a pattern block missing from the level-0 store");
      const int64_t lj = j - an.leaf_off[y];
      bits[boff[b] + (lj >> 6)] |= 1ull << (lj & 63);
    }
  }
  std::vector<std::vector<int32_t>> len(nc), idx(nc);
  std::vector<uint8_t> done(nc, 0);
  for (const auto& batch : lev.batches) {
    for (int32_t s : batch)   // the supports each cluster of the batch is eliminated with
      for (int pass = 0; pass < 2; ++pass)
        for (int32_t q : (pass == 0 ? lev.w[s] : lev.H[s])) {
          if (done[q]) {
            len[s].push_back(-1);
            continue;
          }
          const int64_t b = slot(s, q);
          if (b < 0) fail(HS_E_INTERNAL, "support: block of n(s) or w(s) missing from the store");
          int32_t cnt = 0;
          for (int32_t j = 0; j < size_of(q); ++j)
            if ((bits[boff[b] + (j >> 6)] >> (j & 63)) & 1ull) {
              idx[s].push_back(j);
              ++cnt;
            }
          len[s].push_back(cnt);
        }
    for (int32_t s : batch) {   // the Schur fill of the batch, A_pq -= C_pᵀ C_q on n(s) x n(s)
      const auto& ns = lev.H[s];
      for (int32_t p : ns) {
        if (done[p]) continue;
        for (int32_t q : ns) {
          if (q == p || done[q]) continue;
          const int64_t bd = slot(p, q), bs = slot(s, q);
          if (bd < 0 || bs < 0) continue;   // not held by the store: the update has no target
          for (size_t w = 0; w < nwords(q); ++w) bits[boff[bd] + w] |= bits[boff[bs] + w];
        }
      }
    }
    for (int32_t s : batch) done[s] = 1;
  }
  L0Support& o = an.l0s;
  o.sptr.assign(nc + 1, 0);
  o.iptr.assign(nc + 1, 0);
  for (int32_t s = 0; s < nc; ++s) {
    o.sptr[s + 1] = o.sptr[s] + (int64_t)len[s].size();
    o.iptr[s + 1] = o.iptr[s] + (int64_t)idx[s].size();
  }
  o.len.reserve(o.sptr[nc]);
  o.idx.reserve(o.iptr[nc]);
  for (int32_t s = 0; s < nc; ++s) {
    o.len.insert(o.len.end(), len[s].begin(), len[s].end());
    o.idx.insert(o.idx.end(), idx[s].begin(), idx[s].end());
  }
  o.built = true;
}

}  // namespace hs
