// Multi-GPU decomposition plan (host, integer) — SURVEY §8(e), the reconstruction of the
// parallel algorithm the paper defers to parallel LoRaSp (Thm 2,
// P:719-729).  Mirrors oracle/dist.py (independent implementation, same protocol):
//   * subdomain k of the 2^nsub fixed subdomains (analyze O2.5) is owned by rank k P / 2^nsub;
//     every cluster of a level < L_top lies in one subdomain; parents inherit the owner;
//   * rank g holds block (p, q) iff it owns p or q (cross-owner blocks are duplicated);
//   * a phase-II cluster s is eliminated by its owner, whose record (r, C_s, coarse rows)
//     goes to the owners of n(s) u w(s): they hold every other block the elimination
//     writes (Schur targets (p, q), p, q in n(s); row s blocks (s, q)).
#include <algorithm>

#include "internal.h"

namespace hs {

DistPlan make_plan(const Analysis& an, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) fail(HS_E_INVALID_ARG, "dist plan: bad world/rank");
  const int nsub_log2 = std::min(an.nsub_log2, an.D);
  const int nsub = 1 << nsub_log2;
  if (world > nsub || nsub % world != 0)
    fail(HS_E_INVALID_ARG, "dist plan: world size must divide the number of fixed subdomains");
  DistPlan P;
  P.world = world;
  P.rank = rank;
  P.owner.resize(an.L_top + 1);
  for (int l = 0; l <= an.L_top; ++l) {
    const int d = an.D - l;
    const int nclus = 1 << d;
    auto& o = P.owner[l];
    o.resize(nclus);
    for (int c = 0; c < nclus; ++c) {
      const int sub = c >> std::max(0, d - nsub_log2);
      o[c] = (int32_t)((int64_t)sub * world / nsub);
    }
  }
  return P;
}

std::vector<int32_t> receivers(const Analysis& an, const DistPlan& P, int l, int s) {
  const Level& lev = an.levels[l];
  const int32_t g = P.owner[l][s];
  std::vector<int32_t> r;
  for (const Adj* A : {&lev.H, &lev.w})
    for (int32_t q : (*A)[s]) {
      const int32_t h = P.owner[l][q];
      if (h != g) r.push_back(h);
    }
  std::sort(r.begin(), r.end());
  r.erase(std::unique(r.begin(), r.end()), r.end());
  return r;
}

}  // namespace hs
