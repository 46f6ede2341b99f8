// hs_analyze — clustering, cluster tree and per-level elimination schedule (host, integer).
//
// Paper: clusters are a partition of the graph G_A computed algebraically with
// existing packages; Zoltan geometric partition, clusters of ~100
// (P:812); extruded partition keeps every vertical line in one cluster
// (P:786-798).  Neighbours: A(pi_p, pi_q) != 0, re-applied to A_c at
// every level (Alg. 1).  The readings (RCB, n/w sets, greedy
// independent-set batches, binary tree, structural top) are DESIGN.md Q6-Q11
// (= SURVEY §8(c) O2); the output must equal the oracle's bit for bit.
#include <algorithm>
#include <numeric>

#include "internal.h"

namespace hs {

namespace {

// sorted union into dst (dst sorted, src sorted), skipping `skip`
void merge_into(std::vector<int32_t>& dst, const std::vector<int32_t>& src, int32_t skip,
                std::vector<int32_t>& tmp) {
  tmp.clear();
  tmp.reserve(dst.size() + src.size());
  size_t i = 0, j = 0;
  while (i < dst.size() || j < src.size()) {
    int32_t v;
    if (j >= src.size() || (i < dst.size() && dst[i] < src[j])) {
      v = dst[i++];
    } else if (i >= dst.size() || src[j] < dst[i]) {
      v = src[j++];
      if (v == skip) continue;
    } else {
      v = dst[i++];
      ++j;
    }
    tmp.push_back(v);
  }
  dst.swap(tmp);
}

}  // namespace

Analysis* analyze(int64_t n, const int64_t* rowptr, const int32_t* colind, const double* coords,
                  int32_t coord_dim, const int32_t* column_id, const hs_analyze_opts& opt) {
  if (n <= 0 || !rowptr || !colind) fail(HS_E_INVALID_ARG, "analyze: empty matrix or NULL pattern");
  const bool graph = !coords || coord_dim <= 0;   // coordinate-free: graph bisection (NEXT f4)
  if (graph && column_id) fail(HS_E_UNSUPPORTED, "analyze: graph bisection works on DOF units (no column_id)");
  if (opt.top_log2 < 0 || opt.nsub_log2 < 0 || opt.nsub_log2 > opt.top_log2)
    fail(HS_E_INVALID_ARG, "analyze: need 0 <= nsub_log2 <= top_log2");
  const int64_t nnz = rowptr[n];
  for (int64_t i = 0; i < n; ++i)
    if (rowptr[i + 1] < rowptr[i]) fail(HS_E_INVALID_ARG, "analyze: rowptr not monotone");
  for (int64_t k = 0; k < nnz; ++k)
    if (colind[k] < 0 || colind[k] >= n) fail(HS_E_INVALID_ARG, "analyze: column index out of range");
  // structural symmetry: every (i, j) has (j, i)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int64_t j = colind[k];
      const int32_t* b = colind + rowptr[j];
      const int32_t* e = colind + rowptr[j + 1];
      const int32_t* f = std::lower_bound(b, e, (int32_t)i);
      if (f == e || *f != i) fail(HS_E_NOT_SYMMETRIC, "analyze: pattern is not symmetric");
    }

  auto* an = new Analysis();
  an->n = n;
  an->top_log2 = opt.top_log2;
  an->rowptr.assign(rowptr, rowptr + n + 1);
  an->colind.assign(colind, colind + nnz);

  // ---- units (O2.1) -----------------------------------------------------------------
  int dims;
  std::vector<double> uc;              // unit coordinates, row-major [U][dims]
  std::vector<int64_t> unit_of_dof;    // empty when units are DOFs
  int64_t U;
  if (graph) {
    U = n;
    dims = 0;
  } else if (!column_id) {
    U = n;
    dims = coord_dim;
    uc.assign(coords, coords + n * coord_dim);
  } else {
    std::vector<int64_t> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int64_t a, int64_t b) { return column_id[a] < column_id[b]; });
    dims = std::min(2, (int)coord_dim);
    unit_of_dof.assign(n, -1);
    std::vector<int64_t> first;
    int64_t u = -1;
    for (int64_t t = 0; t < n; ++t) {
      const int64_t i = order[t];
      if (t == 0 || column_id[i] != column_id[order[t - 1]]) {
        ++u;
        first.push_back(i);            // stable sort -> lowest DOF index of the column
      }
      unit_of_dof[i] = u;
    }
    U = u + 1;
    uc.resize(U * dims);
    for (int64_t k = 0; k < U; ++k)
      for (int a = 0; a < dims; ++a) uc[k * dims + a] = coords[first[k] * coord_dim + a];
  }
  const int64_t leaf_units = column_id ? opt.leaf_columns : opt.leaf_size;
  if (leaf_units <= 0) fail(HS_E_INVALID_ARG, "analyze: leaf size must be positive");
  // ---- depth (O2.2) -------------------------------------------------------------------
  int D = 0;
  while (((U + (int64_t(1) << D) - 1) >> D) > leaf_units) ++D;
  if (D > 30) fail(HS_E_UNSUPPORTED, "analyze: tree too deep");
  an->D = D;
  // ---- RCB (O2.3), or recursive BFS bisection without coordinates ----------------------
  std::vector<std::vector<int64_t>> nodes(1);
  nodes[0].resize(U);
  std::iota(nodes[0].begin(), nodes[0].end(), 0);
  if (graph) {
    // At a node with unit set I (ascending): BFS on the induced subgraph from min(I)
    // (neighbours in ascending id, restarting from the smallest unvisited unit when a
    // component is exhausted); from its last unit g the same BFS gives the order; the left
    // child takes the first ceil(|I|/2) units (the paper's "algebraic"
    // clustering P:483-485).
    std::vector<uint8_t> inset(n, 0), seen(n, 0);
    std::vector<int64_t> order, queue;
    auto bfs = [&](const std::vector<int64_t>& I, int64_t start) {
      order.clear();
      queue.clear();
      size_t qh = 0, nxt_start = 0;
      seen[start] = 1;
      order.push_back(start);
      queue.push_back(start);
      while (order.size() < I.size()) {
        if (qh == queue.size()) {
          while (seen[I[nxt_start]]) ++nxt_start;
          const int64_t v = I[nxt_start];
          seen[v] = 1;
          order.push_back(v);
          queue.push_back(v);
        }
        const int64_t u = queue[qh++];
        for (int64_t k = rowptr[u]; k < rowptr[u + 1]; ++k) {
          const int64_t w = colind[k];
          if (inset[w] && !seen[w]) {
            seen[w] = 1;
            order.push_back(w);
            queue.push_back(w);
          }
        }
      }
      for (int64_t v : order) seen[v] = 0;
    };
    for (int d = 0; d < D; ++d) {
      std::vector<std::vector<int64_t>> nxt(nodes.size() * 2);
      for (size_t x = 0; x < nodes.size(); ++x) {
        const auto& I = nodes[x];
        if (I.empty()) continue;
        for (int64_t u : I) inset[u] = 1;
        bfs(I, I[0]);
        const int64_t g = order.back();
        bfs(I, g);
        for (int64_t u : I) inset[u] = 0;
        const size_t h = (I.size() + 1) / 2;
        nxt[2 * x].assign(order.begin(), order.begin() + h);
        nxt[2 * x + 1].assign(order.begin() + h, order.end());
        std::sort(nxt[2 * x].begin(), nxt[2 * x].end());
        std::sort(nxt[2 * x + 1].begin(), nxt[2 * x + 1].end());
      }
      nodes.swap(nxt);
    }
  }
  for (int d = 0; d < (graph ? 0 : D); ++d) {
    std::vector<std::vector<int64_t>> nxt(nodes.size() * 2);
    for (size_t x = 0; x < nodes.size(); ++x) {
      auto& I = nodes[x];
      if (I.empty()) continue;
      int ax = 0;
      double best = -1.0;
      for (int a = 0; a < dims; ++a) {
        double lo = uc[I[0] * dims + a], hi = lo;
        for (int64_t u : I) {
          const double v = uc[u * dims + a];
          lo = std::min(lo, v);
          hi = std::max(hi, v);
        }
        const double ext = hi - lo;
        if (a == 0 || ext > best) { best = ext; ax = a; }   // first maximum = lowest axis on ties
      }
      std::sort(I.begin(), I.end(), [&](int64_t p, int64_t q) {
        const double cp = uc[p * dims + ax], cq = uc[q * dims + ax];
        if (cp < cq) return true;
        if (cq < cp) return false;
        return p < q;
      });
      const size_t h = (I.size() + 1) / 2;
      nxt[2 * x].assign(I.begin(), I.begin() + h);
      nxt[2 * x + 1].assign(I.begin() + h, I.end());
    }
    nodes.swap(nxt);
  }
  const int64_t nleaf = int64_t(1) << D;
  std::vector<int64_t> uleaf(U);
  for (int64_t x = 0; x < nleaf; ++x)
    for (int64_t u : nodes[x]) uleaf[u] = x;
  nodes.clear();
  std::vector<int32_t> dof_leaf(n);
  for (int64_t i = 0; i < n; ++i) dof_leaf[i] = (int32_t)(column_id ? uleaf[unit_of_dof[i]] : uleaf[i]);
  // ---- permutation (O2.4) -------------------------------------------------------------
  an->leaf_off.assign(nleaf + 1, 0);
  for (int64_t i = 0; i < n; ++i) an->leaf_off[dof_leaf[i] + 1]++;
  for (int64_t x = 0; x < nleaf; ++x) an->leaf_off[x + 1] += an->leaf_off[x];
  an->perm.resize(n);
  an->iperm.resize(n);
  {
    std::vector<int64_t> pos(an->leaf_off.begin(), an->leaf_off.end() - 1);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t k = pos[dof_leaf[i]]++;
      an->perm[k] = i;
      an->iperm[i] = k;
    }
  }
  an->L_top = std::max(0, D - opt.top_log2);
  an->nsub_log2 = std::min(opt.nsub_log2, D);
  // ---- H_0 (O2.7) ---------------------------------------------------------------------
  Adj H(nleaf);
  for (int64_t i = 0; i < n; ++i) {
    const int32_t p = dof_leaf[i];
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      const int32_t q = dof_leaf[colind[k]];
      if (q != p) H[p].push_back(q);
    }
  }
  for (auto& h : H) {
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
  }
  // ---- per-level schedule (O2.8, O2.9 / reading R-coarse) --------------------------------
  // F0 = the block pattern of the level's input A_l (H_0 at level 0, then the merge of the
  // previous level's final fill graph).  H = n(s): under R-coarse (coarse_fill = 0) the
  // merged structural neighbours, under O2.9 (coarse_fill = 1) the whole pattern F0.
  if (opt.coarse_fill != 0 && opt.coarse_fill != 1) fail(HS_E_INVALID_ARG, "analyze: coarse_fill must be 0 or 1");
  auto merge = [](const Adj& A, int32_t nclus) {
    Adj M(nclus / 2);
    for (int32_t c = 0; c < nclus; ++c) {
      const int32_t P = c >> 1;
      for (int32_t q : A[c])
        if ((q >> 1) != P) M[P].push_back(q >> 1);
    }
    for (auto& h : M) {
      std::sort(h.begin(), h.end());
      h.erase(std::unique(h.begin(), h.end()), h.end());
    }
    return M;
  };
  Adj F0 = H;
  std::vector<int32_t> tmp;
  for (int l = 0; l < an->L_top; ++l) {
    Level lev;
    const int32_t nclus = (int32_t)(int64_t(1) << (D - l));
    lev.nclus = nclus;
    lev.H = H;
    Adj F = F0;
    lev.interior.assign(nclus, 1);
    for (int32_t s = 0; s < nclus; ++s)
      for (int32_t q : F0[s])
        if (an->subdomain(l, q) != an->subdomain(l, s)) { lev.interior[s] = 0; break; }
    lev.w.assign(nclus, {});
    std::vector<uint8_t> done(nclus, 0), inB(nclus, 0);
    for (int phase = 1; phase <= 2; ++phase) {
      for (;;) {
        std::vector<int32_t> B;
        for (int32_t s = 0; s < nclus; ++s) {
          if (done[s] || (phase == 1 && !lev.interior[s])) continue;
          bool adj = false;
          for (int32_t q : F[s])
            if (inB[q]) { adj = true; break; }
          if (!adj) { B.push_back(s); inB[s] = 1; }
        }
        if (B.empty()) break;
        for (int32_t s : B) {               // w(s) = F-adj(s) \ n(s), before the fill
          auto& w = lev.w[s];
          w.clear();
          std::set_difference(F[s].begin(), F[s].end(), H[s].begin(), H[s].end(), std::back_inserter(w));
        }
        for (int32_t s : B)                 // fill: clique on n(s)
          for (int32_t p : H[s]) merge_into(F[p], H[s], p, tmp);
        for (int32_t s : B) { done[s] = 1; inB[s] = 0; }
        lev.batches.push_back(std::move(B));
        if (phase == 1) lev.nphase1++;
      }
    }
    // A_c's block pattern: parents adjacent iff some children are F_final-adjacent
    Adj Fn = merge(F, nclus);
    Adj Hn = opt.coarse_fill ? Fn : merge(H, nclus);
    lev.Fstart = std::move(F0);
    lev.Ffinal = std::move(F);
    an->levels.push_back(std::move(lev));
    F0 = std::move(Fn);
    H = std::move(Hn);
  }
  an->H_top = std::move(F0);   // the top's whole block pattern (under both readings)
  return an;
}

}  // namespace hs
