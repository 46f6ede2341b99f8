// hs_factor — host driver of Algorithm 1 on one B200.
//
// Per level l = 0 .. L_top-1 and per batch of independent clusters (schedule from
// hs_analyze), the runtime plans descriptors on the host and launches
//   pack (copy2d) -> POTRF -> TRSM (deferred compression) -> CPQR+rotation
//   -> [one D2H of the batch's ranks]
//   -> Schur update (ordered per target tile) + write-back (copy2d, identity)
// then assembles the parent level's blocks (A_c) and finally factors the dense top
// (P:626-628).  The elimination record (G, V, tau, C) stays in device memory for the
// apply, whose plan (descriptors) is built alongside and replayed as a CUDA graph.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <unordered_map>

#include "runtime.h"

namespace hs {

void DevScratch::ensure(size_t bytes) {
  if (bytes <= cap) return;
  if (d) cudaFree(d);
  d = nullptr;
  cap = std::max(bytes, cap * 2);
  HS_CUDA(cudaMalloc(&d, cap));
}
DevScratch::~DevScratch() {
  if (d) cudaFree(d);
}
void HostStage::ensure(size_t bytes) {
  if (bytes <= cap) return;
  if (h) cudaFreeHost(h);
  h = nullptr;
  cap = std::max(bytes, cap * 2);
  HS_CUDA(cudaMallocHost(&h, cap));
}
HostStage::~HostStage() {
  if (h) cudaFreeHost(h);
}

namespace {

// Uploads a set of host vectors into one device scratch region with one memcpy.
struct Upload {
  HostStage stage;
  DevScratch dev;
  std::vector<std::pair<size_t, size_t>> parts;   // (offset, bytes)
  size_t total = 0;
  void reset() {
    parts.clear();
    total = 0;
  }
  template <class T>
  size_t add(const std::vector<T>& v) {
    const size_t off = (total + 255) & ~size_t(255);
    parts.push_back({off, v.size() * sizeof(T)});
    total = off + v.size() * sizeof(T);
    return parts.size() - 1;
  }
  template <class T>
  void copy_in(size_t idx, const std::vector<T>& v) {
    if (!v.empty()) std::memcpy(stage.h + parts[idx].first, v.data(), v.size() * sizeof(T));
  }
  template <class T>
  T* dptr(size_t idx) {
    return reinterpret_cast<T*>(dev.d + parts[idx].first);
  }
  void send(cudaStream_t st) {
    if (total) HS_CUDA(cudaMemcpyAsync(dev.d, stage.h, total, cudaMemcpyHostToDevice, st));
  }
};

struct BlockStore {
  double* d = nullptr;
  std::vector<int32_t> cap;
  std::vector<std::vector<std::pair<int32_t, int64_t>>> rows;   // p -> sorted (q <= p, offset)
  size_t total = 0;

  void build(const std::vector<int32_t>& caps, const Adj& edges) {
    cap = caps;
    const int n = (int)caps.size();
    rows.assign(n, {});
    int64_t off = 0;
    for (int p = 0; p < n; ++p) {
      for (int32_t q : edges[p])
        if (q < p) {
          rows[p].push_back({q, off});
          off += (int64_t)caps[p] * caps[q];
        }
      rows[p].push_back({p, off});
      off += (int64_t)caps[p] * caps[p];
    }
    total = (size_t)off;
    if (total) HS_CUDA(cudaMalloc(&d, total * sizeof(double)));
  }
  int64_t off(int32_t p, int32_t q) const {   // p >= q
    const auto& r = rows[p];
    auto it = std::lower_bound(r.begin(), r.end(), std::make_pair(q, (int64_t)-1));
    if (it == r.end() || it->first != q) return -1;
    return it->second;
  }
  bool has(int32_t p, int32_t q) const { return p >= q ? off(p, q) >= 0 : off(q, p) >= 0; }
  // A(p, q) as (pointer, ld, trans): A(p,q)[i][j] = trans ? ptr[j*ld + i] : ptr[i*ld + j]
  void get(int32_t p, int32_t q, double*& ptr, int32_t& ld, int32_t& trans) const {
    if (p >= q) {
      const int64_t o = off(p, q);
      if (o < 0) fail(HS_E_INTERNAL, "block store: missing block");
      ptr = d + o;
      ld = cap[q];
      trans = 0;
    } else {
      const int64_t o = off(q, p);
      if (o < 0) fail(HS_E_INTERNAL, "block store: missing block");
      ptr = d + o;
      ld = cap[p];
      trans = 1;
    }
  }
  void release() {
    if (d) cudaFree(d);
    d = nullptr;
  }
};

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

void check_status(DevStatus* d_status, DevStatus* h_status, cudaStream_t st) {
  HS_CUDA(cudaMemcpyAsync(h_status, d_status, sizeof(DevStatus), cudaMemcpyDeviceToHost, st));
  HS_CUDA(cudaStreamSynchronize(st));
  if (h_status->flag) {
    char buf[256];
    std::snprintf(buf, sizeof buf, "NOT_SPD: Cholesky breakdown at level %d cluster %d pivot %d value %.17g (P:283)",
                  h_status->level, h_status->cluster, h_status->pivot, h_status->value);
    fail(HS_E_NOT_SPD, buf);
  }
}

}  // namespace
}  // namespace hs

hs_factor_s::~hs_factor_s() {
  using namespace hs;
  auto fr = [](void* p) {
    if (p) cudaFree(p);
  };
  fr(d_rowptr); fr(d_colind); fr(d_vals); fr(d_perm); fr(d_top);
  for (auto& l : lv) { fr(l.arena); fr(l.iarena); }
  fr(ap.d_local); fr(ap.d_nb); fr(ap.d_tgt); fr(ap.d_con); fr(ap.d_y);
  for (auto* p : ap.d_tsrc) fr(p);
  for (auto* p : ap.d_tdst) fr(p);
  if (ap.graph) cudaGraphExecDestroy(ap.graph);
  fr(d_r); fr(d_z); fr(d_p); fr(d_q); fr(d_x); fr(d_b); fr(d_red);
  if (h_red) cudaFreeHost(h_red);
}

namespace hs {

hs_factor_s* factor_create(hs_handle_s* h, const Analysis* an, const double* values, const hs_factor_opts& opt) {
  if (opt.eps < 0 || !std::isfinite(opt.eps)) fail(HS_E_INVALID_ARG, "factor: eps must be finite and >= 0");
  if (opt.dc != 1) fail(HS_E_UNSUPPORTED, "factor: only dc = 1 (deferred compression) is implemented");
  const int64_t n = an->n, nnz = an->rowptr[n];
  // numerical symmetry of the values (A SPD, A_ns = A_sn^T)
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = an->rowptr[i]; k < an->rowptr[i + 1]; ++k) {
      const int64_t j = an->colind[k];
      if (j <= i) continue;
      const int32_t* b = an->colind.data() + an->rowptr[j];
      const int32_t* e = an->colind.data() + an->rowptr[j + 1];
      const int64_t kk = an->rowptr[j] + (std::lower_bound(b, e, (int32_t)i) - b);
      const double a = values[k], t = values[kk];
      if (std::fabs(a - t) > 1e-12 * std::max(std::fabs(a), std::fabs(t)))
        fail(HS_E_NOT_SYMMETRIC, "factor: values are not symmetric");
    }
  cudaStream_t st = h->stream;
  auto* f = new hs_factor_s();
  std::unique_ptr<hs_factor_s> guard(f);
  f->h = h;
  f->an = an;
  f->opt = opt;
  const double t_wall0 = now_s();
  double t_plan = 0.0;
  cudaEvent_t ev0, ev1;
  HS_CUDA(cudaEventCreate(&ev0));
  HS_CUDA(cudaEventCreate(&ev1));
  HS_CUDA(cudaEventRecord(ev0, st));

  HS_CUDA(cudaMalloc(&f->d_rowptr, sizeof(int64_t) * (n + 1)));
  HS_CUDA(cudaMalloc(&f->d_colind, sizeof(int32_t) * std::max<int64_t>(nnz, 1)));
  HS_CUDA(cudaMalloc(&f->d_vals, sizeof(double) * std::max<int64_t>(nnz, 1)));
  HS_CUDA(cudaMalloc(&f->d_perm, sizeof(int64_t) * n));
  HS_CUDA(cudaMemcpyAsync(f->d_rowptr, an->rowptr.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaMemcpyAsync(f->d_colind, an->colind.data(), sizeof(int32_t) * nnz, cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaMemcpyAsync(f->d_vals, values, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaMemcpyAsync(f->d_perm, an->perm.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));

  DevStatus* d_status = nullptr;
  DevStatus h_status{};
  HS_CUDA(cudaMalloc(&d_status, sizeof(DevStatus)));
  std::unique_ptr<void, void (*)(void*)> status_guard(d_status, [](void* p) { cudaFree(p); });
  HS_CUDA(cudaMemsetAsync(d_status, 0, sizeof(DevStatus), st));

  // ---- level-0 blocks from the permuted CSR ------------------------------------------------
  const int nleaf0 = (int)(an->leaf_off.size() - 1);
  std::vector<int32_t> cap(nleaf0);
  for (int c = 0; c < nleaf0; ++c) cap[c] = (int32_t)(an->leaf_off[c + 1] - an->leaf_off[c]);
  BlockStore bs;
  bs.build(cap, an->L_top > 0 ? an->levels[0].Ffinal : an->H_top);
  if (bs.total) HS_CUDA(cudaMemsetAsync(bs.d, 0, bs.total * sizeof(double), st));
  {
    std::vector<int32_t> leaf_of(n);
    for (int c = 0; c < nleaf0; ++c)
      for (int64_t k = an->leaf_off[c]; k < an->leaf_off[c + 1]; ++k) leaf_of[k] = c;
    std::vector<int64_t> map(nnz, -1);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t pi = an->iperm[i];
      const int32_t p = leaf_of[pi];
      for (int64_t k = an->rowptr[i]; k < an->rowptr[i + 1]; ++k) {
        const int64_t pj = an->iperm[an->colind[k]];
        const int32_t q = leaf_of[pj];
        if (p < q) continue;
        const int64_t o = bs.off(p, q);
        if (o < 0) fail(HS_E_INTERNAL, "factor: level-0 block missing");
        map[k] = o + (pi - an->leaf_off[p]) * cap[q] + (pj - an->leaf_off[q]);
      }
    }
    int64_t* d_map = nullptr;
    HS_CUDA(cudaMalloc(&d_map, sizeof(int64_t) * std::max<int64_t>(nnz, 1)));
    HS_CUDA(cudaMemcpyAsync(d_map, map.data(), sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
    launch_scatter(f->d_vals, d_map, nnz, bs.d, st);
    HS_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_map);
  }

  Upload upA, upB;
  int32_t* d_rank = nullptr;
  int32_t* h_rank = nullptr;
  int max_batch = 1;
  for (const auto& lev : an->levels)
    for (const auto& B : lev.batches) max_batch = std::max(max_batch, (int)B.size());
  HS_CUDA(cudaMalloc(&d_rank, sizeof(int32_t) * max_batch));
  HS_CUDA(cudaMallocHost(&h_rank, sizeof(int32_t) * max_batch));
  std::unique_ptr<void, void (*)(void*)> rank_guard(d_rank, [](void* p) { cudaFree(p); });
  std::unique_ptr<void, void (*)(void*)> hrank_guard(h_rank, [](void* p) { cudaFreeHost(p); });

  hs_factor_stats_t& S = f->stats;
  ApplyPlan& ap = f->ap;
  int64_t vbase = 0;
  f->lv.resize(an->L_top);
  ap.batches.resize(an->L_top);
  ap.trans_src.resize(an->L_top);
  ap.trans_dst.resize(an->L_top);

  for (int l = 0; l < an->L_top; ++l) {
    const Level& lev = an->levels[l];
    LevelRT& L = f->lv[l];
    L.nclus = lev.nclus;
    L.cap = cap;
    L.rank.assign(lev.nclus, 0);
    L.kn.assign(lev.nclus, 0);
    L.kw.assign(lev.nclus, 0);
    L.ldB.assign(lev.nclus, 0);
    L.voff.assign(lev.nclus + 1, 0);
    for (int c = 0; c < lev.nclus; ++c) L.voff[c + 1] = L.voff[c] + cap[c];
    L.vlen = L.voff[lev.nclus];
    ap.vbase.push_back(vbase);
    vbase += L.vlen;
    // ---- level arena: G, V (cap^2), tau (cap), nu (bound kw), B (cap x bound(kn + kw)) ----
    std::vector<int64_t> oG(lev.nclus), oV(lev.nclus), oT(lev.nclus), oN(lev.nclus), oB(lev.nclus), oP(lev.nclus);
    int64_t off = 0, ioff = 0;
    for (int s = 0; s < lev.nclus; ++s) {
      const int64_t m = cap[s];
      if (m > MAX_M) {
        char buf[160];
        std::snprintf(buf, sizeof buf, "factor: cluster %d at level %d has %lld DOFs > %d (not supported yet)", s,
                      l, (long long)m, MAX_M);
        fail(HS_E_UNSUPPORTED, buf);
      }
      int64_t bn = 0, bw = 0;
      for (int32_t q : lev.H[s]) bn += cap[q];
      for (int32_t q : lev.w[s]) bw += cap[q];
      oG[s] = off; off += m * m;
      oV[s] = off; off += m * m;
      oT[s] = off; off += m;
      oN[s] = off; off += bw;
      oB[s] = off; off += m * (bn + bw);
      off = (off + 3) & ~int64_t(3);                 // 32-byte alignment
      oP[s] = ioff; ioff += m;
    }
    L.arena_bytes = (size_t)off * sizeof(double);
    HS_CUDA(cudaMalloc(&L.arena, std::max<size_t>(L.arena_bytes, 8)));
    HS_CUDA(cudaMalloc(&L.iarena, std::max<size_t>(sizeof(int32_t) * ioff, 4)));
    L.G.resize(lev.nclus); L.V.resize(lev.nclus); L.tau.resize(lev.nclus); L.B.resize(lev.nclus);
    L.nu.resize(lev.nclus); L.piv.resize(lev.nclus);
    for (int s = 0; s < lev.nclus; ++s) {
      L.G[s] = L.arena + oG[s]; L.V[s] = L.arena + oV[s]; L.tau[s] = L.arena + oT[s];
      L.nu[s] = L.arena + oN[s]; L.B[s] = L.arena + oB[s]; L.piv[s] = L.iarena + oP[s];
    }
    std::vector<int32_t> live = cap;

    for (const auto& Bt : lev.batches) {
      const double tp0 = now_s();
      const int nb = (int)Bt.size();
      std::vector<CopyItem> gather;
      std::vector<CluItem> clu(nb);
      std::vector<TrsmItem> trsm;
      int max_m = 1;
      for (int bi = 0; bi < nb; ++bi) {
        const int32_t s = Bt[bi];
        const int32_t m = live[s];
        int32_t kn = 0, kw = 0;
        for (int32_t q : lev.H[s]) kn += live[q];
        for (int32_t q : lev.w[s]) kw += live[q];
        const int32_t ldB = kn + kw;
        L.kn[s] = kn; L.kw[s] = kw; L.ldB[s] = ldB;
        CluItem& it = clu[bi];
        it.G = L.G[s]; it.V = L.V[s]; it.tau = L.tau[s]; it.B = L.B[s]; it.piv = L.piv[s]; it.nu = L.nu[s];
        it.m = m; it.kw = kw; it.kn = kn; it.ldB = ldB; it.level = l; it.cluster = s;
        max_m = std::max(max_m, m);
        if (m == 0) continue;
        double* p; int32_t ld, tr;
        bs.get(s, s, p, ld, tr);
        gather.push_back(CopyItem{p, L.G[s], ld, m, m, m, tr, 0});
        int32_t col = 0;
        for (int pass = 0; pass < 2; ++pass)
          for (int32_t q : (pass == 0 ? lev.w[s] : lev.H[s])) {
            if (live[q] > 0) {
              bs.get(s, q, p, ld, tr);
              gather.push_back(CopyItem{p, L.B[s] + col, ld, ldB, m, live[q], tr, 0});
            }
            col += live[q];
          }
        for (int32_t c0 = 0; c0 < ldB; c0 += 64) trsm.push_back(TrsmItem{bi, c0, std::min(64, ldB - c0), 0});
        S.flops += (double)m * m * m / 3.0 + (double)m * m * ldB;
        S.flops_phase[1] += (double)m * m * m / 3.0;
        S.flops_phase[2] += (double)m * m * ldB;
      }
      upA.reset();
      const size_t iG = upA.add(gather), iC = upA.add(clu), iT = upA.add(trsm);
      upA.stage.ensure(upA.total);
      upA.dev.ensure(upA.total);
      upA.copy_in(iG, gather); upA.copy_in(iC, clu); upA.copy_in(iT, trsm);
      t_plan += now_s() - tp0;
      upA.send(st);
      launch_copy2d(upA.dptr<CopyItem>(iG), (int)gather.size(), st);
      launch_potrf(upA.dptr<CluItem>(iC), nb, max_m, d_status, st);
      launch_trsm(upA.dptr<CluItem>(iC), upA.dptr<TrsmItem>(iT), (int)trsm.size(), max_m, st);
      launch_cpqr(upA.dptr<CluItem>(iC), nb, opt.eps, opt.eps_relative, d_rank, st);
      HS_CUDA(cudaMemcpyAsync(h_rank, d_rank, sizeof(int32_t) * nb, cudaMemcpyDeviceToHost, st));
      check_status(d_status, &h_status, st);       // synchronises the stream
      const double tp1 = now_s();
      // ---- Schur update, write-back, apply plan ----------------------------------------------
      std::unordered_map<uint64_t, std::vector<SchurContrib>> tgt;   // (p<<32|q) -> contributions
      std::vector<uint64_t> tgt_order;
      std::vector<CopyItem> wb;
      std::vector<double*> id_ptr;
      std::vector<int32_t> id_ld, id_r;
      ApplyBatch abt{};
      abt.local_begin = (int32_t)ap.local.size();
      abt.tgt_begin = (int32_t)ap.tgt.size();
      std::unordered_map<int32_t, std::vector<ApplyContrib>> atgt;
      std::vector<int32_t> atgt_order;
      for (int bi = 0; bi < nb; ++bi) {
        const int32_t s = Bt[bi];
        const int32_t m = live[s], kn = L.kn[s], kw = L.kw[s], ldB = L.ldB[s];
        const int32_t r = m == 0 ? 0 : h_rank[bi];
        L.rank[s] = r;
        S.max_m = std::max(S.max_m, m);
        S.max_rank = std::max(S.max_rank, r);
        const int32_t K = m - r;
        const double* C = L.B[s] + (int64_t)r * ldB + kw;
        // algorithmic flops of CPQR (+ rotation of the n-columns) and Schur
        double fq = 0.0;
        for (int j = 0; j < r; ++j) fq += 4.0 * (m - j) * (double)(kw - j) + 4.0 * (m - j) * (double)kn;
        S.flops += fq + (double)K * kn * (kn + 1);
        S.flops_phase[3] += fq;
        S.flops_phase[4] += (double)K * kn * (kn + 1);
        // neighbour column offsets inside the n-part
        const auto& ns = lev.H[s];
        std::vector<int32_t> noff(ns.size() + 1, 0);
        for (size_t a = 0; a < ns.size(); ++a) noff[a + 1] = noff[a] + live[ns[a]];
        if (K > 0)
          for (size_t a = 0; a < ns.size(); ++a) {
            if (live[ns[a]] == 0) continue;
            for (size_t b = 0; b <= a; ++b) {
              if (live[ns[b]] == 0) continue;
              const uint64_t key = ((uint64_t)(uint32_t)ns[a] << 32) | (uint32_t)ns[b];
              auto itn = tgt.find(key);
              if (itn == tgt.end()) {
                tgt_order.push_back(key);
                itn = tgt.emplace(key, std::vector<SchurContrib>{}).first;
              }
              itn->second.push_back(SchurContrib{C, ldB, K, noff[a], noff[b]});
            }
          }
        // write-back of row s: [I_r | coarse-w | coarse-n]
        if (r > 0) {
          double* p; int32_t ld, tr;
          bs.get(s, s, p, ld, tr);
          id_ptr.push_back(p); id_ld.push_back(ld); id_r.push_back(r);
          int32_t col = 0;
          for (int pass = 0; pass < 2; ++pass)
            for (int32_t q : (pass == 0 ? lev.w[s] : lev.H[s])) {
              if (live[q] > 0) {
                bs.get(s, q, p, ld, tr);
                if (!tr) wb.push_back(CopyItem{L.B[s] + col, p, ldB, ld, r, live[q], 0, 0});
                else wb.push_back(CopyItem{L.B[s] + col, p, ldB, ld, live[q], r, 1, 0});
              }
              col += live[q];
            }
        }
        // apply plan: local item (+ backward neighbour list) and forward scatter contributions
        ApplyLocal al{};
        al.G = L.G[s]; al.V = L.V[s]; al.tau = L.tau[s];
        al.y = nullptr;   // patched with the device base after the factor
        al.C = C; al.ldC = ldB; al.m = m; al.r = r;
        al.nb_begin = (int32_t)ap.nb.size();
        for (size_t a = 0; a < ns.size(); ++a) {
          const int32_t q = ns[a];
          if (live[q] == 0 || K == 0) continue;
          ap.nb.push_back(ApplyNb{reinterpret_cast<const double*>((uintptr_t)(L.voff[q])), noff[a], live[q]});
          auto ita = atgt.find(q);
          if (ita == atgt.end()) {
            atgt_order.push_back(q);
            ita = atgt.emplace(q, std::vector<ApplyContrib>{}).first;
          }
          ita->second.push_back(ApplyContrib{C, reinterpret_cast<const double*>((uintptr_t)(L.voff[s] + r)), ldB,
                                             K, noff[a], 0});
        }
        al.nb_end = (int32_t)ap.nb.size();
        al.y = reinterpret_cast<double*>((uintptr_t)L.voff[s]);
        ap.local.push_back(al);
      }
      // Schur tiles (targets in first-touch order, contributions in source order)
      std::vector<SchurTile> tiles;
      std::vector<SchurContrib> cons;
      for (uint64_t key : tgt_order) {
        const int32_t p = (int32_t)(key >> 32), q = (int32_t)(key & 0xffffffffu);
        const auto& cl = tgt[key];
        const int32_t cb = (int32_t)cons.size();
        cons.insert(cons.end(), cl.begin(), cl.end());
        const int32_t ce = (int32_t)cons.size();
        double* base; int32_t ld, tr;
        bs.get(p, q, base, ld, tr);
        if (tr) fail(HS_E_INTERNAL, "schur: transposed target");
        for (int32_t i0 = 0; i0 < live[p]; i0 += 64)
          for (int32_t j0 = 0; j0 < live[q]; j0 += 64) {
            SchurTile t{};
            t.dst = base + (int64_t)i0 * ld + j0;
            t.ld = ld;
            t.rows = std::min(64, live[p] - i0);
            t.cols = std::min(64, live[q] - j0);
            t.c_begin = cb; t.c_end = ce; t.i0 = i0; t.j0 = j0;
            tiles.push_back(t);
          }
      }
      for (int32_t q : atgt_order) {
        const auto& cl = atgt[q];
        ApplyTarget t{};
        t.yq = reinterpret_cast<double*>((uintptr_t)L.voff[q]);
        t.len = live[q];
        t.c_begin = (int32_t)ap.con.size();
        ap.con.insert(ap.con.end(), cl.begin(), cl.end());
        t.c_end = (int32_t)ap.con.size();
        ap.tgt.push_back(t);
      }
      abt.local_end = (int32_t)ap.local.size();
      abt.tgt_end = (int32_t)ap.tgt.size();
      ap.batches[l].push_back(abt);
      for (int bi = 0; bi < nb; ++bi) live[Bt[bi]] = L.rank[Bt[bi]];
      upB.reset();
      const size_t jT = upB.add(tiles), jC = upB.add(cons), jW = upB.add(wb), jP = upB.add(id_ptr),
                   jL = upB.add(id_ld), jR = upB.add(id_r);
      upB.stage.ensure(upB.total);
      upB.dev.ensure(upB.total);
      upB.copy_in(jT, tiles); upB.copy_in(jC, cons); upB.copy_in(jW, wb);
      upB.copy_in(jP, id_ptr); upB.copy_in(jL, id_ld); upB.copy_in(jR, id_r);
      t_plan += now_s() - tp1;
      upB.send(st);
      launch_schur(upB.dptr<SchurTile>(jT), upB.dptr<SchurContrib>(jC), (int)tiles.size(), st);
      launch_copy2d(upB.dptr<CopyItem>(jW), (int)wb.size(), st);
      launch_identity(upB.dptr<double*>(jP), upB.dptr<int32_t>(jL), upB.dptr<int32_t>(jR), (int)id_ptr.size(), st);
      S.n_batches++;
      if (const char* dd = std::getenv("HS_DEBUG_DUMP")) {   // debug aid: block store after every batch
        HS_CUDA(cudaStreamSynchronize(st));
        char path[512];
        std::snprintf(path, sizeof path, "%s/l%d_b%d.bin", dd, l, (int)ap.batches[l].size() - 1);
        FILE* fp = std::fopen(path, "wb");
        if (fp) {
          std::vector<double> host(bs.total);
          if (bs.total) HS_CUDA(cudaMemcpy(host.data(), bs.d, bs.total * sizeof(double), cudaMemcpyDeviceToHost));
          for (int p = 0; p < lev.nclus; ++p)
            for (const auto& qo : bs.rows[p]) {
              const int32_t q = qo.first;
              int32_t hdr[4] = {p, q, live[p], live[q]};
              std::fwrite(hdr, sizeof hdr, 1, fp);
              for (int i = 0; i < live[p]; ++i)
                std::fwrite(host.data() + qo.second + (int64_t)i * cap[q], sizeof(double), live[q], fp);
            }
          std::fclose(fp);
        }
      }
    }
    // ---- end of level: A_c = parents of [coarse(2P); coarse(2P+1)] -----------------
    const double tp2 = now_s();
    const int nP = lev.nclus / 2;
    std::vector<int32_t> capn(nP);
    for (int P = 0; P < nP; ++P) capn[P] = L.rank[2 * P] + L.rank[2 * P + 1];
    const Adj& En = (l + 1 < an->L_top) ? an->levels[l + 1].Ffinal : an->H_top;
    BlockStore nbs;
    nbs.build(capn, En);
    if (nbs.total) HS_CUDA(cudaMemsetAsync(nbs.d, 0, nbs.total * sizeof(double), st));
    std::vector<CopyItem> asmb;
    for (int P = 0; P < nP; ++P)
      for (const auto& qo : nbs.rows[P]) {
        const int32_t Q = qo.first;
        double* dst = nbs.d + qo.second;
        const int32_t dld = capn[Q];
        for (int a = 0; a < 2; ++a)
          for (int b = 0; b < 2; ++b) {
            const int32_t c = 2 * P + a, d = 2 * Q + b;
            if (L.rank[c] == 0 || L.rank[d] == 0 || !bs.has(c, d)) continue;
            double* p; int32_t ld, tr;
            bs.get(c, d, p, ld, tr);
            const int32_t ro = a ? L.rank[2 * P] : 0, co = b ? L.rank[2 * Q] : 0;
            asmb.push_back(CopyItem{p, dst + (int64_t)ro * dld + co, ld, dld, L.rank[c], L.rank[d], tr, 0});
          }
      }
    // forward vector transition (children's coarse entries -> parent segment)
    int64_t pofs = 0;
    for (int P = 0; P < nP; ++P)
      for (int a = 0; a < 2; ++a) {
        const int32_t c = 2 * P + a;
        for (int32_t i = 0; i < L.rank[c]; ++i) {
          ap.trans_src[l].push_back(L.voff[c] + i);
          ap.trans_dst[l].push_back(pofs++);
        }
      }
    upA.reset();
    const size_t iA = upA.add(asmb);
    upA.stage.ensure(upA.total);
    upA.dev.ensure(upA.total);
    upA.copy_in(iA, asmb);
    t_plan += now_s() - tp2;
    upA.send(st);
    launch_copy2d(upA.dptr<CopyItem>(iA), (int)asmb.size(), st);
    HS_CUDA(cudaStreamSynchronize(st));
    bs.release();
    bs = std::move(nbs);
    nbs.d = nullptr;
    cap = capn;
  }
  // ---- top: dense Cholesky of all live DOFs ----------------------------------
  {
    const int ntc = (int)cap.size();
    std::vector<int64_t> toff(ntc + 1, 0);
    for (int c = 0; c < ntc; ++c) toff[c + 1] = toff[c] + cap[c];
    const int64_t N = toff[ntc];
    f->ntop = N;
    f->top_sizes = cap;
    S.n_top = N;
    ap.vbase.push_back(vbase);
    vbase += N;
    if (N > 0) {
      HS_CUDA(cudaMalloc(&f->d_top, sizeof(double) * N * N));
      HS_CUDA(cudaMemsetAsync(f->d_top, 0, sizeof(double) * N * N, st));
      std::vector<CopyItem> items;
      for (int P = 0; P < ntc; ++P)
        for (const auto& qo : bs.rows[P]) {
          const int32_t Q = qo.first;
          if (cap[P] == 0 || cap[Q] == 0) continue;
          double* src = bs.d + qo.second;
          items.push_back(CopyItem{src, f->d_top + toff[P] * N + toff[Q], cap[Q], (int32_t)N, cap[P], cap[Q], 0, 0});
          if (P != Q)
            items.push_back(CopyItem{src, f->d_top + toff[Q] * N + toff[P], cap[Q], (int32_t)N, cap[Q], cap[P], 1, 0});
        }
      upA.reset();
      const size_t iA = upA.add(items);
      upA.stage.ensure(upA.total);
      upA.dev.ensure(upA.total);
      upA.copy_in(iA, items);
      upA.send(st);
      launch_copy2d(upA.dptr<CopyItem>(iA), (int)items.size(), st);
      dense_potrf(f->d_top, (int)N, (int)N, d_status, an->L_top, nullptr, st);
      check_status(d_status, &h_status, st);
      S.flops += (double)N * N * N / 3.0;
      S.flops_phase[6] += (double)N * N * N / 3.0;
    }
    HS_CUDA(cudaStreamSynchronize(st));
    bs.release();
  }
  HS_CUDA(cudaEventRecord(ev1, st));
  HS_CUDA(cudaEventSynchronize(ev1));
  float ms = 0.f;
  HS_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  S.t_factor_s = ms * 1e-3;
  S.t_phase_s[7] = t_plan;
  S.n_levels = an->L_top;
  // factor bytes: G (m^2/2), V (m r), tau, C ((m - r) kn) per cluster + top (N^2/2)
  double fb = 0.0;
  for (const auto& L : f->lv)
    for (int s = 0; s < L.nclus; ++s) {
      const double m = L.cap[s], r = L.rank[s];
      fb += 8.0 * (m * (m + 1) / 2 + m * r + r + (m - r) * L.kn[s]);
    }
  fb += 8.0 * (double)f->ntop * (f->ntop + 1) / 2;
  S.factor_bytes = fb;
  (void)t_wall0;
  // ---- device apply plan ----------------------------------------------------------------
  ap.vtotal = vbase;
  HS_CUDA(cudaMalloc(&ap.d_y, sizeof(double) * std::max<int64_t>(vbase, 1)));
  // patch vector offsets (stored as integers) into absolute addresses
  std::vector<int64_t> lvl_of_local;
  {
    for (int l = 0; l < an->L_top; ++l) {
      double* base = ap.d_y + ap.vbase[l];
      for (const auto& b : ap.batches[l]) {
        for (int32_t i = b.local_begin; i < b.local_end; ++i) {
          ApplyLocal& a = ap.local[i];
          a.y = base + (uintptr_t)a.y;
          for (int32_t k = a.nb_begin; k < a.nb_end; ++k) ap.nb[k].xq = base + (uintptr_t)ap.nb[k].xq;
        }
        for (int32_t t = b.tgt_begin; t < b.tgt_end; ++t) {
          ApplyTarget& tg = ap.tgt[t];
          tg.yq = base + (uintptr_t)tg.yq;
          for (int32_t c = tg.c_begin; c < tg.c_end; ++c) ap.con[c].yf = base + (uintptr_t)ap.con[c].yf;
        }
      }
    }
  }
  auto up = [&](auto& vec, auto*& dptr) {
    using T = typename std::remove_reference<decltype(vec)>::type::value_type;
    if (vec.empty()) return;
    HS_CUDA(cudaMalloc(&dptr, sizeof(T) * vec.size()));
    HS_CUDA(cudaMemcpyAsync(dptr, vec.data(), sizeof(T) * vec.size(), cudaMemcpyHostToDevice, st));
  };
  up(ap.local, ap.d_local);
  up(ap.nb, ap.d_nb);
  up(ap.tgt, ap.d_tgt);
  up(ap.con, ap.d_con);
  ap.d_tsrc.assign(an->L_top, nullptr);
  ap.d_tdst.assign(an->L_top, nullptr);
  for (int l = 0; l < an->L_top; ++l) {
    // absolute indices into d_y: src at level l, dst at level l+1
    for (auto& v : ap.trans_src[l]) v += ap.vbase[l];
    for (auto& v : ap.trans_dst[l]) v += ap.vbase[l + 1];
    up(ap.trans_src[l], ap.d_tsrc[l]);
    up(ap.trans_dst[l], ap.d_tdst[l]);
  }
  HS_CUDA(cudaStreamSynchronize(st));
  return guard.release();
}

}  // namespace hs
