// hs_apply / hs_pcg host drivers.
//
// Apply = Algorithm 2, captured once per factor as a CUDA graph:
//   permute-in, forward sweep (one dependency-driven task kernel per level; coarse parts go
//   straight into the parent level's segments), top solve, backward sweep (reverse),
//   permute-out.
// PCG (north_star) keeps every scalar on the device; the only host
// synchronisation per iteration is the 8-byte read of ||r||^2 for the stopping test.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "runtime.h"

namespace hs {

namespace {

constexpr int RED_BLOCKS = 296;   // 2 x 148 SMs
constexpr int RED_THREADS = 256;

// scalars layout (device): 0 rho, 1 pq, 2 rr, 3 rz_new, 4 bb
__device__ __forceinline__ double blk_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  double r = 0.0;
  if (threadIdx.x < 32) {
    r = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
  }
  return r;
}

// partial[b] = sum over the block's grid-stride slice of a[i]*b[i]
__global__ void k_dot_partial(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                              double* __restrict__ partial) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += a[i] * b[i];
  acc = blk_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}
// out = sum of the partials in fixed order (deterministic)
__global__ void k_finish(const double* __restrict__ partial, int np, double* out) {
  __shared__ double sh[32];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partial[i];
  acc = blk_sum(acc, sh);
  if (threadIdx.x == 0) *out = acc;
}
// x += alpha p ; r -= alpha q ; alpha = rho / pq ; partial ||r||^2
__global__ void k_update_xr(double* __restrict__ x, double* __restrict__ r, const double* __restrict__ p,
                            const double* __restrict__ q, int64_t n, const double* sc, double* __restrict__ partial) {
  __shared__ double sh[32];
  const double alpha = sc[0] / sc[1];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i] += alpha * p[i];
    const double ri = r[i] - alpha * q[i];
    r[i] = ri;
    acc += ri * ri;
  }
  acc = blk_sum(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}
// p = z + (rz_new / rho) p ; rho = rz_new  (the scalar update is done by block 0 after all reads)
__global__ void k_update_p(double* __restrict__ p, const double* __restrict__ z, int64_t n, const double* sc) {
  const double beta = sc[3] / sc[0];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = z[i] + beta * p[i];
}
__global__ void k_set_rho(double* sc) { sc[0] = sc[3]; }
__global__ void k_zero(double* x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = 0.0;
}
__global__ void k_copy(double* __restrict__ d, const double* __restrict__ s, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[i];
}
__global__ void k_sub(double* __restrict__ d, const double* __restrict__ a, const double* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = a[i] - b[i];
}

// ---- GMRES helpers (NEXT f3): V is column-major, column i at V + i*ldv -----------------
// h[i] = <V_i, w> for i < ncol (a block per column, fixed-order reduction)
__global__ void k_gemv_t(const double* __restrict__ V, int64_t ldv, const double* __restrict__ w, int64_t n,
                         double* __restrict__ h) {
  __shared__ double sh[32];
  const double* v = V + (int64_t)blockIdx.x * ldv;
  double acc = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) acc += v[k] * w[k];
  acc = blk_sum(acc, sh);
  if (threadIdx.x == 0) h[blockIdx.x] = acc;
}
// w += sign * V[:, :ncol] h
__global__ void k_gemv_n(const double* __restrict__ V, int64_t ldv, int ncol, const double* __restrict__ h,
                         double sign, double* __restrict__ w, int64_t n) {
  extern __shared__ double hs_[];
  for (int i = threadIdx.x; i < ncol; i += blockDim.x) hs_[i] = h[i];
  __syncthreads();
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int i = 0; i < ncol; ++i) acc += V[(int64_t)i * ldv + k] * hs_[i];
    w[k] += sign * acc;
  }
}
__global__ void k_scale(double* __restrict__ d, const double* __restrict__ s, double a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = a * s[i];
}
__global__ void k_axpy(double* __restrict__ x, const double* __restrict__ z, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] += z[i];
}

void dot(const double* a, const double* b, int64_t n, double* partial, double* out, cudaStream_t st) {
  k_dot_partial<<<RED_BLOCKS, RED_THREADS, 0, st>>>(a, b, n, partial);
  k_finish<<<1, RED_THREADS, 0, st>>>(partial, RED_BLOCKS, out);
  count_launch(2);
}

long long* g_trace = nullptr;   // HS_APPLY_TRACE (profile_apply only)
int g_trace_level = -1;

ApplyLevelArgs level_args(hs_factor_s* f, int l) {
  ApplyPlan& ap = f->ap;
  const ApplyLevelPlan& P = ap.lv[l];
  const int64_t n = (int64_t)P.src.size();
  ApplyLevelArgs a{};
  a.src = P.d_src;
  a.ftask = P.d_ftask;
  a.ftgt = P.d_ftgt;
  a.pull = P.d_pull;
  a.ctb = P.d_ctb;
  a.contrib = ap.d_contrib + P.contrib_off;
  a.post_cl = P.d_post_cl;
  a.npost = (int32_t)P.post_cl.size();
  a.btask = P.d_btask;
  a.bnb = P.d_bnb;
  a.parts = ap.d_parts;
  a.cnt = ap.d_ctr + P.ctr_off;
  a.bcnt = a.cnt + n;
  a.done = a.cnt + 2 * n;
  a.arr = a.cnt + 3 * n;
  a.ticket = a.cnt + 4 * n;
  a.nftask = (int32_t)P.ftask.size();
  a.nbtask = (int32_t)P.btask.size();
  a.trace = l == g_trace_level ? g_trace : nullptr;
  return a;
}

// Algorithm 2: permute-in, forward sweep (one dependency-driven kernel per level), top
// solve, backward sweep (reverse), permute-out.  The event counters start from zero.
void record_apply(hs_factor_s* f, cudaStream_t st, std::vector<cudaEvent_t>* ev = nullptr) {
  const Analysis* an = f->an;
  ApplyPlan& ap = f->ap;
  const int64_t n = an->n;
  auto mark = [&]() {
    if (!ev) return;
    cudaEvent_t e;
    HS_CUDA(cudaEventCreate(&e));
    HS_CUDA(cudaEventRecord(e, st));
    ev->push_back(e);
  };
  mark();
  if (ap.ctr_total) HS_CUDA(cudaMemsetAsync(ap.d_ctr, 0, sizeof(int32_t) * ap.ctr_total, st));
  // forward contribution slots start empty (all-ones NaN, polled by the consumers)
  if (ap.contrib_total) HS_CUDA(cudaMemsetAsync(ap.d_contrib, 0xFF, sizeof(double) * ap.contrib_total, st));
  // backward results start empty too (polled by the neighbours' backward tasks)
  const int64_t vtot = ap.vbase.back() + f->ntop;   // levels + top
  HS_CUDA(cudaMemsetAsync(ap.d_xb, 0xFF, sizeof(double) * std::max<int64_t>(vtot, 1), st));
  launch_permute(f->d_b, ap.d_y + ap.vbase[0], f->d_perm, n, 0, st);
  for (int l = 0; l < an->L_top; ++l) {
    mark();
    const ApplyLevelPlan& P = ap.lv[l];
    if (P.bsync) {
      const ApplyLevelArgs a = level_args(f, l);
      for (size_t b = 0; b + 1 < P.boff.size(); ++b)
        launch_apply_fwd_batch(a, P.d_bcl + P.boff[b], P.boff[b + 1] - P.boff[b], st);
    } else {
      launch_apply_fwd_level(level_args(f, l), st);
    }
    launch_apply_post_level(level_args(f, l), st);
  }
  mark();
  if (f->ntop > 0) {
    launch_top_solve(ap.d_y + ap.vbase[an->L_top], f->d_top, (int)f->ntop, (int)f->ntop, st);
    HS_CUDA(cudaMemcpyAsync(ap.d_xb + ap.vbase[an->L_top], ap.d_y + ap.vbase[an->L_top], sizeof(double) * f->ntop,
                            cudaMemcpyDeviceToDevice, st));
  }
  for (int l = an->L_top - 1; l >= 0; --l) {
    mark();
    // the level's backward partial sums start empty (polled by the finishing chunks)
    const ApplyLevelPlan& P = ap.lv[l];
    if (P.bsync) {
      const ApplyLevelArgs a = level_args(f, l);
      for (size_t b = P.boff.size() - 1; b-- > 0;)
        launch_apply_bwd_batch(a, P.d_bcl + P.boff[b], P.boff[b + 1] - P.boff[b], st);
      continue;
    }
    if (ap.lv[l].parts) HS_CUDA(cudaMemsetAsync(ap.d_parts, 0xFF, sizeof(double) * ap.lv[l].parts, st));
    launch_apply_bwd_level(level_args(f, l), st);
  }
  mark();
  launch_permute(ap.d_xb + ap.vbase[0], f->d_x, f->d_perm, n, 1, st);
  mark();
}

// HS_PROFILE=1: one eager (non-graph) apply with events at every level boundary
void profile_apply(hs_factor_s* f, cudaStream_t st) {
  std::vector<cudaEvent_t> ev;
  record_apply(f, st, &ev);
  HS_CUDA(cudaStreamSynchronize(st));
  const int L = f->an->L_top;
  auto el = [&](int i) {
    float ms;
    HS_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
    return ms;
  };
  std::fprintf(stderr, "[hs profile] apply (eager): permute-in %.3f ms\n", el(0));
  for (int l = 0; l < L; ++l)
    std::fprintf(stderr, "[hs profile]   fwd level %d: %.3f ms (%zu tasks)\n", l, el(1 + l), f->ap.lv[l].ftask.size());
  std::fprintf(stderr, "[hs profile]   top: %.3f ms (N_top %lld)\n", el(1 + L), (long long)f->ntop);
  for (int k = 0; k < L; ++k)
    std::fprintf(stderr, "[hs profile]   bwd level %d: %.3f ms (%zu tasks)\n", L - 1 - k, el(2 + L + k),
                 f->ap.lv[L - 1 - k].btask.size());
  std::fprintf(stderr, "[hs profile]   permute-out %.3f ms\n", el(2 + 2 * L));
  for (auto e : ev) cudaEventDestroy(e);
  if (const char* tl = std::getenv("HS_APPLY_TRACE")) {   // per-task phase stamps of one level
    const int lt = std::atoi(tl);
    if (lt < 0 || lt >= L) return;
    const ApplyLevelPlan& P = f->ap.lv[lt];
    const size_t nt = P.ftask.size() + P.btask.size();
    HS_CUDA(cudaMalloc(&g_trace, sizeof(long long) * 8 * std::max<size_t>(nt, 1)));
    HS_CUDA(cudaMemset(g_trace, 0, sizeof(long long) * 8 * std::max<size_t>(nt, 1)));
    g_trace_level = lt;
    record_apply(f, st);
    HS_CUDA(cudaStreamSynchronize(st));
    std::vector<long long> tr(8 * nt);
    HS_CUDA(cudaMemcpy(tr.data(), g_trace, sizeof(long long) * 8 * nt, cudaMemcpyDeviceToHost));
    cudaFree(g_trace);
    g_trace = nullptr;
    g_trace_level = -1;
    const size_t nf = P.ftask.size();
    // forward T tasks: claim->wait, wait->pull, pull->gemv, gemv->produce, produce->publish
    double acc[5] = {0, 0, 0, 0, 0};
    int nT = 0;
    long long t0 = LLONG_MAX, t1 = 0;
    for (size_t k = 0; k < nf; ++k) {
      const long long* x = &tr[8 * k];
      t0 = std::min(t0, x[0]);
      t1 = std::max(t1, x[5]);
      if (!P.ftask[k].first) continue;
      ++nT;
      for (int j = 0; j < 5; ++j) acc[j] += (double)(x[j + 1] - x[j]);
    }
    std::fprintf(stderr, "[hs trace] fwd level %d: span %.1f us, %d T tasks, mean ns: wait %.0f pull %.0f gemv %.0f "
                 "produce %.0f publish %.0f\n", lt, (t1 - t0) * 1e-3, nT, acc[0] / nT, acc[1] / nT, acc[2] / nT,
                 acc[3] / nT, acc[4] / nT);
    double bacc[3] = {0, 0, 0};
    int nfin = 0;
    long long b0 = LLONG_MAX, b1 = 0;
    for (size_t k = nf; k < nt; ++k) {
      const long long* x = &tr[8 * k];
      b0 = std::min(b0, x[0]);
      b1 = std::max(b1, std::max(x[3], x[2]));
      if (x[1]) bacc[0] += (double)(x[1] - x[0]);
      if (x[2]) bacc[1] += (double)(x[2] - x[1]);
      if (x[3] && x[2]) {
        bacc[2] += (double)(x[3] - x[2]);
        ++nfin;
      }
    }
    const double nb = (double)(nt - nf);
    std::fprintf(stderr, "[hs trace] bwd level %d: span %.1f us, %zu tasks, mean ns: wait %.0f partial %.0f; finish %.0f (%d)\n",
                 lt, (b1 - b0) * 1e-3, nt - nf, bacc[0] / nb, bacc[1] / nb, nfin ? bacc[2] / nfin : 0.0, nfin);
    // the forward chain: consecutive T tasks, gap between a T's publish and the next T's wait exit
    if (std::getenv("HS_APPLY_TRACE_DUMP")) {
      for (size_t k = nf; k < nt; ++k) {
        const long long* x = &tr[8 * k];
        const BwdTask& bt = P.btask[k - nf];
        int nl = 0, lq = -1;
        for (int b = bt.b0; b < bt.b1; ++b)
          if (P.bnb[b].later) {
            ++nl;
            lq = P.bnb[b].q;
          }
        std::fprintf(stderr, "[hs trace] b %zu s %d chunk %d nc %d later %d lastq %d: %lld %lld %lld %lld\n", k - nf, bt.s,
                     bt.chunk, bt.nc, nl, lq, x[0] - b0, x[1] ? x[1] - b0 : -1, x[2] ? x[2] - b0 : -1,
                     x[3] ? x[3] - b0 : -1);
      }
      for (size_t k = 0; k < nf; ++k) {
        const long long* x = &tr[8 * k];
        std::fprintf(stderr, "[hs trace] f %zu s %d first %d: %lld %lld %lld %lld %lld %lld\n", k, P.ftask[k].s,
                     P.ftask[k].first, x[0] - t0, x[1] - t0, x[2] - t0, x[3] - t0, x[4] - t0, x[5] - t0);
      }
    }
  }
}

void ensure_vectors(hs_factor_s* f) {
  const int64_t n = f->an->n;
  if (f->d_b) return;
  for (double** p : {&f->d_r, &f->d_z, &f->d_p, &f->d_q, &f->d_x, &f->d_b})
    *p = (double*)f->h->cache.alloc(sizeof(double) * std::max<int64_t>(n, 1));
  f->d_red = (double*)f->h->cache.alloc(sizeof(double) * (RED_BLOCKS + 16));
  HS_CUDA(cudaMallocHost(&f->h_red, sizeof(double) * 16));
}

// graph: d_b -> M^{-1} d_b -> d_x
void run_apply_graph(hs_factor_s* f, cudaStream_t st) {
  ApplyPlan& ap = f->ap;
  if (!ap.graph) {
    cudaStream_t cs;
    HS_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t g;
    const int64_t c0 = launch_count();
    HS_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    record_apply(f, cs);
    HS_CUDA(cudaStreamEndCapture(cs, &g));
    ap.graph_kernels = launch_count() - c0;   // captured, not launched
    count_launch(-ap.graph_kernels);
    HS_CUDA(cudaGraphInstantiate(&ap.graph, g, 0));
    cudaGraphDestroy(g);
    cudaStreamDestroy(cs);
  }
  HS_CUDA(cudaGraphLaunch(ap.graph, st));
  count_launch(ap.graph_kernels);
}

}  // namespace

void apply(hs_factor_s* f, const double* d_b, double* d_x) {
  cudaStream_t st = f->h->stream;
  ensure_vectors(f);
  const int64_t n = f->an->n;
  if (d_b != f->d_b) HS_CUDA(cudaMemcpyAsync(f->d_b, d_b, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  if (std::getenv("HS_PROFILE")) profile_apply(f, st);
  run_apply_graph(f, st);
  if (d_x != f->d_x) HS_CUDA(cudaMemcpyAsync(d_x, f->d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
}

void spmv(hs_factor_s* f, const double* d_x, double* d_y) {
  launch_spmv(f->d_rowptr, f->d_colind, f->d_vals, d_x, d_y, f->an->n, f->h->stream);
}

void pcg(hs_factor_s* f, const double* d_bin, double* d_xout, double tol, int maxit, hs_pcg_report* rep) {
  cudaStream_t st = f->h->stream;
  ensure_vectors(f);
  const int64_t n = f->an->n;
  const int G = RED_BLOCKS, T = RED_THREADS;
  double* sc = f->d_red + RED_BLOCKS;   // scalars
  double* part = f->d_red;
  // The apply graph reads d_b (= r) and writes d_x (= z); PCG keeps its own x in d_q's partner.
  double* r = f->d_b;
  double* z = f->d_x;
  double *x = f->d_r, *p = f->d_p, *q = f->d_q;
  cudaEvent_t e0, e1, a0, a1;
  HS_CUDA(cudaEventCreate(&e0)); HS_CUDA(cudaEventCreate(&e1));
  HS_CUDA(cudaEventCreate(&a0)); HS_CUDA(cudaEventCreate(&a1));
  double t_apply = 0.0, t_spmv = 0.0;
  cudaEvent_t s0, s1;
  HS_CUDA(cudaEventCreate(&s0)); HS_CUDA(cudaEventCreate(&s1));
  rep->history_len = 0;
  auto hist = [&](double v) {
    if (rep->history && rep->history_len < rep->history_cap) rep->history[rep->history_len++] = v;
  };
  HS_CUDA(cudaEventRecord(e0, st));
  k_copy<<<G, T, 0, st>>>(r, d_bin, n);
  k_zero<<<G, T, 0, st>>>(x, n);
  dot(r, r, n, part, sc + 4, st);                       // bb
  HS_CUDA(cudaEventRecord(a0, st));
  run_apply_graph(f, st);                               // z = M^{-1} r
  HS_CUDA(cudaEventRecord(a1, st));
  k_copy<<<G, T, 0, st>>>(p, z, n);
  count_launch(3);   // the two copies and the zero
  dot(r, z, n, part, sc + 0, st);                       // rho
  HS_CUDA(cudaMemcpyAsync(f->h_red, sc, sizeof(double) * 5, cudaMemcpyDeviceToHost, st));
  HS_CUDA(cudaStreamSynchronize(st));
  {
    float ms;
    HS_CUDA(cudaEventElapsedTime(&ms, a0, a1));
    t_apply += ms * 1e-3;
  }
  const double bb = f->h_red[4];
  rep->iters = 0;
  rep->converged = 0;
  rep->relres = 1.0;
  hist(bb == 0.0 ? 0.0 : 1.0);
  hs_status err = HS_OK;
  if (bb == 0.0) {
    rep->converged = 1;
    rep->relres = 0.0;
  } else if (!(f->h_red[0] > 0.0)) {
    err = HS_E_PRECOND_NOT_POSITIVE;
  } else {
    const double nb = std::sqrt(bb);
    for (int k = 1; k <= maxit; ++k) {
      HS_CUDA(cudaEventRecord(s0, st));
      launch_spmv(f->d_rowptr, f->d_colind, f->d_vals, p, q, n, st);   // q = A p
      HS_CUDA(cudaEventRecord(s1, st));
      dot(p, q, n, part, sc + 1, st);                                  // pq
      k_update_xr<<<G, T, 0, st>>>(x, r, p, q, n, sc, part);           // x, r, ||r||^2
      k_finish<<<1, T, 0, st>>>(part, G, sc + 2);
      count_launch(2);
      HS_CUDA(cudaMemcpyAsync(f->h_red, sc, sizeof(double) * 3, cudaMemcpyDeviceToHost, st));
      HS_CUDA(cudaStreamSynchronize(st));
      rep->iters = k;
      const double rel = std::sqrt(std::max(f->h_red[2], 0.0)) / nb;
      rep->relres = rel;
      hist(rel);
      {
        float sms;
        HS_CUDA(cudaEventElapsedTime(&sms, s0, s1));
        t_spmv += sms * 1e-3;
      }
      if (!(f->h_red[0] > 0.0)) { err = HS_E_PRECOND_NOT_POSITIVE; break; }
      if (rel <= tol) { rep->converged = 1; break; }
      HS_CUDA(cudaEventRecord(a0, st));
      run_apply_graph(f, st);                                          // z = M^{-1} r
      HS_CUDA(cudaEventRecord(a1, st));
      dot(r, z, n, part, sc + 3, st);                                  // rz_new
      k_update_p<<<G, T, 0, st>>>(p, z, n, sc);
      k_set_rho<<<1, 1, 0, st>>>(sc);
      count_launch(2);
      HS_CUDA(cudaEventSynchronize(a1));
      float ms;
      HS_CUDA(cudaEventElapsedTime(&ms, a0, a1));
      t_apply += ms * 1e-3;
    }
  }
  HS_CUDA(cudaEventRecord(e1, st));
  HS_CUDA(cudaEventSynchronize(e1));
  float ms;
  HS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  rep->t_pcg_s = ms * 1e-3;
  rep->t_apply_s = t_apply;
  rep->t_spmv_s = t_spmv;
  cudaEventDestroy(s0);
  cudaEventDestroy(s1);
  // true residual ||b - A x|| / ||b|| (outside the timed region)
  launch_spmv(f->d_rowptr, f->d_colind, f->d_vals, x, q, n, st);
  k_sub<<<G, T, 0, st>>>(q, d_bin, q, n);
  count_launch(1);
  dot(q, q, n, part, sc + 2, st);
  HS_CUDA(cudaMemcpyAsync(f->h_red, sc, sizeof(double) * 5, cudaMemcpyDeviceToHost, st));
  if (d_xout != x) HS_CUDA(cudaMemcpyAsync(d_xout, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  HS_CUDA(cudaStreamSynchronize(st));
  rep->relres_true = bb > 0 ? std::sqrt(std::max(f->h_red[2], 0.0) / bb) : 0.0;
  cudaEventDestroy(e0); cudaEventDestroy(e1); cudaEventDestroy(a0); cudaEventDestroy(a1);
  if (err != HS_OK) fail(err, "pcg: <r, M^{-1} r> <= 0 (preconditioner not positive)");
  if (!rep->converged) fail(HS_E_NOT_CONVERGED, "pcg: not converged within maxit");
}

// Right-preconditioned restarted GMRES (NEXT f3; the paper's protocol: GMRES(200),
// tol 1e-12, maxit 1000): x0 = 0, A M^{-1} u = b, x = M^{-1} u.  Arnoldi with classical
// Gram-Schmidt applied twice (CGS2: two block projections per step instead of j dependent
// dot products); the Hessenberg column, the Givens rotations and the small triangular
// solve live on the host (one read of j+2 scalars per step).  Iterations = Arnoldi steps.
void gmres(hs_factor_s* f, const double* d_bin, double* d_xout, double tol, int restart, int maxit,
           hs_pcg_report* rep) {
  cudaStream_t st = f->h->stream;
  ensure_vectors(f);
  const int64_t n = f->an->n;
  const int G = RED_BLOCKS, T = RED_THREADS;
  if (restart < 1) fail(HS_E_INVALID_ARG, "gmres: restart must be >= 1");
  DevCache& dc = f->h->cache;
  const int64_t ldv = (n + 31) & ~int64_t(31);
  double* V = (double*)dc.alloc(sizeof(double) * ldv * (restart + 1));
  double* x = (double*)dc.alloc(sizeof(double) * n);
  double* w = (double*)dc.alloc(sizeof(double) * n);
  double* dh = (double*)dc.alloc(sizeof(double) * (2 * (restart + 1) + 8));
  std::vector<double> hh(2 * (restart + 1) + 8);
  double* part = f->d_red;
  double* sc = f->d_red + RED_BLOCKS;
  cudaEvent_t e0, e1;
  HS_CUDA(cudaEventCreate(&e0));
  HS_CUDA(cudaEventCreate(&e1));
  HS_CUDA(cudaEventRecord(e0, st));
  auto norm2 = [&](const double* a) {   // blocking ||a||
    dot(a, a, n, part, sc, st);
    HS_CUDA(cudaMemcpyAsync(f->h_red, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    return std::sqrt(std::max(f->h_red[0], 0.0));
  };
  auto apply_to = [&](const double* v, double* out) {   // out = M^{-1} v
    HS_CUDA(cudaMemcpyAsync(f->d_b, v, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    run_apply_graph(f, st);
    if (out != f->d_x) HS_CUDA(cudaMemcpyAsync(out, f->d_x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  };
  const size_t hsm = sizeof(double) * (restart + 1);
  k_zero<<<G, T, 0, st>>>(x, n);
  count_launch(1);
  const double nb = norm2(d_bin);
  int its = 0;
  double rel = 1.0;
  rep->history_len = 0;
  rep->iters = 0;
  rep->converged = 0;
  if (nb == 0.0) rel = 0.0;
  while (nb > 0.0) {
    // r = b - A x into V_0
    launch_spmv(f->d_rowptr, f->d_colind, f->d_vals, x, w, n, st);
    k_sub<<<G, T, 0, st>>>(w, d_bin, w, n);
    count_launch(1);
    const double beta = norm2(w);
    rel = beta / nb;
    if (rel <= tol || its >= maxit || beta == 0.0) break;
    k_scale<<<G, T, 0, st>>>(V, w, 1.0 / beta, n);
    count_launch(1);
    std::vector<double> H((size_t)(restart + 1) * restart, 0.0), g(restart + 1, 0.0), cs(restart), sn(restart);
    auto Hij = [&](int i, int j) -> double& { return H[(size_t)i * restart + j]; };
    g[0] = beta;
    int k = 0;
    for (int j = 0; j < restart; ++j) {
      ++its;
      apply_to(V + (int64_t)j * ldv, f->d_x);                              // z = M^{-1} v_j
      launch_spmv(f->d_rowptr, f->d_colind, f->d_vals, f->d_x, w, n, st);   // w = A z
      for (int pass = 0; pass < 2; ++pass) {                                // CGS2
        k_gemv_t<<<j + 1, T, 0, st>>>(V, ldv, w, n, dh + pass * (restart + 1));
        k_gemv_n<<<G, T, hsm, st>>>(V, ldv, j + 1, dh + pass * (restart + 1), -1.0, w, n);
        count_launch(2);
      }
      dot(w, w, n, part, dh + 2 * (restart + 1), st);
      HS_CUDA(cudaMemcpyAsync(hh.data(), dh, sizeof(double) * (2 * (restart + 1) + 1), cudaMemcpyDeviceToHost, st));
      HS_CUDA(cudaStreamSynchronize(st));
      for (int i = 0; i <= j; ++i) Hij(i, j) = hh[i] + hh[restart + 1 + i];
      const double hn = std::sqrt(std::max(hh[2 * (restart + 1)], 0.0));
      Hij(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {   // previous rotations
        const double t = cs[i] * Hij(i, j) + sn[i] * Hij(i + 1, j);
        Hij(i + 1, j) = -sn[i] * Hij(i, j) + cs[i] * Hij(i + 1, j);
        Hij(i, j) = t;
      }
      const double den = std::hypot(Hij(j, j), Hij(j + 1, j));
      cs[j] = den == 0.0 ? 1.0 : Hij(j, j) / den;
      sn[j] = den == 0.0 ? 0.0 : Hij(j + 1, j) / den;
      Hij(j, j) = den;
      Hij(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      k = j + 1;
      rel = std::fabs(g[j + 1]) / nb;
      if (rel <= tol || its >= maxit || hn == 0.0) break;
      k_scale<<<G, T, 0, st>>>(V + (int64_t)(j + 1) * ldv, w, 1.0 / hn, n);
      count_launch(1);
    }
    // y = H(0:k, 0:k)^{-1} g(0:k); x += M^{-1} V y
    std::vector<double> y(k);
    for (int i = k - 1; i >= 0; --i) {
      double t = g[i];
      for (int c = i + 1; c < k; ++c) t -= Hij(i, c) * y[c];
      y[i] = t / Hij(i, i);
    }
    HS_CUDA(cudaMemcpyAsync(dh, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
    k_zero<<<G, T, 0, st>>>(w, n);
    k_gemv_n<<<G, T, hsm, st>>>(V, ldv, k, dh, 1.0, w, n);
    count_launch(2);
    apply_to(w, f->d_x);
    k_axpy<<<G, T, 0, st>>>(x, f->d_x, n);
    count_launch(1);
    HS_CUDA(cudaStreamSynchronize(st));   // y (pageable) consumed; dh reusable
    if (rel <= tol || its >= maxit) break;
  }
  HS_CUDA(cudaEventRecord(e1, st));
  HS_CUDA(cudaEventSynchronize(e1));
  float ms;
  HS_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  rep->t_pcg_s = ms * 1e-3;
  rep->t_apply_s = 0.0;
  rep->t_spmv_s = 0.0;
  rep->iters = its;
  rep->relres = rel;
  rep->converged = rel <= tol ? 1 : 0;
  // true residual
  launch_spmv(f->d_rowptr, f->d_colind, f->d_vals, x, w, n, st);
  k_sub<<<G, T, 0, st>>>(w, d_bin, w, n);
  count_launch(1);
  const double rn = norm2(w);
  rep->relres_true = nb > 0 ? rn / nb : 0.0;
  HS_CUDA(cudaMemcpyAsync(d_xout, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  HS_CUDA(cudaStreamSynchronize(st));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  for (void* p : {(void*)V, (void*)x, (void*)w, (void*)dh}) dc.free(p);
  if (!rep->converged) fail(HS_E_NOT_CONVERGED, "gmres: not converged within maxit");
}

}  // namespace hs
