// extern "C" entry points of libhsolve (include/hsolve.h).  Every call translates
// internal exceptions into hs_status; nothing throws across the ABI.
#include <cuda_runtime.h>

#include <mutex>
#include <string>

#include "runtime.h"

namespace {
std::mutex g_mu;
std::string g_err;   // last error when no handle is available

void set_err(hs_handle h, const std::string& m) {
  if (h) h->err = m;
  std::lock_guard<std::mutex> lk(g_mu);
  g_err = m;
}

template <class F>
hs_status guarded(hs_handle h, F&& fn) {
  try {
    fn();
    return HS_OK;
  } catch (const hs::Error& e) {
    set_err(h, e.what());
    return e.status;
  } catch (const std::bad_alloc&) {
    set_err(h, "host out of memory");
    return HS_E_OOM;
  } catch (const std::exception& e) {
    set_err(h, e.what());
    return HS_E_INTERNAL;
  } catch (...) {
    set_err(h, "unknown error");
    return HS_E_INTERNAL;
  }
}

void require_device(hs_handle h) {
  if (!h) hs::fail(HS_E_INVALID_ARG, "NULL handle");
  HS_CUDA(cudaSetDevice(h->device));
}

template <class T>
void export_vec(const std::vector<T>& v, int64_t* out, int64_t cap, int64_t* len) {
  if (len) *len = (int64_t)v.size();
  if (out)
    for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)v.size()); ++i) out[i] = (int64_t)v[i];
}
void export_adj(const hs::Adj& a, bool ptr, int64_t* out, int64_t cap, int64_t* len) {
  std::vector<int64_t> v;
  if (ptr) {
    v.push_back(0);
    for (const auto& r : a) v.push_back(v.back() + (int64_t)r.size());
  } else {
    for (const auto& r : a) v.insert(v.end(), r.begin(), r.end());
  }
  export_vec(v, out, cap, len);
}
}  // namespace

extern "C" {

const char* hs_status_string(hs_status s) {
  switch (s) {
    case HS_OK: return "HS_OK";
    case HS_E_INVALID_ARG: return "HS_E_INVALID_ARG";
    case HS_E_DIM: return "HS_E_DIM";
    case HS_E_NOT_SYMMETRIC: return "HS_E_NOT_SYMMETRIC";
    case HS_E_NOT_SPD: return "HS_E_NOT_SPD";
    case HS_E_COLUMN_SPLIT: return "HS_E_COLUMN_SPLIT";
    case HS_E_PRECOND_NOT_POSITIVE: return "HS_E_PRECOND_NOT_POSITIVE";
    case HS_E_NOT_CONVERGED: return "HS_E_NOT_CONVERGED";
    case HS_E_OOM: return "HS_E_OOM";
    case HS_E_CUDA: return "HS_E_CUDA";
    case HS_E_NCCL: return "HS_E_NCCL";
    case HS_E_NO_DEVICE: return "HS_E_NO_DEVICE";
    case HS_E_UNSUPPORTED: return "HS_E_UNSUPPORTED";
    case HS_E_INTERNAL: return "HS_E_INTERNAL";
  }
  return "HS_E_?";
}

const char* hs_last_error(hs_handle h) {
  if (h) return h->err.c_str();
  std::lock_guard<std::mutex> lk(g_mu);
  return g_err.c_str();
}

static hs_status create_impl(hs_handle* out, int device, int world_size, int rank, const void* nccl_unique_id,
                             void* loopback);

hs_status hs_create(hs_handle* out, int device, int world_size, int rank, const void* nccl_unique_id) {
  return create_impl(out, device, world_size, rank, nccl_unique_id, nullptr);
}

hs_status hs_loopback_world_create(int32_t world, void** out) {
  return guarded(nullptr, [&] {
    if (!out || world < 2) hs::fail(HS_E_INVALID_ARG, "hs_loopback_world_create: need world >= 2");
    *out = hs::loop_world_create(world);
  });
}

void hs_loopback_world_destroy(void* w) {
  if (w) hs::loop_world_destroy((hs::LoopWorld*)w);
}

hs_status hs_create_loopback(hs_handle* out, int device, void* world, int32_t rank) {
  if (!world) return HS_E_INVALID_ARG;
  return create_impl(out, device, hs::loop_world_size((hs::LoopWorld*)world), rank, nullptr, world);
}

static hs_status create_impl(hs_handle* out, int device, int world_size, int rank, const void* nccl_unique_id,
                             void* loopback) {
  return guarded(nullptr, [&] {
    if (!out) hs::fail(HS_E_INVALID_ARG, "hs_create: NULL out");
    *out = nullptr;
    if (world_size < 1 || rank < 0 || rank >= world_size) hs::fail(HS_E_INVALID_ARG, "hs_create: bad world/rank");
    if (world_size > 1 && !nccl_unique_id && !loopback)
      hs::fail(HS_E_INVALID_ARG, "hs_create: world_size > 1 needs an NCCL id");
    int nd = 0;
    if (cudaGetDeviceCount(&nd) != cudaSuccess || nd == 0) {
      cudaGetLastError();
      hs::fail(HS_E_NO_DEVICE, "hs_create: no CUDA device (there is no CPU fallback)");
    }
    if (device < 0 || device >= nd) hs::fail(HS_E_INVALID_ARG, "hs_create: bad device ordinal");
    auto* h = new hs_handle_s();
    h->device = device;
    HS_CUDA(cudaSetDevice(device));
    HS_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
    HS_CUDA(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    HS_CUDA(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
    HS_CUDA(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
    h->upA.dev.dc = &h->cache;
    h->upB.dev.dc = &h->cache;
    h->upC.dev.dc = &h->cache;
    h->world = world_size;
    h->rank = rank;
    if (world_size > 1 && loopback) {
      h->comm = hs::comm_loopback((hs::LoopWorld*)loopback, rank);
    } else if (world_size > 1) {
      try {
        h->comm = hs::comm_init(world_size, rank, nccl_unique_id);
      } catch (...) {
        cudaStreamDestroy(h->stream);
        cudaStreamDestroy(h->side);
        delete h;
        throw;
      }
    }
    *out = h;
  });
}

hs_status hs_nccl_unique_id(void* out128) {
  return guarded(nullptr, [&] {
    if (!out128) hs::fail(HS_E_INVALID_ARG, "hs_nccl_unique_id: NULL out");
    hs::nccl_unique_id(out128);
  });
}

hs_status hs_set_stream(hs_handle h, void* stream) {
  return guarded(h, [&] {
    require_device(h);
    // cached memory is reused in host order, which is only stream-ordered on one stream:
    // drain the old stream before switching
    if (h->stream) HS_CUDA(cudaStreamSynchronize(h->stream));
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    if (stream) {
      h->stream = (cudaStream_t)stream;
      h->own_stream = false;
    } else {
      HS_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
      h->own_stream = true;
    }
  });
}

void hs_destroy(hs_handle h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  // release the staging buffers while their stream is still alive (stream-ordered frees)
  for (hs::Upload* u : {&h->upA, &h->upB, &h->upC}) {
    if (u->dev.d) h->cache.free(u->dev.d);
    u->dev.d = nullptr;
    u->dev.cap = 0;
  }
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (h->side) cudaStreamSynchronize(h->side);
  if (h->h_rank) cudaFreeHost(h->h_rank);
  if (h->pub) cudaFreeHost(h->pub);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  h->cache.trim();
  if (h->comm) hs::comm_destroy(h->comm);
  delete h;
}

hs_status hs_analyze(hs_handle h, int64_t n, const int64_t* rowptr, const int32_t* colind, const double* coords,
                     int32_t coord_dim, const int32_t* column_id, const hs_analyze_opts* opt, hs_analysis* out) {
  return guarded(h, [&] {
    if (!out || !opt) hs::fail(HS_E_INVALID_ARG, "hs_analyze: NULL argument");
    *out = nullptr;
    auto* a = new hs_analysis_s();
    try {
      a->an = hs::analyze(n, rowptr, colind, coords, coord_dim, column_id, *opt);
    } catch (...) {
      delete a;
      throw;
    }
    *out = a;
  });
}

hs_status hs_analysis_get_info(hs_analysis a, hs_analysis_info* info) {
  return guarded(nullptr, [&] {
    if (!a || !a->an || !info) hs::fail(HS_E_INVALID_ARG, "hs_analysis_get_info: NULL argument");
    info->n = a->an->n;
    info->depth = a->an->D;
    info->L_top = a->an->L_top;
    info->nsub_log2 = a->an->nsub_log2;
    info->top_log2 = a->an->top_log2;
  });
}

hs_status hs_analysis_export(hs_analysis a, int32_t key, int32_t level, int64_t* out, int64_t cap, int64_t* len) {
  return guarded(nullptr, [&] {
    if (!a || !a->an) hs::fail(HS_E_INVALID_ARG, "hs_analysis_export: NULL analysis");
    const hs::Analysis& an = *a->an;
    auto lev = [&]() -> const hs::Level& {
      if (level < 0 || level >= an.L_top) hs::fail(HS_E_INVALID_ARG, "hs_analysis_export: bad level");
      return an.levels[level];
    };
    switch (key) {
      case HS_EXP_PERM: export_vec(an.perm, out, cap, len); break;
      case HS_EXP_LEAF_OFF: export_vec(an.leaf_off, out, cap, len); break;
      case HS_EXP_H_PTR: export_adj(lev().H, true, out, cap, len); break;
      case HS_EXP_H_IDX: export_adj(lev().H, false, out, cap, len); break;
      case HS_EXP_W_PTR: export_adj(lev().w, true, out, cap, len); break;
      case HS_EXP_W_IDX: export_adj(lev().w, false, out, cap, len); break;
      case HS_EXP_BATCH_PTR: export_adj(lev().batches, true, out, cap, len); break;
      case HS_EXP_BATCH_IDX: export_adj(lev().batches, false, out, cap, len); break;
      case HS_EXP_INTERIOR: export_vec(lev().interior, out, cap, len); break;
      case HS_EXP_F_PTR: export_adj(lev().Ffinal, true, out, cap, len); break;
      case HS_EXP_F_IDX: export_adj(lev().Ffinal, false, out, cap, len); break;
      case HS_EXP_NPHASE1: export_vec(std::vector<int64_t>{lev().nphase1}, out, cap, len); break;
      case HS_EXP_HTOP_PTR: export_adj(an.H_top, true, out, cap, len); break;
      case HS_EXP_HTOP_IDX: export_adj(an.H_top, false, out, cap, len); break;
      case HS_EXP_FS_PTR: export_adj(lev().Fstart, true, out, cap, len); break;
      case HS_EXP_FS_IDX: export_adj(lev().Fstart, false, out, cap, len); break;
      default: hs::fail(HS_E_INVALID_ARG, "hs_analysis_export: bad key");
    }
  });
}

hs_status hs_dist_plan_export(hs_analysis a, int32_t world, int32_t rank, int32_t key, int32_t level, int64_t* out,
                              int64_t cap, int64_t* len) {
  return guarded(nullptr, [&] {
    if (!a || !a->an) hs::fail(HS_E_INVALID_ARG, "hs_dist_plan_export: NULL analysis");
    const hs::Analysis& an = *a->an;
    const hs::DistPlan P = hs::make_plan(an, world, rank);
    if (level < 0 || level > an.L_top || (key != HS_DEXP_OWNER && level >= an.L_top))
      hs::fail(HS_E_INVALID_ARG, "hs_dist_plan_export: bad level");
    std::vector<int64_t> v;
    switch (key) {
      case HS_DEXP_OWNER: v.assign(P.owner[level].begin(), P.owner[level].end()); break;
      case HS_DEXP_RECV_PTR:
      case HS_DEXP_RECV: {
        const hs::Level& lev = an.levels[level];
        std::vector<int64_t> ptr(1, 0), idx;
        std::vector<uint8_t> phase2(lev.nclus, 0);
        for (size_t b = lev.nphase1; b < lev.batches.size(); ++b)
          for (int32_t s : lev.batches[b]) phase2[s] = 1;
        for (int s = 0; s < lev.nclus; ++s) {
          if (phase2[s])
            for (int32_t h : hs::receivers(an, P, level, s)) idx.push_back(h);
          ptr.push_back((int64_t)idx.size());
        }
        v = key == HS_DEXP_RECV_PTR ? ptr : idx;
        break;
      }
      case HS_DEXP_HELD_PTR:
      case HS_DEXP_HELD: {
        const hs::Level& lev = an.levels[level];
        std::vector<int64_t> ptr(1, 0), idx;
        for (int p = 0; p < lev.nclus; ++p) {
          for (int32_t q : lev.Ffinal[p])
            if (q < p && P.holds(level, p, q)) idx.push_back(q);
          if (P.holds(level, p, p)) idx.push_back(p);
          ptr.push_back((int64_t)idx.size());
        }
        v = key == HS_DEXP_HELD_PTR ? ptr : idx;
        break;
      }
      default: hs::fail(HS_E_INVALID_ARG, "hs_dist_plan_export: bad key");
    }
    if (len) *len = (int64_t)v.size();
    if (out)
      for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)v.size()); ++i) out[i] = v[i];
  });
}

void hs_analysis_destroy(hs_analysis a) {
  if (!a) return;
  if (a->an && a->an->dev >= 0) {
    cudaSetDevice(a->an->dev);
    for (void* p : {(void*)a->an->d_rowptr, (void*)a->an->d_colind, (void*)a->an->d_perm, (void*)a->an->d_map,
                    (void*)a->an->d_tmap})
      if (p) cudaFree(p);
  }
  if (a->an && a->an->maps_pinned) {
    cudaHostUnregister(a->an->h_map.data());
    cudaHostUnregister(a->an->h_tmap.data());
  }
  if (a->an && a->an->l0s.d_idx) {
    cudaSetDevice(a->an->l0s.dev);
    cudaFree(a->an->l0s.d_idx);
  }
  delete a->an;
  delete a;
}

hs_status hs_factor_create(hs_handle h, hs_analysis a, const double* values, const hs_factor_opts* opt,
                           hs_factor* out) {
  return guarded(h, [&] {
    if (!out) hs::fail(HS_E_INVALID_ARG, "hs_factor_create: NULL out");
    *out = nullptr;
    if (!a || !a->an || !values || !opt) hs::fail(HS_E_INVALID_ARG, "hs_factor_create: NULL argument");
    require_device(h);
    *out = hs::factor_create(h, a->an, values, *opt);
  });
}

hs_status hs_factor_get_stats(hs_factor f, hs_factor_stats_t* st) {
  return guarded(f ? f->h : nullptr, [&] {
    if (!f || !st) hs::fail(HS_E_INVALID_ARG, "hs_factor_get_stats: NULL argument");
    *st = f->stats;
  });
}

hs_status hs_factor_export(hs_factor f, int32_t key, int32_t level, int64_t* out, int64_t cap, int64_t* len) {
  return guarded(f ? f->h : nullptr, [&] {
    if (!f) hs::fail(HS_E_INVALID_ARG, "hs_factor_export: NULL factor");
    if (key == HS_FEXP_TOP) {
      export_vec(f->top_sizes, out, cap, len);
      return;
    }
    if (level < 0 || level >= (int)f->lv.size()) hs::fail(HS_E_INVALID_ARG, "hs_factor_export: bad level");
    const hs::LevelRT& L = f->lv[level];
    switch (key) {
      case HS_FEXP_RANKS: export_vec(L.rank, out, cap, len); break;
      case HS_FEXP_LIVE0: export_vec(L.cap, out, cap, len); break;
      case HS_FEXP_KN: export_vec(L.kn, out, cap, len); break;
      case HS_FEXP_KW: export_vec(L.kw, out, cap, len); break;
      case HS_FEXP_PIV_PTR: {
        std::vector<int64_t> p(L.nclus + 1, 0);
        for (int s = 0; s < L.nclus; ++s) p[s + 1] = p[s] + L.rank[s];
        export_vec(p, out, cap, len);
        break;
      }
      case HS_FEXP_PIV: {
        require_device(f->h);
        std::vector<int64_t> v;
        for (int s = 0; s < L.nclus; ++s) {
          std::vector<int32_t> tmp(L.rank[s]);
          if (L.rank[s] && !L.piv[s])
            hs::fail(HS_E_UNSUPPORTED, "hs_factor_export: pivots of clusters eliminated on another rank stay there");
          if (L.rank[s])
            HS_CUDA(cudaMemcpy(tmp.data(), L.piv[s], sizeof(int32_t) * L.rank[s], cudaMemcpyDeviceToHost));
          v.insert(v.end(), tmp.begin(), tmp.end());
        }
        export_vec(v, out, cap, len);
        break;
      }
      default: hs::fail(HS_E_INVALID_ARG, "hs_factor_export: bad key");
    }
  });
}

hs_status hs_factor_export_cluster(hs_factor f, int32_t key, int32_t level, int32_t cluster, double* out,
                                   int64_t cap, int64_t* len) {
  return guarded(f ? f->h : nullptr, [&] {
    if (!f) hs::fail(HS_E_INVALID_ARG, "hs_factor_export_cluster: NULL factor");
    if (level < 0 || level >= (int)f->lv.size()) hs::fail(HS_E_INVALID_ARG, "hs_factor_export_cluster: bad level");
    const hs::LevelRT& L = f->lv[level];
    if (cluster < 0 || cluster >= L.nclus) hs::fail(HS_E_INVALID_ARG, "hs_factor_export_cluster: bad cluster");
    const int64_t m = L.cap[cluster], r = L.rank[cluster];
    std::vector<double> v;
    auto dev = [&](const double* p, int64_t cnt) {
      v.resize(cnt);
      if (cnt) HS_CUDA(cudaMemcpy(v.data(), p, sizeof(double) * cnt, cudaMemcpyDeviceToHost));
    };
    require_device(f->h);
    HS_CUDA(cudaStreamSynchronize(f->h->stream));
    if (key != HS_CEXP_SHAPE && m > 0 && !L.G[cluster])
      hs::fail(HS_E_UNSUPPORTED, "hs_factor_export_cluster: per-cluster records are freed after each batch; "
                                 "factor with HS_KEEP_RECORDS=1 in the environment to keep them");
    switch (key) {
      case HS_CEXP_SHAPE:
        v = {(double)m, (double)r, (double)L.kw[cluster], (double)L.kn[cluster], (double)L.ldB[cluster]};
        break;
      case HS_CEXP_G: dev(L.G[cluster], m * m); break;
      case HS_CEXP_V: dev(L.V[cluster], r * m); break;
      case HS_CEXP_TAU: dev(L.tau[cluster], r); break;
      case HS_CEXP_B: dev(L.B[cluster], m * L.ldB[cluster]); break;
      default: hs::fail(HS_E_INVALID_ARG, "hs_factor_export_cluster: bad key");
    }
    if (len) *len = (int64_t)v.size();
    if (out)
      for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)v.size()); ++i) out[i] = v[i];
  });
}

void hs_factor_destroy(hs_factor f) {
  if (!f) return;
  cudaSetDevice(f->h->device);
  delete f;
}

static void io_in(hs_factor f, const double* v, double* dtmp, int32_t on_device, cudaStream_t st) {
  HS_CUDA(cudaMemcpyAsync(dtmp, v, sizeof(double) * f->an->n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
}

hs_status hs_apply(hs_factor f, const double* b, double* x, int32_t on_device) {
  return guarded(f ? f->h : nullptr, [&] {
    if (!f || !b || !x) hs::fail(HS_E_INVALID_ARG, "hs_apply: NULL argument");
    require_device(f->h);
    cudaStream_t st = f->h->stream;
    const int64_t n = f->an->n;
    double* din = nullptr;
    din = (double*)f->h->cache.alloc(sizeof(double) * n);
    io_in(f, b, din, on_device, st);
    if (f->ds) hs::dist_apply(f, din, din);   // world > 1: collective, every rank passes b and gets x
    else hs::apply(f, din, din);
    HS_CUDA(cudaMemcpyAsync(x, din, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    f->h->cache.free(din);
    HS_CUDA(cudaStreamSynchronize(st));
  });
}

hs_status hs_spmv(hs_factor f, const double* x, double* y, int32_t on_device) {
  return guarded(f ? f->h : nullptr, [&] {
    if (!f || !x || !y) hs::fail(HS_E_INVALID_ARG, "hs_spmv: NULL argument");
    require_device(f->h);
    cudaStream_t st = f->h->stream;
    const int64_t n = f->an->n;
    double *dx = nullptr, *dy = nullptr;
    dx = (double*)f->h->cache.alloc(sizeof(double) * n);
    dy = (double*)f->h->cache.alloc(sizeof(double) * n);
    io_in(f, x, dx, on_device, st);
    if (f->ds) hs::dist_spmv_global(f, dx, dy);
    else hs::spmv(f, dx, dy);
    HS_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    f->h->cache.free(dx);
    f->h->cache.free(dy);
    HS_CUDA(cudaStreamSynchronize(st));
  });
}

int64_t hs_launch_count(void) { return hs::launch_count(); }

hs_status hs_pcg(hs_factor f, const double* b, double* x, double tol, int32_t maxit, int32_t on_device,
                 hs_pcg_report* rep) {
  hs_status s_inner = HS_OK;
  const hs_status s = guarded(f ? f->h : nullptr, [&] {
    if (!f || !b || !x || !rep) hs::fail(HS_E_INVALID_ARG, "hs_pcg: NULL argument");
    if (!(tol >= 0) || maxit < 0) hs::fail(HS_E_INVALID_ARG, "hs_pcg: bad tol/maxit");
    require_device(f->h);
    cudaStream_t st = f->h->stream;
    const int64_t n = f->an->n;
    double *db = nullptr, *dx = nullptr;
    db = (double*)f->h->cache.alloc(sizeof(double) * n);
    dx = (double*)f->h->cache.alloc(sizeof(double) * n);
    io_in(f, b, db, on_device, st);
    try {
      if (f->ds) hs::dist_pcg(f, db, dx, tol, maxit, rep);   // world > 1: collective
      else hs::pcg(f, db, dx, tol, maxit, rep);
    } catch (const hs::Error& e) {
      s_inner = e.status;
      if (e.status != HS_E_NOT_CONVERGED) {
        f->h->cache.free(db);
        f->h->cache.free(dx);
        throw;
      }
      f->h->err = e.what();
    }
    HS_CUDA(cudaMemcpyAsync(x, dx, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    f->h->cache.free(db);
    f->h->cache.free(dx);
    HS_CUDA(cudaStreamSynchronize(st));
  });
  return s != HS_OK ? s : s_inner;
}

hs_status hs_gmres(hs_factor f, const double* b, double* x, double tol, int32_t restart, int32_t maxit,
                   int32_t on_device, hs_pcg_report* rep) {
  hs_status s_inner = HS_OK;
  const hs_status s = guarded(f ? f->h : nullptr, [&] {
    if (!f || !b || !x || !rep) hs::fail(HS_E_INVALID_ARG, "hs_gmres: NULL argument");
    if (!(tol >= 0) || maxit < 0 || restart < 1) hs::fail(HS_E_INVALID_ARG, "hs_gmres: bad tol/restart/maxit");
    if (f->ds) hs::fail(HS_E_UNSUPPORTED, "hs_gmres: the distributed solve runs PCG (hs_pcg)");
    require_device(f->h);
    cudaStream_t st = f->h->stream;
    const int64_t n = f->an->n;
    double* db = (double*)f->h->cache.alloc(sizeof(double) * n);
    double* dx = (double*)f->h->cache.alloc(sizeof(double) * n);
    io_in(f, b, db, on_device, st);
    try {
      hs::gmres(f, db, dx, tol, restart, maxit, rep);
    } catch (const hs::Error& e) {
      s_inner = e.status;
      if (e.status != HS_E_NOT_CONVERGED) {
        f->h->cache.free(db);
        f->h->cache.free(dx);
        throw;
      }
      f->h->err = e.what();
    }
    HS_CUDA(cudaMemcpyAsync(x, dx, sizeof(double) * n, on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    f->h->cache.free(db);
    f->h->cache.free(dx);
  });
  return s != HS_OK ? s : s_inner;
}

}  // extern "C"
