// Internal structures of libhsolve (host side).  Not part of the ABI.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hsolve.h"

namespace hs {

// An exception that carries an hs_status across internal code; translated to a
// status code at the ABI (capi.cpp).  Never crosses the C boundary.
struct Error : std::runtime_error {
  hs_status status;
  Error(hs_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void fail(hs_status s, const std::string& m) { throw Error(s, m); }

using Adj = std::vector<std::vector<int32_t>>;   // sorted adjacency lists

struct Level {
  int32_t nclus = 0;
  Adj H;                       // H_l: structural block pattern of A_l; n(s) = H[s]
  Adj w;                       // w(s) at elimination time
  std::vector<std::vector<int32_t>> batches;
  int32_t nphase1 = 0;
  std::vector<uint8_t> interior;   // all of Fstart-adj(s) in s's subdomain
  Adj Fstart;                  // block pattern of the level's input A_l (= H under coarse_fill = 1)
  Adj Ffinal;                  // fill graph after the level
};

// Structural column supports of the level-0 blocks as each cluster is eliminated (support.cpp)
struct L0Support {
  bool built = false;
  // cluster s: entries sptr[s] .. sptr[s+1] of len, one per q of w(s) then n(s) (the B_s
  // column order): the number of supported columns of q, or -1 (q eliminated before s: its
  // coarse columns, dense); the supported local columns, ascending, at idx[iptr[s] ..]
  std::vector<int64_t> sptr, iptr;
  std::vector<int32_t> len, idx;
  int32_t* d_idx = nullptr;   // idx on device dev (l0_support_device; freed with the analysis)
  int dev = -1;
};

struct Analysis {
  int64_t n = 0;
  int32_t D = 0, L_top = 0, top_log2 = 3, nsub_log2 = 3;
  std::vector<int64_t> perm;       // perm[new] = old
  std::vector<int64_t> iperm;      // iperm[old] = new
  std::vector<int64_t> leaf_off;   // 2^D + 1
  std::vector<Level> levels;       // 0 .. L_top-1
  Adj H_top;
  // the pattern, kept for hs_factor (values come later)
  std::vector<int64_t> rowptr;
  std::vector<int32_t> colind;
  // device cache of the pattern (filled by the first factor; freed by hs_analysis_destroy)
  int dev = -1;
  int map_world = 1, map_rank = 0;   // the (world, rank) the cached level-0 scatter map is for
  int64_t* d_rowptr = nullptr;
  int32_t* d_colind = nullptr;
  int64_t* d_perm = nullptr;
  int64_t* d_map = nullptr;     // CSR entry -> offset in the level-0 block store (-1: upper)
  int64_t* d_tmap = nullptr;    // CSR entry (i,j) -> index of (j,i) (value symmetry check)
  // large patterns: host copies of the two maps, so that a factor that needs the device memory
  // (record space active) can drop d_map / d_tmap after its level-0 scatter and the next
  // factor uploads them again instead of recomputing them
  std::vector<int64_t> h_map, h_tmap;
  bool maps_pinned = false;     // h_map / h_tmap registered with cudaHostRegister
  L0Support l0s;                // built by the first factor that restricts level 0 to the supports
  int32_t subdomain(int32_t level, int32_t c) const { return c >> ((D - level) - nsub_log2); }
};

// Multi-GPU decomposition plan (dist.cpp).
struct DistPlan {
  int world = 1, rank = 0;
  std::vector<std::vector<int32_t>> owner;   // [level 0..L_top][cluster] -> owning rank
  bool own(int l, int c) const { return owner[l][c] == rank; }
  bool holds(int l, int p, int q) const { return owner[l][p] == rank || owner[l][q] == rank; }
};
DistPlan make_plan(const Analysis& an, int world, int rank);
// ranks other than the owner that receive the elimination record of cluster s of level l
std::vector<int32_t> receivers(const Analysis& an, const DistPlan& P, int l, int s);

void build_l0_support(Analysis& an);   // fills an.l0s (idempotent, thread-safe)
// an.l0s.idx on the device (uploaded once per analysis and device; thread-safe)
const int32_t* l0_support_device(Analysis& an, int device);

Analysis* analyze(int64_t n, const int64_t* rowptr, const int32_t* colind, const double* coords,
                  int32_t coord_dim, const int32_t* column_id, const hs_analyze_opts& opt);

}  // namespace hs
