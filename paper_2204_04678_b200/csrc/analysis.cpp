// Tile-level symbolic analysis (host, one-time per pattern).  See analysis.hpp.
#include "analysis.hpp"

#include <algorithm>
#include <thread>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <queue>
#include <tuple>
#include <stdexcept>

namespace pinla {

static constexpr int64_t kChunkFactor = 16;  // max update pairs per chained chunk
static constexpr int64_t kGroup = 32;        // pairs per parallel partial group
static constexpr int64_t kChainKeep = 32;    // newest pairs kept in the chain
static constexpr int64_t kDiagKeep = 32;     // the same for diagonal tiles
static constexpr int64_t kDiagGroup = 0;
static constexpr int64_t kRunMin = 8;       // same-level pair runs this long are grouped
static constexpr int64_t kRunGroup = 8;      //   into groups of this many pairs   // off: no measured gain on c2 (tunable)
static constexpr int kPrioClasses = 8;          // ready-queue priority classes
static constexpr int64_t kSelGroup = 4;         // selinv grouped tiles: pairs per parallel group
static constexpr int64_t kSelKeep = 1;          // selinv grouped tiles: newest pair kept in the chain
static constexpr int64_t kSelRunGroup = 8;      // other tiles: the oldest same-readiness run
                                                //   (>= 8 pairs) goes to groups of 8
static constexpr int64_t kSelWindow = 16;       // group buffers recycled after >= 16 columns
static constexpr int64_t kSelPoolMin = 1024;
static constexpr int64_t kChunkSolve = 32;   // max tile GEMVs per forward-solve task

int64_t Analysis::tid_of(int32_t I, int32_t J) const {
  auto b = tile_row.begin() + colptr[J], e = tile_row.begin() + colptr[J + 1];
  auto it = std::lower_bound(b, e, I);
  if (it == e || *it != I) return -1;
  return (int64_t)(it - tile_row.begin());
}

int64_t Analysis::pad_of_perm(int64_t j) const {
  auto it = std::upper_bound(tstart.begin(), tstart.end(), j);
  int64_t t = (int64_t)(it - tstart.begin()) - 1;
  return t * TB + (j - tstart[t]);
}

// intersection of two ascending K lists (with tids) restricted to K < kmax
static void intersect(const int32_t* ka, const int32_t* ta, int64_t na, const int32_t* kb,
                      const int32_t* tb, int64_t nb, int32_t kmax, std::vector<int32_t>& oa,
                      std::vector<int32_t>& ob) {
  bool swap = na > nb;
  if (swap) { std::swap(ka, kb); std::swap(ta, tb); std::swap(na, nb); }
  int64_t j = 0;
  for (int64_t i = 0; i < na; ++i) {
    int32_t k = ka[i];
    if (k >= kmax) break;
    // gallop in b
    if (j < nb && kb[j] < k) {
      int64_t step = 1, lo = j;
      while (lo + step < nb && kb[lo + step] < k) { lo += step; step <<= 1; }
      int64_t hi = std::min(nb, lo + step + 1);
      j = std::lower_bound(kb + lo, kb + hi, k) - kb;
    }
    if (j < nb && kb[j] == k) {
      if (swap) { oa.push_back(tb[j]); ob.push_back(ta[i]); }
      else { oa.push_back(ta[i]); ob.push_back(tb[j]); }
    }
  }
}

// geometric chunk sizes from the end of a list: 1, 1, 2, 4, 8, 16, 16, ...
// chunk sizes from the newest pair.  mode 3: 1, 4, 8, 16, ... (factor default,
// measured best on c2-c5); 4: 1, 8, 16, ... (selinv default); 0: 1, 1, 2, 4,
// ...; 1: 1, 2, 4, ...; 2: all cap; 5: 1, 3, 6, 12, ...
static void chunk_sizes(int64_t count, int64_t cap, std::vector<int32_t>& sizes, int mode) {
  sizes.clear();
  int64_t left = count, sz = 1;
  int k = 0;
  while (left > 0) {
    const int64_t take = std::min(left, sz);
    sizes.push_back((int32_t)take);
    left -= take;
    ++k;
    if (mode == 0 && k >= 2) sz = std::min<int64_t>(sz * 2, cap);
    if (mode == 1) sz = std::min<int64_t>(sz * 2, cap);
    if (mode == 2) sz = cap;
    if (mode == 3 && k == 1) sz = std::min<int64_t>(4, cap);
    if (mode == 3 && k >= 2) sz = std::min<int64_t>(sz * 2, cap);
    if (mode == 4 && k == 1) sz = std::min<int64_t>(8, cap);
    if (mode == 4 && k >= 2) sz = std::min<int64_t>(sz * 2, cap);
    if (mode == 5 && k == 1) sz = std::min<int64_t>(3, cap);
    if (mode == 5 && k >= 2) sz = std::min<int64_t>(sz * 2, cap);
  }
  if (sizes.empty()) sizes.push_back(0);
  std::reverse(sizes.begin(), sizes.end());
}

// successor CSR + ready list from per-task dependency lists
static void build_succ(std::vector<std::vector<int32_t>>& deps, std::vector<int32_t>& ndep,
                       std::vector<int32_t>& succ_ptr, std::vector<int32_t>& succ,
                       std::vector<int32_t>& ready0) {
  const int64_t ntask = (int64_t)deps.size();
  ndep.assign(ntask, 0);
  succ_ptr.assign(ntask + 1, 0);
  par_for(ntask, [&](int64_t i0, int64_t i1) {  // each list is its own
    for (int64_t i = i0; i < i1; ++i) {
      std::sort(deps[i].begin(), deps[i].end());
      deps[i].erase(std::unique(deps[i].begin(), deps[i].end()), deps[i].end());
      ndep[i] = (int32_t)deps[i].size();
    }
  });
  for (int64_t i = 0; i < ntask; ++i)
    for (int32_t p : deps[i]) succ_ptr[p + 1]++;
  for (int64_t i = 0; i < ntask; ++i) succ_ptr[i + 1] += succ_ptr[i];
  succ.assign(succ_ptr[ntask], 0);
  std::vector<int32_t> w(succ_ptr.begin(), succ_ptr.end() - 1);
  for (int64_t i = 0; i < ntask; ++i)
    for (int32_t p : deps[i]) succ[w[p]++] = (int32_t)i;
  ready0.clear();
  for (int64_t i = 0; i < ntask; ++i)
    if (ndep[i] == 0) ready0.push_back((int32_t)i);
}

// list-schedule simulation: `workers` workers, highest bottom level first;
// returns the start order (a topological order)
static void list_schedule(const std::vector<int32_t>& ndep, const std::vector<int32_t>& succ_ptr,
                          const std::vector<int32_t>& succ, const std::vector<int32_t>& ready0,
                          const std::vector<double>& cost, int workers,
                          std::vector<int32_t>& order_out) {
  const int64_t ntask = (int64_t)ndep.size();
  std::vector<int32_t> topo;
  {
    std::vector<int32_t> indeg(ndep.begin(), ndep.end());
    topo = ready0;
    for (size_t k = 0; k < topo.size(); ++k)
      for (int32_t q = succ_ptr[topo[k]]; q < succ_ptr[topo[k] + 1]; ++q)
        if (--indeg[succ[q]] == 0) topo.push_back(succ[q]);
  }
  if ((int64_t)topo.size() != ntask) throw std::runtime_error("task graph is not a DAG");
  std::vector<double> bl(ntask, 0.0);
  for (int64_t k = ntask - 1; k >= 0; --k) {
    const int32_t t = topo[k];
    double m = 0.0;
    for (int32_t q = succ_ptr[t]; q < succ_ptr[t + 1]; ++q) m = std::max(m, bl[succ[q]]);
    bl[t] = cost[t] + m;
  }
  std::vector<int32_t> indeg(ndep.begin(), ndep.end());
  std::priority_queue<std::pair<double, int32_t>> ready;
  std::priority_queue<std::pair<double, int32_t>, std::vector<std::pair<double, int32_t>>,
                      std::greater<std::pair<double, int32_t>>> running;
  for (int32_t t : ready0) ready.push({bl[t], t});
  order_out.clear();
  order_out.reserve(ntask);
  double now = 0.0;
  int busy = 0;
  const int P = std::max(1, workers);
  while ((int64_t)order_out.size() < ntask) {
    while (busy < P && !ready.empty()) {
      const int32_t t = ready.top().second;
      ready.pop();
      order_out.push_back(t);
      running.push({now + cost[t], t});
      ++busy;
    }
    if (running.empty()) break;
    const auto ev = running.top();
    running.pop();
    --busy;
    now = ev.first;
    for (int32_t q = succ_ptr[ev.second]; q < succ_ptr[ev.second + 1]; ++q)
      if (--indeg[succ[q]] == 0) ready.push({bl[succ[q]], succ[q]});
  }
}


void analyze_tiles(Analysis& A, int64_t n, const int64_t* indptr, const int64_t* indices,
                   const int64_t* perm, int64_t n_dense, const int64_t* tile_bounds,
                   int64_t n_tile_bounds, int workers, int solve_group_cap, int solve_links,
                   int factor_lane) {
  PhaseClock clk;
  A.n = n;
  A.n_main = n - n_dense;
  A.perm.assign(perm, perm + n);
  A.iperm.assign(n, -1);
  for (int64_t j = 0; j < n; ++j) {
    if (perm[j] < 0 || perm[j] >= n || A.iperm[perm[j]] != -1)
      throw std::runtime_error("ordering is not a permutation");
    A.iperm[perm[j]] = j;
  }
  // tile boundaries: 64-chunks of the main range, then of the dense range
  A.tstart.clear();
  if (tile_bounds && n_tile_bounds >= 2) {
    A.tstart.assign(tile_bounds, tile_bounds + n_tile_bounds);
    if (A.tstart.front() != 0 || A.tstart.back() != n)
      throw std::runtime_error("tile bounds must cover [0, n)");
    bool has_main = false;
    for (size_t t = 0; t + 1 < A.tstart.size(); ++t) {
      int64_t a = A.tstart[t], b = A.tstart[t + 1];
      if (b <= a || b - a > TB) throw std::runtime_error("tiles must hold 1..64 rows");
      if (a < A.n_main && b > A.n_main) throw std::runtime_error("a tile straddles the dense tail");
      has_main |= (b == A.n_main);
    }
    if (A.n_main > 0 && !has_main) throw std::runtime_error("no tile boundary at the dense tail");
  } else {
    for (int64_t s = 0; s < A.n_main; s += TB) A.tstart.push_back(s);
    for (int64_t s = A.n_main; s < n; s += TB) A.tstart.push_back(s);
    A.tstart.push_back(n);
  }
  const int32_t NT = (int32_t)A.tstart.size() - 1;
  A.NT = NT;
  std::vector<int32_t> tile_of(n);
  for (int32_t t = 0; t < NT; ++t)
    for (int64_t j = A.tstart[t]; j < A.tstart[t + 1]; ++j) tile_of[j] = t;

  clk.mark("tile bounds");
  // tile pattern of Q (lower)
  std::vector<std::vector<int32_t>> qcol(NT);
  for (int64_t c = 0; c < n; ++c) {
    for (int64_t p = indptr[c]; p < indptr[c + 1]; ++p) {
      int64_t r = indices[p];
      int64_t pr = A.iperm[r], pc = A.iperm[c];
      int32_t TI = tile_of[std::max(pr, pc)], TJ = tile_of[std::min(pr, pc)];
      qcol[TJ].push_back(TI);
    }
  }
  clk.mark("tile pattern of Q");
  // block symbolic elimination: pat(J) = Q(J) U (pat(child) \ child)
  std::vector<std::vector<int32_t>> pend(NT), pat(NT);
  for (int32_t J = 0; J < NT; ++J) {
    std::vector<int32_t>& S = pat[J];
    S.swap(qcol[J]);
    S.insert(S.end(), pend[J].begin(), pend[J].end());
    std::vector<int32_t>().swap(pend[J]);
    S.push_back(J);
    std::sort(S.begin(), S.end());
    S.erase(std::unique(S.begin(), S.end()), S.end());
    if (S.front() != J) throw std::runtime_error("tile pattern above the diagonal");
    if (S.size() > 1) {
      int32_t parent = S[1];
      pend[parent].insert(pend[parent].end(), S.begin() + 1, S.end());
    }
  }
  A.colptr.assign(NT + 1, 0);
  for (int32_t J = 0; J < NT; ++J) A.colptr[J + 1] = A.colptr[J] + (int32_t)pat[J].size();
  A.nT = A.colptr[NT];
  A.tile_row.resize(A.nT);
  A.tile_col.resize(A.nT);
  for (int32_t J = 0; J < NT; ++J) {
    std::copy(pat[J].begin(), pat[J].end(), A.tile_row.begin() + A.colptr[J]);
    std::fill(A.tile_col.begin() + A.colptr[J], A.tile_col.begin() + A.colptr[J + 1], J);
    std::vector<int32_t>().swap(pat[J]);
  }
  clk.mark("symbolic elimination");
  // row form (K ascending because columns are visited in order)
  A.rowptr.assign(NT + 1, 0);
  for (int64_t t = 0; t < A.nT; ++t) A.rowptr[A.tile_row[t] + 1]++;
  for (int32_t I = 0; I < NT; ++I) A.rowptr[I + 1] += A.rowptr[I];
  A.row_col.resize(A.nT);
  A.row_tid.resize(A.nT);
  {
    std::vector<int32_t> w(A.rowptr.begin(), A.rowptr.end() - 1);
    for (int64_t t = 0; t < A.nT; ++t) {
      int32_t I = A.tile_row[t];
      int32_t q = w[I]++;
      A.row_col[q] = A.tile_col[t];
      A.row_tid[q] = (int32_t)t;
    }
  }
  clk.mark("row form");
  // levels
  A.flevel.assign(NT, 0);
  for (int32_t J = 0; J < NT; ++J) {
    int32_t lv = 0;
    for (int32_t q = A.rowptr[J]; q < A.rowptr[J + 1]; ++q) {
      int32_t K = A.row_col[q];
      if (K < J) lv = std::max(lv, A.flevel[K] + 1);
    }
    A.flevel[J] = lv;
  }
  A.blevel.assign(NT, 0);
  for (int32_t J = NT - 1; J >= 0; --J) {
    int32_t lv = 0;
    for (int32_t q = A.colptr[J] + 1; q < A.colptr[J + 1]; ++q)
      lv = std::max(lv, A.blevel[A.tile_row[q]] + 1);
    A.blevel[J] = lv;
  }

  clk.mark("levels");
  // The selected-inversion DAG only reads the tile pattern: it is built on
  // a second host thread while this one builds the factor and solve DAGs.
  auto build_selinv = [&]() {
  // ---------------- selected inversion DAG ----------------
  A.s_pa.clear();
  A.s_pb.clear();
  A.s_mode.clear();
  A.s_chunk_rng.assign(1, 0);
  A.s_chunk_tile.clear();
  A.s_chunk_flags.clear();
  A.s_last_chunk.assign(A.nT, -1);
  A.s_grp_rng.assign(1, 0);
  A.s_grp_tile.clear();
  A.s_tile_grp_ptr.assign(A.nT + 1, 0);
  {
    std::vector<int32_t> gpa, gpb, gmode;
    std::vector<int32_t> s_first_chunk(A.nT, 0);
    // per-tile lists in parallel tile ranges (each range appends to its own
    // Local), then concatenated in tile order with the offsets shifted:
    // identical to one serial pass
    struct Local {
      int64_t t0 = 0;
      std::vector<int32_t> gpa, gpb, gmode, grp_tile, pa, pb, mode, chunk_tile, chunk_flags;
      std::vector<int64_t> grp_end, chunk_end;
      std::vector<int32_t> ng_of, first_of, last_of;
    };
    auto process = [&](int64_t t, Local& L, std::vector<std::tuple<int32_t, int32_t, int32_t, int32_t>>& pl,
                       std::vector<int32_t>& sizes) {
      const int32_t I = A.tile_row[t], J = A.tile_col[t];
      pl.clear();
      for (int32_t q = A.colptr[J] + 1; q < A.colptr[J + 1]; ++q) {
        const int32_t K = A.tile_row[q];
        // keys order the pairs oldest first (chunks run in list order)
        if (I != J) {
          // Sigma(I,K) (or Sigma(K,I)^T) * L(K,J); newest dependency = smallest
          // min(I,K); among K >= I (all read column I) Sigma(I,I) is the last of
          // that column to finish, so it sorts after the others
          const bool trans = K > I;
          const int32_t sid = trans ? (int32_t)A.tid_of(K, I) : (int32_t)A.tid_of(I, K);
          // within column I (K > I), its first sub-diagonal Sigma(I+1, I) is
          // the last off-diagonal to finish (it waits for Sigma(I+1, I+1)):
          // it sorts after the other K > I and before Sigma(I, I)
          const bool sub1 = trans && sid == A.colptr[I] + 1;
          pl.emplace_back(-4 * std::min(I, K) + (K == I ? 2 : (sub1 ? 1 : 0)), sid, q,
                          (trans ? 2 : 0) | 4);
        } else {
          // L(K,J)^T * Sigma(K,J); Sigma(J+1,J) (smallest K) is the newest
          pl.emplace_back(-K, q, q, 1 | 2);
        }
      }
      std::stable_sort(pl.begin(), pl.end(),
                       [](const auto& x, const auto& y) { return std::get<0>(x) < std::get<0>(y); });
      size_t first = 0;
      L.ng_of[t - L.t0] = 0;
      // the diagonal tile and the first sub-diagonal tile of a column read
      // (almost) only the newest column: their lists go to parallel groups
      // Every other tile: its oldest pairs all read column I (K >= I share one
      // readiness key) and become ready together; chained they would run
      // back to back on the critical path, so that run goes to groups too.
      const bool first_sub = (int64_t)t == (int64_t)A.colptr[J] + 1;
      static const int64_t selg = getenv("PINLA_SEL_GROUP") ? atoll(getenv("PINLA_SEL_GROUP")) : kSelGroup;  // tuning
      size_t ng = 0, gsz = selg;
      size_t ngrouped = 0;  // pairs [0, ngrouped) go to groups
      // pairs kept in the tile's own chain: the newest readiness key (the
      // diagonal tile: Sigma(J+1,J); the first sub-diagonal (J+1,J):
      // Sigma(J+1,J+1) and Sigma(J+2,J+1)^T, the two last of column J+1)
      size_t keep = kSelKeep;
      if (I == J && pl.size() >= 2) keep = 2;  // Sigma(J+1,J) and Sigma(J+2,J) finish last
      if (first_sub && pl.size() >= 2) {
        keep = 0;
        while (keep < pl.size() && std::get<0>(pl[pl.size() - 1 - keep]) > std::get<0>(pl[0])) ++keep;
        keep = std::max<size_t>(keep, 1);
      }
      bool split = false;  // group sums in a pair-less first chunk, off the chain
      if ((I == J || first_sub) && (int64_t)pl.size() > selg + (int64_t)keep) {
        ngrouped = pl.size() - keep;
        ng = (ngrouped + selg - 1) / selg;
        split = true;
      } else if (I != J) {
        size_t run = 0;
        while (run < pl.size() && std::get<0>(pl[run]) == std::get<0>(pl[0])) ++run;
        static const int64_t rung = getenv("PINLA_SEL_RUN_GROUP") ? atoll(getenv("PINLA_SEL_RUN_GROUP")) : kSelRunGroup;  // tuning
        if ((int64_t)run >= rung) {
          gsz = rung;
          ngrouped = run;  // the whole run (the last group may be smaller)
          ng = (run + gsz - 1) / gsz;
        }
      }
      if (ng > 0) {
        for (size_t g = 0; g < ng; ++g) {
          for (size_t u = g * gsz; u < std::min(ngrouped, (g + 1) * gsz); ++u) {
            L.gpa.push_back(std::get<1>(pl[u]));
            L.gpb.push_back(std::get<2>(pl[u]));
            L.gmode.push_back(std::get<3>(pl[u]));
          }
          L.grp_end.push_back((int64_t)L.gpa.size());
          L.grp_tile.push_back((int32_t)t);
          L.ng_of[t - L.t0]++;
        }
        first = ngrouped;
      }
      for (size_t u = first; u < pl.size(); ++u) {
        L.pa.push_back(std::get<1>(pl[u]));
        L.pb.push_back(std::get<2>(pl[u]));
        L.mode.push_back(std::get<3>(pl[u]));
      }
      static const int smode = getenv("PINLA_SEL_CHUNK_MODE") ? atoi(getenv("PINLA_SEL_CHUNK_MODE")) : 4;  // tuning
      chunk_sizes((int64_t)(pl.size() - first), kChunkFactor, sizes, smode);
      if (split && !sizes.empty() && sizes[0] > 0) sizes.insert(sizes.begin(), 0);
      L.first_of[t - L.t0] = (int32_t)L.chunk_tile.size();
      for (size_t c = 0; c < sizes.size(); ++c) {
        L.chunk_end.push_back((L.chunk_end.empty() ? 0 : L.chunk_end.back()) + sizes[c]);
        L.chunk_tile.push_back((int32_t)t);
        L.chunk_flags.push_back((c == 0 ? 1 : 0) | (c + 1 == sizes.size() ? 2 : 0));
      }
      L.last_of[t - L.t0] = (int32_t)L.chunk_tile.size() - 1;
        };
    const int nloc = (int)std::max<int64_t>(1, std::min<int64_t>(64, A.nT / 4096));
    std::vector<Local> locs(nloc);
    par_for(nloc, [&](int64_t r0, int64_t r1) {
      std::vector<std::tuple<int32_t, int32_t, int32_t, int32_t>> pl;  // (key, a, b, mode)
      std::vector<int32_t> sizes;
      for (int64_t r = r0; r < r1; ++r) {
        Local& L = locs[r];
        L.t0 = A.nT * r / nloc;
        const int64_t t1 = A.nT * (r + 1) / nloc;
        L.ng_of.assign(t1 - L.t0, 0);
        L.first_of.assign(t1 - L.t0, 0);
        L.last_of.assign(t1 - L.t0, 0);
        for (int64_t t = L.t0; t < t1; ++t) process(t, L, pl, sizes);
      }
    }, 1);
    for (const Local& L : locs) {
      const int64_t pa_off = (int64_t)A.s_pa.size(), ch_off = (int64_t)A.s_chunk_tile.size();
      const int64_t g_off = (int64_t)gpa.size();
      A.s_pa.insert(A.s_pa.end(), L.pa.begin(), L.pa.end());
      A.s_pb.insert(A.s_pb.end(), L.pb.begin(), L.pb.end());
      A.s_mode.insert(A.s_mode.end(), L.mode.begin(), L.mode.end());
      for (int64_t e : L.chunk_end) A.s_chunk_rng.push_back(pa_off + e);
      A.s_chunk_tile.insert(A.s_chunk_tile.end(), L.chunk_tile.begin(), L.chunk_tile.end());
      A.s_chunk_flags.insert(A.s_chunk_flags.end(), L.chunk_flags.begin(), L.chunk_flags.end());
      gpa.insert(gpa.end(), L.gpa.begin(), L.gpa.end());
      gpb.insert(gpb.end(), L.gpb.begin(), L.gpb.end());
      gmode.insert(gmode.end(), L.gmode.begin(), L.gmode.end());
      for (int64_t e : L.grp_end) A.s_grp_rng.push_back(g_off + e);
      A.s_grp_tile.insert(A.s_grp_tile.end(), L.grp_tile.begin(), L.grp_tile.end());
      for (size_t k = 0; k < L.ng_of.size(); ++k) {
        const int64_t t = L.t0 + (int64_t)k;
        A.s_tile_grp_ptr[t + 1] = A.s_tile_grp_ptr[t] + L.ng_of[k];
        s_first_chunk[t] = (int32_t)(ch_off + L.first_of[k]);
        A.s_last_chunk[t] = (int32_t)(ch_off + L.last_of[k]);
      }
    }
    A.s_nchunk = (int64_t)A.s_chunk_tile.size();
    A.s_ngrp = (int32_t)A.s_grp_tile.size();
    // group pairs live after the chunk pairs
    const int64_t goff = (int64_t)A.s_pa.size();
    A.s_pa.insert(A.s_pa.end(), gpa.begin(), gpa.end());
    A.s_pb.insert(A.s_pb.end(), gpb.begin(), gpb.end());
    A.s_mode.insert(A.s_mode.end(), gmode.begin(), gmode.end());
    for (auto& v : A.s_grp_rng) v += goff;
    // tasks: chunks [0, nchunk), groups [nchunk, nchunk + ngrp)
    const int64_t ntask = A.s_nchunk + A.s_ngrp;
    std::vector<std::vector<int32_t>> deps(ntask);
    std::vector<double> cost(ntask);
    auto pair_deps = [&](int64_t u, std::vector<int32_t>& d) {
      if (!(A.s_mode[u] & 1)) d.push_back(A.s_last_chunk[A.s_pa[u]]);
      if (!(A.s_mode[u] & 4)) d.push_back(A.s_last_chunk[A.s_pb[u]]);
    };
    par_for(A.s_nchunk, [&](int64_t c0, int64_t c1) {  // per-chunk lists
    for (int64_t c = c0; c < c1; ++c) {
      std::vector<int32_t>& d = deps[c];
      for (int64_t u = A.s_chunk_rng[c]; u < A.s_chunk_rng[c + 1]; ++u) pair_deps(u, d);
      if (!(A.s_chunk_flags[c] & 1)) d.push_back((int32_t)c - 1);
      else
        for (int32_t g = A.s_tile_grp_ptr[A.s_chunk_tile[c]]; g < A.s_tile_grp_ptr[A.s_chunk_tile[c] + 1]; ++g)
          d.push_back((int32_t)(A.s_nchunk + g));
      {
        const int32_t t = A.s_chunk_tile[c];
        const bool dg = A.tile_row[t] == A.tile_col[t];
        cost[c] = 5.0 + 4.5 * (double)(A.s_chunk_rng[c + 1] - A.s_chunk_rng[c]) +
                  ((A.s_chunk_flags[c] & 2) ? (dg ? 25.0 : 10.0) : 0.0) +
                  ((A.s_chunk_flags[c] & 1) ? 1.0 * (A.s_tile_grp_ptr[t + 1] - A.s_tile_grp_ptr[t]) : 0.0);
      }
    }
    });
    // group scratch ring: columns in processing order (descending J) take the
    // next buffers; a buffer's previous user is >= kSelWindow columns earlier
    // (higher J), whose consumer chunk cannot depend on this column: acyclic
    std::vector<int32_t> prev_user(A.s_ngrp, -1);
    {
      int64_t maxpc = 0;
      for (int32_t J = 0; J < NT; ++J)
        maxpc = std::max<int64_t>(maxpc, A.s_tile_grp_ptr[A.colptr[J + 1]] - A.s_tile_grp_ptr[A.colptr[J]]);
      const int64_t R = std::min<int64_t>(A.s_ngrp, std::max<int64_t>(kSelPoolMin, kSelWindow * maxpc));
      A.s_ngbuf = (int32_t)std::max<int64_t>(R, 1);
      A.s_grp_buf.assign(A.s_ngrp, 0);
      std::vector<int32_t> owner(A.s_ngbuf, -1);
      int64_t ptr = 0;
      for (int32_t J = NT - 1; J >= 0; --J)
        for (int32_t g = A.s_tile_grp_ptr[A.colptr[J]]; g < A.s_tile_grp_ptr[A.colptr[J + 1]]; ++g) {
          const int32_t b = (int32_t)ptr;
          ptr = (ptr + 1) % A.s_ngbuf;
          prev_user[g] = owner[b];
          owner[b] = g;
          A.s_grp_buf[g] = b;
        }
    }
    for (int32_t g = 0; g < A.s_ngrp; ++g) {
      if (prev_user[g] >= 0) deps[A.s_nchunk + g].push_back(s_first_chunk[A.s_grp_tile[prev_user[g]]]);
      for (int64_t u = A.s_grp_rng[g]; u < A.s_grp_rng[g + 1]; ++u) pair_deps(u, deps[A.s_nchunk + g]);
      cost[A.s_nchunk + g] = 5.0 + 4.5 * (double)(A.s_grp_rng[g + 1] - A.s_grp_rng[g]);
    }
    build_succ(deps, A.s_ndep, A.s_succ_ptr, A.s_succ, A.s_ready0);
    // the 128-thread selinv kernel runs in ready-queue (FIFO) mode; the
    // warp-specialised one (and PINLA_SELINV_SCHED=s) claims in this static
    // list-schedule order
    A.s_order.clear();
    list_schedule(A.s_ndep, A.s_succ_ptr, A.s_succ, A.s_ready0, cost, 296, A.s_order);
    // the per-column chain (last chunks of the diagonal and first sub-diagonal
    // tiles) runs as continuations of the task that readies it
    A.s_hot.assign(ntask, 0);
    for (int64_t c = 0; c < A.s_nchunk; ++c) {
      const int32_t t = A.s_chunk_tile[c];
      const int32_t J = A.tile_col[t];
      if ((A.s_chunk_flags[c] & 2) && (A.tile_row[t] == J || t == A.colptr[J] + 1)) A.s_hot[c] = 1;
    }
    A.selinv_tasks.clear();
    for (int64_t c = 0; c < A.s_nchunk; ++c) A.selinv_tasks.push_back({0, 0, (int32_t)c, 0});
    for (int32_t g = 0; g < A.s_ngrp; ++g) A.selinv_tasks.push_back({1, 0, g, 0});
  }

  };
  std::thread sel_thread(build_selinv);
  // factor update pairs (left-looking, K ascending) cut into chained chunks
  A.upd_a.clear();
  A.upd_b.clear();
  A.chunk_rng.assign(1, 0);
  A.chunk_tile.clear();
  A.chunk_flags.clear();
  A.last_chunk.assign(A.nT, -1);
  A.grp_rng.assign(1, 0);
  A.grp_tile.clear();
  A.chunk_grp_ptr.assign(1, 0);
  std::vector<int32_t> ga, gb;  // group pairs, stored before the chunk pairs
  int32_t first_arrow = NT;
  int64_t diag_keep = kDiagKeep, diag_group = kDiagGroup;
  if (const char* e = getenv("PINLA_DIAG_GROUP")) {  // "keep,group" (tuning)
    long k = 0, g = 0;
    if (sscanf(e, "%ld,%ld", &k, &g) == 2) { diag_keep = k; diag_group = g; }
  }
  int64_t run_min = kRunMin;
  if (const char* e = getenv("PINLA_RUN_GROUP")) run_min = atol(e);  // 0: off (tuning)
  for (int32_t t = 0; t < NT; ++t)
    if (A.tstart[t] >= A.n_main) { first_arrow = t; break; }
  // Chunk sizes of the chained updates.  With chunk continuations a boundary is
  // only a potential split point, but each still costs a task hand-off, and
  // small early chunks only pay when operands arrive late (chain-bound DAGs).
  // Deep DAGs (time-major block-tridiagonal orderings) with wide time blocks
  // (>= 48 tiles per tile row: c3, c4) therefore keep one pair for the newest
  // operand and cut the rest into 32-pair chunks when several theta-slots are
  // resident (throughput-bound: c4 x 3 28.5 -> 30.7 TF/s, c3 x 3 29.3 -> 30.3)
  // and into 16-pair chunks for one slot (c4 x 1 29.1 -> 30.1, c3 x 1 28.0 ->
  // 28.6).  Shallow nested-dissection DAGs (c2 bench 569 -> 523 f-evals/s with
  // 32-pair chunks) and narrow blocks (c5, 37 tiles per row: its single-slot
  // launches -- the serial evaluations between the batches of a fit -- are
  // chain-bound, 22.7 -> 18.2 / 12.3 TF/s with 16- / 32-pair chunks) keep the
  // latency-oriented 1, 4, 8, 16, 16, ...  Sweeps: profiles/chunk_sweep_cont_r02.txt,
  // profiles/chunk_sweep_final_r02.txt.  The chunking only moves the points where
  // a running sum may leave the registers: the factor is bitwise the same for
  // every choice (tests/test_gpu_modes.py).
  int32_t fdepth0 = 0;
  for (int32_t I = 0; I < NT; ++I) fdepth0 = std::max(fdepth0, A.flevel[I] + 1);
  const bool wide_deep = 4LL * fdepth0 > NT && A.nT >= 48LL * NT;
  const bool throughput_dag = wide_deep && workers < 296;  // several resident slots
  const int64_t fcap = getenv("PINLA_CHUNK_CAP") ? atoll(getenv("PINLA_CHUNK_CAP"))
                                                 : (throughput_dag ? 32 : kChunkFactor);  // tuning
  const int fmode = getenv("PINLA_CHUNK_MODE") ? atoi(getenv("PINLA_CHUNK_MODE")) : (wide_deep ? 2 : 3);  // tuning
  {
    const bool order_by_level = !getenv("PINLA_PAIR_ORDER_K");  // tuning: K order
    const bool split_first_sub = !getenv("PINLA_NO_SPLIT");     // tuning
    // a group segment: pairs [u0, u1) of the tile's list, consumed by the
    // chunk that starts at chain position `at` (chain = pairs not grouped)
    struct Seg { int64_t u0, u1, gsz, at; };
    // per-tile lists in parallel tile ranges (each range appends to its own
    // Local), then concatenated in tile order with the offsets shifted:
    // identical to one serial pass
    struct Local {
      int64_t t0 = 0;
      std::vector<int32_t> upd_a, upd_b, chunk_tile, chunk_flags, ga, gb, grp_tile, chunk_grp_end, last_of;
      std::vector<int64_t> chunk_end, grp_end;
    };
    struct Scratch {
      std::vector<int32_t> pa, pb, sizes, cut, ord, tmp_a, tmp_b;
      std::vector<Seg> segs;
      std::vector<char> grouped;
    };
    auto process = [&](int64_t t, Local& L, Scratch& S) {
      std::vector<int32_t>&pa = S.pa, &pb = S.pb, &sizes = S.sizes, &cut = S.cut, &ord = S.ord,
                          &tmp_a = S.tmp_a, &tmp_b = S.tmp_b;
      std::vector<Seg>& segs = S.segs;
      std::vector<char>& grouped = S.grouped;
      const int32_t I = A.tile_row[t], J = A.tile_col[t];
      pa.clear();
      pb.clear();
      intersect(&A.row_col[A.rowptr[I]], &A.row_tid[A.rowptr[I]], A.rowptr[I + 1] - A.rowptr[I],
                &A.row_col[A.rowptr[J]], &A.row_tid[A.rowptr[J]], A.rowptr[J + 1] - A.rowptr[J],
                J, pa, pb);
      // chain order = readiness order: by the elimination level of column K
      // (sibling subtrees interleave instead of running one after the other)
      if (order_by_level && pa.size() > 1) {
        ord.resize(pa.size());
        for (size_t u = 0; u < pa.size(); ++u) ord[u] = (int32_t)u;
        std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
          return A.flevel[A.tile_col[pa[x]]] < A.flevel[A.tile_col[pa[y]]];
        });
        tmp_a.resize(pa.size());
        tmp_b.resize(pa.size());
        for (size_t u = 0; u < pa.size(); ++u) { tmp_a[u] = pa[ord[u]]; tmp_b[u] = pb[ord[u]]; }
        pa.swap(tmp_a);
        pb.swap(tmp_b);
      }
      const int64_t np = (int64_t)pa.size();
      segs.clear();
      grouped.assign(np, 0);
      const bool arrow = I >= first_arrow;
      if (arrow) {
        // arrow-row tiles with long lists: the oldest pairs go to parallel
        // groups of kGroup pairs, the newest kChainKeep stay in the chain
        if (np > kChainKeep + kGroup) segs.push_back({0, ((np - kChainKeep) / kGroup) * kGroup, kGroup, 0});
      } else if (I == J && diag_group > 0 && np > diag_keep + diag_group) {
        segs.push_back({0, ((np - diag_keep) / diag_group) * diag_group, diag_group, 0});
      } else if (run_min > 0) {
        // pairs whose column K sits at the same elimination level become
        // ready together (sibling subtrees finish at once); chained they
        // would run back to back, so each such run is summed by parallel
        // groups that the chunk after the run adds in
        int64_t u = 0;
        while (u < np) {
          int64_t v = u + 1;
          const int32_t lv = A.flevel[A.tile_col[pa[u]]];
          while (v < np && A.flevel[A.tile_col[pa[v]]] == lv) ++v;
          if (v - u >= run_min) segs.push_back({u, v, kRunGroup, 0});
          u = v;
        }
      }
      for (auto& sg : segs)
        for (int64_t u = sg.u0; u < sg.u1; ++u) grouped[u] = 1;
      // chain positions: number of chain pairs before each segment
      {
        int64_t pos = 0, u = 0;
        for (auto& sg : segs) {
          for (; u < sg.u0; ++u) pos += grouped[u] ? 0 : 1;
          sg.at = pos;
          u = sg.u1;
        }
      }
      for (int64_t u = 0; u < np; ++u)
        if (!grouped[u]) {
          L.upd_a.push_back(pa[u]);
          L.upd_b.push_back(pb[u]);
        }
      const int64_t nchain = np - (int64_t)std::count(grouped.begin(), grouped.end(), (char)1);
      // chunk sizes from the end: 1, 1, 2, 4, 8, 16, 16, ... with forced cuts
      // where groups are added in (a run at the end gets an empty last chunk)
      chunk_sizes(nchain, fcap, sizes, fmode);
      cut.assign(1, 0);
      for (int32_t sz : sizes) cut.push_back(cut.back() + sz);
      for (auto& sg : segs) cut.push_back(sg.at);
      std::sort(cut.begin(), cut.end());
      cut.erase(std::unique(cut.begin(), cut.end()), cut.end());
      bool tail_run = false;
      for (auto& sg : segs) tail_run |= (sg.at == nchain && nchain > 0);
      // first sub-diagonal tiles sit on the column chain (diag J -> TRSM of
      // (J+1,J) -> diag J+1): their finalize chunk carries no pair, the
      // newest pair runs before L_JJ is ready
      if (split_first_sub && I == J + 1 && nchain > 0) tail_run = true;
      // chunk k covers chain pairs [cut[k], cut[k+1]); plus an empty chunk at
      // nchain when a run ends the list (or the list is empty)
      std::vector<std::pair<int64_t, int64_t>> ch;
      for (size_t k = 0; k + 1 < cut.size(); ++k) ch.push_back({cut[k], cut[k + 1]});
      if (ch.empty() || tail_run) ch.push_back({nchain, nchain});
      const int64_t base = L.chunk_end.empty() ? 0 : L.chunk_end.back();
      for (size_t k = 0; k < ch.size(); ++k) {
        L.chunk_end.push_back(base + ch[k].second);
        L.chunk_tile.push_back((int32_t)t);
        L.chunk_flags.push_back((k == 0 ? 1 : 0) | (k + 1 == ch.size() ? 2 : 0));
        // groups consumed by this chunk: the segments positioned at its start
        for (auto& sg : segs) {
          if (sg.at != ch[k].first) continue;
          for (int64_t g0 = sg.u0; g0 < sg.u1; g0 += sg.gsz) {
            for (int64_t u = g0; u < std::min(sg.u1, g0 + sg.gsz); ++u) {
              L.ga.push_back(pa[u]);
              L.gb.push_back(pb[u]);
            }
            L.grp_end.push_back((int64_t)L.ga.size());
            L.grp_tile.push_back((int32_t)t);
          }
        }
        L.chunk_grp_end.push_back((int32_t)L.grp_tile.size());
      }
      L.last_of[t - L.t0] = (int32_t)L.chunk_tile.size() - 1;
        };
    const int nloc = (int)std::max<int64_t>(1, std::min<int64_t>(64, A.nT / 4096));
    std::vector<Local> locs(nloc);
    par_for(nloc, [&](int64_t r0, int64_t r1) {
      Scratch S;
      for (int64_t r = r0; r < r1; ++r) {
        Local& L = locs[r];
        L.t0 = A.nT * r / nloc;
        const int64_t t1 = A.nT * (r + 1) / nloc;
        L.last_of.assign(t1 - L.t0, 0);
        for (int64_t t = L.t0; t < t1; ++t) process(t, L, S);
      }
    }, 1);
    for (const Local& L : locs) {
      const int64_t upd_off = (int64_t)A.upd_a.size(), ch_off = (int64_t)A.chunk_tile.size();
      const int64_t ga_off = (int64_t)ga.size(), grp_off = (int64_t)A.grp_tile.size();
      A.upd_a.insert(A.upd_a.end(), L.upd_a.begin(), L.upd_a.end());
      A.upd_b.insert(A.upd_b.end(), L.upd_b.begin(), L.upd_b.end());
      for (int64_t e : L.chunk_end) A.chunk_rng.push_back(upd_off + e);
      A.chunk_tile.insert(A.chunk_tile.end(), L.chunk_tile.begin(), L.chunk_tile.end());
      A.chunk_flags.insert(A.chunk_flags.end(), L.chunk_flags.begin(), L.chunk_flags.end());
      for (int32_t e : L.chunk_grp_end) A.chunk_grp_ptr.push_back((int32_t)(grp_off + e));
      ga.insert(ga.end(), L.ga.begin(), L.ga.end());
      gb.insert(gb.end(), L.gb.begin(), L.gb.end());
      for (int64_t e : L.grp_end) A.grp_rng.push_back(ga_off + e);
      A.grp_tile.insert(A.grp_tile.end(), L.grp_tile.begin(), L.grp_tile.end());
      for (size_t k = 0; k < L.last_of.size(); ++k) A.last_chunk[L.t0 + (int64_t)k] = (int32_t)(ch_off + L.last_of[k]);
    }
    A.nchunk = (int64_t)A.chunk_tile.size();
    A.ngrp = (int32_t)A.grp_tile.size();
    // one pair array: chunk pairs first (as indexed by chunk_rng), group
    // pairs after them (grp_rng offset by the chunk pair count)
    const int64_t off = (int64_t)A.upd_a.size();
    A.upd_a.insert(A.upd_a.end(), ga.begin(), ga.end());
    A.upd_b.insert(A.upd_b.end(), gb.begin(), gb.end());
    for (auto& v : A.grp_rng) v += off;
  }

  clk.mark("update pairs + chunks");
  // ---------------- task lists ----------------
  auto sort_tasks = [](std::vector<TileTask>& v) {
    std::stable_sort(v.begin(), v.end(),
                     [](const TileTask& x, const TileTask& y) { return x.level < y.level; });
  };
  A.factor_tasks.clear();
  for (int64_t c = 0; c < A.nchunk; ++c) {
    const int32_t J = A.tile_col[A.chunk_tile[c]];
    A.factor_tasks.push_back({0, 0, (int32_t)c, A.flevel[J]});
  }
  for (int32_t g = 0; g < A.ngrp; ++g) A.factor_tasks.push_back({1, 0, g, 0});
  sort_tasks(A.factor_tasks);

  // dependency graph of the factor tasks for the ready-queue scheduler:
  // chunk c waits for the LAST chunk of every tile its pairs read, for the
  // previous chunk of its own tile, and (last chunk of an off-diagonal
  // tile) for the last chunk of the diagonal tile of its column.
  {
    const int64_t ntask = (int64_t)A.factor_tasks.size();
    std::vector<int32_t> task_of_chunk(A.nchunk), task_of_grp(std::max(A.ngrp, 1));
    for (int64_t i = 0; i < ntask; ++i) {
      if (A.factor_tasks[i].type == 0) task_of_chunk[A.factor_tasks[i].id] = (int32_t)i;
      else task_of_grp[A.factor_tasks[i].id] = (int32_t)i;
    }
    std::vector<std::vector<int32_t>> deps(ntask);
    par_for(ntask, [&](int64_t i0, int64_t i1) {  // each task's list is its own
    for (int64_t i = i0; i < i1; ++i) {
      std::vector<int32_t>& d = deps[i];
      if (A.factor_tasks[i].type == 1) {
        const int32_t g = A.factor_tasks[i].id;
        for (int64_t u = A.grp_rng[g]; u < A.grp_rng[g + 1]; ++u) {
          d.push_back(task_of_chunk[A.last_chunk[A.upd_a[u]]]);
          d.push_back(task_of_chunk[A.last_chunk[A.upd_b[u]]]);
        }
        std::sort(d.begin(), d.end());
        d.erase(std::unique(d.begin(), d.end()), d.end());
        continue;
      }
      const int32_t c = A.factor_tasks[i].id;
      const int32_t t = A.chunk_tile[c];
      for (int32_t g = A.chunk_grp_ptr[c]; g < A.chunk_grp_ptr[c + 1]; ++g) d.push_back(task_of_grp[g]);
      for (int64_t u = A.chunk_rng[c]; u < A.chunk_rng[c + 1]; ++u) {
        d.push_back(task_of_chunk[A.last_chunk[A.upd_a[u]]]);
        d.push_back(task_of_chunk[A.last_chunk[A.upd_b[u]]]);
      }
      if (!(A.chunk_flags[c] & 1)) d.push_back(task_of_chunk[c - 1]);
      if ((A.chunk_flags[c] & 2) && A.tile_row[t] != A.tile_col[t])
        d.push_back(task_of_chunk[A.last_chunk[A.colptr[A.tile_col[t]]]]);
      std::sort(d.begin(), d.end());
      d.erase(std::unique(d.begin(), d.end()), d.end());
    }
    });
    clk.mark("factor deps");
    A.f_ndep.assign(ntask, 0);
    A.f_succ_ptr.assign(ntask + 1, 0);
    for (int64_t i = 0; i < ntask; ++i) {
      A.f_ndep[i] = (int32_t)deps[i].size();
      for (int32_t p : deps[i]) A.f_succ_ptr[p + 1]++;
    }
    for (int64_t i = 0; i < ntask; ++i) A.f_succ_ptr[i + 1] += A.f_succ_ptr[i];
    A.f_succ.assign(A.f_succ_ptr[ntask], 0);
    std::vector<int32_t> w(A.f_succ_ptr.begin(), A.f_succ_ptr.end() - 1);
    for (int64_t i = 0; i < ntask; ++i)
      for (int32_t p : deps[i]) A.f_succ[w[p]++] = (int32_t)i;
    A.f_ready0.clear();
    for (int64_t i = 0; i < ntask; ++i)
      if (A.f_ndep[i] == 0) A.f_ready0.push_back((int32_t)i);
    clk.mark("factor succ CSR");
    // bottom levels (estimated remaining path length, in pair-GEMM units)
    std::vector<int32_t> order;
    {
      std::vector<int32_t> indeg(A.f_ndep.begin(), A.f_ndep.end());
      order = A.f_ready0;
      for (size_t k = 0; k < order.size(); ++k) {
        const int32_t t = order[k];
        for (int32_t q = A.f_succ_ptr[t]; q < A.f_succ_ptr[t + 1]; ++q)
          if (--indeg[A.f_succ[q]] == 0) order.push_back(A.f_succ[q]);
      }
    }
    // cost model (microseconds, measured on B200 with 2 CTAs per SM):
    // ~5 us fixed per task, ~4.5 us per pair GEMM, ~45 us for a diagonal
    // POTRI, ~5 us for an off-diagonal TRSM
    std::vector<double> cost(ntask), bl(ntask, 0.0);
    for (int64_t t = 0; t < ntask; ++t) {
      const TileTask& tk = A.factor_tasks[t];
      if (tk.type == 1) {
        cost[t] = 5.0 + 4.5 * (double)(A.grp_rng[tk.id + 1] - A.grp_rng[tk.id]);
      } else {
        const int32_t c = tk.id, tt = A.chunk_tile[c];
        cost[t] = 5.0 + 4.5 * (double)(A.chunk_rng[c + 1] - A.chunk_rng[c]);
        if (A.chunk_flags[c] & 2) cost[t] += (A.tile_row[tt] == A.tile_col[tt]) ? 45.0 : 5.0;
      }
    }
    for (int64_t k = (int64_t)order.size() - 1; k >= 0; --k) {
      const int32_t t = order[k];
      double m = 0.0;
      for (int32_t q = A.f_succ_ptr[t]; q < A.f_succ_ptr[t + 1]; ++q) m = std::max(m, bl[A.f_succ[q]]);
      bl[t] = cost[t] + m;
    }
    clk.mark("factor bottom levels");
    // list-schedule simulation with `workers` workers, highest bottom level
    // first; the start order becomes the GPU claim order
    double makespan = 0.0;
    {
      std::vector<int32_t> indeg(A.f_ndep.begin(), A.f_ndep.end());
      std::priority_queue<std::pair<double, int32_t>> ready;  // (bl, task)
      std::priority_queue<std::pair<double, int32_t>, std::vector<std::pair<double, int32_t>>,
                          std::greater<std::pair<double, int32_t>>> running;  // (finish, task)
      // Claim priority: the bottom level; for throughput-bound DAGs optionally
      // quantised into bands of R tile rows' worth of critical path, with the
      // tasks of a band ordered by blocks of C tile columns (PINLA_FACTOR_LOCALITY
      // = "R,C"): the tasks running together then cover an R x (k C) patch of
      // output tiles that shares its operand tile rows in L2, instead of a slanted
      // wavefront of tiles with distinct operands.  Any priority gives a
      // topological claim order (tasks are taken from the simulated READY set).
      std::vector<double> prio_v;
      const double* prio = bl.data();
      {
        int R = 0, C = 4;
        if (const char* e = getenv("PINLA_FACTOR_LOCALITY")) sscanf(e, "%d,%d", &R, &C);
        if (R > 0 && C > 0 && throughput_dag) {
          double bm = 1e-9;
          for (double v : bl) bm = std::max(bm, v);
          const double wb = R * bm / std::max(1, fdepth0);  // R levels of the critical path
          prio_v.resize(ntask);
          for (int64_t t = 0; t < ntask; ++t) {
            const TileTask& tk = A.factor_tasks[t];
            const int32_t tile = tk.type == 1 ? A.grp_tile[tk.id] : A.chunk_tile[tk.id];
            const double band = std::floor(bl[t] / wb);
            const double frac = (bl[t] - band * wb) / wb;
            prio_v[t] = band * 1e9 + (double)(NT / C + 1 - A.tile_col[tile] / C) * 1e3 + std::min(999.0, frac * 999.0);
          }
          prio = prio_v.data();
        }
      }
      for (int32_t t : A.f_ready0) ready.push({prio[t], t});
      A.f_order.clear();
      A.f_order.reserve(ntask);
      double now = 0.0;
      int busy = 0;
      const int P = std::max(1, workers);
      while ((int64_t)A.f_order.size() < ntask) {
        while (busy < P && !ready.empty()) {
          const int32_t t = ready.top().second;
          ready.pop();
          A.f_order.push_back(t);
          running.push({now + cost[t], t});
          ++busy;
        }
        if (running.empty()) break;  // cannot happen for a DAG
        const auto ev = running.top();
        running.pop();
        --busy;
        now = ev.first;
        const int32_t t = ev.second;
        for (int32_t q = A.f_succ_ptr[t]; q < A.f_succ_ptr[t + 1]; ++q)
          if (--indeg[A.f_succ[q]] == 0) ready.push({prio[A.f_succ[q]], A.f_succ[q]});
      }
      if ((int64_t)A.f_order.size() != ntask) throw std::runtime_error("factor task graph is not a DAG");
      makespan = now;
    }
    clk.mark("factor list schedule");
    double blmax = 1e-9;
    for (double v : bl) blmax = std::max(blmax, v);
    // critical lane (Analysis::f_nlane): lane tasks move to the end of the
    // claim order, keeping their relative (topological) order
    A.f_nlane = 0;
    // (only for one long chain: a deep DAG — forward depth > NT/4, as in the
    // time-major block-tridiagonal orderings — whose critical path dominates)
    int32_t depth = 0;
    for (int32_t I = 0; I < NT; ++I) depth = std::max(depth, A.flevel[I] + 1);
    // Since the warp-specialised kernel (one CTA per SM, producer run-ahead,
    // continuations, publisher warp) the lane no longer pays: off is 4-5 %
    // faster on c3 x 1, c4 x 1, c5 x 2 / x 3 and equal on c5 x 1
    // (profiles/lane_ab_r02.txt).  It stays available with PINLA_FACTOR_LANE=1.
    if (factor_lane == 1) {
      std::vector<char> lane(ntask, 0);
      for (int64_t t = 0; t < ntask; ++t) {
        const TileTask& tk = A.factor_tasks[t];
        if (tk.type != 0 || !(A.chunk_flags[tk.id] & 2)) continue;
        const int32_t tt = A.chunk_tile[tk.id];
        const int32_t J = A.tile_col[tt];
        if (A.tile_row[tt] == J || tt == A.colptr[J] + 1) lane[t] = 1;
      }
      std::vector<int32_t> o2;
      o2.reserve(ntask);
      for (int32_t t : A.f_order)
        if (!lane[t]) o2.push_back(t);
      for (int32_t t : A.f_order)
        if (lane[t]) o2.push_back(t);
      A.f_nlane = (int32_t)(ntask - (int64_t)std::count(lane.begin(), lane.end(), 0));
      A.f_order.swap(o2);
    }
    A.f_chain_ratio = blmax / std::max(makespan, 1e-9);
    A.f_depth = depth;
    if (getenv("PINLA_VERBOSE"))
      fprintf(stderr, "pinla: factor DAG depth %d of %d tile rows, critical path / makespan %.3f (P = %d), lane tasks %d\n",
              depth, NT, A.f_chain_ratio, std::max(1, workers), A.f_nlane);
    A.f_prio.assign(ntask, 0);
    for (int64_t t = 0; t < ntask; ++t) {
      int c = (int)((1.0 - bl[t] / blmax) * kPrioClasses);
      A.f_prio[t] = std::min(std::max(c, 0), kPrioClasses - 1);
    }
    // renumber the base tasks in claim order: the claim index is then the
    // task id itself (no order[] indirection on the GPU's claim path)
    {
      std::vector<int32_t> nid(ntask);
      for (int64_t k = 0; k < ntask; ++k) nid[A.f_order[k]] = (int32_t)k;
      std::vector<TileTask> ft(ntask);
      std::vector<int32_t> nd(ntask), pr(ntask), sp(ntask + 1, 0), su(A.f_succ.size());
      for (int64_t t = 0; t < ntask; ++t) {
        ft[nid[t]] = A.factor_tasks[t];
        nd[nid[t]] = A.f_ndep[t];
        pr[nid[t]] = A.f_prio[t];
        sp[nid[t] + 1] = A.f_succ_ptr[t + 1] - A.f_succ_ptr[t];
      }
      for (int64_t t = 0; t < ntask; ++t) sp[t + 1] += sp[t];
      par_for(ntask, [&](int64_t t0, int64_t t1) {  // each task writes its own range
        for (int64_t t = t0; t < t1; ++t) {
          int32_t w = sp[nid[t]];
          for (int32_t q = A.f_succ_ptr[t]; q < A.f_succ_ptr[t + 1]; ++q) su[w++] = nid[A.f_succ[q]];
          std::sort(su.begin() + sp[nid[t]], su.begin() + w);
        }
      });
      for (auto& r : A.f_ready0) r = nid[r];
      std::sort(A.f_ready0.begin(), A.f_ready0.end());
      A.factor_tasks.swap(ft);
      A.f_ndep.swap(nd);
      A.f_prio.swap(pr);
      A.f_succ_ptr.swap(sp);
      A.f_succ.swap(su);
      for (int64_t k = 0; k < ntask; ++k) A.f_order[k] = (int32_t)k;
    }
  }

  clk.mark("factor DAG + list schedule");
  // solves, right-looking: P(I,K) = L(I,K) y_K as its own task once y_K is
  // final (type 1, id = tile), row task F(I) sums them (type 0, id = I);
  // backward Q(I,J) = L(I,J)^T x_I (type 3, id = tile), B(J) (type 2, id = J)
  // Products are grouped (Analysis::sg_*): a group task waits for the
  // vector of its newest tile (its task level) and streams its tiles in
  // readiness order.
  A.solve_tasks.clear();
  A.sg_lo.clear();
  A.sg_hi.clear();
  A.sg_line.clear();
  A.sf_ptr.assign(NT + 1, 0);
  A.sb_ptr.assign(NT + 1, 0);
  // group cap: long tile-row chains (time-major block-tridiagonal orderings,
  // forward depth ~ NT/2) stream many tiles per row behind the chain, so large
  // groups; shallow nested-dissection DAGs keep groups short (latency)
  int32_t fdepth = 0;
  for (int32_t I = 0; I < NT; ++I) fdepth = std::max(fdepth, A.flevel[I] + 1);
  const bool chain = 4LL * fdepth > NT;
  const int32_t gcap = solve_group_cap > 0 ? solve_group_cap : (chain ? 16 : 4);
  A.solve_links = solve_links >= 0 ? std::min(solve_links, 2) : (chain ? 2 : 0);
  const int32_t nex = std::max(1, A.solve_links);  // products computed inside the row task
  for (int32_t I = 0; I < NT; ++I) A.solve_tasks.push_back({0, 0, I, 3 * A.flevel[I]});
  for (int32_t I = 0; I < NT; ++I) {
    // the newest off-diagonal K of row I (the link) is computed inside the
    // row task; the others [q0, e) are cut from the newest end: 1, 2, 4, ...
    const int32_t q0 = A.rowptr[I];
    int32_t e = A.rowptr[I + 1] - 1 - nex;
    std::vector<std::pair<int32_t, int32_t>> gs;
    for (int32_t sz = 1; e > q0; sz = std::min(2 * sz, gcap)) {
      const int32_t lo = std::max(q0, e - sz);
      gs.push_back({lo, e});
      e = lo;
    }
    A.sf_ptr[I] = (int32_t)A.sg_lo.size();
    for (auto it = gs.rbegin(); it != gs.rend(); ++it) {
      const int32_t g = (int32_t)A.sg_lo.size();
      A.sg_lo.push_back(it->first);
      A.sg_hi.push_back(it->second);
      A.sg_line.push_back(I);
      int32_t lv = 0;  // the group waits for every y_K it reads
      for (int32_t q = it->first; q < it->second; ++q) lv = std::max(lv, A.flevel[A.row_col[q]]);
      A.solve_tasks.push_back({1, 0, g, 3 * lv + 1});
    }
  }
  A.sf_ptr[NT] = (int32_t)A.sg_lo.size();
  sort_tasks(A.solve_tasks);
  {
    std::vector<TileTask> bw;
    for (int32_t J = 0; J < NT; ++J) {
      bw.push_back({2, 0, J, 3 * A.blevel[J]});
      // the nearest off-diagonal I of column J (the link) is handled inside
      // the column task; the others [colptr[J]+2, end) are cut from the
      // nearest end
      const int32_t q1 = A.colptr[J + 1];
      int32_t b = A.colptr[J] + 1 + nex;
      std::vector<std::pair<int32_t, int32_t>> gs;
      for (int32_t sz = 1; b < q1; sz = std::min(2 * sz, gcap)) {
        const int32_t hi = std::min(q1, b + sz);
        gs.push_back({b, hi});
        b = hi;
      }
      A.sb_ptr[J] = (int32_t)A.sg_lo.size();
      for (auto it = gs.rbegin(); it != gs.rend(); ++it) {
        const int32_t g = (int32_t)A.sg_lo.size();
        A.sg_lo.push_back(it->first);
        A.sg_hi.push_back(it->second);
        A.sg_line.push_back(J);
        int32_t lv = 0;
        for (int32_t q = it->first; q < it->second; ++q) lv = std::max(lv, A.blevel[A.tile_row[q]]);
        bw.push_back({3, 0, g, 3 * lv + 1});
      }
    }
    A.sb_ptr[NT] = (int32_t)A.sg_lo.size();
    sort_tasks(bw);
    A.solve_tasks.insert(A.solve_tasks.end(), bw.begin(), bw.end());
  }
  A.n_sgrp = (int32_t)A.sg_lo.size();

  clk.mark("solve tasks");
  sel_thread.join();
  clk.mark("selinv DAG (overlapped)");
  // ---------------- accounting ----------------
  const int64_t g = 2LL * TB * TB * TB;  // one tile GEMM
  int64_t pairs = (int64_t)A.upd_a.size();
  int64_t offdiag = A.nT - NT;
  A.factor_flops = pairs * g + offdiag * g + (int64_t)NT * (2LL * TB * TB * TB / 3);
  int64_t sel = 0;
  for (int32_t J = 0; J < NT; ++J) {
    int64_t c = A.colptr[J + 1] - A.colptr[J];
    sel += c * (c - 1) * g + (c - 1) * g + 2 * g;  // off-diag tasks + diag task
  }
  A.selinv_flops = sel;
  A.solve_bytes = 2LL * (A.nT + NT) * TB * TB * 8;
  {
    auto r8 = [&](int32_t t) { return (int64_t)((A.tstart[t + 1] - A.tstart[t] + 7) & ~7); };
    auto r4 = [&](int32_t t) { return (int64_t)((A.tstart[t + 1] - A.tstart[t] + 3) & ~3); };
    int64_t lim = 0;
    for (int64_t c = 0; c < A.nchunk; ++c) {
      const int32_t t = A.chunk_tile[c];
      const int32_t I = A.tile_row[t], J = A.tile_col[t];
      for (int64_t u = A.chunk_rng[c]; u < A.chunk_rng[c + 1]; ++u)
        lim += 2 * r8(I) * r8(J) * r4(A.tile_col[A.upd_a[u]]);
      if ((A.chunk_flags[c] & 2) && I != J) lim += 2 * r8(I) * r8(J) * r4(J);
    }
    for (int32_t g = 0; g < A.ngrp; ++g) {
      const int32_t t = A.grp_tile[g];
      for (int64_t u = A.grp_rng[g]; u < A.grp_rng[g + 1]; ++u)
        lim += 2 * r8(A.tile_row[t]) * r8(A.tile_col[t]) * r4(A.tile_col[A.upd_a[u]]);
    }
    A.factor_flops_limited = lim + (int64_t)NT * (2LL * TB * TB * TB / 3);
  }

  A.pad_of_orig.assign(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    int64_t j = A.iperm[i];
    int32_t t = tile_of[j];
    A.pad_of_orig[i] = (int64_t)t * TB + (j - A.tstart[t]);
  }
  clk.mark("accounting");
}

}  // namespace pinla
