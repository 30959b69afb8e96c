// Host-side one-time structural analysis for the tile-DAG engine.
//
// Replaces the reference's per-pattern analyze() (cholesky.py:88-137:
// ordering -> permuted row form -> etree -> column patterns) with a
// TILE-level symbolic factorization: the permuted index range is cut into
// tiles of TB=64 rows (dense trailing "arrow" vertices get their own tiles),
// the tile pattern of L is the block elimination of the tile pattern of Q,
// and every numeric pass (factor / solve / selinv) becomes a list of
// dependency-ordered tile tasks executed by one persistent kernel.
#pragma once
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <cstdlib>
#include <exception>
#include <thread>
#include <vector>

namespace pinla {

constexpr int TB = 64;  // tile edge

// phase timings on stderr with PINLA_VERBOSE=1 (tuning)
struct PhaseClock {
  bool on = getenv("PINLA_VERBOSE") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "  %-36s %8.3f s\n", what, std::chrono::duration<double>(now - t).count());
    t = now;
  }
};



// Host parallel-for over [0, n) in contiguous ranges for the build's
// per-column / per-entry / per-tile loops.  Every index writes its own
// outputs, so the results do not depend on the thread count; the first
// exception of any range is rethrown after the join.
template <class F>
inline void par_for(int64_t n, F&& fn, int64_t grain = 1 << 13) {
  // PINLA_BUILD_THREADS caps the threads (testing: results are identical)
  static const int64_t hw = getenv("PINLA_BUILD_THREADS")
                                ? std::max(1, atoi(getenv("PINLA_BUILD_THREADS")))
                                : (int64_t)std::max(1u, std::thread::hardware_concurrency());
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>({hw, 16, (n + grain - 1) / grain}));
  if (nt <= 1) {
    fn((int64_t)0, n);
    return;
  }
  std::vector<std::exception_ptr> err(nt);
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t)
    th.emplace_back([&, t] {
      try {
        fn(n * t / nt, n * (t + 1) / nt);
      } catch (...) {
        err[t] = std::current_exception();
      }
    });
  try {
    fn((int64_t)0, n / nt);
  } catch (...) {
    err[0] = std::current_exception();
  }
  for (auto& x : th) x.join();
  for (auto& e : err)
    if (e) std::rethrow_exception(e);
}

struct TileTask {  // 16 bytes, uploaded as int4
  int32_t type;    // task type (kernel specific)
  int32_t slot;    // filled per launch from slot-agnostic list (see engine)
  int32_t id;      // tile id / partial id / tile row
  int32_t level;
};

struct Analysis {
  int64_t n = 0, n_main = 0;
  int32_t NT = 0;                      // tile rows/cols
  std::vector<int64_t> tstart;         // NT+1 permuted boundaries
  std::vector<int64_t> perm, iperm;    // perm[new] = old
  // tile pattern of L, column-major; diagonal tile first in each column
  std::vector<int32_t> colptr;         // NT+1
  std::vector<int32_t> tile_row;       // nT
  std::vector<int32_t> tile_col;       // nT
  int64_t nT = 0;
  // row form (K ascending, includes the diagonal tile last)
  std::vector<int32_t> rowptr, row_col, row_tid;
  // levels
  std::vector<int32_t> flevel;  // forward (factor/forward-solve) column level
  std::vector<int32_t> blevel;  // backward (selinv/backward-solve) level
  // factor: left-looking update pairs of every tile (K ascending), cut into
  // chained in-place chunks whose sizes grow geometrically away from the
  // last pair (1, 4, 8, 16, 16, ...): chunk c of tile t accumulates
  // pairs [chunk_rng[c], chunk_rng[c+1]) into the tile's own buffer after
  // chunk c-1; the last chunk also runs the tile's POTRF / TRSM.
  std::vector<int32_t> upd_a, upd_b;   // tile ids: C(I,J) -= L[a] * L[b]^T
  std::vector<int64_t> chunk_rng;      // nchunk+1 pair ranges
  std::vector<int32_t> chunk_tile;     // owning tile
  std::vector<int32_t> chunk_flags;    // bit0 first chunk, bit1 last chunk
  std::vector<int32_t> last_chunk;     // nT: last chunk of each tile
  int64_t nchunk = 0;
  // parallel partial groups (arrow-row tiles with long update lists): group
  // g sums pairs [grp_rng[g], grp_rng[g+1]) of tile grp_tile[g] into its own
  // scratch tile; the tile's first chunk subtracts its groups in order
  std::vector<int64_t> grp_rng;        // ngrp+1
  std::vector<int32_t> grp_tile;       // ngrp
  std::vector<int32_t> chunk_grp_ptr;  // nchunk+1 -> groups a chunk adds in at its start
  int32_t ngrp = 0;
  // solve product groups: group g sums the GEMVs of tiles [sg_lo[g], sg_hi[g])
  // of one row (forward: row-form positions, K ascending) or one column
  // (backward: column positions = tile ids, streamed I descending) into one
  // partial vector.  Sizes grow geometrically away from the chain link
  // (1, 2, 4, ... up to the cap; 0 = by DAG shape), so a row task sums a handful of
  // partials instead of one per tile.  Forward groups first (row I owns
  // [sf_ptr[I], sf_ptr[I+1]), oldest first), then backward ones (column J
  // owns [sb_ptr[J], sb_ptr[J+1]), farthest first; ids offset by the forward
  // count).
  std::vector<int32_t> sg_lo, sg_hi, sg_line, sf_ptr, sb_ptr;
  int32_t n_sgrp = 0;
  // chain links fused into the row / column tasks (0: one link multiplied
  // by L then Linv; 1 or 2: the newest one or two off-diagonal products via
  // precomputed M = Linv_I L(I,K) tiles, excluded from the groups)
  int32_t solve_links = 0;
  // task lists (slot-agnostic; slot field = 0, expanded per launch)
  std::vector<TileTask> factor_tasks, solve_tasks, selinv_tasks;
  // dynamic-scheduling graphs over factor_tasks: dependency counts, successor
  // CSR and the initially ready tasks (indices into factor_tasks)
  std::vector<int32_t> f_ndep, f_succ_ptr, f_succ, f_ready0;
  std::vector<int32_t> f_prio;   // priority class per factor task (0 = most critical)
  std::vector<int32_t> f_order;  // claim order: simulated list schedule (critical path first)
  // critical lane: on chain-bound DAGs (critical path > half the simulated
  // makespan) the last chunks of the diagonal tiles and of the nearest
  // sub-diagonal tile of each column are numbered LAST (f_nlane tasks, in
  // list-schedule order) and claimed only by the lane CTAs, which run
  // nothing else (the POTRI chain does not share its SM with bulk updates)
  int32_t f_nlane = 0;
  double f_chain_ratio = 0.0;  // simulated critical path / makespan of the factor DAG
  int32_t f_depth = 0;         // levels of the factor DAG (tile-column levels)
  // selected inversion: chained chunks over per-tile pair lists.  pair u:
  // op(A)(i,k) from tile s_pa[u], op(B)(k,n) from tile s_pb[u]; s_mode[u]
  // bit0 A from L (else Sigma), bit1 A transposed, bit2 B from L, bit3 B
  // transposed.  Chunk flags as for the factor (bit0 first, bit1 last).
  std::vector<int32_t> s_pa, s_pb, s_mode;
  std::vector<int64_t> s_chunk_rng;
  std::vector<int32_t> s_chunk_tile, s_chunk_flags, s_last_chunk;
  std::vector<int32_t> s_ndep, s_succ_ptr, s_succ, s_ready0, s_order;
  int64_t s_nchunk = 0;
  // parallel partial groups of the diagonal tiles' lists (all their inputs
  // finish together): group g sums pairs [s_grp_rng[g], s_grp_rng[g+1]) of
  // tile s_grp_tile[g] into scratch; the tile's first chunk adds them
  std::vector<int64_t> s_grp_rng;
  std::vector<int32_t> s_grp_tile, s_tile_grp_ptr;
  int32_t s_ngrp = 0;
  // group scratch is a ring of s_ngbuf tiles: group g writes buffer s_grp_buf[g]
  // (reuse ordered by a DAG edge from the previous user's consumer)
  std::vector<int32_t> s_grp_buf;
  std::vector<int32_t> s_hot;  // [selinv task] chain-critical (continuation) tasks
  int32_t s_ngbuf = 0;
  // flop / byte accounting
  int64_t factor_flops = 0, selinv_flops = 0, solve_bytes = 0;
  int64_t factor_flops_limited = 0;  // flops the M/N/K-limited tile kernels execute
  int64_t tid_of(int32_t I, int32_t J) const;  // -1 if absent
  // padded layout helpers
  int64_t pad_of_perm(int64_t j) const;        // permuted index -> padded pos
  std::vector<int64_t> pad_of_orig;            // original index -> padded pos
  int64_t npad() const { return (int64_t)NT * TB; }
};

// Build the analysis for the lower-CSC pattern (original order) and ordering.
// n_dense trailing entries of perm form the arrow tiles.
void analyze_tiles(Analysis& A, int64_t n, const int64_t* indptr, const int64_t* indices,
                   const int64_t* perm, int64_t n_dense, const int64_t* tile_bounds = nullptr,
                   int64_t n_tile_bounds = 0, int workers = 296, int solve_group_cap = 0,
                   int solve_links = -1, int factor_lane = -1);

}  // namespace pinla
