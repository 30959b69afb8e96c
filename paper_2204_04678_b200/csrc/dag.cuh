// Argument blocks of the persistent tile-DAG kernels (device pointers only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pinla {

// Scheduler of the factorization DAG.  Task instance i = s * ntask + t
// (slot s, base task t).  Instances are claimed with ONE fetch-and-add in a
// host-computed list-schedule order (critical path first, slots
// interleaved); a claimed instance waits on its own dependency counter,
// which its producers count down when they finish.  The order is
// topological, so no claimed instance can wait on an unclaimed one.
constexpr int kQueues = 8;
struct DagQueue {
  int ntask;              // base tasks
  const int* ndep0;       // [ntask] dependency counts
  const int* succ_ptr;    // [ntask+1]
  const int* succ;        // successor base tasks
  const int* prio;        // [ntask] priority class
  int nready0;
  int* cnt;               // [S*ntask] remaining dependencies (init per launch)
  unsigned long long* queue;  // unused (reserved)
  int* ctr;               // [0]: claim counter
  int cap;
  unsigned epoch;
  const int* act_slots;   // [nact] active slot ids
  int nact;
  const int* order;       // [ntask] claim order (simulated list schedule)
  int fifo;               // 1: ready-queue mode (no claimed task ever waits)
  int* fqueue;            // [S*ntask] FIFO entries (-1 = not yet pushed)
  const int* ready0;      // [nready0] initially ready base tasks (FIFO mode)
  const int* hot;         // [ntask] or null: run by the CTA that readies it (FIFO mode)
  int* claimed;           // [S*ntask] or null: epoch tag of the launch that claimed the instance
                          // (warp-specialised factor kernel: chunk continuations, factor_ws.cu)
  int nlane;              // factor: the last nlane base tasks form the critical lane (list mode)
  int lane_ctas;          // CTAs that publish their SM for the lane (<= kLaneCtasMax)
};
// critical lane of the factor kernel: CTAs 0..kLaneCtas-1 and every CTA that
// shares an SM with one of them claim only lane tasks (ctr[2]: lane claim
// counter, ctr[3..3+kLaneCtas): SM id + 1 of lane CTA k, written at start)
constexpr int kLaneCtas = 8;      // default lane_ctas
constexpr int kLaneCtasMax = 12;  // ctr[3 .. 3 + lane_ctas)
#ifndef PINLA_LANE_CORES
#define PINLA_LANE_CORES 1
#endif
constexpr int kLaneCoRes = PINLA_LANE_CORES;  // co-resident CTAs: 1 join the lane, 2 exit

// Everything a factor task needs before its first tile load, in one
// 96-byte record per base task (fetched while the task's dependency counter
// is awaited, instead of a chain of dependent index loads).
struct __align__(16) FTask {
  int type;           // 0 chunk, 1 parallel partial group
  int id;             // chunk id / group id
  int tid;            // output tile (chunk) or the group's tile
  int flags;          // chunk flags: bit0 first chunk, bit1 last chunk
  int I, J, mI, nJ;   // tile row/col and their heights
  long long u0, u1;   // update pair range
  long long q0, q1;   // Q(I,J) entries of the tile (first chunk)
  int g0, g1;         // groups added in at the start of the chunk
  int succ0, succ1;   // successor range (q.succ)
  int pa0, pb0;       // first pair's tiles (-1: no pair)
  int k0;             // K extent of the first pair
  int next;           // inner chunk: base task of the next chunk of the same tile (its only
                      // successor) when that chunk may run as a continuation, else -1
};
static_assert(sizeof(FTask) == 96, "FTask layout");

struct FactorArgs {
  const FTask* rec;   // [n_base] task records
  const int* upd_k;   // [npairs] K extent (row count of tile column K) per pair
  int S;              // slots in the launch (task index = base * S + slot)
  int64_t n_base;     // base tasks
  const int4* tasks;  // (type, -, id, level)
  double* L;          // [S][nT][64*64]  (running sums, then the factor)
  double* Linv;       // [S][NT][64*64]
  int64_t nT;
  int NT;
  const int* tile_row;
  const int* tile_col;
  const int64_t* tstart;
  const int* upd_a;
  const int* upd_b;
  const int64_t* chunk_rng;  // [nchunk+1]
  const int* chunk_tile;     // [nchunk]
  const int* chunk_flags;    // [nchunk] bit0 first, bit1 last
  const int* tbsz;           // [NT] rows of each tile (<= 64)
  const int64_t* grp_rng;    // [ngrp+1]
  const int* grp_tile;       // [ngrp]
  const int* chunk_grp_ptr;  // [nchunk+1] groups added at the start of a chunk
  double* G;                 // [S][ngrp][64*64] group partial sums
  int ngrp;
  const int64_t* qptr;       // [nT+1]
  const int* qloc;           // [nq]
  const double* qv;          // [S][nq]
  int64_t nq;
  const int64_t* diagq;  // [NT*64]
  int* status;           // [S]  INT_MAX = ok, else failing permuted row
  double rel_tol;
  unsigned long long* trace;  // debug: [total tasks][8] (claim, pairs done, end, smid, pop start,
                              // setup done, finalize math done, stores done) or null
  double flops_per_level;     // executed flops of one slot / levels of the factor DAG (kernel choice)
  DagQueue q;
};

struct SolveArgs {
  int S;
  int64_t n_base;
  const int4* tasks;
  int* counter;
  int epoch;
  const int* active;
  // every vector exchanged between tasks is in "LL" form: 128 words per
  // tile row, word k = (tag << 32) | 32-bit half (k & 1) of value k >> 1; a
  // consumer polls the data itself (no producer fence, no flag -> data round
  // trip, no counters)
  unsigned long long* llY;  // [S][NT][128]
  unsigned long long* llX;  // [S][NT][128]
  unsigned long long* llP;  // [S][n_grp][128] product-group partials (fwd tag 2E, bwd 2E+1)
  const int4* grp;          // [n_grp] (lo, hi, row / column, -): see Analysis::sg_*
  int n_grp;
  const int* fgp;           // [NT+1] forward groups of row I (oldest first)
  const int* bgp;           // [NT+1] backward groups of column J (farthest first)
  const double* L;
  const double* Linv;
  int64_t nT;
  int NT;
  const int* tile_row;
  const int* tile_col;
  const int* colptr;
  const int* rowptr;   // [NT+1] row form of the tile pattern (K ascending)
  const int* row_tid;  // [nT]
  const int* row_col;  // [nT]
  const double* b;   // [S][NT*64]
  double* x;         // [S][NT*64] (plain copy of x for the caller)
  // chain-link tiles (null: off), from link_tiles_kernel: M[s][k][NT] with
  // k = 0/1 forward Linv_I L(I,l) for the newest / second-newest column l of
  // row I, k = 2/3 backward L(l,J) Linv_J for the nearest / second-nearest
  // row l of column J.  The row task applies Linv to everything else before
  // its links arrive; each chain step is then one 64x64 GEMV.
  const double* M;
  int nlinks;  // 1 or 2 links per row / column when M is set
  unsigned long long* trace;  // debug: [tasks][8] (claim, rhs, psum, -, ready, end, smid, -) or null
};

// chain-link tiles after a factorization (see SolveArgs::M)
struct LinkArgs {
  int S;
  int nlink;
  const int4* links;  // (k: 0/1 fwd, 2/3 bwd; row or column; link tile; link source)
  const int* active;
  const double* L;
  const double* Linv;
  double* M;          // [S][4][NT][64*64]
  int64_t nT;
  int NT;
  const int* tbsz;
};

struct SelinvArgs {
  int S;
  int64_t n_base;
  const int4* tasks;
  const int* lslot;  // [S] factor slot feeding selinv slot s
  const double* L;
  const double* Linv;
  double* Sg;        // [S][nT][64*64]
  const int* tbsz;   // [NT]
  int64_t nT;
  int NT;
  const int* tile_row;
  const int* tile_col;
  const int* pa;
  const int* pb;
  const int* mode;
  const int64_t* chunk_rng;
  const int* chunk_tile;
  const int* chunk_flags;
  const int64_t* grp_rng;   // [ngrp+1]
  const int* grp_tile;      // [ngrp]
  const int* tile_grp_ptr;  // [nT+1]
  double* G;                // [S][ngbuf][64*64] group scratch ring
  int ngrp;
  const int* gbuf;          // [ngrp] ring buffer of each group
  int ngbuf;
  unsigned long long* trace;  // debug: [tasks][4] (t_claimed, t_ready, t_end, smid) or null
  int SL;                     // factor slots behind L / Linv (tensor-map extents)
  double flops_per_level;     // selinv flops / levels of the DAG (kernel choice)
  DagQueue q;
};

size_t dag_smem_bytes();
cudaError_t launch_factor(const FactorArgs& a, cudaStream_t st);
// warp-specialised factor kernel (factor_ws.cu): producer warp + TMA bulk
// box loads + 8 MMA warps per SM; PINLA_FACTOR_WS = 0 never, 1 (default) for
// DAGs without a critical lane, 2 always
int factor_ws_mode();
cudaError_t launch_factor_ws(const FactorArgs& a, cudaStream_t st);
cudaError_t launch_queue_init(const DagQueue& q, int S, cudaStream_t st);
cudaError_t launch_solve(const SolveArgs& a, cudaStream_t st);
cudaError_t launch_link_tiles(const LinkArgs& a, cudaStream_t st);
cudaError_t launch_selinv(const SelinvArgs& a, cudaStream_t st);
// warp-specialised selected inversion (selinv_ws.cu, the default);
// PINLA_SELINV_WS=0 selects the 128-thread kernel
int selinv_ws_mode();
cudaError_t launch_selinv_ws(const SelinvArgs& a, cudaStream_t st);
cudaError_t launch_selinv_diag(const double* Sg, int64_t nT, int NT, const int* colptr,
                               double* var_pad, cudaStream_t st);

}  // namespace pinla
