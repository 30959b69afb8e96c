// Persistent tile-DAG kernels: numeric factorization, forward/backward
// solves and Takahashi selected inversion, each ONE launch per call over all
// theta slots of the batch.
//
// Scheduling: the host builds a dependency-ordered (topological) task list
// once per pattern (analysis.cpp); every CTA claims the next task with one
// atomicAdd and spins on the ready flags of the tiles it reads.  A task only
// ever waits on tasks with a smaller index, which were claimed by running
// CTAs, so the scheme cannot deadlock whatever the residency.  Each output
// tile is produced by exactly one task with a fixed accumulation order, so
// results are bitwise reproducible run to run and independent of the slot
// count and of the number of GPUs a batch is sharded over.
//
// Reference counterparts (/root/reference/pkg/src/parinla):
//   factor_kernel  <- kernels.factor_range (kernels.py:99-143) under
//                     run_tree_tasks (runtime.py:180-268); pivot rule
//                     d > 1e-13 * Q_jj (cholesky.py:31-32, kernels.py:138);
//                     log det = 2 sum log L_jj (cholesky.py:321)
//   solve_kernel   <- solve_lower / solve_lower_t (kernels.py:146-165)
//   selinv_kernel  <- selinv_range (kernels.py:185-246), root-first schedule
//                     (cholesky.py:378-391), block Takahashi form
#include <algorithm>
#include <climits>
#include <cstdio>

#include "dag.cuh"
#include "tile.cuh"
#include "potri.cuh"

namespace pinla {

// ---------------------------------------------------------------------------
// in-tile dense kernels (smem, 128 threads)

// row-major global tile from an ld-65 smem tile
__device__ __forceinline__ void tile_store_ld(double* G, const double* S, int ld) {
  for (int e = threadIdx.x; e < kTB * kTB; e += kThreads) __stcg(G + e, S[(e >> 6) * ld + (e & 63)]);
}

__device__ __forceinline__ int claim(int* counter) {
  __shared__ int sh_task;
  if (threadIdx.x == 0) sh_task = atomicAdd(counter, 1);
  __syncthreads();
  int t = sh_task;
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------
// factorization

// ---------------------------------------------------------------------------
// ready-queue scheduler

// dependency / ready-slot polls spin this many times before backing off
// with __nanosleep (tuning: -DPINLA_SPIN_SLEEP_AFTER=N via make EXTRA=...)
#ifndef PINLA_SPIN_SLEEP_AFTER
#define PINLA_SPIN_SLEEP_AFTER 4
#endif
constexpr int kSpinSleepAfter = PINLA_SPIN_SLEEP_AFTER;

__global__ void queue_init_kernel(DagQueue q, int S) {
  const int64_t n = (int64_t)S * q.ntask;
  const int64_t ninit = (int64_t)q.nact * q.nready0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    q.cnt[i] = q.ndep0[i % q.ntask];
    if (q.fifo) {
      int v = -1;
      if (i < ninit) v = q.act_slots[i / q.nready0] * q.ntask + q.ready0[i % q.nready0];
      q.fqueue[i] = v;
    }
  }
  if (q.fifo && blockIdx.x == 0 && threadIdx.x == 0) q.ctr[1] = (int)ninit;
}

cudaError_t launch_queue_init(const DagQueue& q, int S, cudaStream_t st) {
  const int64_t n = (int64_t)S * q.ntask;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  cudaMemsetAsync(q.ctr, 0, (2 * kQueues + 1) * sizeof(int), st);
  queue_init_kernel<<<blocks < 1 ? 1 : blocks, 256, 0, st>>>(q, S);
  return cudaGetLastError();
}

__device__ __forceinline__ int ld_relaxed_int(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// claim the next instance in the precomputed list-schedule order (one
// fetch-and-add, slots interleaved) and wait until its dependency counter
// reaches zero; -1 when all instances are claimed.  The order is
// topological, so every awaited producer was claimed earlier by a running
// CTA: no deadlock.
//
// FIFO mode with continuations: a CTA whose completion readies a `hot` task
// runs it next itself (no queue latency on the chain) and leaves a skip marker
// (-2) in the FIFO so that every instance still fills exactly one position.
__device__ __forceinline__ int* queue_cont_slot() {
  __shared__ int cont;
  return &cont;
}
__device__ __forceinline__ void queue_start() {
  if (threadIdx.x == 0) *queue_cont_slot() = -1;
  __syncthreads();
}
__device__ __forceinline__ int queue_pop(const DagQueue& q) {
  __shared__ int sh_inst;
  if (threadIdx.x == 0) {
    const int total = q.nact * q.ntask;
    int inst = -1;
    int* cont = queue_cont_slot();
    if (*cont >= 0) {
      inst = *cont;
      *cont = -1;
      const int pos = atomicAdd(q.ctr + 1, 1);
      st_release(q.fqueue + pos, -2);
    } else {
      for (;;) {
        const int idx = atomicAdd(q.ctr, 1);
        inst = -1;
        if (idx >= total) break;
        if (q.fifo) {
          int spins = 0;
          while ((inst = ld_acquire(q.fqueue + idx)) == -1) { if (++spins > kSpinSleepAfter) __nanosleep(32); }
          if (inst == -2) continue;  // taken as a continuation
        } else {
          const int t = q.order[idx / q.nact];
          inst = q.act_slots[idx % q.nact] * q.ntask + t;
          int spins = 0;
          while (ld_acquire(q.cnt + inst) != 0) {
            if (++spins > kSpinSleepAfter) __nanosleep(32);
          }
        }
        break;
      }
    }
    sh_inst = inst;
  }
  __syncthreads();
  const int r = sh_inst;
  __syncthreads();
  return r;
}

// queue_pop for the factor kernel: the claimed task's record (6 x 16 B) is
// fetched by thread 0 while its dependency counter is awaited and handed to
// the CTA through shared memory
__device__ __forceinline__ int queue_pop_rec(const DagQueue& q, const FTask* rec, FTask* srec,
                                             bool lane) {
  __shared__ int sh_inst;
  if (threadIdx.x == 0) {
    const int nbase = lane ? q.nlane : q.ntask - q.nlane;  // lane tasks are numbered last
    const int t0 = lane ? q.ntask - q.nlane : 0;
    const int total = q.nact * nbase;
    int inst = -1;
    int* cont = queue_cont_slot();
    int4 r[6];
    auto fetch = [&](int t) {
      const int4* p = reinterpret_cast<const int4*>(rec + t);
#pragma unroll
      for (int k = 0; k < 6; ++k) r[k] = __ldg(p + k);
    };
    if (*cont >= 0) {
      inst = *cont;
      *cont = -1;
      fetch(inst % q.ntask);
      const int pos = atomicAdd(q.ctr + 1, 1);
      st_release(q.fqueue + pos, -2);
    } else {
      for (;;) {
        const int idx = atomicAdd(q.ctr + (lane ? 2 : 0), 1);
        inst = -1;
        if (idx >= total) break;
        if (q.fifo) {
          int spins = 0;
          while ((inst = ld_acquire(q.fqueue + idx)) == -1) { if (++spins > kSpinSleepAfter) __nanosleep(32); }
          if (inst == -2) continue;  // taken as a continuation
          fetch(inst % q.ntask);
        } else {
          const int t = t0 + idx / q.nact;  // base tasks are numbered in claim order
          inst = q.act_slots[idx % q.nact] * q.ntask + t;
          fetch(t);  // in flight during the wait
          int spins = 0;
          while (ld_acquire(q.cnt + inst) != 0) {
            if (++spins > kSpinSleepAfter) __nanosleep(32);
          }
        }
        break;
      }
    }
    if (inst >= 0) {
      int4* d = reinterpret_cast<int4*>(srec);
#pragma unroll
      for (int k = 0; k < 6; ++k) d[k] = r[k];
    }
    sh_inst = inst;
  }
  __syncthreads();
  const int r = sh_inst;
  __syncthreads();
  return r;
}

// publish this CTA's writes, then count down the successors of `inst`
// (successor range [s0, s1) of q.succ)
// (successor ids prefetched into `ssucc` by succ_prefetch when s1 - s0 <=
// kSuccPre, so the tail of a task has no dependent global load)
constexpr int kSuccPre = kThreads;
// pair lists of up to kPairPre update pairs are staged in smem per task
constexpr int kPairPre = kThreads;
__device__ __forceinline__ void succ_prefetch(const DagQueue& q, int s0, int s1, int* ssucc) {
  if (s1 - s0 <= kSuccPre && threadIdx.x < s1 - s0) ssucc[threadIdx.x] = __ldg(q.succ + s0 + threadIdx.x);
}
// (the CTA barrier orders every thread's tile stores before the successor
// decrements; each decrement is a gpu-scope release, which is cumulative
// over those stores: the __syncthreads + release pattern of CUTLASS's
// semaphore, without a membar in every thread)
__device__ __forceinline__ void queue_complete_rng(const DagQueue& q, int inst, int s0, int s1,
                                                   const int* ssucc) {
  __syncthreads();
  const int base = inst - inst % q.ntask;
  const bool pre = s1 - s0 <= kSuccPre;
  for (int k = s0 + threadIdx.x; k < s1; k += blockDim.x) {
    const int u = base + (pre ? ssucc[k - s0] : q.succ[k]);
    if (q.fifo) {
      if (atom_dec_acq_rel(q.cnt + u) == 1) {
        if (!(q.hot && q.hot[u % q.ntask] && atomicCAS(queue_cont_slot(), -1, u) == -1)) {
          const int pos = atomicAdd(q.ctr + 1, 1);
          st_release(q.fqueue + pos, u);
        }
      }
    } else {
      red_dec_release(q.cnt + u);
    }
  }
  __syncthreads();
}

// publish this CTA's writes, then count down the successors of `inst`
__device__ __forceinline__ void queue_complete(const DagQueue& q, int inst) {
  __threadfence();
  __syncthreads();
  const int t = inst % q.ntask;
  const int base = inst - t;
  for (int k = q.succ_ptr[t] + threadIdx.x; k < q.succ_ptr[t + 1]; k += blockDim.x) {
    const int u = base + q.succ[k];
    if (q.fifo) {
      if (atom_dec_acq_rel(q.cnt + u) == 1) {
        if (!(q.hot && q.hot[u % q.ntask] && atomicCAS(queue_cont_slot(), -1, u) == -1)) {
          const int pos = atomicAdd(q.ctr + 1, 1);
          st_release(q.fqueue + pos, u);
        }
      }
    } else {
      red_dec_release(q.cnt + u);  // no return value to wait for
    }
  }
  __syncthreads();
}

// acc += sign * sum_g T[idx[g]] for g in [g0, g1), in order; the tiles stream
// through two smem buffers (buf2: 2 tiles) with one load in flight
__device__ __forceinline__ void sum_tiles_async(Frag& acc, double* buf2, const double* base,
                                                const int* idx, int g0, int g1, double sign) {
  if (g0 >= g1) return;
  tile_load_async(buf2, base + (int64_t)idx[g0] * kTileElems);
  cp_async_commit();
  for (int g = g0; g < g1; ++g) {
    const int b = (g - g0) & 1;
    if (g + 1 < g1) {
      tile_load_async(buf2 + (b ^ 1) * kSmemTile, base + (int64_t)idx[g + 1] * kTileElems);
      cp_async_commit();
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_group<0>();
    }
    __syncthreads();
    frag_axpy(acc, buf2 + b * kSmemTile, sign);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// factorization (left-looking tile tasks, dynamically scheduled)

// smem: C tile + stage area (4 half operands = 2 pipeline stages); the
// stage area doubles as two full tiles (As, Bs) outside the pair loop
constexpr int kFactorSmem = kSmemTile + 4 * kHalfElems;
static_assert(4 * kHalfElems >= 2 * kSmemTile - 2 * kTB * 0, "stage area too small");

__global__ void __launch_bounds__(kThreads, 2) factor_kernel(FactorArgs a) {
  extern __shared__ __align__(16) double smem[];
  double* C = smem;
  double* stage = smem + kSmemTile;
  double* Bs = stage + kSmemTile;
  __shared__ double qd[kTB];
  __shared__ int sh_fail;
  __shared__ FTask tk;
  __shared__ int ssucc[kSuccPre];
  __shared__ int sp_a[kPairPre], sp_b[kPairPre], sp_k[kPairPre];
  const int ntask = a.q.ntask;
  queue_start();
  // critical-lane role (DagQueue::nlane): CTAs 0..kLaneCtas-1 publish their
  // SM; a CTA on one of those SMs joins the lane (kLaneCoRes = 1) or exits
  // (kLaneCoRes = 2: the lane CTA runs its POTRI chain on an otherwise idle SM) (all CTAs of a persistent
  // grid are resident, and the lowest block ids are dispatched first)
  __shared__ int sh_lane;
  if (threadIdx.x == 0) {
    int lane = 0;
    if (a.q.nlane > 0 && !a.q.fifo) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      if ((int)blockIdx.x < a.q.lane_ctas) {
        st_release(a.q.ctr + 3 + blockIdx.x, (int)smid + 1);
        lane = 1;
      } else {
        for (int k = 0; k < a.q.lane_ctas && k < (int)gridDim.x; ++k) {
          int v;
          while ((v = ld_acquire(a.q.ctr + 3 + k)) == 0) __nanosleep(64);
          if (v == (int)smid + 1) lane = kLaneCoRes;
        }
      }
    }
    sh_lane = lane;
  }
  __syncthreads();
  if (sh_lane == 2) return;  // co-resident with a lane CTA: leave its SM to the chain
  const bool lane = sh_lane != 0;
  for (;;) {
    const unsigned long long t_pop = a.trace ? globaltimer() : 0ull;
    const int inst = queue_pop_rec(a.q, a.rec, &tk, lane);
    if (inst < 0) break;
    const unsigned long long t_claim = a.trace ? globaltimer() : 0ull;
    const int s = inst / ntask;
    const bool skip = *((volatile const int*)(a.status + s)) != INT_MAX;
    const int I = tk.I, J = tk.J, mI = tk.mI, nJ = tk.nJ;
    succ_prefetch(a.q, tk.succ0, tk.succ1, ssucc);
    // the task's pair list (tile ids, K extents) staged in smem up front: the
    // pair pipeline then issues its tile loads without a dependent global
    // index read per half-step (long-scoreboard stalls in the c4 profile)
    const bool pre_pairs = tk.u1 - tk.u0 <= kPairPre;
    if (pre_pairs && threadIdx.x < tk.u1 - tk.u0) {
      sp_a[threadIdx.x] = __ldg(a.upd_a + tk.u0 + threadIdx.x);
      sp_b[threadIdx.x] = __ldg(a.upd_b + tk.u0 + threadIdx.x);
      sp_k[threadIdx.x] = __ldg(a.upd_k + tk.u0 + threadIdx.x);
    }
    __syncthreads();
    const int* upa = pre_pairs ? sp_a : a.upd_a;
    const int* upb = pre_pairs ? sp_b : a.upd_b;
    const int* upk = pre_pairs ? sp_k : a.upd_k;
    const int64_t u0 = pre_pairs ? 0 : tk.u0, u1 = pre_pairs ? tk.u1 - tk.u0 : tk.u1;
    double* Ls = a.L + (int64_t)s * a.nT * kTileElems;
    if (tk.type == 1) {  // parallel partial group of an arrow-row tile
      if (!skip) {
        Frag acc;
        frag_zero(acc);
        const int iss = pair_pipe_prologue(stage, Ls, upa, upb, u0, u1, mI, nJ, tk.pa0,
                                           tk.pb0, tk.k0);
        pair_pipe_run2(acc, stage, Ls, upa, upb, u0, u1, upk, mI, nJ, 1.0, iss);
        frag_store_global(acc, a.G + ((int64_t)s * a.ngrp + tk.id) * kTileElems);
      }
      queue_complete_rng(a.q, inst, tk.succ0, tk.succ1, ssucc);
      continue;
    }
    const int tid = tk.tid;
    const int flags = tk.flags;
    double* Lt = Ls + (int64_t)tid * kTileElems;
    if (!skip) {
      Frag acc;
      // finalize without pairs of an off-diagonal tile: Linv_J (ready, it is
      // a dependency) streams in from the start
      const bool pre_linv = (flags & 2) && I != J && u0 == u1;
      // diagonal finalize: the pivot-rule reference values Q_jj load early
      if ((flags & 2) && I == J && threadIdx.x < kTB) {
        const int64_t dq = a.diagq[(int64_t)J * kTB + threadIdx.x];
        qd[threadIdx.x] = dq >= 0 ? a.qv[(int64_t)s * a.nq + dq] : -1.0;
      }
      if (pre_linv) {
        tile_load_async(Bs, a.Linv + ((int64_t)s * a.NT + J) * kTileElems);
        cp_async_commit();
      }
      int iss;
      if (flags & 1) {  // first chunk: start from Q(I,J)
        // the first two half-steps of the pair pipeline and this thread's
        // first Q entry are in flight while C is cleared
        iss = pair_pipe_prologue(stage, Ls, upa, upb, u0, u1, mI, nJ, tk.pa0, tk.pb0, tk.k0);
        const double* qv = a.qv + (int64_t)s * a.nq;
        const int64_t e0 = tk.q0 + threadIdx.x;
        int loc0 = 0;
        double val0 = 0.0;
        if (e0 < tk.q1) {
          loc0 = a.qloc[e0];
          val0 = qv[e0];
        }
        tile_zero(C);
        __syncthreads();
        if (e0 < tk.q1) C[(loc0 >> 6) * kLD + (loc0 & 63)] = val0;
        for (int64_t e = e0 + kThreads; e < tk.q1; e += kThreads) {
          const int loc = a.qloc[e];
          C[(loc >> 6) * kLD + (loc & 63)] = qv[e];
        }
        __syncthreads();
        frag_load(acc, C);
      } else {  // continue the running sum kept in the tile buffer
        tile_load_async(C, Lt);
        cp_async_commit();
        iss = pair_pipe_prologue(stage, Ls, upa, upb, u0, u1, mI, nJ, tk.pa0, tk.pb0, tk.k0);
        if (iss == 2) cp_async_wait_group<2>();
        else if (iss == 1) cp_async_wait_group<1>();
        else cp_async_wait_group<0>();
        __syncthreads();
        frag_load(acc, C);
      }
      __syncthreads();
      if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 5] = globaltimer();
      // parallel partial groups of a run that ends before this chunk's pairs
      for (int g = tk.g0; g < tk.g1; ++g) {
        tile_load(C, a.G + ((int64_t)s * a.ngrp + g) * kTileElems);
        frag_axpy(acc, C, -1.0);
        __syncthreads();
      }
      pair_pipe_run2(acc, stage, Ls, upa, upb, u0, u1, upk, mI, nJ, -1.0, iss);
      if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 1] = globaltimer();
      if (!(flags & 2)) {
        frag_store_global(acc, Lt);
      } else if (I == J) {
        double* W = stage;               // 64 x 65
        double* X = stage + kTB * kLDW;  // 64 x 65
        frag_store_ld(acc, W, kLDW);
        const int nb = mI;
        __syncthreads();
        for (int e = threadIdx.x; e < kTB * kTB; e += kThreads) {
          int r = e >> 6, cc = e & 63;
          if (r >= nb || cc >= nb) W[r * kLDW + cc] = (r == cc) ? 1.0 : 0.0;
        }
        __syncthreads();
        tile_potri(W, X, qd, nb, a.rel_tol, &sh_fail, C);  // C is idle here
        if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 6] = globaltimer();
        if (threadIdx.x == 0 && sh_fail < kTB) atomicMin(a.status + s, (int)(a.tstart[J] + sh_fail));
        tile_store_ld(Lt, W, kLDW);
        tile_store_ld(a.Linv + ((int64_t)s * a.NT + J) * kTileElems, X, kLDW);
        if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 7] = globaltimer();
      } else {
        if (!pre_linv) {
          tile_load_async(Bs, a.Linv + ((int64_t)s * a.NT + J) * kTileElems);
          cp_async_commit();
        }
        frag_store(acc, C);
        cp_async_wait_all();
        __syncthreads();
        Frag x;
        frag_zero(x);
        frag_mma<false, true>(x, C, Bs, 1.0, mI, nJ, nJ);  // X = C * Linv^T
        if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 6] = globaltimer();
        frag_store_global(x, Lt);
        if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 7] = globaltimer();
      }
    }
    queue_complete_rng(a.q, inst, tk.succ0, tk.succ1, ssucc);
    if (a.trace && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      a.trace[(int64_t)inst * 8 + 0] = t_claim;
      a.trace[(int64_t)inst * 8 + 2] = globaltimer();
      a.trace[(int64_t)inst * 8 + 3] = smid;
      a.trace[(int64_t)inst * 8 + 4] = t_pop;
    }
  }
}

// ---------------------------------------------------------------------------
// triangular solves

// v[i] (+)= sign * sum_k T[i][k] u[k]   (T global row-major tile)
__device__ __forceinline__ void gemv_acc(double* v, const double* T, const double* u, double sign,
                                         bool assign) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const double u0 = u[l], u1 = u[l + 32];
#pragma unroll 4
  for (int r = 0; r < 16; ++r) {
    const int i = w * 16 + r;
    double s = __ldcg(T + i * kTB + l) * u0 + __ldcg(T + i * kTB + l + 32) * u1;
    s = warp_sum(s);
    if (l == 0) v[i] = assign ? sign * s : v[i] + sign * s;
  }
  __syncthreads();
}
// v[k] (+)= sign * sum_i T[i][k] u[i]
__device__ __forceinline__ void gemvT_acc(double* v, const double* T, const double* u, double sign,
                                          bool assign, double* part) {
  const int j = threadIdx.x & 63, h = threadIdx.x >> 6;
  double s = 0.0;
#pragma unroll 8
  for (int i = h * 32; i < h * 32 + 32; ++i) s += __ldcg(T + i * kTB + j) * u[i];
  part[h * kTB + j] = s;
  __syncthreads();
  if (threadIdx.x < kTB) {
    const double t = part[j] + part[kTB + j];
    v[j] = assign ? sign * t : v[j] + sign * t;
  }
  __syncthreads();
}
__device__ __forceinline__ void vec_load(double* v, const double* g) {
  if (threadIdx.x < kTB) v[threadIdx.x] = __ldcg(g + threadIdx.x);
  __syncthreads();
}
__device__ __forceinline__ void vec_store(double* g, const double* v) {
  if (threadIdx.x < kTB) __stcg(g + threadIdx.x, v[threadIdx.x]);
}

// smem tiles of the solve: leading dimension 66 (16-byte aligned rows for
// cp.async; 2-way conflicts at most for row-per-thread dots)
constexpr int kLDS = 66;
__device__ __forceinline__ void stile_load_async(double* S, const double* G) {
  for (int c = threadIdx.x; c < kTileElems / 2; c += kThreads) {
    const int r = c >> 5, col = (c & 31) * 2;
    cp_async16(S + r * kLDS + col, G + r * kTB + col);
  }
}
// out[i] = sum_k T[i][k] u[k]  (two threads per row, 32 products each)
// (4 independent FMA chains per thread: the tile-row chain runs through
// these, so latency matters more than instruction count)
__device__ __forceinline__ double sgemv_row(const double* T, const double* u) {
  const int i = threadIdx.x >> 1, h = threadIdx.x & 1;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int k = h * 32; k < h * 32 + 32; k += 4) {
    s0 = fma(T[i * kLDS + k], u[k], s0);
    s1 = fma(T[i * kLDS + k + 1], u[k + 1], s1);
    s2 = fma(T[i * kLDS + k + 2], u[k + 2], s2);
    s3 = fma(T[i * kLDS + k + 3], u[k + 3], s3);
  }
  double s = (s0 + s1) + (s2 + s3);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;  // valid in both threads of the pair, row i
}
// out[j] = sum_i T[i][j] u[i]
__device__ __forceinline__ double sgemvT_col(const double* T, const double* u) {
  const int j = threadIdx.x >> 1, h = threadIdx.x & 1;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
  for (int i = h * 32; i < h * 32 + 32; i += 4) {
    s0 = fma(T[i * kLDS + j], u[i], s0);
    s1 = fma(T[(i + 1) * kLDS + j], u[i + 1], s1);
    s2 = fma(T[(i + 2) * kLDS + j], u[i + 2], s2);
    s3 = fma(T[(i + 3) * kLDS + j], u[i + 3], s3);
  }
  double s = (s0 + s1) + (s2 + s3);
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  return s;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// all 128 threads: value `v` of row threadIdx.x >> 1 (held by both threads
// of the pair) -> the 128 LL words of a tile row
__device__ __forceinline__ void ll_store(unsigned long long* w, double v, unsigned epoch) {
  const int k = threadIdx.x;
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const unsigned half = (k & 1) ? (unsigned)(bits >> 32) : (unsigned)bits;
  st_relaxed_u64(w + k, ((unsigned long long)epoch << 32) | half);
}
// all 128 threads: wait for the 128 LL words of a tile row, u[r] = value r
__device__ __forceinline__ void ll_load(const unsigned long long* w, unsigned epoch, double* u) {
  const int k = threadIdx.x;
  unsigned long long x;
  while ((unsigned)((x = ld_relaxed_u64(w + k)) >> 32) != epoch) {
  }
  const unsigned half = (unsigned)x;
  const unsigned other = __shfl_xor_sync(0xffffffffu, half, 1);
  if (!(k & 1)) u[k >> 1] = __hiloint2double((int)other, (int)half);
}

// Accumulate acc -= sum of the LL partial vectors ids[0..n) (tile ids into
// llP) in list order, consuming each as soon as its 128 words carry `tag`
// (progressive: the row task keeps pace with the products of its row, so
// only the last partials remain when its chain link arrives).  Thread k owns
// word k (half k & 1 of value k >> 1); both threads of a pair end with the
// same acc.  A window of kWin partials is in flight per thread.
constexpr int kWin = 8;
__device__ __forceinline__ double ll_value(unsigned long long w) {
  const unsigned half = (unsigned)w;
  const unsigned other = __shfl_xor_sync(0xffffffffu, half, 1);
  return (threadIdx.x & 1) ? __hiloint2double((int)half, (int)other)
                           : __hiloint2double((int)other, (int)half);
}
template <class IdAt>
__device__ __forceinline__ double ll_sum_partials(double acc, const unsigned long long* llP, IdAt id_at,
                                                  int n, unsigned tag) {
  const int k = threadIdx.x;
  for (int e0 = 0; e0 < n; e0 += kWin) {
    unsigned long long w[kWin];
#pragma unroll
    for (int j = 0; j < kWin; ++j)
      if (e0 + j < n) w[j] = ld_relaxed_u64(llP + (int64_t)id_at(e0 + j) * 2 * kTB + k);
#pragma unroll
    for (int j = 0; j < kWin; ++j) {
      if (e0 + j < n) {
        while ((unsigned)(w[j] >> 32) != tag) w[j] = ld_relaxed_u64(llP + (int64_t)id_at(e0 + j) * 2 * kTB + k);
        acc -= ll_value(w[j]);
      }
    }
  }
  return acc;
}

// Forward/backward triangular solves over the tile pattern, right-looking,
// with every inter-task value in LL form (no fences, flags or counters):
//   P(I,K) = L(I,K) y_K            (type 1, one tile)   -> llP[tile], tag 2E
//   F(I):  y_I = Linv_I (b_I - sum_K P(I,K) - L(I,link) y_link)   (type 0)
//   Q(I,J) = L(I,J)^T x_I          (type 3, one tile)   -> llP[tile], tag 2E+1
//   B(J):  x_J = Linv_J^T (y_J - sum_I Q(I,J) - L(link,J)^T x_link) (type 2)
// The newest product of a row (nearest of a column) is the chain link and is
// computed inside the row task from a prefetched tile.  Partials are summed
// in a fixed order (K ascending / I descending): results are deterministic.
__global__ void __launch_bounds__(kThreads) solve_kernel(SolveArgs a) {
  extern __shared__ __align__(16) double ssm[];
  double* Ti = ssm;               // L^-1 (or its transpose use) of the block
  double* Tl = ssm + kTB * kLDS;  // the chain-link tile
  double* T3 = ssm + 2 * kTB * kLDS;  // second link tile (two-link mode)
  __shared__ double v[kTB], u[kTB], u2[kTB];
  const int64_t total = a.n_base * a.S;
  const int64_t npad = (int64_t)a.NT * kTB;
  const unsigned E = (unsigned)a.epoch;
  for (;;) {
    const int64_t task = claim(a.counter);
    if (task >= total) break;
    const int4 tk = a.tasks[task / a.S];
    const int s = (int)(task % a.S);
    if (!a.active[s]) continue;
    const unsigned long long t_claim = a.trace ? globaltimer() : 0ull;
    const double* Ls = a.L + (int64_t)s * a.nT * kTileElems;
    const double* Li = a.Linv + (int64_t)s * a.NT * kTileElems;
    unsigned long long* lY = a.llY + (int64_t)s * a.NT * 2 * kTB;
    unsigned long long* lX = a.llX + (int64_t)s * a.NT * 2 * kTB;
    unsigned long long* lP = a.llP + (int64_t)s * a.n_grp * 2 * kTB;
    double* xs = a.x + (int64_t)s * npad;
    if (tk.x == 1 || tk.x == 3) {
      // product group: its tiles stream through the two smem tiles (one load
      // in flight) while their input vectors are awaited; the GEMVs sum in
      // a fixed order (forward K ascending, backward I descending)
      const int4 gr = a.grp[tk.z];
      const bool fwd = tk.x == 1;
      const int cnt = gr.y - gr.x;
      auto tile_at = [&](int e) -> int {  // e-th tile of the group in stream order
        return fwd ? a.row_tid[gr.x + e] : gr.y - 1 - e;
      };
      stile_load_async(Ti, Ls + (int64_t)tile_at(0) * kTileElems);
      cp_async_commit();
      double pv = 0.0;
      for (int e = 0; e < cnt; ++e) {
        double* cur = (e & 1) ? Tl : Ti;
        if (e + 1 < cnt) {
          stile_load_async((e & 1) ? Ti : Tl, Ls + (int64_t)tile_at(e + 1) * kTileElems);
          cp_async_commit();
        }
        const int t = tile_at(e);
        ll_load(fwd ? lY + (int64_t)a.tile_col[t] * 2 * kTB : lX + (int64_t)a.tile_row[t] * 2 * kTB,
                E, u);
        if (e + 1 < cnt)
          cp_async_wait_group<1>();
        else
          cp_async_wait_all();
        __syncthreads();
        if (a.trace && threadIdx.x == 0 && e == 0) a.trace[task * 8 + 4] = globaltimer();
        pv += fwd ? sgemv_row(cur, u) : sgemvT_col(cur, u);
        __syncthreads();  // u and cur are rewritten next round
      }
      ll_store(lP + (int64_t)tk.z * 2 * kTB, pv, fwd ? 2 * E : 2 * E + 1);
    } else {
      const bool fwd = tk.x == 0;
      const int I = tk.z;
      int q0, q1, link_tile, link_src;
      if (fwd) {
        q0 = a.rowptr[I];
        q1 = a.rowptr[I + 1] - 1;  // off-diagonals [q0, q1), the newest is the link
        link_tile = q1 > q0 ? a.row_tid[q1 - 1] : -1;
        link_src = q1 > q0 ? a.row_col[q1 - 1] : -1;
      } else {
        q0 = a.colptr[I] + 1;
        q1 = a.colptr[I + 1];  // off-diagonals [q0, q1), the nearest is the link
        link_tile = q1 > q0 ? q0 : -1;
        link_src = q1 > q0 ? a.tile_row[q0] : -1;
      }
      const bool has_link = link_tile >= 0;
      const int g0 = fwd ? a.fgp[I] : a.bgp[I];
      const int np = (fwd ? a.fgp[I + 1] : a.bgp[I + 1]) - g0;  // product-group partials
      const bool mlink = a.M != nullptr && has_link;
      // second link (two-link mode): second-newest column / second-nearest row
      const bool link2 = mlink && a.nlinks == 2 && q1 - q0 >= 2;
      const int link2_src = link2 ? (fwd ? a.row_col[q1 - 2] : a.tile_row[q0 + 1]) : -1;
      const double* Mbase = a.M + (int64_t)s * 4 * a.NT * kTileElems;
      stile_load_async(Ti, Li + (int64_t)I * kTileElems);
      if (mlink)
        stile_load_async(Tl, Mbase + ((int64_t)(fwd ? 0 : 2) * a.NT + I) * kTileElems);
      else if (has_link)
        stile_load_async(Tl, Ls + (int64_t)link_tile * kTileElems);
      if (link2) stile_load_async(T3, Mbase + ((int64_t)(fwd ? 1 : 3) * a.NT + I) * kTileElems);
      cp_async_commit();
      // right-hand side: b_I (forward) or y_J (backward, LL)
      double acc;
      if (fwd) {
        acc = __ldcg(a.b + (int64_t)s * npad + (int64_t)I * kTB + (threadIdx.x >> 1));
      } else {
        unsigned long long w;
        const unsigned long long* p = lY + (int64_t)I * 2 * kTB + threadIdx.x;
        while ((unsigned)((w = ld_relaxed_u64(p)) >> 32) != E) {
        }
        acc = ll_value(w);
      }
      if (a.trace && threadIdx.x == 0) a.trace[task * 8 + 1] = globaltimer();
      const unsigned tag = fwd ? 2 * E : 2 * E + 1;
      // partials in readiness order (oldest / farthest group first)
      acc = ll_sum_partials(acc, lP, [&](int e) { return g0 + e; }, np, tag);
      if (a.trace && threadIdx.x == 0) a.trace[task * 8 + 2] = globaltimer();
      if ((threadIdx.x & 1) == 0) v[threadIdx.x >> 1] = acc;
      if (mlink) {
        // Linv applied off the chain; the chain step is z = vp - M u_link
        cp_async_wait_all();
        __syncthreads();
        double vp = fwd ? sgemv_row(Ti, v) : sgemvT_col(Ti, v);
        if (link2) {
          ll_load(fwd ? lY + (int64_t)link2_src * 2 * kTB : lX + (int64_t)link2_src * 2 * kTB, E, u2);
          __syncthreads();
          vp -= fwd ? sgemv_row(T3, u2) : sgemvT_col(T3, u2);
        }
        ll_load(fwd ? lY + (int64_t)link_src * 2 * kTB : lX + (int64_t)link_src * 2 * kTB, E, u);
        __syncthreads();
        if (a.trace && threadIdx.x == 0) a.trace[task * 8 + 4] = globaltimer();
        const double z = vp - (fwd ? sgemv_row(Tl, u) : sgemvT_col(Tl, u));
        ll_store((fwd ? lY : lX) + (int64_t)I * 2 * kTB, z, E);
        if (!fwd && (threadIdx.x & 1) == 0) __stcg(xs + (int64_t)I * kTB + (threadIdx.x >> 1), z);
        goto task_done;
      }
      // the chain link: poll its LL words directly
      if (has_link) ll_load(fwd ? lY + (int64_t)link_src * 2 * kTB : lX + (int64_t)link_src * 2 * kTB, E, u);
      cp_async_wait_all();
      __syncthreads();
      if (a.trace && threadIdx.x == 0) a.trace[task * 8 + 4] = globaltimer();
      if (has_link) {
        const double pl = fwd ? sgemv_row(Tl, u) : sgemvT_col(Tl, u);
        if ((threadIdx.x & 1) == 0) v[threadIdx.x >> 1] -= pl;
        __syncthreads();
      }
      const double z = fwd ? sgemv_row(Ti, v) : sgemvT_col(Ti, v);
      ll_store((fwd ? lY : lX) + (int64_t)I * 2 * kTB, z, E);
      if (!fwd && (threadIdx.x & 1) == 0) __stcg(xs + (int64_t)I * kTB + (threadIdx.x >> 1), z);
    }
  task_done:
    if (a.trace && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      a.trace[task * 8 + 0] = t_claim;
      a.trace[task * 8 + 5] = globaltimer();
      a.trace[task * 8 + 6] = smid;
    }
  }
}

// chain-link tiles for the solve (one CTA per (link, slot)):
//   forward row I:     M_I = Linv_I L(I,l)      (rows of I x rows of l)
//   backward column J: N_J = L(l,J) Linv_J      (rows of l x rows of J)
// so that Linv_I (r - L(I,link) y_link) = Linv_I r - M_I y_link and
// Linv_J^T (r - L(link,J)^T x_link) = Linv_J^T r - N_J^T x_link.
__global__ void __launch_bounds__(kThreads) link_tiles_kernel(LinkArgs a) {
  extern __shared__ __align__(16) double lsm[];
  double* As = lsm;
  double* Bs = lsm + kSmemTile;
  const int s = blockIdx.y;
  if (!a.active[s]) return;
  const int4 lk = a.links[blockIdx.x];
  const double* Ls = a.L + (int64_t)s * a.nT * kTileElems;
  const double* Li = a.Linv + (int64_t)s * a.NT * kTileElems;
  const int I = lk.y;
  const int mI = a.tbsz[I], ms = a.tbsz[lk.w];
  const bool fwd = lk.x < 2;
  tile_load_async(As, fwd ? Li + (int64_t)I * kTileElems : Ls + (int64_t)lk.z * kTileElems);
  tile_load_async(Bs, fwd ? Ls + (int64_t)lk.z * kTileElems : Li + (int64_t)I * kTileElems);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  Frag f;
  frag_zero(f);
  if (fwd)
    frag_mma<false, false>(f, As, Bs, 1.0, mI, ms, mI);
  else
    frag_mma<false, false>(f, As, Bs, 1.0, ms, mI, mI);
  frag_store_global(f, a.M + (((int64_t)s * 4 + lk.x) * a.NT + I) * kTileElems);
}

// ---------------------------------------------------------------------------
// selected inversion (block Takahashi):
//   Sigma(I,J) = -[ sum_{K in col(J), K>J} Sigma(I,K) L(K,J) ] Linv_J       (I > J)
//   Sigma(J,J) = Linv_J^T [ Linv_J - sum_{K>J} L(K,J)^T Sigma(K,J) ]

__global__ void __launch_bounds__(kThreads, 2) selinv_kernel(SelinvArgs a) {
  extern __shared__ __align__(16) double smem[];
  double* C = smem;
  double* stage = smem + kSmemTile;
  double* As = stage;
  double* Bs = stage + kSmemTile;
  const int ntask = a.q.ntask;
  __shared__ int sp_a[kPairPre], sp_b[kPairPre], sp_m[kPairPre], sp_k[kPairPre];
  // stage pairs [u0, u1) (operand tiles, modes, K extents) in smem when they
  // fit: no dependent global index chain (mode -> tile -> tile row -> height)
  // per half-step of the pair pipeline
  auto stage_pairs = [&](int64_t u0, int64_t u1, const int*& pa, const int*& pb, const int*& md,
                         const int*& kx, int64_t& b0, int64_t& b1) {
    const bool pre = u1 - u0 <= kPairPre;
    if (pre && threadIdx.x < u1 - u0) {
      const int64_t u = u0 + threadIdx.x;
      const int m = __ldg(a.mode + u), ta = __ldg(a.pa + u), tb = __ldg(a.pb + u);
      sp_a[threadIdx.x] = ta;
      sp_b[threadIdx.x] = tb;
      sp_m[threadIdx.x] = m;
      sp_k[threadIdx.x] = a.tbsz[a.tile_row[(m & 1) ? ta : tb]];
    }
    __syncthreads();
    pa = pre ? sp_a : a.pa;
    pb = pre ? sp_b : a.pb;
    md = pre ? sp_m : a.mode;
    kx = pre ? sp_k : nullptr;
    b0 = pre ? 0 : u0;
    b1 = pre ? u1 - u0 : u1;
  };
  queue_start();
  for (;;) {
    const unsigned long long t_c0 = a.trace ? globaltimer() : 0ull;
    const int inst = queue_pop(a.q);
    if (inst < 0) break;
    const unsigned long long t_c1 = a.trace ? globaltimer() : 0ull;
    if (a.trace && threadIdx.x == 0) {
      a.trace[(int64_t)inst * 4 + 0] = t_c0;
      a.trace[(int64_t)inst * 4 + 1] = t_c1;
    }
    const int s = inst / ntask;
    const int4 tk = a.tasks[inst % ntask];
    const int ls = a.lslot[s];
    if (tk.x == 1) {  // parallel partial group of a diagonal tile
      const int g = tk.z, gt = a.grp_tile[g];
      const int mIg = a.tbsz[a.tile_row[gt]], nJg = a.tbsz[a.tile_col[gt]];
      Frag acc;
      frag_zero(acc);
      const int *spa, *spb, *smd, *skx;
      int64_t b0, b1;
      stage_pairs(a.grp_rng[g], a.grp_rng[g + 1], spa, spb, smd, skx, b0, b1);
      pair_gemm_modes(acc, stage, a.L + (int64_t)ls * a.nT * kTileElems,
                      a.Sg + (int64_t)s * a.nT * kTileElems, spa, spb, smd, b0, b1, a.tile_row,
                      a.tbsz, skx, mIg, nJg, 1.0);
      frag_store_global(acc, a.G + ((int64_t)s * a.ngbuf + a.gbuf[g]) * kTileElems);
      queue_complete(a.q, inst);
      if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 4 + 2] = globaltimer();
      continue;
    }
    const int c = tk.z;
    const int tid = a.chunk_tile[c];
    const int flags = a.chunk_flags[c];
    const int I = a.tile_row[tid], J = a.tile_col[tid];
    const int mI = a.tbsz[I], nJ = a.tbsz[J];
    const double* Ls = a.L + (int64_t)ls * a.nT * kTileElems;
    const double* Li = a.Linv + (int64_t)ls * a.NT * kTileElems;
    double* Ss = a.Sg + (int64_t)s * a.nT * kTileElems;
    double* St = Ss + (int64_t)tid * kTileElems;
    Frag acc;
    if (flags & 1) {
      frag_zero(acc);
      sum_tiles_async(acc, stage, a.G + (int64_t)s * a.ngbuf * kTileElems, a.gbuf,
                      a.tile_grp_ptr[tid], a.tile_grp_ptr[tid + 1], 1.0);
    } else {
      tile_load(C, St);
      frag_load(acc, C);
      __syncthreads();
    }
    {
      const int *spa, *spb, *smd, *skx;
      int64_t b0, b1;
      stage_pairs(a.chunk_rng[c], a.chunk_rng[c + 1], spa, spb, smd, skx, b0, b1);
      pair_gemm_modes(acc, stage, Ls, Ss, spa, spb, smd, b0, b1, a.tile_row, a.tbsz, skx,
                      I == J ? nJ : mI, nJ, 1.0);
    }
    if (!(flags & 2)) {
      frag_store_global(acc, St);
    } else if (I != J) {
      // Sigma(I,J) = -(sum_K Sigma(I,K) L(K,J)) Linv_J
      frag_store(acc, C);
      tile_load(Bs, Li + (int64_t)J * kTileElems);
      Frag x;
      frag_zero(x);
      frag_mma<false, false>(x, C, Bs, -1.0, mI, nJ, nJ);
      frag_store_global(x, St);
    } else {
      // Sigma(J,J) = Linv_J^T (Linv_J - sum_K L(K,J)^T Sigma(K,J)), symmetrized
      frag_store(acc, C);
      tile_load(As, Li + (int64_t)J * kTileElems);
      for (int e = threadIdx.x; e < kSmemTile; e += kThreads) C[e] = As[e] - C[e];
      __syncthreads();
      Frag x;
      frag_zero(x);
      frag_mma<true, false>(x, As, C, 1.0);
      frag_store(x, Bs);
      __syncthreads();
      for (int e = threadIdx.x; e < kTB * kTB; e += kThreads) {
        const int r = e >> 6, cc = e & 63;
        C[r * kLD + cc] = 0.5 * (Bs[r * kLD + cc] + Bs[cc * kLD + r]);
      }
      __syncthreads();
      tile_store(St, C);
    }
    queue_complete(a.q, inst);
    if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 4 + 2] = globaltimer();
  }
}

// diag(Sigma) of slot s -> var_pad[NT*64]
__global__ void selinv_diag_kernel(const double* Sg, int64_t nT, int NT, const int* colptr,
                                   double* var_pad) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)NT * kTB) return;
  int J = (int)(i / kTB), r = (int)(i % kTB);
  var_pad[i] = Sg[(int64_t)colptr[J] * kTileElems + r * kTB + r];
}

// ---------------------------------------------------------------------------
// launchers

static int g_sm_count = 0;

// Persistent grid of `want` CTAs per SM.  The kernels are designed for that
// residency (the list schedule assumes it); if registers or shared memory
// ever stop fitting, say so once instead of silently serialising CTAs.
template <class Kernel>
static int persistent_grid(Kernel kernel, int want, size_t smem, const char* name) {
  if (g_sm_count == 0) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
  if (occ < want) {
    fprintf(stderr, "pinla: %s fits %d CTA(s)/SM, designed for %d\n", name, occ, want);
    return g_sm_count * (occ > 0 ? occ : 1);
  }
  return g_sm_count * want;
}

size_t dag_smem_bytes() { return 3 * kSmemTile * sizeof(double); }
static size_t factor_smem_bytes() { return kFactorSmem * sizeof(double); }

cudaError_t launch_factor(const FactorArgs& a, cudaStream_t st) {
  // The warp-specialised kernel (factor_ws.cu) is the default.  Launches
  // that are bound by the POTRI -> TRSM chain -- critical lane on and little
  // work per DAG level: c5 with one resident slot -- keep the 128-thread
  // kernel, whose two CTAs per lane SM turn the chain around faster.
  // Measured (profiles/ws_matrix_r02.txt; work per level at 25 TF/s): c5 x 1
  // slot 28 us: 128-thread kernel 11 % faster; c3 x 1 74 us, c5 x 3 83 us,
  // c4 x 1 94 us and every lane-less launch: warp-specialised 5-7 % faster.
  // PINLA_FACTOR_WS = 0 never, 2 always.
  const bool chain_bound = a.q.nlane > 0 && a.q.nact * a.flops_per_level < 1.2e9;
  if (!a.q.fifo && (factor_ws_mode() == 2 || (factor_ws_mode() == 1 && !chain_bound)))
    return launch_factor_ws(a, st);
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)factor_smem_bytes());
    grid = persistent_grid(factor_kernel, 2, factor_smem_bytes(), "factor_kernel");
  }
  cudaError_t e = launch_queue_init(a.q, a.S, st);
  if (e != cudaSuccess) return e;
  factor_kernel<<<grid, kThreads, factor_smem_bytes(), st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_solve(const SolveArgs& a, cudaStream_t st) {
  // two smem tiles (3 CTAs/SM); three in two-link mode (2 CTAs/SM)
  static int grid2 = 0, grid3 = 0;
  const int smem2 = 2 * kTB * kLDS * (int)sizeof(double), smem3 = 3 * kTB * kLDS * (int)sizeof(double);
  if (!grid2) {
    cudaFuncSetAttribute(solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem3);
    grid2 = persistent_grid(solve_kernel, 3, smem2, "solve_kernel");
    grid3 = persistent_grid(solve_kernel, 2, smem3, "solve_kernel (two links)");
  }
  const bool three = a.M != nullptr && a.nlinks == 2;
  cudaMemsetAsync(a.counter, 0, sizeof(int), st);
  solve_kernel<<<three ? grid3 : grid2, kThreads, three ? smem3 : smem2, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_link_tiles(const LinkArgs& a, cudaStream_t st) {
  const int smem = 2 * kSmemTile * (int)sizeof(double);
  static bool init = false;
  if (!init) {
    cudaFuncSetAttribute(link_tiles_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    init = true;
  }
  if (a.nlink == 0) return cudaSuccess;
  link_tiles_kernel<<<dim3(a.nlink, a.S), kThreads, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_selinv(const SelinvArgs& a, cudaStream_t st) {
  // The warp-specialised kernel (selinv_ws.cu, list-schedule order) is the
  // default: c3 204 -> 193 ms, c4 1471 -> 1406 ms, c5 665 -> 458 ms
  // (profiles/ws_matrix_r02.txt); the chain-bound c5 gains most, because a
  // task owns the whole DMMA pipe of its SM and its operands are prefetched
  // by the producer warp.  PINLA_SELINV_WS=0 selects the 128-thread kernel
  // with its ready queue and continuations.
  if (a.q.order && selinv_ws_mode() != 0)
    return launch_selinv_ws(a, st);
  static int grid = 0;
  if (!grid) {
    cudaFuncSetAttribute(selinv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)factor_smem_bytes());
    grid = persistent_grid(selinv_kernel, 2, factor_smem_bytes(), "selinv_kernel");
  }
  cudaError_t e = launch_queue_init(a.q, a.S, st);
  if (e != cudaSuccess) return e;
  selinv_kernel<<<grid, kThreads, factor_smem_bytes(), st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_selinv_diag(const double* Sg, int64_t nT, int NT, const int* colptr,
                               double* var_pad, cudaStream_t st) {
  int64_t n = (int64_t)NT * kTB;
  selinv_diag_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(Sg, nT, NT, colptr, var_pad);
  return cudaGetLastError();
}

}  // namespace pinla
