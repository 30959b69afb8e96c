// Warp-specialised numeric factorization (the default factor kernel).
//
// Same task DAG, task records and arithmetic as dag.cu's 128-thread
// factor_kernel (bitwise identical factors: every output element sees the
// same operation sequence), different execution shape: ONE CTA per SM with
//   * warp 8, the producer: claims the next task in the list-schedule order
//     (one fetch-and-add), waits for its dependency counter, publishes the
//     task record to the MMA warps through a two-entry task-slot ring and
//     streams the task's operands -- running-sum tile, group partials, the
//     half-K operand pairs, L_JJ^-1 -- into a 4-stage shared-memory ring with
//     TMA box loads (cp.async.bulk.tensor.2d through tensor maps over the L,
//     L^-1 and group arrays + mbarrier complete_tx): 16 columns x (tile
//     height) rows per box, hardware-swizzled (128B span, 32B atoms) so the
//     DMMA fragment loads are bank-conflict free without padding;
//   * warps 0-7, the MMA team: all eight work on the same 64x64 output tile
//     (32x16 per warp, DMMA.8x8x4), wait on a stage's `full` mbarrier, run its
//     8 k-steps and release it with one arrive per warp.  No CTA-wide barrier
//     and no global load inside the pair loop.
//   * warp 9, the publisher: waits until the MMA warps have issued a task's
//     stores (pfull mbarrier) and counts the task's successors down with
//     gpu-scope releases, so the fence drain is off the MMA team's path.
// The producer runs ahead across task boundaries (bounded by the ring), so the
// claim, the dependency wait and the first operand loads of task n+1 overlap
// the math and the finalize (TRSM / POTRI) of task n, and a task owns the
// whole DMMA pipe of its SM: its latency is half that of the two-CTA design.
//
// Reference counterpart: kernels.factor_range (kernels.py:99-143) under
// run_tree_tasks (runtime.py:180-268); pivot rule kernels.py:138.
#include <cuda.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "dag.cuh"
#include "potri.cuh"
#include "tile.cuh"
#include "ws.cuh"

namespace pinla {

constexpr int kWsStages = 4;
// Publisher warp (warp 9): the completion of a task -- gpu-scope release of its
// tile stores + successor decrements -- runs beside the MMA team instead of at
// the end of its task: the eight MMA warps hand their stores over through the
// slot's `pfull` barrier and go on with the next task while the fence drains.
#ifndef PINLA_WS_PUBLISHER
#define PINLA_WS_PUBLISHER 1
#endif
constexpr int kFwsThreads = kWsThreads + (PINLA_WS_PUBLISHER ? 32 : 0);
#ifndef PINLA_WS_SLOTS
#define PINLA_WS_SLOTS 2
#endif
constexpr int kWsSlots = PINLA_WS_SLOTS;  // task-slot ring: how many tasks the producer may run ahead
#ifndef PINLA_WS_POTRI_ROT
#define PINLA_WS_POTRI_ROT 96
#endif
// POTRI chain role on MMA warp 1: the producer (warp 8) polls on warp 0's scheduler partition
constexpr int kWsPotriRot = PINLA_WS_POTRI_ROT;
constexpr int kWsPre = 128;  // pair K extents / successor ids staged per task slot

struct __align__(16) WsSlot {
  FTask rec;
  int inst;  // -1: no more tasks
  int skip;  // the slot's factorization already failed: completion only
  int cont_prev;  // continuation of the previous task on this SM: the accumulators hold the running sum
  int cont_next;  // the next chunk of this tile follows on this SM: no store, no publish
  unsigned long long t_pop, t_ready;  // trace: claimed / dependencies met (producer clock)
  int sk[kWsPre];     // K extent per pair (lists of <= kWsPre pairs)
  int ssucc[kWsPre];  // successor base tasks (<= kWsPre)
};

// dynamic smem (1 KB aligned): ring | C (swizzled tile; W of the POTRI at ld 65) | X (64 x 65) |
// POTRI scratch
constexpr int kWsSmemDoubles = kWsStages * kWsStageElems + kSmemTile + kTB * kLDW + kPotriScratch;
constexpr size_t kWsSmemBytes = (size_t)kWsSmemDoubles * sizeof(double) + 1024;

// Tensor maps of one launch: the L array with box heights 8, 16, .., 64 (a
// pair operand of a short tile row loads only its rows), L^-1 and the group
// partial sums with full-height boxes.  Rows of a map = all tiles of all slots.
struct WsMaps {
  CUtensorMap Lh[8];
  CUtensorMap Linv;
  CUtensorMap G;
};

__device__ __forceinline__ void ws_tile_store_ld(double* G, const double* S, int ld) {
  for (int e = threadIdx.x; e < kTB * kTB; e += kWsConsumers) __stcg(G + e, S[(e >> 6) * ld + (e & 63)]);
}

// The POTRI of a diagonal tile as a real call: its register needs (tile rows
// held in registers) stay out of the allocation of the MMA loops.
__device__ __noinline__ void ws_potri(double* W, double* X, const double* qd, int nb, double rel_tol, int* sh_fail,
                                      double* scratch) {
  tile_potri(W, X, qd, nb, rel_tol, sh_fail, scratch, WsSync128(), kWsPotriRot);
}

__global__ void __launch_bounds__(kFwsThreads, 1)
    factor_ws_kernel(FactorArgs a, const __grid_constant__ WsMaps maps) {
  extern __shared__ __align__(1024) double smem_raw[];
  double* smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw)) / 8;
  double* ring = smem;
  double* C = ring + kWsStages * kWsStageElems;
  double* X = C + kSmemTile;
  double* scratch = X + kTB * kLDW;
  __shared__ unsigned long long full[kWsStages], empty[kWsStages], sfull[kWsSlots], sempty[kWsSlots];
  __shared__ unsigned long long sdec[kWsSlots];  // the task's continuation decision (cont_next) is written
  __shared__ unsigned long long pfull[kWsSlots];  // the MMA warps' stores of the task are issued (publisher)
  __shared__ WsSlot slots[kWsSlots];
  __shared__ int pclaim[4];
  __shared__ int ppa[kWsPre], ppb[kWsPre], pkk[kWsPre];  // producer: staged pair records
  __shared__ double qd[kTB];
  __shared__ int sh_fail;
  const int ntask = a.q.ntask;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kWsStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kWsConsumers / 32);
    }
    for (int i = 0; i < kWsSlots; ++i) {
      mbar_init(sfull + i, 1);
      mbar_init(sempty + i, kWsConsumers / 32 + (PINLA_WS_PUBLISHER ? 1 : 0));
      mbar_init(sdec + i, 1);
      mbar_init(pfull + i, kWsConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

#if PINLA_WS_PUBLISHER
  if (threadIdx.x >= kWsThreads) {
    // ----------------------------------------------------------- publisher
    // per task: wait until the producer published the slot and every MMA warp
    // has issued its stores (pfull: cta-scope release / acquire), then count
    // the successors down; each decrement is a gpu-scope release, cumulative
    // over the MMA warps' stores observed through the barrier
    RingCur pc{0, 0u};
    for (;;) {
      mbar_wait(sfull + pc.st, pc.ph);
      const WsSlot& sl = slots[pc.st];
      const int inst = sl.inst;
      if (inst < 0) break;
      mbar_wait(pfull + pc.st, pc.ph);
      if (!sl.cont_next) {
        const int base = inst - inst % ntask;
        const int succ0 = sl.rec.succ0, succ1 = sl.rec.succ1;
        const bool pre = succ1 - succ0 <= kWsPre;
        for (int k = succ0 + lane; k < succ1; k += 32)
          red_dec_release(a.q.cnt + base + (pre ? sl.ssucc[k - succ0] : a.q.succ[k]));
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + pc.st);
      pc.advance(kWsSlots);
    }
    return;
  }
#endif
  if (threadIdx.x >= kWsConsumers) {
    // ------------------------------------------------------------ producer
    RingCur rc{0, 1u};  // waits `empty`: a fresh barrier passes parity 1
    RingCur sc{0, 1u};
    // critical lane (DagQueue::nlane): the first lane_ctas CTAs (one SM each)
    // claim only the lane tasks, which are numbered last
    const bool lane_cta = a.q.nlane > 0 && (int)blockIdx.x < a.q.lane_ctas;
    const int nbase = a.q.nlane > 0 ? (lane_cta ? a.q.nlane : ntask - a.q.nlane) : ntask;
    const int t0 = lane_cta ? ntask - a.q.nlane : 0;
    const int total = a.q.nact * nbase;
    int* ctr = a.q.ctr + (lane_cta ? 2 : 0);
    // Chunk continuations (a.q.claimed): an inner chunk's only successor is the
    // next chunk of the same tile (FTask::next).  When that chunk waits for
    // nothing else once this one's loads are issued, the producer claims it too
    // (an exchange on the instance's claim tag; whoever meets the tag later in
    // the list order skips the instance) and runs it right after: the running
    // sum stays in the MMA warps' accumulators -- no tile store, fence, counter
    // hand-off and reload between the two.  Same operation order per element,
    // so the factor is unchanged bit for bit.  The decision is taken AFTER the
    // task's loads are queued (off the consumers' path) and handed over through
    // the slot's `sdec` barrier, which the MMA warps pass at the end of the task.
    const int tag = (int)a.q.epoch;
    int next_inst = -1, next_t = 0;  // lane 0: continuation decided for the next iteration
    FTask tkn;                       // record of FTask::next, fetched ahead
    tkn.next = -1;
    for (;;) {
      const unsigned long long t_pop = a.trace ? globaltimer() : 0ull;
      if (lane == 0) {
        int inst = -1, t = 0, cont = 0, cnt0 = 1;
        if (next_inst >= 0) {
          inst = next_inst;
          t = next_t;
          cont = 1;
          next_inst = -1;
        } else {
          for (;;) {
            const int idx = atomicAdd(ctr, 1);
            if (idx >= total) {
              inst = -1;
              break;
            }
            t = t0 + idx / a.q.nact;  // base tasks are numbered in claim order
            inst = a.q.act_slots[idx % a.q.nact] * ntask + t;
            // the record prefetch, the claim-tag exchange and the first look at
            // the dependency counter are in flight together
            asm volatile("prefetch.global.L2 [%0];" ::"l"(a.rec + t));
            const int old = a.q.claimed ? atomicExch(a.q.claimed + inst, tag) : 0;
            cnt0 = ld_acquire(a.q.cnt + inst);
            if (!a.q.claimed || old != tag) break;  // ours
          }
        }
        pclaim[0] = inst;
        pclaim[1] = t;
        pclaim[2] = cont;
        pclaim[3] = cnt0;
      }
      __syncwarp();
      const int inst = pclaim[0], t = pclaim[1], cont = pclaim[2], cnt0 = pclaim[3];
      __syncwarp();  // every lane has read the claim before lane 0 writes the next one
      mbar_wait(sempty + sc.st, sc.ph);
      WsSlot& sl = slots[sc.st];
      if (inst < 0) {
        if (lane == 0) {
          sl.inst = -1;
          mbar_arrive(sfull + sc.st);
        }
        break;
      }
      // the 96-byte record is in flight during the dependency wait (a
      // continuation's record was fetched while its predecessor was dispatched)
      FTask tk;
      if (cont) {
        tk = tkn;
      } else {
        const int4* p = reinterpret_cast<const int4*>(a.rec + t);
        int4* d = reinterpret_cast<int4*>(&tk);
#pragma unroll
        for (int k = 0; k < 6; ++k) d[k] = __ldg(p + k);
      }
      const int s = inst / ntask;
      const int64_t npair = tk.u1 - tk.u0;
      const int nsucc = tk.succ1 - tk.succ0;
      if (lane == 0) sl.rec = tk;
      // the first block of pair records is staged once, for the MMA warps (K
      // extents in the slot) and for lane 0's load loop below (lane 0 is done
      // with the previous task's block)
      const int nb0 = npair < kWsPre ? (int)npair : kWsPre;
      for (int k = lane; k < nb0; k += 32) {
        const int kk = __ldg(a.upd_k + tk.u0 + k);
        ppa[k] = __ldg(a.upd_a + tk.u0 + k);
        ppb[k] = __ldg(a.upd_b + tk.u0 + k);
        pkk[k] = kk;
        if (npair <= kWsPre) sl.sk[k] = kk;
      }
      if (nsucc <= kWsPre)
        for (int k = lane; k < nsucc; k += 32) sl.ssucc[k] = __ldg(a.q.succ + tk.succ0 + k);
      if (lane == 0) {
        if (!cont && cnt0 != 0) {  // (a continuation was taken with every other dependency met)
          int spins = 0;
          while (ld_acquire(a.q.cnt + inst) != 0) {
            if (++spins > 4) __nanosleep(32);
          }
        }
        const int skip = *((volatile const int*)(a.status + s)) != INT_MAX;
        sl.inst = inst;
        sl.skip = skip;
        sl.cont_prev = cont;
        if (a.trace) {
          sl.t_pop = t_pop;
          sl.t_ready = globaltimer();
        }
      }
      __syncwarp();
      const int skip = sl.skip;
      if (lane == 0) mbar_arrive(sfull + sc.st);
      unsigned long long* const dec = sdec + sc.st;
      sc.advance(kWsSlots);
      const bool may_cont = a.q.claimed && !skip && tk.next >= 0;
      if (may_cont) {  // the successor chunk's record, in flight behind this task's loads
        const int4* p = reinterpret_cast<const int4*>(a.rec + tk.next);
        int4* d = reinterpret_cast<int4*>(&tkn);
#pragma unroll
        for (int k = 0; k < 6; ++k) d[k] = __ldg(p + k);
      }
      // lane 0: take the next chunk of the tile if nothing but this task holds
      // it back, and tell the MMA warps.  First tried when the ring is full for
      // the first time (the producer would only wait for a free stage then, and
      // a taken continuation's loads follow this task's without a gap), again
      // (`last`) when all loads are queued.
      bool decided = false;
      auto decide = [&](bool last) {
        if (decided) return;
        int cn = 0;
        if (may_cont) {
          const int inst2 = s * ntask + tk.next;
          if (ld_acquire(a.q.cnt + inst2) == 1 && atomicExch(a.q.claimed + inst2, tag) != tag) {
            cn = 1;
            next_inst = inst2;
            next_t = tk.next;
          }
        }
        if (!cn && !last && may_cont) return;  // the successor still waits for another operand: ask again later
        sl.cont_next = cn;
        mbar_arrive(dec);
        decided = true;
      };
      if (skip) {
        if (lane == 0) decide(true);
        continue;
      }
      fence_proxy_async();
      const int mI = tk.mI, nJ = tk.nJ;
      // Lane 0 alone drives the ring (waits for a free stage, arms the `full`
      // barrier, issues the TMA loads); the other lanes only stage the next
      // block of pair records in shared memory between two __syncwarp()s (no
      // warp shuffles from lane-divergent code).
      // (column, row) coordinates in the maps: row = (slot tile index) * 64
      auto put_tile = [&](const CUtensorMap* m, int64_t tile) {  // lane 0
        mbar_wait(empty + rc.st, rc.ph);
        mbar_expect_tx(full + rc.st, kTB * kTB * 8);
        double* dst = ring + rc.st * kWsStageElems;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          tma_load_2d(dst + b * kBoxElems, m, b * kBoxCols, (int)(tile * kTB), full + rc.st);
        rc.advance(kWsStages);
      };
      const int ra = (mI + 7) & ~7, rb = (nJ + 7) & ~7;
      const CUtensorMap* ma = maps.Lh + (ra / 8 - 1);
      const CUtensorMap* mb = maps.Lh + (rb / 8 - 1);
      const int64_t tbase = (int64_t)s * a.nT;
      auto put_half = [&](int ta, int tb, int kh, int kext) {  // lane 0
        const int klim = min(32, kext - kh * 32);
        const int nbox = (klim + kBoxCols - 1) / kBoxCols;
        mbar_wait(empty + rc.st, rc.ph);
        mbar_expect_tx(full + rc.st, (unsigned)(nbox * (ra + rb) * kBoxCols * 8));
        double* dst = ring + rc.st * kWsStageElems;
        for (int b = 0; b < nbox; ++b) {
          tma_load_2d(dst + b * kBoxElems, ma, kh * 32 + b * kBoxCols, (int)((tbase + ta) * kTB), full + rc.st);
          tma_load_2d(dst + (2 + b) * kBoxElems, mb, kh * 32 + b * kBoxCols, (int)((tbase + tb) * kTB),
                      full + rc.st);
        }
        rc.advance(kWsStages);
      };
      if (lane == 0 && tk.type == 0) {
        if (!(tk.flags & 1) && !cont) put_tile(maps.Lh + 7, tbase + tk.tid);  // the running sum
        for (int g = tk.g0; g < tk.g1; ++g) put_tile(&maps.G, (int64_t)s * a.ngrp + g);
      }
      int nput = 0;        // lane 0: pair stages queued so far
      bool tried = false;  // lane 0: the early continuation check ran
      for (int64_t ub = tk.u0; ub < tk.u1; ub += kWsPre) {
        const int nb = tk.u1 - ub < kWsPre ? (int)(tk.u1 - ub) : kWsPre;
        __syncwarp();  // lane 0 is done with the previous block
        if (ub != tk.u0)  // (the first block was staged with the task record)
          for (int k = lane; k < nb; k += 32) {
            ppa[k] = __ldg(a.upd_a + ub + k);
            ppb[k] = __ldg(a.upd_b + ub + k);
            pkk[k] = __ldg(a.upd_k + ub + k);
          }
        __syncwarp();
        if (lane == 0)
          for (int j = 0; j < nb; ++j) {
            const int kk = pkk[j];
            put_half(ppa[j], ppb[j], 0, kk);
            if (kk > 32) put_half(ppa[j], ppb[j], 1, kk);
            if ((nput += kk > 32 ? 2 : 1) >= kWsStages && !tried) {
              tried = true;
              decide(false);
            }
          }
      }
      if (lane == 0 && tk.type == 0 && (tk.flags & 2) && tk.I != tk.J)
        put_tile(&maps.Linv, (int64_t)s * a.NT + tk.J);
      if (lane == 0) decide(true);
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------------------- MMA team
  RingCur rc{0, 0u};
  RingCur sc{0, 0u};
  const int warp = threadIdx.x >> 5;
#ifdef PINLA_WS_TRACE_WAIT
  long long ring_wait = 0;  // diagnostic build: clocks this thread spent waiting for ring stages in the task
#endif
  auto wait_item = [&]() -> double* {
#ifdef PINLA_WS_TRACE_WAIT
    const long long t_in = clock64();
    mbar_wait(full + rc.st, rc.ph);
    ring_wait += clock64() - t_in;
#else
    mbar_wait(full + rc.st, rc.ph);
#endif
    return ring + rc.st * kWsStageElems;
  };
  auto release_item = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + rc.st);
    rc.advance(kWsStages);
  };
  Frag8 acc;  // lives across tasks: a continued chunk starts from its predecessor's sum
  for (;;) {
    mbar_wait(sfull + sc.st, sc.ph);
    const WsSlot& sl = slots[sc.st];
    const int inst = sl.inst;
    if (inst < 0) break;
    const int s = inst / ntask;
    const bool skip = sl.skip != 0;
    const bool cont_prev = sl.cont_prev != 0;
    bool cont_next = false;
    const int type = sl.rec.type, flags = sl.rec.flags;
    const int I = sl.rec.I, J = sl.rec.J, mI = sl.rec.mI, nJ = sl.rec.nJ;
    const int64_t u0 = sl.rec.u0, u1 = sl.rec.u1;
#if !PINLA_WS_PUBLISHER
    const int succ0 = sl.rec.succ0, succ1 = sl.rec.succ1;
#endif
    double* Ls = a.L + (int64_t)s * a.nT * kTileElems;
    if (!skip) {
      // a chunk task (type 0) subtracts its pair products: acc holds the
      // NEGATED running sum until the pair loop ends (see ws_mma_swz)
      const bool fin = type == 0 && (flags & 2);
      if (cont_prev) {
        // acc already holds the negated running sum of this tile
      } else if (type == 1 || !(flags & 1)) {
        if (type == 1) {
          ws_zero(acc);
        } else {
          const double* b = wait_item();  // the running sum
          ws_load_swz(acc, b);
          release_item();
          ws_neg(acc);
        }
      } else if (sl.rec.q1 == sl.rec.q0) {  // first chunk of a pure fill tile: Q(I,J) = 0
        ws_zero(acc);
      } else {  // first chunk: start from Q(I,J)
        const double* qv = a.qv + (int64_t)s * a.nq;
        const int64_t q0 = sl.rec.q0, q1 = sl.rec.q1;
        const int64_t e0 = q0 + threadIdx.x;
        int loc0 = 0;
        double val0 = 0.0;
        if (e0 < q1) {
          loc0 = a.qloc[e0];
          val0 = qv[e0];
        }
        ws_cbar();  // every warp is past the previous task's reads of C (no barrier ends a task)
        for (int i = threadIdx.x; i < kTileElems; i += kWsConsumers) C[i] = 0.0;
        ws_cbar();
        if (e0 < q1) C[swz(loc0 >> 6, loc0 & 63)] = -val0;
        for (int64_t e = e0 + kWsConsumers; e < q1; e += kWsConsumers) {
          const int loc = a.qloc[e];
          C[swz(loc >> 6, loc & 63)] = -qv[e];
        }
        ws_cbar();
        ws_load_swz(acc, C);
      }
      // diagonal finalize: the pivot-rule reference values Q_jj
      if (fin && I == J && threadIdx.x < kTB) {
        const int64_t dq = a.diagq[(int64_t)J * kTB + threadIdx.x];
        qd[threadIdx.x] = dq >= 0 ? a.qv[(int64_t)s * a.nq + dq] : -1.0;
      }
      if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 5] = globaltimer();
      if (type == 0)
        for (int g = sl.rec.g0; g < sl.rec.g1; ++g) {
          const double* b = wait_item();
          ws_axpy_swz(acc, b, 1.0);
          release_item();
        }
      {
        const bool pre = u1 - u0 <= kWsPre;
        const int np = (int)(u1 - u0);
        for (int u = 0; u < np; ++u) {
          const int kk = pre ? sl.sk[u] : __ldg(a.upd_k + u0 + u);
          const int nh = kk > 32 ? 2 : 1;
          for (int kh = 0; kh < nh; ++kh) {
            const double* b = wait_item();
            ws_mma_swz<32>(acc, b, b + 2 * kBoxElems, mI, nJ, min(32, kk - kh * 32));
            release_item();
          }
        }
      }
      if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 1] = globaltimer();
#ifdef PINLA_WS_TRACE_WAIT
      if (a.trace && threadIdx.x == 0 && !fin) a.trace[(int64_t)inst * 8 + 6] = (unsigned long long)ring_wait;
      ring_wait = 0;
#endif
      mbar_wait(sdec + sc.st, sc.ph);
      cont_next = sl.cont_next != 0;
      if (cont_next) {
        // the next chunk of this tile runs next on this SM, from the accumulators
      } else if (type == 1) {
        ws_store_global(acc, a.G + ((int64_t)s * a.ngrp + sl.rec.id) * kTileElems);
      } else {
        ws_neg(acc);
        double* Lt = Ls + (int64_t)sl.rec.tid * kTileElems;
        if (!fin) {
          ws_store_global(acc, Lt);
        } else if (I == J) {
          double* W = C;  // 64 x 65
          ws_cbar();      // every warp is past its own reads of C
          ws_store(acc, W, kLDW);
          ws_cbar();
          const int nb = mI;
          for (int e = threadIdx.x; e < kTB * kTB; e += kWsConsumers) {
            const int r = e >> 6, cc = e & 63;
            if (r >= nb || cc >= nb) W[r * kLDW + cc] = (r == cc) ? 1.0 : 0.0;
          }
          ws_cbar();
          if (warp < 4) ws_potri(W, X, qd, nb, a.rel_tol, &sh_fail, scratch);
          ws_cbar();
          if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 6] = globaltimer();
          if (threadIdx.x == 0 && sh_fail < kTB) atomicMin(a.status + s, (int)(a.tstart[J] + sh_fail));
          ws_tile_store_ld(Lt, W, kLDW);
          ws_tile_store_ld(a.Linv + ((int64_t)s * a.NT + J) * kTileElems, X, kLDW);
          if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 7] = globaltimer();
        } else {
          ws_cbar();
          ws_store_swz(acc, C);
          ws_cbar();
          const double* b = wait_item();  // L_JJ^-1
          Frag8 x;
          ws_zero(x);
          ws_mma_swz<64>(x, C, b, mI, nJ, nJ);  // X = C * Linv^T
          release_item();
          if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 6] = globaltimer();
          ws_store_global(x, Lt);
          if (a.trace && threadIdx.x == 0) a.trace[(int64_t)inst * 8 + 7] = globaltimer();
        }
      }
    }
    if (skip) mbar_wait(sdec + sc.st, sc.ph);  // (every phase of the barrier is passed; cont_next = 0)
#if PINLA_WS_PUBLISHER
    // hand the task's stores to the publisher warp (which counts the successors down)
    __syncwarp();
    if (lane == 0) mbar_arrive(pfull + sc.st);
#else
    // publish: the team barrier orders every thread's tile stores before the
    // successor decrements; each decrement is a gpu-scope release, cumulative
    // over those stores
    if (!cont_next) {
      ws_cbar();
      const int base = inst - inst % ntask;
      const bool pre = succ1 - succ0 <= kWsPre;
      for (int k = succ0 + threadIdx.x; k < succ1; k += kWsConsumers)
        red_dec_release(a.q.cnt + base + (pre ? sl.ssucc[k - succ0] : a.q.succ[k]));
    }
#endif
    if (a.trace && threadIdx.x == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
      a.trace[(int64_t)inst * 8 + 0] = sl.t_ready;
      a.trace[(int64_t)inst * 8 + 2] = globaltimer();
      a.trace[(int64_t)inst * 8 + 3] = smid;
      a.trace[(int64_t)inst * 8 + 4] = sl.t_pop;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(sempty + sc.st);
    sc.advance(kWsSlots);
  }
}

int factor_ws_mode() {  // read per launch (the GPU tests switch kernels between engines)
  const char* e = getenv("PINLA_FACTOR_WS");
  return e ? atoi(e) : 1;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) p = nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}
// rows x 64 fp64 array of row-major 64x64 tiles; box = 16 columns x box_rows
static bool make_map(CUtensorMap* m, const double* base, uint64_t rows, uint32_t box_rows) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)kTB, rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)kTB * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)kBoxCols, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim, gstride, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t launch_factor_ws(const FactorArgs& a, cudaStream_t st) {
  static int grid = 0;
  const size_t smem = kWsSmemBytes;
  if (!grid) {
    cudaError_t e = cudaFuncSetAttribute(factor_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, factor_ws_kernel, kFwsThreads, smem);
    if (occ < 1) {
      fprintf(stderr, "pinla: factor_ws_kernel does not fit an SM (smem %zu)\n", smem);
      return cudaErrorLaunchOutOfResources;
    }
    grid = sms;
  }
  // tensor maps, cached on (L, Linv, G, extents): one encode per handle shape
  struct Key {
    const void *L, *Linv, *G;
    int64_t nT;
    int NT, ngrp, S;
    bool operator==(const Key& o) const {
      return L == o.L && Linv == o.Linv && G == o.G && nT == o.nT && NT == o.NT && ngrp == o.ngrp && S == o.S;
    }
  };
  static Key ckey{};
  static WsMaps cmaps;
  const Key key{a.L, a.Linv, a.G, a.nT, a.NT, a.ngrp, a.S};
  if (!(key == ckey)) {
    bool ok = true;
    for (int h = 0; h < 8 && ok; ++h) ok = make_map(&cmaps.Lh[h], a.L, (uint64_t)a.S * a.nT * kTB, 8 * (h + 1));
    ok = ok && make_map(&cmaps.Linv, a.Linv, (uint64_t)a.S * a.NT * kTB, kTB);
    ok = ok && (a.G && a.ngrp > 0 ? make_map(&cmaps.G, a.G, (uint64_t)a.S * a.ngrp * kTB, kTB)
                                  : make_map(&cmaps.G, a.Linv, (uint64_t)a.S * a.NT * kTB, kTB));
    if (!ok) {
      fprintf(stderr, "pinla: cuTensorMapEncodeTiled failed\n");
      return cudaErrorInvalidValue;
    }
    ckey = key;
  }
  cudaError_t e = launch_queue_init(a.q, a.S, st);
  if (e != cudaSuccess) return e;
  factor_ws_kernel<<<grid, kFwsThreads, smem, st>>>(a, cmaps);
  return cudaGetLastError();
}

}  // namespace pinla
