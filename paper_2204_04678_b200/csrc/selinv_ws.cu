// Warp-specialised selected inversion (block Takahashi), the default selinv
// kernel: the same tasks, pair lists and arithmetic as dag.cu's 128-thread
// selinv_kernel (bitwise identical Sigma), run like factor_ws.cu: ONE CTA per
// SM, a producer warp that claims tasks in the list-schedule order, waits for
// their dependency counters and streams operands through a 4-stage
// shared-memory ring with TMA box loads (tensor maps over the L, Sigma, L^-1
// and group arrays, 128B-span / 32B-atom swizzle), and 8 MMA warps that share
// one 64x64 output tile (32x16 per warp, DMMA.8x8x4).
//
//   Sigma(I,J) = -[ sum_{K in col(J), K>J} Sigma(I,K) L(K,J) ] Linv_J       (I > J)
//   Sigma(J,J) = Linv_J^T [ Linv_J - sum_{K>J} L(K,J)^T Sigma(K,J) ]
//
// A pair's operands come from L or Sigma, plain or transposed (mode bits of
// analysis.cpp): a plain operand is staged as rows x 16-column k boxes, a
// transposed one as 32 k-rows x 16-column boxes; both fragment patterns are
// bank-conflict free in the swizzled layout (ws.cuh).
//
// Reference counterpart: kernels.selinv_range (kernels.py:185-246), root-first
// schedule (cholesky.py:378-391).
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "dag.cuh"
#include "tile.cuh"
#include "ws.cuh"

namespace pinla {

constexpr int kSwStages = 4;
constexpr int kSwSlots = 2;
constexpr int kSwPre = 128;
constexpr int kHalfBox = 32 * kBoxCols;  // doubles of a 32 k-row x 16-column box

struct __align__(16) SelSlot {
  int inst, type, id, tid;
  int flags, I, J, mI;
  int nJ, mlim, nlim, ls;
  int g0, g1, succ0, succ1;
  long long u0, u1;
  int sm[kSwPre];     // pair modes
  int sk[kSwPre];     // pair K extents
  int ssucc[kSwPre];  // successor base tasks
};

struct SwMaps {
  CUtensorMap Lh[8], Sh[8];  // L / Sigma: 16 columns x 8(h+1) rows
  CUtensorMap Lk, Sk;        // L / Sigma: 16 columns x 32 rows (k-row staging of transposed operands)
  CUtensorMap Linv, G;       // full-height boxes
};

// dynamic smem (1 KB aligned): ring | C | T
constexpr size_t kSwSmemBytes = (size_t)(kSwStages * kWsStageElems + 2 * kTileElems) * sizeof(double) + 1024;

// f += op(A) op(B) over k < klim.  TA: A staged by k-rows (A(i,k) = tile[k][i], boxes of 16 i-columns,
// `kbox` doubles apart); else by rows i in boxes of 16 k-columns.  TB: B staged by k-rows
// (B(k,n) = tile[k][n]); else by rows n (B(k,n) = tile[n][k]).
template <bool TA, bool TB, int KFULL>
__device__ __forceinline__ void ws_mma_gen(Frag8& f, const double* A, const double* B, int mlim, int nlim,
                                           int klim, int kbox) {
  int r0, c0, g, t;
  ws_origin(r0, c0, g, t);
  if (r0 >= mlim || c0 >= nlim) return;
  const int mb = min(4, (mlim - r0 + 7) >> 3);
  const int nb = min(2, (nlim - c0 + 7) >> 3);
  const int xg = g & 3, gh = g >> 2;
  // per-thread bases; the k-dependent part is added per step
  const double* Ap = TA ? A + (r0 >> 4) * kbox + t * kBoxCols + xg : A + (r0 + g) * kBoxCols + t;
  const double* Bp = TB ? B + (c0 >> 4) * kbox + t * kBoxCols + xg : B + (c0 + g) * kBoxCols + t;
  auto a_ptr = [&](int mi, int k0) -> const double* {
    if (TA) return Ap + (mi >> 1) * kbox + k0 * kBoxCols + ((((mi & 1) * 2 + gh) ^ t) << 2);
    return Ap + (k0 >> 4) * kBoxElems + mi * 8 * kBoxCols + ((((k0 >> 2) & 3) ^ xg) << 2);
  };
  auto b_ptr = [&](int ni, int k0) -> const double* {
    if (TB) return Bp + k0 * kBoxCols + (((ni * 2 + gh) ^ t) << 2);
    return Bp + (k0 >> 4) * kBoxElems + ni * 8 * kBoxCols + ((((k0 >> 2) & 3) ^ xg) << 2);
  };
  auto a_at = [&](int mi, int k0) -> double { return *a_ptr(mi, k0); };
  auto b_at = [&](int ni, int k0) -> double { return *b_ptr(ni, k0); };
  if (mb == 4 && nb == 2 && klim == KFULL) {
#if PINLA_WS_PREFETCH
    // fragments of k-step s+1 loaded before the DMMAs of step s (see ws_mma_swz)
    double a[2][4], b[2][2];
    auto frag_load = [&](int buf, int k0) {
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[buf][mi] = lds_f64(a_ptr(mi, k0));
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[buf][ni] = lds_f64(b_ptr(ni, k0));
    };
    frag_load(0, 0);
#pragma unroll
    for (int k0 = 0; k0 < KFULL; k0 += 4) {
      const int cur = (k0 >> 2) & 1;
      if (k0 + 4 < KFULL) frag_load(cur ^ 1, k0 + 4);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(f.c[mi][ni], a[cur][mi], b[cur][ni]);
    }
#else
#pragma unroll
    for (int k0 = 0; k0 < KFULL; k0 += 4) {
      double a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = a_at(mi, k0);
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = b_at(ni, k0);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
    }
#endif
    return;
  }
  for (int k0 = 0; k0 < klim; k0 += 4) {
    double a[4], b[2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = mi < mb ? a_at(mi, k0) : 0.0;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = ni < nb ? b_at(ni, k0) : 0.0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
  }
}

__global__ void __launch_bounds__(kWsThreads, 1)
    selinv_ws_kernel(SelinvArgs a, const __grid_constant__ SwMaps maps) {
  extern __shared__ __align__(1024) double smem_raw[];
  double* smem = smem_raw + (((smem_u32(smem_raw) + 1023u) & ~1023u) - smem_u32(smem_raw)) / 8;
  double* ring = smem;
  double* C = ring + kSwStages * kWsStageElems;
  double* T = C + kTileElems;
  __shared__ unsigned long long full[kSwStages], empty[kSwStages], sfull[kSwSlots], sempty[kSwSlots];
  __shared__ SelSlot slots[kSwSlots];
  __shared__ int pclaim[2];
  __shared__ int ppa[kSwPre], ppb[kSwPre], pmd[kSwPre], pkk[kSwPre];  // producer: staged pair records
  const int ntask = a.q.ntask;
  const int lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kSwStages; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kWsConsumers / 32);
    }
    for (int i = 0; i < kSwSlots; ++i) {
      mbar_init(sfull + i, 1);
      mbar_init(sempty + i, kWsConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (threadIdx.x >= kWsConsumers) {
    // ------------------------------------------------------------ producer
    RingCur rc{0, 1u};
    RingCur sc{0, 1u};
    const int total = a.q.nact * ntask;
    for (;;) {
      if (lane == 0) {
        int inst = -1, t = 0;
        const int idx = atomicAdd(a.q.ctr, 1);
        if (idx < total) {
          t = a.q.order[idx / a.q.nact];
          inst = a.q.act_slots[idx % a.q.nact] * ntask + t;
        }
        pclaim[0] = inst;
        pclaim[1] = t;
      }
      __syncwarp();
      const int inst = pclaim[0], t = pclaim[1];
      __syncwarp();  // every lane has read the claim before lane 0 writes the next one
      mbar_wait(sempty + sc.st, sc.ph, 1);
      SelSlot& sl = slots[sc.st];
      if (inst < 0) {
        if (lane == 0) {
          sl.inst = -1;
          mbar_arrive(sfull + sc.st);
        }
        break;
      }
      const int s = inst / ntask;
      if (lane == 0) {
        // the task's scalars (a few dependent index loads) are in flight
        // before the dependency wait
        const int4 tk = __ldg(a.tasks + t);
        const int type = tk.x == 1 ? 1 : 0, id = tk.z;
        const int tid = type ? __ldg(a.grp_tile + id) : __ldg(a.chunk_tile + id);
        const int I = __ldg(a.tile_row + tid), J = __ldg(a.tile_col + tid);
        const int mI = __ldg(a.tbsz + I), nJ = __ldg(a.tbsz + J);
        const int flags = type ? 0 : __ldg(a.chunk_flags + id);
        sl.type = type;
        sl.id = id;
        sl.tid = tid;
        sl.flags = flags;
        sl.I = I;
        sl.J = J;
        sl.mI = mI;
        sl.nJ = nJ;
        sl.mlim = type ? mI : (I == J ? nJ : mI);
        sl.nlim = nJ;
        sl.ls = __ldg(a.lslot + s);
        sl.u0 = type ? __ldg(a.grp_rng + id) : __ldg(a.chunk_rng + id);
        sl.u1 = type ? __ldg(a.grp_rng + id + 1) : __ldg(a.chunk_rng + id + 1);
        sl.g0 = (!type && (flags & 1)) ? __ldg(a.tile_grp_ptr + tid) : 0;
        sl.g1 = (!type && (flags & 1)) ? __ldg(a.tile_grp_ptr + tid + 1) : 0;
        sl.succ0 = __ldg(a.q.succ_ptr + t);
        sl.succ1 = __ldg(a.q.succ_ptr + t + 1);
        sl.inst = inst;
      }
      __syncwarp();
      const int type = sl.type, flags = sl.flags, tid = sl.tid, J = sl.J;
      const int mlim = sl.mlim, nlim = sl.nlim, ls = sl.ls;
      const long long u0 = sl.u0, u1 = sl.u1;
      const int g0 = sl.g0, g1 = sl.g1, succ0 = sl.succ0, succ1 = sl.succ1;
      const bool pre = u1 - u0 <= kSwPre;
      auto kext_of = [&](int md, int pa, int pb) {
        return __ldg(a.tbsz + __ldg(a.tile_row + ((md & 1) ? pa : pb)));
      };
      if (pre)
        for (int k = lane; k < (int)(u1 - u0); k += 32) {
          const int md = __ldg(a.mode + u0 + k);
          sl.sm[k] = md;
          sl.sk[k] = kext_of(md, __ldg(a.pa + u0 + k), __ldg(a.pb + u0 + k));
        }
      if (succ1 - succ0 <= kSwPre)
        for (int k = lane; k < succ1 - succ0; k += 32) sl.ssucc[k] = __ldg(a.q.succ + succ0 + k);
      if (lane == 0) {
        int spins = 0;
        while (ld_acquire(a.q.cnt + inst) != 0) {
          if (++spins > 4) __nanosleep(32);
#ifdef PINLA_WS_WATCHDOG_DEP
          if (spins > (1 << 22)) {
            ws_dbg_record(100 + ld_acquire(a.q.cnt + inst), inst);
            for (int i = 0; i < 2000; ++i) __nanosleep(1000000);
            __trap();
          }
#endif
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(sfull + sc.st);
      sc.advance(kSwSlots);
      fence_proxy_async();
      const int64_t lbase = (int64_t)ls * a.nT, sbase = (int64_t)s * a.nT;
      // Lane 0 alone drives the ring (waits for a free stage, arms the `full`
      // barrier, issues the TMA loads); the other lanes only stage the next
      // block of pair records in shared memory between two __syncwarp()s.
      // (An earlier version broadcast the records with __shfl_sync from
      // inside lane-divergent code and deadlocked inside the warp.)
      auto put_tile = [&](const CUtensorMap* m, int64_t tile) {  // lane 0
        mbar_wait(empty + rc.st, rc.ph, 2);
        mbar_expect_tx(full + rc.st, kTB * kTB * 8);
        double* dst = ring + rc.st * kWsStageElems;
#pragma unroll
        for (int b = 0; b < 4; ++b)
          tma_load_2d(dst + b * kBoxElems, m, b * kBoxCols, (int)(tile * kTB), full + rc.st);
        rc.advance(kSwStages);
      };
      const int ra = (mlim + 7) & ~7, rb = (nlim + 7) & ~7;
      const int nia = (mlim + kBoxCols - 1) / kBoxCols, nib = (nlim + kBoxCols - 1) / kBoxCols;
      auto put_half = [&](int md, int pa, int pb, int kh, int kext) {  // lane 0
        const int klim = min(32, kext - kh * 32);
        const int nbox = (klim + kBoxCols - 1) / kBoxCols;
        const bool aL = md & 1, aT = md & 2, bL = md & 4, bN = !(md & 8);  // bN: B staged by k-rows
        const unsigned bytes = (unsigned)((aT ? nia * 32 : nbox * ra) + (bN ? nib * 32 : nbox * rb)) * kBoxCols * 8u;
        mbar_wait(empty + rc.st, rc.ph, 3);
        mbar_expect_tx(full + rc.st, bytes);
        double* dst = ring + rc.st * kWsStageElems;
        const int ya = (int)(((aL ? lbase : sbase) + pa) * kTB), yb = (int)(((bL ? lbase : sbase) + pb) * kTB);
        if (aT) {
          const CUtensorMap* m = aL ? &maps.Lk : &maps.Sk;
          for (int b = 0; b < nia; ++b) tma_load_2d(dst + b * kHalfBox, m, b * kBoxCols, ya + kh * 32, full + rc.st);
        } else {
          const CUtensorMap* m = (aL ? maps.Lh : maps.Sh) + (ra / 8 - 1);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(dst + b * kBoxElems, m, kh * 32 + b * kBoxCols, ya, full + rc.st);
        }
        double* dstb = dst + 2 * kBoxElems;
        if (bN) {
          const CUtensorMap* m = bL ? &maps.Lk : &maps.Sk;
          for (int b = 0; b < nib; ++b) tma_load_2d(dstb + b * kHalfBox, m, b * kBoxCols, yb + kh * 32, full + rc.st);
        } else {
          const CUtensorMap* m = (bL ? maps.Lh : maps.Sh) + (rb / 8 - 1);
          for (int b = 0; b < nbox; ++b)
            tma_load_2d(dstb + b * kBoxElems, m, kh * 32 + b * kBoxCols, yb, full + rc.st);
        }
        rc.advance(kSwStages);
      };
      if (lane == 0 && type == 0) {
        if (flags & 1) {
          for (int g = g0; g < g1; ++g) put_tile(&maps.G, (int64_t)s * a.ngbuf + __ldg(a.gbuf + g));
        } else {
          put_tile(maps.Sh + 7, sbase + tid);  // the running sum
        }
      }
      for (long long ub = u0; ub < u1; ub += kSwPre) {
        const int nb = u1 - ub < kSwPre ? (int)(u1 - ub) : kSwPre;
        __syncwarp();  // lane 0 is done with the previous block
        for (int k = lane; k < nb; k += 32) {
          const int md = __ldg(a.mode + ub + k), pa = __ldg(a.pa + ub + k), pb = __ldg(a.pb + ub + k);
          ppa[k] = pa;
          ppb[k] = pb;
          pmd[k] = md;
          pkk[k] = pre ? sl.sk[k] : kext_of(md, pa, pb);
        }
        __syncwarp();
        if (lane == 0)
          for (int j = 0; j < nb; ++j) {
            const int kk = pkk[j];
            put_half(pmd[j], ppa[j], ppb[j], 0, kk);
            if (kk > 32) put_half(pmd[j], ppa[j], ppb[j], 1, kk);
          }
      }
      if (lane == 0 && type == 0 && (flags & 2)) put_tile(&maps.Linv, (int64_t)ls * a.NT + J);
      __syncwarp();
    }
    return;
  }

  // ---------------------------------------------------------------- MMA team
  RingCur rc{0, 0u};
  RingCur sc{0, 0u};
  auto wait_item = [&]() -> double* {
    mbar_wait(full + rc.st, rc.ph, 4);
    return ring + rc.st * kWsStageElems;
  };
  auto release_item = [&]() {
    __syncwarp();
    if (lane == 0) mbar_arrive(empty + rc.st);
    rc.advance(kSwStages);
  };
  for (;;) {
    mbar_wait(sfull + sc.st, sc.ph, 5);
    const SelSlot& sl = slots[sc.st];
    const int inst = sl.inst;
    if (inst < 0) break;
    const unsigned long long t_c = a.trace ? globaltimer() : 0ull;
    const int s = inst / ntask;
    const int type = sl.type, flags = sl.flags, I = sl.I, J = sl.J;
    const int mI = sl.mI, nJ = sl.nJ, mlim = sl.mlim, nlim = sl.nlim;
    const long long u0 = sl.u0, u1 = sl.u1;
    Frag8 acc;
    if (type == 1 || (flags & 1)) {
      ws_zero(acc);
      for (int g = sl.g0; g < sl.g1; ++g) {
        const double* b = wait_item();
        ws_axpy_swz(acc, b, 1.0);
        release_item();
      }
    } else {
      const double* b = wait_item();
      ws_load_swz(acc, b);
      release_item();
    }
    {
      const bool pre = u1 - u0 <= kSwPre;
      const int np = (int)(u1 - u0);
      for (int u = 0; u < np; ++u) {
        int md, kk;
        if (pre) {
          md = sl.sm[u];
          kk = sl.sk[u];
        } else {
          md = __ldg(a.mode + u0 + u);
          kk = __ldg(a.tbsz + __ldg(a.tile_row + ((md & 1) ? __ldg(a.pa + u0 + u) : __ldg(a.pb + u0 + u))));
        }
        const int nh = kk > 32 ? 2 : 1;
        for (int kh = 0; kh < nh; ++kh) {
          const double* b = wait_item();
          const int klim = min(32, kk - kh * 32);
          const double* B = b + 2 * kBoxElems;
          if (md & 2) {
            if (md & 8) ws_mma_gen<true, false, 32>(acc, b, B, mlim, nlim, klim, kHalfBox);
            else ws_mma_gen<true, true, 32>(acc, b, B, mlim, nlim, klim, kHalfBox);
          } else {
            if (md & 8) ws_mma_gen<false, false, 32>(acc, b, B, mlim, nlim, klim, kHalfBox);
            else ws_mma_gen<false, true, 32>(acc, b, B, mlim, nlim, klim, kHalfBox);
          }
          release_item();
        }
      }
    }
    if (type == 1) {
      ws_store_global(acc, a.G + ((int64_t)s * a.ngbuf + a.gbuf[sl.id]) * kTileElems);
    } else {
      double* St = a.Sg + ((int64_t)s * a.nT + sl.tid) * kTileElems;
      if (!(flags & 2)) {
        ws_store_global(acc, St);
      } else if (I != J) {
        // Sigma(I,J) = -(sum_K Sigma(I,K) L(K,J)) Linv_J
        ws_cbar();
        ws_store_swz(acc, C);
        ws_cbar();
        const double* b = wait_item();  // Linv_J
        Frag8 x;
        ws_zero(x);
        ws_mma_gen<false, true, 64>(x, C, b, mI, nJ, nJ, kBoxElems);
        release_item();
        ws_neg(x);
        ws_store_global(x, St);
      } else {
        // Sigma(J,J) = Linv_J^T (Linv_J - sum_K L(K,J)^T Sigma(K,J)), symmetrized
        ws_cbar();
        ws_store_swz(acc, C);
        const double* b = wait_item();  // Linv_J
        ws_cbar();
        for (int e = threadIdx.x; e < kTileElems; e += kWsConsumers) C[e] = b[e] - C[e];
        ws_cbar();
        Frag8 x;
        ws_zero(x);
        ws_mma_gen<true, true, 64>(x, b, C, kTB, kTB, kTB, kBoxElems);
        release_item();
        ws_store_swz(x, T);
        ws_cbar();
        for (int e = threadIdx.x; e < kTileElems; e += kWsConsumers) {
          const int r = e >> 6, cc = e & 63;
          __stcg(St + e, 0.5 * (T[swz(r, cc)] + T[swz(cc, r)]));
        }
      }
    }
    ws_cbar();
    {
      const int base = inst - inst % ntask;
      const int succ0 = sl.succ0, succ1 = sl.succ1;
      const bool pre = succ1 - succ0 <= kSwPre;
      for (int k = succ0 + threadIdx.x; k < succ1; k += kWsConsumers)
        red_dec_release(a.q.cnt + base + (pre ? sl.ssucc[k - succ0] : a.q.succ[k]));
    }
    if (a.trace && threadIdx.x == 0) {
      a.trace[(int64_t)inst * 4 + 0] = t_c;
      a.trace[(int64_t)inst * 4 + 1] = t_c;
      a.trace[(int64_t)inst * 4 + 2] = globaltimer();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(sempty + sc.st);
    sc.advance(kSwSlots);
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                  CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                  CUtensorMapFloatOOBfill);
// rows x 64 fp64 array of row-major 64x64 tiles; box = 16 columns x box_rows, 128B-span / 32B-atom swizzle
bool ws_make_tile_map(void* m, const double* base, uint64_t rows, uint32_t box_rows) {
  static EncodeTiledFn enc = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess) p = nullptr;
    return (EncodeTiledFn)p;
  }();
  if (!enc) return false;
  const cuuint64_t gdim[2] = {(cuuint64_t)kTB, rows};
  const cuuint64_t gstride[1] = {(cuuint64_t)kTB * sizeof(double)};
  const cuuint32_t box[2] = {(cuuint32_t)kBoxCols, box_rows};
  const cuuint32_t es[2] = {1, 1};
  return enc(static_cast<CUtensorMap*>(m), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), gdim,
             gstride, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int selinv_ws_mode() {  // PINLA_SELINV_WS = 0: 128-thread kernel; otherwise (default) this one
  const char* e = getenv("PINLA_SELINV_WS");
  return e ? atoi(e) : 1;
}

cudaError_t launch_selinv_ws(const SelinvArgs& a0, cudaStream_t st) {
  static int grid = 0;
  if (!grid) {
    cudaError_t e = cudaFuncSetAttribute(selinv_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kSwSmemBytes);
    if (e != cudaSuccess) return e;
    int dev, sms = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, selinv_ws_kernel, kWsThreads, kSwSmemBytes);
    if (occ < 1) {
      fprintf(stderr, "pinla: selinv_ws_kernel does not fit an SM (smem %zu)\n", kSwSmemBytes);
      return cudaErrorLaunchOutOfResources;
    }
    grid = sms;
  }
  SelinvArgs a = a0;
  a.q.fifo = 0;  // list-schedule order (q.order), dependency counters
  a.q.hot = nullptr;
  struct Key {
    const void *L, *Linv, *Sg, *G;
    int64_t nT;
    int NT, ngbuf, S, SL;
    bool operator==(const Key& o) const {
      return L == o.L && Linv == o.Linv && Sg == o.Sg && G == o.G && nT == o.nT && NT == o.NT &&
             ngbuf == o.ngbuf && S == o.S && SL == o.SL;
    }
  };
  static Key ckey{};
  static SwMaps cmaps;
  const Key key{a.L, a.Linv, a.Sg, a.G, a.nT, a.NT, a.ngbuf, a.S, a.SL};
  if (!(key == ckey)) {
    bool ok = true;
    const uint64_t lrows = (uint64_t)a.SL * a.nT * kTB, srows = (uint64_t)a.S * a.nT * kTB;
    for (int h = 0; h < 8 && ok; ++h)
      ok = ws_make_tile_map(&cmaps.Lh[h], a.L, lrows, 8 * (h + 1)) &&
           ws_make_tile_map(&cmaps.Sh[h], a.Sg, srows, 8 * (h + 1));
    ok = ok && ws_make_tile_map(&cmaps.Lk, a.L, lrows, 32) && ws_make_tile_map(&cmaps.Sk, a.Sg, srows, 32);
    ok = ok && ws_make_tile_map(&cmaps.Linv, a.Linv, (uint64_t)a.SL * a.NT * kTB, kTB);
    ok = ok && ws_make_tile_map(&cmaps.G, a.G, (uint64_t)a.S * a.ngbuf * kTB, kTB);
    if (!ok) {
      fprintf(stderr, "pinla: cuTensorMapEncodeTiled failed (selinv)\n");
      return cudaErrorInvalidValue;
    }
    ckey = key;
  }
  cudaError_t e = launch_queue_init(a.q, a.S, st);
  if (e != cudaSuccess) return e;
#ifdef PINLA_WS_DBGBUF
  static int* hdbg = nullptr;
  if (!hdbg) {
    cudaHostAlloc(&hdbg, 4096, cudaHostAllocMapped);
    int* ddbg = nullptr;
    cudaHostGetDevicePointer(&ddbg, hdbg, 0);
    cudaMemcpyToSymbol(g_ws_dbg, &ddbg, sizeof(ddbg));
  }
  for (int i = 0; i < 1024; ++i) hdbg[i] = 0;
#endif
  selinv_ws_kernel<<<grid, kWsThreads, kSwSmemBytes, st>>>(a, cmaps);
  if (getenv("PINLA_SYNC_DEBUG")) {
    cudaError_t se = cudaStreamSynchronize(st);
    fprintf(stderr, "pinla: selinv_ws_kernel sync: %s\n", cudaGetErrorString(se));
  }
#ifdef PINLA_WS_DBGBUF
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    fprintf(stderr, "pinla watchdog: %d waiters (tag, block, thread, x):", hdbg[0]);
    for (int i = 0; i < hdbg[0] && i < 60; ++i)
      fprintf(stderr, " (%d,%d,%d,%d)", hdbg[4 + 4 * i], hdbg[5 + 4 * i], hdbg[6 + 4 * i], hdbg[7 + 4 * i]);
    fprintf(stderr, "\npinla watchdog: consumers (block: inst, items, type*1000+flags*100+npairs, last done):");
    for (int b = 0; b < 148; ++b)
      if (hdbg[256 + 4 * b] != -2 || true)
        fprintf(stderr, " [%d: %d %d %d %d]", b, hdbg[256 + 4 * b], hdbg[257 + 4 * b], hdbg[258 + 4 * b],
                hdbg[259 + 4 * b]);
    fprintf(stderr, "\n");
  }
#endif
  return cudaGetLastError();
}

}  // namespace pinla
