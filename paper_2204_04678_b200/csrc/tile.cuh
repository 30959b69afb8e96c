// Device primitives for the tile-DAG engine (sm_100a, fp64).
//
// * 64x64 fp64 tiles staged in shared memory with a padded leading dimension
//   of 68 doubles: every DMMA fragment load (plain or transposed access) is
//   bank-conflict free for the 64-bit half-warp wavefronts.
// * 128 threads = 4 warps per CTA; warp w owns the 32x32 output sub-tile at
//   rows (w>>1)*32, cols (w&1)*32 as 4x4 blocks of the m8n8k4 fp64 MMA
//   (SASS DMMA.8x8x4 — the fp64 tensor path of sm_100a; tcgen05 has no f64
//   kind).  The 32 accumulator doubles live in registers.
// * Inter-CTA dependencies: one int flag per produced tile, set with a
//   release store to the launch's epoch and polled with acquire loads.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace pinla {

constexpr int kTB = 64;
constexpr int kLD = 68;
constexpr int kThreads = 128;
constexpr int kTileElems = kTB * kTB;
constexpr int kSmemTile = kTB * kLD;  // doubles

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int atom_dec_acq_rel(int* p) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], -1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

__device__ __forceinline__ void red_dec_release(int* p) {
  asm volatile("red.release.gpu.global.add.s32 [%0], -1;" ::"l"(p) : "memory");
}

// all threads: wait until *flag == epoch (one poller, then CTA barrier)
__device__ __forceinline__ void wait_flag(const int* flag, int epoch) {
  if (threadIdx.x == 0) {
    int spins = 0;
    while (ld_acquire(flag) != epoch) {
      if (++spins > 4) __nanosleep(64);
    }
  }
  __syncthreads();
}
__device__ __forceinline__ void wait_flag2(const int* f1, const int* f2, int epoch) {
  if (threadIdx.x == 0) {
    int spins = 0;
    while (ld_acquire(f1) != epoch) { if (++spins > 4) __nanosleep(64); }
    while (ld_acquire(f2) != epoch) { if (++spins > 4) __nanosleep(64); }
  }
  __syncthreads();
}
// all threads: publish this CTA's global writes, then set the flag
__device__ __forceinline__ void set_flag(int* flag, int epoch) {
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) st_release(flag, epoch);
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// global row-major 64x64 tile -> padded smem tile (async; caller commits/waits)
__device__ __forceinline__ void tile_load_async(double* S, const double* G) {
  for (int c = threadIdx.x; c < kTileElems / 2; c += kThreads) {
    int r = c >> 5, col = (c & 31) * 2;
    cp_async16(S + r * kLD + col, G + r * kTB + col);
  }
}
__device__ __forceinline__ void tile_load(double* S, const double* G) {
  tile_load_async(S, G);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
}
__device__ __forceinline__ void tile_store(double* G, const double* S) {
  for (int c = threadIdx.x; c < kTileElems / 2; c += kThreads) {
    int r = c >> 5, col = (c & 31) * 2;
    double2 v = make_double2(S[r * kLD + col], S[r * kLD + col + 1]);
    __stcg(reinterpret_cast<double2*>(G + r * kTB + col), v);
  }
}
__device__ __forceinline__ void tile_zero(double* S) {
  for (int i = threadIdx.x; i < kSmemTile; i += kThreads) S[i] = 0.0;
}

struct Frag {
  double c[4][4][2];
};

__device__ __forceinline__ void frag_zero(Frag& f) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) f.c[i][j][0] = f.c[i][j][1] = 0.0;
}

__device__ __forceinline__ void warp_origin(int& r0, int& c0, int& g, int& t) {
  int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  r0 = (w >> 1) * 32;
  c0 = (w & 1) * 32;
  g = lane >> 2;
  t = lane & 3;
}

// f = S (smem tile)
__device__ __forceinline__ void frag_load(Frag& f, const double* S) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const double* p = S + (r0 + mi * 8 + g) * kLD + c0 + ni * 8 + 2 * t;
      f.c[mi][ni][0] = p[0];
      f.c[mi][ni][1] = p[1];
    }
}
// f += sign * S
__device__ __forceinline__ void frag_axpy(Frag& f, const double* S, double sign) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const double* p = S + (r0 + mi * 8 + g) * kLD + c0 + ni * 8 + 2 * t;
      f.c[mi][ni][0] += sign * p[0];
      f.c[mi][ni][1] += sign * p[1];
    }
}
// S = f (smem tile)
__device__ __forceinline__ void frag_store(const Frag& f, double* S) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      double* p = S + (r0 + mi * 8 + g) * kLD + c0 + ni * 8 + 2 * t;
      p[0] = f.c[mi][ni][0];
      p[1] = f.c[mi][ni][1];
    }
}
// S (leading dimension ld, scalar stores) = f
__device__ __forceinline__ void frag_store_ld(const Frag& f, double* S, int ld) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      double* p = S + (r0 + mi * 8 + g) * ld + c0 + ni * 8 + 2 * t;
      p[0] = f.c[mi][ni][0];
      p[1] = f.c[mi][ni][1];
    }
}
// global row-major tile = f
__device__ __forceinline__ void frag_store_global(const Frag& f, double* G) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      double* p = G + (r0 + mi * 8 + g) * kTB + c0 + ni * 8 + 2 * t;
      __stcg(reinterpret_cast<double2*>(p), make_double2(f.c[mi][ni][0], f.c[mi][ni][1]));
    }
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// f += sign * op(A) * op(B) over K = 64.
//   op(A)(i,k) = TA ? A[k][i] : A[i][k]
//   op(B)(k,n) = TBt ? B[n][k] : B[k][n]
// Only rows i < mlim, columns n < nlim and k < klim are touched (limits are
// tile heights/widths: padded rows/cols of a tile are zero, so skipping them
// is exact).  All limits are warp-uniform, so the skips do not diverge.
template <bool TA, bool TBt>
__device__ __forceinline__ void frag_mma(Frag& f, const double* A, const double* B, double sign,
                                         int mlim = kTB, int nlim = kTB, int klim = kTB) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
  if (r0 >= mlim || c0 >= nlim) return;
  const int mb = min(4, (mlim - r0 + 7) >> 3);
  const int nbk = min(4, (nlim - c0 + 7) >> 3);
  if (mb == 4 && nbk == 4) {
#pragma unroll 4
    for (int k0 = 0; k0 < klim; k0 += 4) {
      double a[4], b[4];
      const int k = k0 + t;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        int i = r0 + mi * 8 + g;
        a[mi] = sign * (TA ? A[k * kLD + i] : A[i * kLD + k]);
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        int nn = c0 + ni * 8 + g;
        b[ni] = TBt ? B[nn * kLD + k] : B[k * kLD + nn];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
    }
    return;
  }
  for (int k0 = 0; k0 < klim; k0 += 4) {
    double a[4], b[4];
    const int k = k0 + t;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      int i = r0 + mi * 8 + g;
      a[mi] = mi < mb ? sign * (TA ? A[k * kLD + i] : A[i * kLD + k]) : 0.0;
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      int nn = c0 + ni * 8 + g;
      b[ni] = ni < nbk ? (TBt ? B[nn * kLD + k] : B[k * kLD + nn]) : 0.0;
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
        if (mi < mb && ni < nbk) dmma(f.c[mi][ni], a[mi], b[ni]);
  }
}

// global row-major tile rows [0, nrows) -> padded smem tile (async)
__device__ __forceinline__ void tile_load_rows_async(double* S, const double* G, int nrows) {
  const int lim = ((nrows + 7) & ~7) * (kTB / 2);
  for (int c = threadIdx.x; c < lim; c += kThreads) {
    int r = c >> 5, col = (c & 31) * 2;
    cp_async16(S + r * kLD + col, G + r * kTB + col);
  }
}

// ---------------------------------------------------------------------------
// half-K pipeline stages for C -= A B^T with A = L(I,K), B = L(J,K) (both
// row-major, k contiguous).  A stage holds 32 k-columns of A and B in
// [64][kLDH] arrays; kLDH = 36 keeps the DMMA fragment loads conflict free.
constexpr int kLDH = 36;
constexpr int kHalfElems = kTB * kLDH;  // doubles per operand half

__device__ __forceinline__ void half_load_async(double* S, const double* G, int nrows, int khalf) {
  const int rows = (nrows + 7) & ~7;
  for (int c = threadIdx.x; c < rows * 8; c += kThreads) {
    const int r = c >> 3, col = (c & 7) * 4;
    cp_async16(S + r * kLDH + col, G + r * kTB + khalf * 32 + col);
    cp_async16(S + r * kLDH + col + 2, G + r * kTB + khalf * 32 + col + 2);
  }
}

// f += sign * A[i][k] B[n][k] over k < klim (<= 32) of one half stage
__device__ __forceinline__ void frag_mma_half(Frag& f, const double* A, const double* B, double sign,
                                              int mlim, int nlim, int klim) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
  if (r0 >= mlim || c0 >= nlim) return;
  const int mb = min(4, (mlim - r0 + 7) >> 3);
  const int nbk = min(4, (nlim - c0 + 7) >> 3);
  if (mb == 4 && nbk == 4 && klim == 32) {
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      double a[4], b[4];
      const int k = k0 + t;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = sign * A[(r0 + mi * 8 + g) * kLDH + k];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) b[ni] = B[(c0 + ni * 8 + g) * kLDH + k];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
    }
    return;
  }
  for (int k0 = 0; k0 < klim; k0 += 4) {
    double a[4], b[4];
    const int k = k0 + t;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = mi < mb ? sign * A[(r0 + mi * 8 + g) * kLDH + k] : 0.0;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b[ni] = ni < nbk ? B[(c0 + ni * 8 + g) * kLDH + k] : 0.0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
        if (mi < mb && ni < nbk) dmma(f.c[mi][ni], a[mi], b[ni]);
  }
}

// k-rows [32*khalf, 32*khalf+32) of a row-major tile -> [32][kLD] stage buffer
__device__ __forceinline__ void half_rows_load_async(double* S, const double* G, int khalf) {
  for (int c = threadIdx.x; c < 32 * 32; c += kThreads) {
    const int r = c >> 5, col = (c & 31) * 2;
    cp_async16(S + r * kLD + col, G + (khalf * 32 + r) * kTB + col);
  }
}

// f += sign * op(A) op(B) over one half stage (k < klim <= 32):
//   TA: A staged [k][i] (ld kLD) else [i][k] (ld kLDH)
//   TBt: B staged [n][k] (ld kLDH) else [k][n] (ld kLD)
template <bool TA, bool TBt>
__device__ __forceinline__ void frag_mma_half2(Frag& f, const double* A, const double* B,
                                               double sign, int mlim, int nlim, int klim) {
  int r0, c0, g, t;
  warp_origin(r0, c0, g, t);
  if (r0 >= mlim || c0 >= nlim) return;
  const int mb = min(4, (mlim - r0 + 7) >> 3);
  const int nbk = min(4, (nlim - c0 + 7) >> 3);
  if (mb == 4 && nbk == 4 && klim == 32) {
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) {
      double a[4], b[4];
      const int k = k0 + t;
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int i = r0 + mi * 8 + g;
        a[mi] = sign * (TA ? A[k * kLD + i] : A[i * kLDH + k]);
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) {
        const int nn = c0 + ni * 8 + g;
        b[ni] = TBt ? B[nn * kLDH + k] : B[k * kLD + nn];
      }
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
    }
    return;
  }
  // partial tile: the blocks outside (mi >= mb or ni >= nbk) run on zero
  // operands instead of being predicated off (exact: they add +0 to
  // accumulators that are never stored), so the DMMAs need no per-block
  // predicate + warp re-convergence; the K loop is unrolled when full
  auto kstep = [&](int k0) {
    double a[4], b[4];
    const int k = k0 + t;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) {
      const int i = r0 + mi * 8 + g;
      a[mi] = mi < mb ? sign * (TA ? A[k * kLD + i] : A[i * kLDH + k]) : 0.0;
    }
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) {
      const int nn = c0 + ni * 8 + g;
      b[ni] = ni < nbk ? (TBt ? B[nn * kLDH + k] : B[k * kLD + nn]) : 0.0;
    }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
  };
  if (klim == 32) {
#pragma unroll
    for (int k0 = 0; k0 < 32; k0 += 4) kstep(k0);
  } else {
    for (int k0 = 0; k0 < klim; k0 += 4) kstep(k0);
  }
}

template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// acc += sign * sum over pairs u in [u0, u1) of L[ua[u]] L[ub[u]]^T, with a
// two-stage cp.async pipeline over half-K stages (stage buffer = 4 halves)
// stage 0 of the pair pipeline (issued early so that it overlaps other loads)
__device__ __forceinline__ void pair_pipe_issue0(double* stage, const double* Ls, const int* ua,
                                                 const int* ub, int64_t u0, int64_t u1, int mI,
                                                 int nJ) {
  if (u0 >= u1) return;
  half_load_async(stage, Ls + (int64_t)ua[u0] * kTileElems, mI, 0);
  half_load_async(stage + kHalfElems, Ls + (int64_t)ub[u0] * kTileElems, nJ, 0);
  cp_async_commit();
}

// the pair loop proper, stage 0 already issued
__device__ __forceinline__ void pair_pipe_run(Frag& acc, double* stage, const double* Ls,
                                              const int* ua, const int* ub, int64_t u0, int64_t u1,
                                              const int* uk, int mI, int nJ, double sign) {
  // half-steps: (pair, khalf); a pair with K width <= 32 has one half
  auto nhalf = [&](int64_t u) { return uk[u] > 32 ? 2 : 1; };
  if (u0 >= u1) return;
  int64_t u = u0;
  int kh = 0;
  int buf = 0;
  for (;;) {
    // next half-step
    int64_t nu = u;
    int nkh = kh + 1;
    if (nkh >= nhalf(u)) {
      nu = u + 1;
      nkh = 0;
    }
    const bool more = nu < u1;
    if (more) {
      double* nb = stage + (buf ^ 1) * 2 * kHalfElems;
      half_load_async(nb, Ls + (int64_t)ua[nu] * kTileElems, mI, nkh);
      half_load_async(nb + kHalfElems, Ls + (int64_t)ub[nu] * kTileElems, nJ, nkh);
      cp_async_commit();
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_group<0>();
    }
    __syncthreads();
    const int kK = uk[u];
    const int klim = min(32, kK - kh * 32);
    double* cb = stage + buf * 2 * kHalfElems;
    frag_mma_half(acc, cb, cb + kHalfElems, sign, mI, nJ, klim);
    __syncthreads();
    if (!more) break;
    u = nu;
    kh = nkh;
    buf ^= 1;
  }
}

// stage 0 with the first pair's tiles already known (task record)
__device__ __forceinline__ void pair_pipe_issue0_t(double* stage, const double* Ls, int ta, int tb,
                                                   int mI, int nJ) {
  if (ta < 0) return;
  half_load_async(stage, Ls + (int64_t)ta * kTileElems, mI, 0);
  half_load_async(stage + kHalfElems, Ls + (int64_t)tb * kTileElems, nJ, 0);
  cp_async_commit();
}

// Two-stages-ahead variant: the prologue issues half-steps 0 and 1 (one
// cp.async group each) as soon as the task record is known; the loop then
// always has the next half-step in flight and refills a buffer right after
// it is consumed.  Half-step i lives in buffer i & 1.
struct PairCur {
  int64_t u;
  int kh;
};
__device__ __forceinline__ bool pair_cur_next(PairCur& c, const int* uk, int64_t u1) {
  if (c.kh == 0 && uk[c.u] > 32) {
    c.kh = 1;
    return true;
  }
  ++c.u;
  c.kh = 0;
  return c.u < u1;
}
__device__ __forceinline__ void pair_issue(double* buf, const double* Ls, int ta, int tb, int mI,
                                           int nJ, int kh) {
  half_load_async(buf, Ls + (int64_t)ta * kTileElems, mI, kh);
  half_load_async(buf + kHalfElems, Ls + (int64_t)tb * kTileElems, nJ, kh);
  cp_async_commit();
}
// returns the number of half-steps issued (0, 1 or 2); k0 = K extent of the
// first pair, (ta0, tb0) its tiles (task record)
__device__ __forceinline__ int pair_pipe_prologue(double* stage, const double* Ls, const int* ua,
                                                  const int* ub, int64_t u0, int64_t u1, int mI,
                                                  int nJ, int ta0, int tb0, int k0) {
  if (u0 >= u1) return 0;
  pair_issue(stage, Ls, ta0, tb0, mI, nJ, 0);
  if (k0 > 32) {
    pair_issue(stage + 2 * kHalfElems, Ls, ta0, tb0, mI, nJ, 1);
    return 2;
  }
  if (u0 + 1 < u1) {
    pair_issue(stage + 2 * kHalfElems, Ls, ua[u0 + 1], ub[u0 + 1], mI, nJ, 0);
    return 2;
  }
  return 1;
}
// the loop; `extra` = cp.async groups committed AFTER the prologue's that
// must also be complete before the first half-step runs (0 here: callers
// wait for their own groups first)
__device__ __forceinline__ void pair_pipe_run2(Frag& acc, double* stage, const double* Ls,
                                               const int* ua, const int* ub, int64_t u0, int64_t u1,
                                               const int* uk, int mI, int nJ, double sign,
                                               int issued) {
  if (u0 >= u1) return;
  PairCur cur{u0, 0};
  PairCur nxt2 = cur;  // half-step i + 2 (next to issue)
  bool more2 = pair_cur_next(nxt2, uk, u1) && (issued < 2 ? false : pair_cur_next(nxt2, uk, u1));
  int buf = 0;
  for (;;) {
    PairCur nx = cur;
    const bool has_next = pair_cur_next(nx, uk, u1);
    if (has_next) cp_async_wait_group<1>();
    else cp_async_wait_group<0>();
    __syncthreads();
    const int klim = min(32, uk[cur.u] - cur.kh * 32);
    double* cb = stage + buf * 2 * kHalfElems;
    frag_mma_half(acc, cb, cb + kHalfElems, sign, mI, nJ, klim);
    __syncthreads();
    if (more2) {
      pair_issue(cb, Ls, ua[nxt2.u], ub[nxt2.u], mI, nJ, nxt2.kh);
      more2 = pair_cur_next(nxt2, uk, u1);
    }
    if (!has_next) break;
    cur = nx;
    buf ^= 1;
  }
}

__device__ __forceinline__ void pair_gemm_pipelined(Frag& acc, double* stage, const double* Ls,
                                                    const int* ua, const int* ub, int64_t u0,
                                                    int64_t u1, const int* uk, int mI, int nJ,
                                                    double sign) {
  pair_pipe_issue0(stage, Ls, ua, ub, u0, u1, mI, nJ);
  pair_pipe_run(acc, stage, Ls, ua, ub, u0, u1, uk, mI, nJ, sign);
}

// Generic pipelined pair loop with per-pair operand modes (selected
// inversion): acc += sign * sum_u op(A_u) op(B_u).  mode bit0: A from Lsrc
// (else Ssrc), bit1: A transposed (staged by k-rows), bit2: B from Lsrc,
// bit3: B transposed (staged by k-columns).  The k extent of pair u is the
// row count of its L operand's tile row.
__device__ __forceinline__ void pair_gemm_modes(Frag& acc, double* stage, const double* Lsrc,
                                                const double* Ssrc, const int* pa, const int* pb,
                                                const int* mode, int64_t u0, int64_t u1,
                                                const int* tile_row, const int* tbsz,
                                                const int* kx, int mI, int nJ, double sign) {
  if (u0 >= u1) return;
  auto kext = [&](int64_t u) {  // kx: precomputed K extents (smem), else derived
    if (kx) return kx[u];
    const int lt = (mode[u] & 1) ? pa[u] : pb[u];
    return tbsz[tile_row[lt]];
  };
  auto issue = [&](double* buf, int64_t u, int kh) {
    const int md = mode[u];
    const double* Ag = ((md & 1) ? Lsrc : Ssrc) + (int64_t)pa[u] * kTileElems;
    const double* Bg = ((md & 4) ? Lsrc : Ssrc) + (int64_t)pb[u] * kTileElems;
    if (md & 2) half_rows_load_async(buf, Ag, kh);
    else half_load_async(buf, Ag, mI, kh);
    if (md & 8) half_load_async(buf + kHalfElems, Bg, nJ, kh);
    else half_rows_load_async(buf + kHalfElems, Bg, kh);
    cp_async_commit();
  };
  int64_t u = u0;
  int kh = 0;
  int buf = 0;
  issue(stage, u, 0);
  for (;;) {
    int64_t nu = u;
    int nkh = kh + 1;
    if (nkh >= (kext(u) > 32 ? 2 : 1)) {
      nu = u + 1;
      nkh = 0;
    }
    const bool more = nu < u1;
    if (more) {
      issue(stage + (buf ^ 1) * 2 * kHalfElems, nu, nkh);
      cp_async_wait_group<1>();
    } else {
      cp_async_wait_group<0>();
    }
    __syncthreads();
    const int klim = min(32, kext(u) - kh * 32);
    double* cb = stage + buf * 2 * kHalfElems;
    const int md = mode[u];
    if (md & 2) {
      if (md & 8) frag_mma_half2<true, true>(acc, cb, cb + kHalfElems, sign, mI, nJ, klim);
      else frag_mma_half2<true, false>(acc, cb, cb + kHalfElems, sign, mI, nJ, klim);
    } else {
      if (md & 8) frag_mma_half2<false, true>(acc, cb, cb + kHalfElems, sign, mI, nJ, klim);
      else frag_mma_half2<false, false>(acc, cb, cb + kHalfElems, sign, mI, nJ, klim);
    }
    __syncthreads();
    if (!more) break;
    u = nu;
    kh = nkh;
    buf ^= 1;
  }
}

// deterministic warp sum (fixed butterfly)
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace pinla
