// Warp-specialised CTA primitives of the tile-DAG kernels (sm_100a).
//
// One CTA per SM: 8 MMA warps (256 threads) share ONE 64x64 output tile, each
// owning the 32x16 sub-tile at rows (w >> 2) * 32, cols (w & 3) * 16 as 4x2
// blocks of the m8n8k4 fp64 MMA (SASS DMMA.8x8x4); a ninth warp is the
// producer: it claims tasks, waits for their dependencies and moves the
// operand tiles global -> shared with the TMA engine (cp.async.bulk.tensor box
// loads through tensor maps, SASS UTMALDG) into a ring of stages guarded by
// full / empty mbarriers.  The producer runs ahead across task boundaries, so a task's
// claim, dependency wait and first operand loads overlap the previous task's
// math; the MMA warps never issue a global load or a CTA-wide barrier inside
// the pair loop.
#pragma once
#include <cstdio>

#include "tile.cuh"

namespace pinla {

constexpr int kWsConsumers = 256;              // 8 MMA warps
constexpr int kWsThreads = kWsConsumers + 32;  // + the producer warp
// Shared-memory tile format of the warp-specialised kernels: a 64x64 tile is
// four TMA boxes of 16 columns x 64 rows (8 KB each, rows of 128 B), loaded
// with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B: the 32-byte atom (4 doubles) a of
// row r lands at atom a ^ (r & 3) (measured image: profiles/
// tma_swizzle_probe_r02.txt).  A DMMA fragment load -- 4 consecutive rows x 4
// consecutive k per half-warp, plain or transposed -- then touches every bank
// exactly once without any padding.
constexpr int kBoxCols = 16;
constexpr int kBoxElems = kTB * kBoxCols;      // doubles per box (8 KB)
constexpr int kWsStageElems = 4 * kBoxElems;   // ring stage: one tile, or half-K of A + half-K of B
// double index of element (r, c) of a swizzled 64x64 tile
__device__ __forceinline__ int swz(int r, int c) {
  return (c >> 4) * kBoxElems + r * kBoxCols + ((((c >> 2) & 3) ^ (r & 3)) << 2) + (c & 3);
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
// One try_wait per loop iteration, the loop in C++ (try_wait suspends the
// thread in hardware up to a time limit, so this is not a busy poll).
// -DPINLA_WS_WATCHDOG: a wait that lasts > 2 s records (tag, block, thread,
// parity) in g_ws_dbg and traps (`tag` names the call site).
#if defined(PINLA_WS_WATCHDOG) || defined(PINLA_WS_WATCHDOG_DEP)
#define PINLA_WS_DBGBUF 1
#endif
#ifdef PINLA_WS_DBGBUF
// host-mapped record (readable by the CPU after the trap): [0] count, then (tag, block, thread, parity)
static __device__ int* g_ws_dbg;
__device__ __forceinline__ void ws_dbg_record(int tag, int x) {
  int* d = g_ws_dbg;
  const int slot = atomicAdd(d, 1);
  if (slot < 60) {
    d[4 + 4 * slot] = tag;
    d[5 + 4 * slot] = blockIdx.x;
    d[6 + 4 * slot] = threadIdx.x;
    d[7 + 4 * slot] = x;
  }
  __threadfence_system();
}
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity, int tag = 0) {
  unsigned ok = 0;
#ifdef PINLA_WS_WATCHDOG
  const unsigned long long t_in = globaltimer();
#endif
  while (!ok) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
#ifdef PINLA_WS_WAIT_SLEEP
    if (!ok) __nanosleep(PINLA_WS_WAIT_SLEEP);
#endif
#ifdef PINLA_WS_WAIT_TIMER
    if (!ok && globaltimer() == 0ull) __trap();
#endif
#ifdef PINLA_WS_WATCHDOG
    if (!ok && globaltimer() - t_in > 2000000000ull) {
      ws_dbg_record(tag, (int)parity);
      for (int i = 0; i < 2000; ++i) __nanosleep(1000000);  // let the other waiters record themselves
      __trap();
    }
#endif
  }
  (void)tag;
}
// TMA 2-D box load global -> shared through a tensor map (SASS UTMALDG),
// completion counted in bytes on `bar`; (x, y) = (column, row) of the box
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
      "%3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
// order this thread's earlier generic-proxy accesses (the dependency acquire)
// before its later async-proxy (TMA) reads
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// named barriers: 1 = the 256 MMA threads, 2 = MMA warps 0-3 (the POTRI team)
__device__ __forceinline__ void ws_cbar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
struct WsSync128 {
  __device__ __forceinline__ void operator()() const { asm volatile("bar.sync 2, 128;" ::: "memory"); }
};

#ifndef PINLA_WS_PREFETCH
#define PINLA_WS_PREFETCH 1
#endif
// shared-memory fp64 load that the compiler keeps in program order relative to
// the (volatile) DMMAs
__device__ __forceinline__ double lds_f64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

struct Frag8 {
  double c[4][2][2];
};
__device__ __forceinline__ void ws_origin(int& r0, int& c0, int& g, int& t) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  r0 = (w >> 2) * 32;
  c0 = (w & 3) * 16;
  g = lane >> 2;
  t = lane & 3;
}
__device__ __forceinline__ void ws_zero(Frag8& f) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) f.c[i][j][0] = f.c[i][j][1] = 0.0;
}
// f = S (smem tile, leading dimension ld)
__device__ __forceinline__ void ws_store(const Frag8& f, double* S, int ld) {
  int r0, c0, g, t;
  ws_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      double* p = S + (r0 + mi * 8 + g) * ld + c0 + ni * 8 + 2 * t;
      p[0] = f.c[mi][ni][0];
      p[1] = f.c[mi][ni][1];
    }
}
// swizzled-tile forms: f = S, f += sign * S, S = f
__device__ __forceinline__ void ws_load_swz(Frag8& f, const double* S) {
  int r0, c0, g, t;
  ws_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const double2 v = *reinterpret_cast<const double2*>(S + swz(r0 + mi * 8 + g, c0 + ni * 8 + 2 * t));
      f.c[mi][ni][0] = v.x;
      f.c[mi][ni][1] = v.y;
    }
}
__device__ __forceinline__ void ws_axpy_swz(Frag8& f, const double* S, double sign) {
  int r0, c0, g, t;
  ws_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const double2 v = *reinterpret_cast<const double2*>(S + swz(r0 + mi * 8 + g, c0 + ni * 8 + 2 * t));
      f.c[mi][ni][0] += sign * v.x;
      f.c[mi][ni][1] += sign * v.y;
    }
}
__device__ __forceinline__ void ws_store_swz(const Frag8& f, double* S) {
  int r0, c0, g, t;
  ws_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni)
      *reinterpret_cast<double2*>(S + swz(r0 + mi * 8 + g, c0 + ni * 8 + 2 * t)) =
          make_double2(f.c[mi][ni][0], f.c[mi][ni][1]);
}
// global row-major tile = f
__device__ __forceinline__ void ws_store_global(const Frag8& f, double* G) {
  int r0, c0, g, t;
  ws_origin(r0, c0, g, t);
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      double* p = G + (r0 + mi * 8 + g) * kTB + c0 + ni * 8 + 2 * t;
      __stcg(reinterpret_cast<double2*>(p), make_double2(f.c[mi][ni][0], f.c[mi][ni][1]));
    }
}

__device__ __forceinline__ void ws_neg(Frag8& f) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      f.c[i][j][0] = -f.c[i][j][0];
      f.c[i][j][1] = -f.c[i][j][1];
    }
}

// f += A B^T over k < klim, A(i,k) and B(n,k) in swizzled boxes of 16
// k-columns (box b of A at A + b * kBoxElems, same for B).  Only rows
// i < mlim and columns n < nlim matter (padding is zero); blocks outside run
// on zero operands (exact: they add +0 to accumulators that hold the
// padding's zero), so there is no per-block predicate.  k runs in the same
// order as in the 128-thread kernels: the factors are bitwise identical.
// There is no sign argument on purpose: a runtime sign costs one DMUL per A
// fragment on the very pipe the DMMAs use (measured: 20 % math-pipe-throttle
// stalls); a subtracting caller keeps the NEGATED sum in f instead (exact).
template <int KFULL>
__device__ __forceinline__ void ws_mma_swz(Frag8& f, const double* A, const double* B, int mlim,
                                           int nlim, int klim) {
  int r0, c0, g, t;
  ws_origin(r0, c0, g, t);
  if (r0 >= mlim || c0 >= nlim) return;
  const int mb = min(4, (mlim - r0 + 7) >> 3);
  const int nb = min(2, (nlim - c0 + 7) >> 3);
  const int xg = g & 3;
  const double* Ar = A + (r0 + g) * kBoxCols + t;
  const double* Br = B + (c0 + g) * kBoxCols + t;
  if (mb == 4 && nb == 2 && klim == KFULL) {
#if PINLA_WS_PREFETCH
    // fragments of k-step s+1 are loaded (volatile: kept in program order)
    // before the 8 DMMAs of step s, so a warp never waits for a shared-memory
    // load between DMMAs; the operation order per accumulator is unchanged
    double a[2][4], b[2][2];
    auto frag_load = [&](int buf, int k0) {
      const int off = (k0 >> 4) * kBoxElems + ((((k0 >> 2) & 3) ^ xg) << 2);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[buf][mi] = lds_f64(Ar + off + mi * 8 * kBoxCols);
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[buf][ni] = lds_f64(Br + off + ni * 8 * kBoxCols);
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
      const int off = (k0 >> 4) * kBoxElems + ((((k0 >> 2) & 3) ^ xg) << 2);
      double a[4], b[2];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) a[mi] = Ar[off + mi * 8 * kBoxCols];
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) b[ni] = Br[off + ni * 8 * kBoxCols];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
    }
#endif
    return;
  }
  for (int k0 = 0; k0 < klim; k0 += 4) {
    const int off = (k0 >> 4) * kBoxElems + ((((k0 >> 2) & 3) ^ xg) << 2);
    double a[4], b[2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi) a[mi] = mi < mb ? Ar[off + mi * 8 * kBoxCols] : 0.0;
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) b[ni] = ni < nb ? Br[off + ni * 8 * kBoxCols] : 0.0;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 2; ++ni) dmma(f.c[mi][ni], a[mi], b[ni]);
  }
}

// ring cursor shared by the producer and consumer sides (stage, phase parity)
struct RingCur {
  int st;
  unsigned ph;
  __device__ __forceinline__ void advance(int nstages) {
    if (++st == nstages) {
      st = 0;
      ph ^= 1u;
    }
  }
};

}  // namespace pinla
