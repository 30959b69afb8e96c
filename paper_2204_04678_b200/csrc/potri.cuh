// In-tile fused Cholesky + inverse of the diagonal tiles of the
// factorization (the only non-GEMM work on the critical path).
//
// Blocked over four 16-column panels with warp roles (see tile_potri):
//   * warp 0 runs the chain: 16x16 Cholesky (rows in registers, columns
//     broadcast through smem, next pivot recomputed redundantly), 16x16
//     inverse (2x8 blocked + DMMA), update of the next diagonal block;
//   * warps 1-3 solve the panel below by substitution, update the rest of
//     the trailing part on the DMMA pipe (m8n8k4) and assemble the
//     off-diagonal blocks of L^-1 by recursive doubling,
//       X21 = -X22 (L21 X11),  as soon as their inputs exist.
// Pivot rule of the reference: fail when d <= 1e-13 * Q_jj
// (kernels.py:138), the first failing row is reported.
#pragma once
#include "tile.cuh"

namespace pinla {

constexpr int kLDW = 65;  // odd stride: row-per-thread access is conflict free
constexpr int kLDT = 33;
constexpr int kPotriScratch = 32 * kLDT + 16 * 17 + kTB + 16 + 72;  // doubles of caller smem (16B aligned)

// 16x16 lower block at B (ld): Cholesky in place (strict upper set to zero).
// One warp; lanes 0..15 own rows (lanes 16..31 mirror them).  rdiag[r] = 1/L_rr.
// Each step broadcasts the scaled column through shared memory (xc: 16
// doubles, 16-byte aligned; one store per lane, paired 16-byte broadcast
// reads), and every lane recomputes the next pivot
// d_{j+1} = a_{j+1,j+1} - (a_{j+1,j}/L_jj)^2 from lane j+1's two values,
// shuffled one step ahead (bit-identical to lane j+1's own update).
// Measured 2.5k cycles per call vs 3.1k for an all-shuffle version.
__device__ __forceinline__ void warp_chol16(double* B, int ld, const double* qd, int nrem,
                                            double rel_tol, int* sh_fail, int rowbase,
                                            double* rdiag, double* xc) {
  const int lane = threadIdx.x & 31;
  const int r = lane & 15;
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (k <= r) ? B[r * ld + k] : 0.0;
  double d = __shfl_sync(0xffffffffu, a[0], 0);
  double nx_a = __shfl_sync(0xffffffffu, a[0], 1);  // a_{j+1,j}
  double nx_d = __shfl_sync(0xffffffffu, a[1], 1);  // a_{j+1,j+1}
  double myd = 0.0, myil = 0.0;  // this lane's pivot and 1 / L_rr
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double il = rsqrt(d);
    if (r == j) { myd = d; myil = il; }
    const double lrj = (r > j) ? a[j] * il : (r == j ? d * il : 0.0);
    a[j] = lrj;
    double dn = 0.0;
    if (j < 15) {
      const double l1 = nx_a * il;
      dn = fma(-l1, l1, nx_d);
    }
    if (lane < 16) xc[r] = lrj;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 16; k += 2) {
      if (k + 1 > j) {
        const double2 pk = *reinterpret_cast<const double2*>(xc + k);
        if (k > j) {
          const double u = fma(-lrj, pk.x, a[k]);
          a[k] = (r >= k) ? u : a[k];
        }
        const double u = fma(-lrj, pk.y, a[k + 1]);
        a[k + 1] = (r >= k + 1) ? u : a[k + 1];
      }
    }
    __syncwarp();
    if (j + 2 < 16) {
      nx_a = __shfl_sync(0xffffffffu, a[j + 1], j + 2);
      nx_d = __shfl_sync(0xffffffffu, a[j + 2], j + 2);
    }
    d = dn;
  }
  if (lane < 16) {
    rdiag[r] = myil;
    if (r < nrem) {
      const double q = qd[r];
      if (q <= 0.0 || !(myd > rel_tol * q)) atomicMin(sh_fail, rowbase + r);
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) B[r * ld + k] = a[k];
  }
  __syncwarp();
}

// inverse of the lower 16x16 block L (ld) -> Bi (ld), one warp, blocked 2x8:
// lanes 0-7 / 8-15 invert the two 8x8 diagonal halves in parallel (column per
// lane, forward substitution, two partial sums), then
// X21 = -X22 (L21 X11) by two chained DMMA products through tmp (8 x 9).
// Measured 1.1k cycles per call vs 2.0k for a 16-step column substitution.
__device__ __forceinline__ void warp_trtri16(const double* L, int ld, double* Bi, int ldi,
                                             const double* rdiag, double* tmp) {
  const int lane = threadIdx.x & 31;
  const int h = (lane >> 3) & 1, c = lane & 7;
  const int o = 8 * h;
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double s0 = (i == c) ? 1.0 : 0.0, s1 = 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) {
      if (k & 1) s1 = fma(-L[(o + i) * ld + o + k], x[k], s1);
      else s0 = fma(-L[(o + i) * ld + o + k], x[k], s0);
    }
    x[i] = (i >= c) ? (s0 + s1) * rdiag[o + i] : 0.0;
  }
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      Bi[(o + i) * ldi + o + c] = x[i];
      if (h == 0) Bi[i * ldi + 8 + c] = 0.0;  // strict upper block
    }
  }
  __syncwarp();
  const int g = lane >> 2, t4 = lane & 3;
  double t[2] = {0.0, 0.0};
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4) dmma(t, L[(8 + g) * ld + k0 + t4], Bi[(k0 + t4) * ldi + g]);
  tmp[g * 9 + 2 * t4] = t[0];
  tmp[g * 9 + 2 * t4 + 1] = t[1];
  __syncwarp();
  double xo[2] = {0.0, 0.0};
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4)
    dmma(xo, -Bi[(8 + g) * ldi + 8 + k0 + t4], tmp[(k0 + t4) * 9 + g]);
  Bi[(8 + g) * ldi + 2 * t4] = xo[0];
  Bi[(8 + g) * ldi + 2 * t4 + 1] = xo[1];
  __syncwarp();
}

#ifdef POTRI_PROFILE
__device__ long long g_potri_phase[16];
#define PMARK(k)                                                   \
  do {                                                             \
    __syncthreads();                                               \
    if (threadIdx.x == 0) atomicAdd((unsigned long long*)&g_potri_phase[k], (unsigned long long)(clock64() - t_last)); \
    t_last = clock64();                                            \
  } while (0)
#else
#define PMARK(k) do {} while (0)
#endif

// Two independent 8x8 blocks c0 += alpha A0 B0, c1 += alpha A1 B1 on the
// DMMA pipe, interleaved to hide its latency.  A(i,k) = A[i * lda + k];
// B(k,j) = B[j * ldb + k] when kBT, else B[k * ldb + j].  Block 0 runs
// k in [k0a, k1), block 1 k in [k0b, k1) (k0a <= k0b: leading zero chunks of
// a triangular operand are skipped).
template <bool kBT>
__device__ __forceinline__ void mma8_acc2(double (&c0)[2], double (&c1)[2], const double* A0,
                                          const double* A1, int lda, const double* B0,
                                          const double* B1, int ldb, int k0a, int k0b, int k1,
                                          double alpha) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  int k = k0a;
  for (; k < k0b; k += 4) {
    const double av = alpha * A0[g * lda + k + t4];
    const double bv = kBT ? B0[g * ldb + k + t4] : B0[(k + t4) * ldb + g];
    dmma(c0, av, bv);
  }
#pragma unroll 2
  for (; k < k1; k += 4) {
    const double a0 = alpha * A0[g * lda + k + t4];
    const double b0 = kBT ? B0[g * ldb + k + t4] : B0[(k + t4) * ldb + g];
    const double a1 = alpha * A1[g * lda + k + t4];
    const double b1 = kBT ? B1[g * ldb + k + t4] : B1[(k + t4) * ldb + g];
    dmma(c0, a0, b0);
    dmma(c1, a1, b1);
  }
}

__device__ __forceinline__ void st8(double* D, int ld, const double (&acc)[2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  D[g * ld + 2 * t4] = acc[0];
  D[g * ld + 2 * t4 + 1] = acc[1];
}
__device__ __forceinline__ void ld8(double (&acc)[2], const double* D, int ld) {
  const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  acc[0] = D[g * ld + 2 * t4];
  acc[1] = D[g * ld + 2 * t4 + 1];
}

// W (ld 65): lower part of the updated diagonal tile, padded rows/cols set to
// identity.  Out: W = L (strict upper zero), X = L^-1 (ld 65).
// scratch: kPotriScratch doubles of shared memory (the caller's idle buffer).
//
// Warp roles.  Warp 0 runs the chain: chol16(p) -> trtri16(p) -> update of
// the next diagonal block -> chol16(p+1).  Warps 1-3 meanwhile solve the
// panel below (substitution with 1/L_jj, no inverse needed), do the rest of
// the trailing update and every piece of the recursive-doubling inverse as
// soon as its inputs exist:
//   S3(0): T_A = L10 X00          S3(1): X10 = -X11 T_A
//   S2(2): T2 = L[32:64][0:32] X[0:32][0:32]
//   S3(2): T_B = L32 X22, X[32:48][0:32] = -X22 T2[0:16]
//   end:   X32 = -X33 T_B ; X[48:64][0:32] = -[X32 X33] T2
struct SyncCta {
  __device__ __forceinline__ void operator()() const { __syncthreads(); }
};
// `sync` is the barrier of the 128 calling threads: the whole CTA in the
// 128-thread kernels, a named barrier of MMA warps 0-3 in the warp-specialised
// factor kernel.  `tid0` (a multiple of 32) rotates the warp roles: role
// warp = ((threadIdx.x + tid0) & 127) >> 5, so the chain role can sit on a
// scheduler partition that no polling warp shares.
template <class Sync = SyncCta>
__device__ void tile_potri(double* W, double* X, const double* qd, int nb, double rel_tol,
                           int* sh_fail, double* scratch, Sync sync = Sync(), int tid0 = 0) {
#ifdef POTRI_PROFILE
  long long t_last = clock64();
#endif
  double* T2 = scratch;                     // 32 x kLDT
  double* TB = scratch + 32 * kLDT;         // 16 x 17 (T_A, later T_B)
  double* rdiag = TB + 16 * 17;             // 64
  double* xc = rdiag + kTB;                 // 16 (chol16 column broadcast, 16B aligned)
  double* tt = xc + 16;                     // 8 x 9 (trtri16)
  constexpr int kLDB = 17;
  const int tid = (threadIdx.x + tid0) & (kThreads - 1);
  const int warp = tid >> 5;
  if (tid == 0) *sh_fail = kTB;
  // strictly upper 16x16 blocks of W and X are zero (the rest is written below)
  for (int e = tid; e < 6 * 256; e += kThreads) {
    const int b = e >> 8, q = e & 255;
    const int bi = b < 3 ? 0 : (b < 5 ? 1 : 2);
    const int bj = b < 3 ? b + 1 : (b < 5 ? b - 1 : 3);
    const int off = (16 * bi + (q >> 4)) * kLDW + 16 * bj + (q & 15);
    W[off] = 0.0;
    X[off] = 0.0;
  }
  if (warp == 0) warp_chol16(W, kLDW, qd, nb, rel_tol, sh_fail, 0, rdiag, xc);
  sync();
  PMARK(0);
  for (int p = 0; p < 3; ++p) {
    const int o = 16 * p;
    // ---- S2: inverse of the new diagonal block | panel by substitution
    if (warp == 0) {
      warp_trtri16(W + o * kLDW + o, kLDW, X + o * kLDW + o, kLDW, rdiag + o, tt);
    } else {
      const int nrow = kTB - o - 16;
      const int i = tid - 32;
      if (i < nrow) {
        const int r = o + 16 + i;
        double v[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          double s0 = W[r * kLDW + o + c], s1 = 0.0;
#pragma unroll
          for (int k = 0; k < c; ++k) {
            if (k & 1) s1 = fma(-v[k], W[(o + c) * kLDW + o + k], s1);
            else s0 = fma(-v[k], W[(o + c) * kLDW + o + k], s0);
          }
          v[c] = (s0 + s1) * rdiag[o + c];
        }
#pragma unroll
        for (int c = 0; c < 16; ++c) W[r * kLDW + o + c] = v[c];
      }
      if (p == 2 && warp >= 2) {
        // T2 = L[32:64][0:32] X[0:32][0:32]: 16 blocks, two per step, 2 warps
        for (int t = warp - 2; t < 8; t += 2) {
          const int sr = t >> 1, sc0 = 2 * (t & 1), sc1 = sc0 + 1;
          double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
          const double* A = W + (32 + 8 * sr) * kLDW;
          mma8_acc2<false>(c0, c1, A, A, kLDW, X + 8 * sc0, X + 8 * sc1, kLDW, 8 * sc0, 8 * sc1,
                           32, 1.0);
          st8(T2 + (8 * sr) * kLDT + 8 * sc0, kLDT, c0);
          st8(T2 + (8 * sr) * kLDT + 8 * sc1, kLDT, c1);
        }
      }
    }
    sync();
    PMARK(1);
    // ---- S3: next diagonal block + chol16 | rest of the trailing update
    const int ob = 2 * p + 2;  // first 8-row block of the trailing region
    if (warp == 0) {
      // blocks (ob,ob), (ob+1,ob), (ob+1,ob+1) of the next diagonal tile
      double* D0 = W + (8 * ob) * kLDW + 8 * ob;
      double* D1 = W + (8 * ob + 8) * kLDW + 8 * ob;
      double* D2 = W + (8 * ob + 8) * kLDW + 8 * ob + 8;
      double c0[2], c1[2], c2[2], c3[2];
      ld8(c0, D0, kLDW);
      ld8(c1, D1, kLDW);
      ld8(c2, D2, kLDW);
      c3[0] = c3[1] = 0.0;
      mma8_acc2<true>(c0, c1, W + (8 * ob) * kLDW + o, W + (8 * ob + 8) * kLDW + o, kLDW,
                      W + (8 * ob) * kLDW + o, W + (8 * ob) * kLDW + o, kLDW, 0, 0, 16, -1.0);
      mma8_acc2<true>(c2, c3, W + (8 * ob + 8) * kLDW + o, W + (8 * ob + 8) * kLDW + o, kLDW,
                      W + (8 * ob + 8) * kLDW + o, W + (8 * ob + 8) * kLDW + o, kLDW, 0, 16, 16,
                      -1.0);
      st8(D0, kLDW, c0);
      st8(D1, kLDW, c1);
      st8(D2, kLDW, c2);
      __syncwarp();
      warp_chol16(W + (o + 16) * kLDW + o + 16, kLDW, qd + o + 16, nb - o - 16, rel_tol, sh_fail,
                  o + 16, rdiag + o + 16, xc);
    } else {
      const int w = warp - 1;  // 0..2
      // trailing blocks (a, b): a in [ob+2, 8), b in [ob, a]
      const int na = 8 - (ob + 2);
      int nblk = 0;
      for (int x = 0; x < na; ++x) nblk += (ob + 2 + x) - ob + 1;
      for (int b0 = 2 * w; b0 < nblk; b0 += 6) {
        const int b1 = b0 + 1 < nblk ? b0 + 1 : b0;
        int ia = ob + 2, rem = b0;
        while (rem >= ia - ob + 1) { rem -= ia - ob + 1; ++ia; }
        const int ja = ob + rem;
        int ib = ob + 2;
        rem = b1;
        while (rem >= ib - ob + 1) { rem -= ib - ob + 1; ++ib; }
        const int jb = ob + rem;
        double* D0 = W + (8 * ia) * kLDW + 8 * ja;
        double* D1 = W + (8 * ib) * kLDW + 8 * jb;
        double c0[2], c1[2];
        ld8(c0, D0, kLDW);
        ld8(c1, D1, kLDW);
        mma8_acc2<true>(c0, c1, W + (8 * ia) * kLDW + o, W + (8 * ib) * kLDW + o, kLDW,
                        W + (8 * ja) * kLDW + o, W + (8 * jb) * kLDW + o, kLDW, 0, 0, 16, -1.0);
        st8(D0, kLDW, c0);
        if (b1 != b0) st8(D1, kLDW, c1);
      }
      if (p == 0) {
        // T_A = L10 X00 (X00 lower triangular: column block sc from k = 8 sc)
        for (int t = w; t < 2; t += 3) {
          const int sr = t;
          double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
          const double* A = W + (16 + 8 * sr) * kLDW;
          mma8_acc2<false>(c0, c1, A, A, kLDW, X, X + 8, kLDW, 0, 8, 16, 1.0);
          st8(TB + (8 * sr) * kLDB, kLDB, c0);
          st8(TB + (8 * sr) * kLDB + 8, kLDB, c1);
        }
      } else if (p == 1) {
        // X10 = -X11 T_A (X11 lower triangular: row block sr uses k < 8 (sr + 1))
        for (int t = w; t < 2; t += 3) {
          const int sr = t;
          double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
          const double* A = X + (16 + 8 * sr) * kLDW + 16;
          mma8_acc2<false>(c0, c1, A, A, kLDW, TB, TB + 8, kLDB, 0, 0, 8 * (sr + 1), -1.0);
          st8(X + (16 + 8 * sr) * kLDW, kLDW, c0);
          st8(X + (16 + 8 * sr) * kLDW + 8, kLDW, c1);
        }
      } else {
        // T_B = L32 X22 (2 tasks) and X[32:48][0:32] = -X22 T2[0:16] (4 tasks)
        for (int t = w; t < 6; t += 3) {
          double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
          if (t < 2) {
            const int sr = t;
            const double* A = W + (48 + 8 * sr) * kLDW + 32;
            mma8_acc2<false>(c0, c1, A, A, kLDW, X + 32 * kLDW + 32, X + 32 * kLDW + 40, kLDW, 0,
                             8, 16, 1.0);
            st8(TB + (8 * sr) * kLDB, kLDB, c0);
            st8(TB + (8 * sr) * kLDB + 8, kLDB, c1);
          } else {
            const int q = t - 2, sr = q >> 1, sc0 = 2 * (q & 1), sc1 = sc0 + 1;
            const double* A = X + (32 + 8 * sr) * kLDW + 32;
            mma8_acc2<false>(c0, c1, A, A, kLDW, T2 + 8 * sc0, T2 + 8 * sc1, kLDT, 0, 0,
                             8 * (sr + 1), -1.0);
            st8(X + (32 + 8 * sr) * kLDW + 8 * sc0, kLDW, c0);
            st8(X + (32 + 8 * sr) * kLDW + 8 * sc1, kLDW, c1);
          }
        }
      }
    }
    sync();
    PMARK(2);
  }
  // ---- last diagonal block: inverse, then the two remaining products
  if (warp == 0) warp_trtri16(W + 48 * kLDW + 48, kLDW, X + 48 * kLDW + 48, kLDW, rdiag + 48, tt);
  sync();
  PMARK(3);
  {
    // X32 = -X33 T_B: 4 blocks, one per warp
    const int sr = warp >> 1, sc = warp & 1;
    double c0[2] = {0.0, 0.0};
    const int lane = tid & 31, g = lane >> 2, t4 = lane & 3;
#pragma unroll 2
    for (int k = 0; k < 8 * (sr + 1); k += 4) {
      const double av = -X[(48 + 8 * sr + g) * kLDW + 48 + k + t4];
      const double bv = TB[(k + t4) * kLDB + 8 * sc + g];
      dmma(c0, av, bv);
    }
    st8(X + (48 + 8 * sr) * kLDW + 32 + 8 * sc, kLDW, c0);
  }
  sync();
  {
    // X[48:64][0:32] = -[X32 X33] T2: 8 blocks, two per warp
    const int sr = warp >> 1, sc0 = 2 * (warp & 1), sc1 = sc0 + 1;
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
    const double* A = X + (48 + 8 * sr) * kLDW + 32;
    mma8_acc2<false>(c0, c1, A, A, kLDW, T2 + 8 * sc0, T2 + 8 * sc1, kLDT, 0, 0,
                     16 + 8 * (sr + 1), -1.0);
    st8(X + (48 + 8 * sr) * kLDW + 8 * sc0, kLDW, c0);
    st8(X + (48 + 8 * sr) * kLDW + 8 * sc1, kLDW, c1);
  }
  sync();
  PMARK(4);
}

}  // namespace pinla
