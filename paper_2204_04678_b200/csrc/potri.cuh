// In-tile fused Cholesky + inverse of the diagonal tiles of the
// factorization (the only non-GEMM work on the critical path).
//
// Blocked over four 16-column panels:
//   * the 16x16 diagonal block of a panel is factored by one warp (lanes own
//     rows in registers; the pivot and the scaled column are exchanged
//     through shared memory with __syncwarp, no CTA barrier);
//   * the panel below is solved row-per-thread by substitution;
//   * the trailing lower part is updated with register-accumulated dots;
//   * afterwards the four 16x16 diagonal inverses run in parallel (one warp
//     each, column-per-lane forward substitution with broadcast reads) and
//     the off-diagonal blocks of L^-1 are assembled block row by block row:
//       X_ip = -Linv_ii * sum_{k=p}^{i-1} L_ik X_kp.
// Pivot rule of the reference: fail when d <= 1e-13 * Q_jj
// (kernels.py:138), the first failing row is reported.
#pragma once
#include "tile.cuh"

namespace pinla {

constexpr int kLDW = 65;  // odd stride: row-per-thread access is conflict free

// 16x16 lower block at B (ld): Cholesky in place.  One warp; lanes 0..15
// own rows (lanes 16..31 mirror them).  xch: 17 doubles of warp scratch.
__device__ __forceinline__ void warp_chol16(double* B, int ld, const double* qd, int nrem,
                                            double rel_tol, int* sh_fail, int rowbase,
                                            double* xch, double* rdiag) {
  const int lane = threadIdx.x & 31;
  const int r = lane & 15;
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (k <= r) ? B[r * ld + k] : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (lane == j) xch[16] = a[j];
    __syncwarp();
    const double d = xch[16];
    if (lane == 0 && j < nrem) {
      const double q = qd[j];
      if ((q <= 0.0 || !(d > rel_tol * q)) && *sh_fail > rowbase + j) atomicMin(sh_fail, rowbase + j);
    }
    const double il = rsqrt(d);
    const double l = d * il;
    const double lrj = (r > j) ? a[j] * il : (r == j ? l : 0.0);
    a[j] = lrj;
    if (lane == j) rdiag[j] = il;  // 1 / L_jj for the panel solves and inverses
    __syncwarp();
    if (lane < 16) xch[lane] = lrj;
    __syncwarp();
#pragma unroll
    for (int k = j + 1; k < 16; ++k)
      if (r >= k) a[k] = fma(-lrj, xch[k], a[k]);
    __syncwarp();
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k)
      if (k <= r) B[r * ld + k] = a[k];
  }
  __syncwarp();
}

// inverse of the lower 16x16 block L (ld) -> Bi (ld); lane c < 16 computes
// column c by forward substitution (reads of L are warp broadcasts)
__device__ __forceinline__ void warp_trtri16(const double* L, int ld, double* Bi, int ldi,
                                             const double* rdiag) {
  const int lane = threadIdx.x & 31;
  const int c = lane & 15;
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) s = fma(-L[i * ld + k], x[k], s);
    x[i] = (i >= c) ? s * rdiag[i] : 0.0;
  }
  if (lane < 16) {
#pragma unroll
    for (int i = 0; i < 16; ++i) Bi[i * ldi + c] = x[i];
  }
  __syncwarp();
}

// W (ld 65): lower part of the updated diagonal tile, padded rows/cols set to
// identity.  Out: W = L (strict upper zero), X = L^-1 (ld 65).
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
__device__ void tile_potri(double* W, double* X, const double* qd, int nb, double rel_tol,
                           int* sh_fail) {
#ifdef POTRI_PROFILE
  long long t_last = clock64();
#endif
  __shared__ double T[48 * 17];
  __shared__ double xch[4][17];
  __shared__ double rdiag[kTB];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) *sh_fail = kTB;
  for (int e = tid; e < kTB * kTB; e += kThreads) X[(e >> 6) * kLDW + (e & 63)] = 0.0;
  __syncthreads();
  for (int p = 0; p < 4; ++p) {
    const int o = 16 * p;
    if (warp == 0)
      warp_chol16(W + o * kLDW + o, kLDW, qd + o, nb - o, rel_tol, sh_fail, o, xch[0], rdiag + o);
    __syncthreads();
    PMARK(0);
    if (p == 3) break;
    // panel: row r solves L[r][o..o+16) from A[r][o..o+16) by substitution
    const int nrow = kTB - o - 16;
    if (tid < nrow) {
      const int r = o + 16 + tid;
      double v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        double s = W[r * kLDW + o + c];
#pragma unroll
        for (int k = 0; k < c; ++k) s = fma(-v[k], W[(o + c) * kLDW + o + k], s);
        v[c] = s * rdiag[o + c];
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) W[r * kLDW + o + c] = v[c];
    }
    __syncthreads();
    PMARK(1);
    // trailing update of the lower part: W[r][k] -= sum_c L[r][o+c] L[k][o+c]
    const int ntri = nrow * (nrow + 1) / 2;
    for (int e0 = tid; e0 < ntri; e0 += 2 * kThreads) {
      // lower-triangle index -> (rr, kk), two independent elements per pass
      int rr0 = (int)((sqrtf(8.0f * e0 + 1.0f) - 1.0f) * 0.5f);
      while ((rr0 + 1) * (rr0 + 2) / 2 <= e0) ++rr0;
      while (rr0 * (rr0 + 1) / 2 > e0) --rr0;
      const int kk0 = e0 - rr0 * (rr0 + 1) / 2;
      const int e1 = e0 + kThreads;
      int rr1 = rr0, kk1 = kk0;
      const bool two = e1 < ntri;
      if (two) {
        rr1 = (int)((sqrtf(8.0f * e1 + 1.0f) - 1.0f) * 0.5f);
        while ((rr1 + 1) * (rr1 + 2) / 2 <= e1) ++rr1;
        while (rr1 * (rr1 + 1) / 2 > e1) --rr1;
        kk1 = e1 - rr1 * (rr1 + 1) / 2;
      }
      const int r0 = o + 16 + rr0, k0 = o + 16 + kk0, r1 = o + 16 + rr1, k1 = o + 16 + kk1;
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        s0 = fma(W[r0 * kLDW + o + c], W[k0 * kLDW + o + c], s0);
        s1 = fma(W[r1 * kLDW + o + c], W[k1 * kLDW + o + c], s1);
      }
      W[r0 * kLDW + k0] -= s0;
      if (two) W[r1 * kLDW + k1] -= s1;
    }
    __syncthreads();
    PMARK(2);
  }
  // diagonal 16x16 inverses, one warp each
  warp_trtri16(W + (16 * warp) * kLDW + 16 * warp, kLDW, X + (16 * warp) * kLDW + 16 * warp, kLDW,
               rdiag + 16 * warp);
  __syncthreads();
  PMARK(3);
  // block inverse assembly, block rows i = 1..3 in order
  for (int bi = 1; bi < 4; ++bi) {
    const int ri = 16 * bi;
    for (int e = tid; e < bi * 256; e += kThreads) {
      const int p = e >> 8, row = (e >> 4) & 15, col = e & 15;
      const int cc = 16 * p + col;
      double s = 0.0;
      for (int k = 16 * p; k < ri; ++k) s = fma(W[(ri + row) * kLDW + k], X[k * kLDW + cc], s);
      T[(p * 16 + row) * 17 + col] = s;
    }
    __syncthreads();
    for (int e = tid; e < bi * 256; e += kThreads) {
      const int p = e >> 8, row = (e >> 4) & 15, col = e & 15;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < 16; ++k) s = fma(X[(ri + row) * kLDW + ri + k], T[(p * 16 + k) * 17 + col], s);
      X[(ri + row) * kLDW + 16 * p + col] = -s;
    }
    __syncthreads();
  }
  PMARK(4);
  for (int e = tid; e < kTB * kTB; e += kThreads) {
    const int r = e >> 6, c = e & 63;
    if (c > r) W[r * kLDW + c] = 0.0;
  }
  __syncthreads();
}

}  // namespace pinla
