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
                                            double* xch) {
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
    const double l = sqrt(d);
    const double il = 1.0 / l;
    const double lrj = (r > j) ? a[j] * il : (r == j ? l : 0.0);
    a[j] = lrj;
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
__device__ __forceinline__ void warp_trtri16(const double* L, int ld, double* Bi, int ldi) {
  const int lane = threadIdx.x & 31;
  const int c = lane & 15;
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double s = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) s = fma(-L[i * ld + k], x[k], s);
    x[i] = (i >= c) ? s / L[i * ld + i] : 0.0;
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
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) *sh_fail = kTB;
  for (int e = tid; e < kTB * kTB; e += kThreads) X[(e >> 6) * kLDW + (e & 63)] = 0.0;
  __syncthreads();
  for (int p = 0; p < 4; ++p) {
    const int o = 16 * p;
    if (warp == 0)
      warp_chol16(W + o * kLDW + o, kLDW, qd + o, nb - o, rel_tol, sh_fail, o, xch[0]);
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
        v[c] = s / W[(o + c) * kLDW + o + c];
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) W[r * kLDW + o + c] = v[c];
    }
    __syncthreads();
    PMARK(1);
    // trailing update of the lower part: W[r][k] -= sum_c L[r][o+c] L[k][o+c]
    for (int e = tid; e < nrow * nrow; e += kThreads) {
      const int rr = e / nrow, kk = e - rr * nrow;
      if (kk > rr) continue;
      const int r = o + 16 + rr, k = o + 16 + kk;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 16; ++c) s = fma(W[r * kLDW + o + c], W[k * kLDW + o + c], s);
      W[r * kLDW + k] -= s;
    }
    __syncthreads();
    PMARK(2);
  }
  // diagonal 16x16 inverses, one warp each
  warp_trtri16(W + (16 * warp) * kLDW + 16 * warp, kLDW, X + (16 * warp) * kLDW + 16 * warp, kLDW);
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
