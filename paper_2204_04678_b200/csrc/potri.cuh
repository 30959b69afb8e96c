// In-tile fused Cholesky + inverse of the diagonal tiles of the
// factorization (the only non-GEMM work on the critical path).
//
// Blocked over four 16-column panels.  The 16x16 diagonal block of a panel
// is factored AND inverted by one warp with register rows and shuffles (no
// CTA barrier inside); the panel TRSM, the trailing update and the block
// inverse assembly are short register-accumulated dot products separated
// by ~15 CTA barriers in total.  Pivot rule of the reference: fail when
// d <= 1e-13 * Q_jj (kernels.py:138), first failing row reported.
#pragma once
#include "tile.cuh"

namespace pinla {

constexpr int kLDW = 65;  // odd stride: row-per-thread access is conflict free

// 16x16 lower block at B (ld) -> L in place; its inverse -> Bi (ld).
// Executed by one full warp; lanes 0..15 own rows.
__device__ __forceinline__ void warp_potri16(double* B, int ld, double* Bi, int ldi,
                                             const double* qd, int nrem, double rel_tol,
                                             int* sh_fail, int rowbase) {
  const int lane = threadIdx.x & 31;
  const int r = lane & 15;
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (k <= r) ? B[r * ld + k] : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = __shfl_sync(0xffffffffu, a[j], j);
    if (lane == 0 && j < nrem) {
      const double q = qd[j];
      if ((q <= 0.0 || !(d > rel_tol * q)) && *sh_fail > rowbase + j) atomicMin(sh_fail, rowbase + j);
    }
    const double l = sqrt(d);
    const double il = 1.0 / l;
    const double lrj = (r > j) ? a[j] * il : (r == j ? l : 0.0);
    a[j] = lrj;
#pragma unroll
    for (int k = j + 1; k < 16; ++k) {
      const double lkj = __shfl_sync(0xffffffffu, lrj, k);
      if (r >= k) a[k] = fma(-lrj, lkj, a[k]);
    }
  }
  // column c = r of the inverse: x[i] = (delta_ic - sum_{c<=k<i} L[i][k] x[k]) / L[i][i]
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double s = (i == r) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) {
      const double lik = __shfl_sync(0xffffffffu, a[k], i);
      s = fma(-lik, x[k], s);
    }
    const double lii = __shfl_sync(0xffffffffu, a[i], i);
    x[i] = (i >= r) ? s / lii : 0.0;
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k <= r) B[r * ld + k] = a[k];
      Bi[k * ldi + r] = x[k];  // column r of the inverse
    }
  }
  __syncwarp();
}

// W (ld 65): lower part of the updated diagonal tile, padded rows/cols set to
// identity.  Out: W = L (strict upper zero), X = L^-1 (ld 65).
__device__ void tile_potri(double* W, double* X, const double* qd, int nb, double rel_tol,
                           int* sh_fail) {
  __shared__ double T[48 * 17];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (tid == 0) *sh_fail = kTB;
  for (int e = tid; e < kTB * kTB; e += kThreads) X[(e >> 6) * kLDW + (e & 63)] = 0.0;
  __syncthreads();
  for (int p = 0; p < 4; ++p) {
    const int o = 16 * p;
    if (warp == 0)
      warp_potri16(W + o * kLDW + o, kLDW, X + o * kLDW + o, kLDW, qd + o, nb - o, rel_tol, sh_fail, o);
    __syncthreads();
    if (p == 3) break;
    // panel TRSM: L[r][o+c] = sum_{k<=c} A[r][o+k] * Linv_pp[c][k], rows r >= o+16
    const int nrow = kTB - o - 16;
    for (int e = tid; e < nrow * 16; e += kThreads) {
      const int rr = e >> 4, c = e & 15, r = o + 16 + rr;
      double s = 0.0;
      for (int k = 0; k <= c; ++k) s = fma(W[r * kLDW + o + k], X[(o + c) * kLDW + o + k], s);
      T[rr * 17 + c] = s;
    }
    __syncthreads();
    for (int e = tid; e < nrow * 16; e += kThreads) {
      const int rr = e >> 4, c = e & 15;
      W[(o + 16 + rr) * kLDW + o + c] = T[rr * 17 + c];
    }
    __syncthreads();
    // trailing update of the lower part: W[r][k] -= sum_c L[r][o+c] L[k][o+c]
    for (int e = tid; e < nrow * nrow; e += kThreads) {
      const int rr = e / nrow, kk = e % nrow;
      if (kk > rr) continue;
      const int r = o + 16 + rr, k = o + 16 + kk;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < 16; ++c) s = fma(W[r * kLDW + o + c], W[k * kLDW + o + c], s);
      W[r * kLDW + k] -= s;
    }
    __syncthreads();
  }
  // block inverse assembly, block rows i = 1..3 in order:
  //   X_ip = -Linv_ii * sum_{k=p}^{i-1} L_ik X_kp      (p < i)
  for (int bi = 1; bi < 4; ++bi) {
    const int ri = 16 * bi;
    // T[(p, row, col)] = sum_k L[ri+row][16p..ri) X[16p..ri)[16p+col]
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
  // strict upper triangle of L is zero
  for (int e = tid; e < kTB * kTB; e += kThreads) {
    const int r = e >> 6, c = e & 63;
    if (c > r) W[r * kLDW + c] = 0.0;
  }
  __syncthreads();
}

}  // namespace pinla
