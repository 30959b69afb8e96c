// Time the pieces of the tile POTRI in isolation.
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2204_04678_b200/csrc/potri.cuh"
using namespace pinla;

template <int MODE>
__device__ __forceinline__ void warp16(double* B, int ld, double* Bi, int ldi) {
  const int lane = threadIdx.x & 31;
  const int r = lane & 15;
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (k <= r) ? B[r * ld + k] : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const double d = __shfl_sync(0xffffffffu, a[j], j);
    double l, il;
    if (MODE == 0) { l = sqrt(d); il = 1.0 / l; }
    else { il = rsqrt(d); l = d * il; }
    const double lrj = (r > j) ? a[j] * il : (r == j ? l : 0.0);
    a[j] = lrj;
#pragma unroll
    for (int k = j + 1; k < 16; ++k) {
      const double lkj = __shfl_sync(0xffffffffu, lrj, k);
      if (r >= k) a[k] = fma(-lrj, lkj, a[k]);
    }
  }
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
    x[i] = (i >= r) ? (MODE == 0 ? s / lii : s * (1.0 / lii)) : 0.0;
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (k <= r) B[r * ld + k] = a[k];
      Bi[k * ldi + r] = x[k];
    }
  }
  __syncwarp();
}

// smem-exchange variant: lanes own rows, column values broadcast via smem
__device__ __forceinline__ void warp16_smem(double* B, int ld, double* Bi, int ldi, double* col) {
  const int lane = threadIdx.x & 31;
  const int r = lane & 15;
  double a[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) a[k] = (k <= r) ? B[r * ld + k] : 0.0;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    if (lane == j) col[16] = a[j];
    __syncwarp();
    const double d = col[16];
    const double il = rsqrt(d);
    const double l = d * il;
    const double lrj = (r > j) ? a[j] * il : (r == j ? l : 0.0);
    a[j] = lrj;
    __syncwarp();
    if (lane < 16) col[lane] = lrj;
    __syncwarp();
#pragma unroll
    for (int k = j + 1; k < 16; ++k)
      if (r >= k) a[k] = fma(-lrj, col[k], a[k]);
    __syncwarp();
  }
  if (lane < 16) {
#pragma unroll
    for (int k = 0; k < 16; ++k) if (k <= r) B[r * ld + k] = a[k];
  }
  __syncwarp();
}

template <int MODE>
__global__ void k16(const double* A, double* out, int reps) {
  __shared__ double B[4][16 * 17], Bi[4][16 * 17];
  const int w = threadIdx.x >> 5;
  for (int e = threadIdx.x; e < 4 * 256; e += blockDim.x) {
    int b = e >> 8, i = (e >> 4) & 15, j = e & 15;
    B[b][i * 17 + j] = A[(blockIdx.x * 4 + b) * 256 + i * 16 + j];
  }
  __syncthreads();
  __shared__ double colbuf[4][32];
  for (int r = 0; r < reps; ++r) {
    if (MODE == 2) warp16_smem(B[w], 17, Bi[w], 17, colbuf[w]);
    else warp16<MODE>(B[w], 17, Bi[w], 17);
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 4 * 256; e += blockDim.x) out[blockIdx.x * 1024 + e] = B[e >> 8][(e & 255)] + Bi[e >> 8][e & 255];
}

int main() {
  int nb = 296;
  std::vector<double> A(nb * 1024);
  for (int t = 0; t < nb * 4; ++t)
    for (int i = 0; i < 16; ++i)
      for (int j = 0; j < 16; ++j) A[t * 256 + i * 16 + j] = (i == j ? 20.0 : 0.0) + 1.0 / (1 + abs(i - j));
  double *dA, *dO;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dO, A.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      if (mode == 0) k16<0><<<nb, 128>>>(dA, dO, 64);
      else if (mode == 1) k16<1><<<nb, 128>>>(dA, dO, 64);
      else k16<2><<<nb, 128>>>(dA, dO, 64);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("mode %d (%s): %.3f us per warp16 call\n", mode, mode == 2 ? "smem chol only" : (mode ? "rsqrt" : "ieee div/sqrt"), ms * 1e3 / 64);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
