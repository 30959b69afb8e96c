// Microbenchmark of the diagonal-tile POTRI (one CTA per tile).
#include <cstdio>
#include <vector>
#include <cmath>
// POTRI_PROFILE defined by -DPOTRI_PROFILE
#include "../paper_2204_04678_b200/csrc/potri.cuh"
using namespace pinla;

__global__ void k_potri(const double* A, double* L, double* Li, int ntiles, int reps) {
  extern __shared__ double sm[];
  double* W = sm;
  double* X = sm + kTB * kLDW;
  __shared__ double qd[kTB];
  __shared__ int fail;
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    for (int r = 0; r < reps; ++r) {
      for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) W[(e >> 6) * kLDW + (e & 63)] = A[(size_t)t * 4096 + e];
      if (threadIdx.x < kTB) qd[threadIdx.x] = A[(size_t)t * 4096 + threadIdx.x * 65];
      __syncthreads();
      tile_potri(W, X, qd, 64, 1e-13, &fail, X + kTB * kLDW);
    }
    for (int e = threadIdx.x; e < kTB * kTB; e += blockDim.x) {
      L[(size_t)t * 4096 + e] = W[(e >> 6) * kLDW + (e & 63)];
      Li[(size_t)t * 4096 + e] = X[(e >> 6) * kLDW + (e & 63)];
    }
    __syncthreads();
  }
}

#ifndef GRID
#define GRID 296
#endif
int main() {
  const int nt = 296 * 4;
  std::vector<double> A((size_t)nt * 4096);
  for (int t = 0; t < nt; ++t)
    for (int i = 0; i < 64; ++i)
      for (int j = 0; j < 64; ++j)
        A[(size_t)t * 4096 + i * 64 + j] = (i == j ? 70.0 : 0.0) + 1.0 / (1.0 + std::abs(i - j) + 0.01 * t);
  double *dA, *dL, *dLi;
  cudaMalloc(&dA, A.size() * 8); cudaMalloc(&dL, A.size() * 8); cudaMalloc(&dLi, A.size() * 8);
  cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice);
  size_t smem = (2 * kTB * kLDW + kPotriScratch) * 8;
  cudaFuncSetAttribute(k_potri, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int reps : {1, 4}) {
    k_potri<<<GRID, 128, smem>>>(dA, dL, dLi, nt, reps);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    k_potri<<<GRID, 128, smem>>>(dA, dL, dLi, nt, reps);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("reps %d: %.1f us per tile per CTA (2 CTA/SM, %d tiles)\n", reps, ms * 1e3 / (nt / 296.0) / reps, nt);
  }
  // check L * L^T = A and L * Li = I for tile 0
  std::vector<double> L(4096), Li(4096);
  cudaMemcpy(L.data(), dL, 4096 * 8, cudaMemcpyDeviceToHost);
  cudaMemcpy(Li.data(), dLi, 4096 * 8, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0;
  for (int i = 0; i < 64; ++i)
    for (int j = 0; j <= i; ++j) {
      double s = 0, s2 = 0;
      for (int k = 0; k < 64; ++k) { s += L[i * 64 + k] * L[j * 64 + k]; s2 += L[i * 64 + k] * Li[k * 64 + j]; }
      e1 = fmax(e1, fabs(s - A[i * 64 + j]));
      e2 = fmax(e2, fabs(s2 - (i == j)));
    }
#ifdef POTRI_PROFILE
  long long ph[16];
  cudaMemcpyFromSymbol(ph, g_potri_phase, sizeof(ph));
  const char* nm[5] = {"chol16(0)", "S2 x3 (trtri|panel)", "S3 x3 (chol|trailing)", "trtri16(3)", "tail products"};
  double tot = 0; for (int k = 0; k < 5; ++k) tot += ph[k];
  for (int k = 0; k < 5; ++k) printf("  %-12s %5.1f%%  %.0f cycles/tile\n", nm[k], 100.0 * ph[k] / tot, (double)ph[k] / (nt * 5.0));
#endif
  printf("max |LL^T - A| = %.3e, max |L Linv - I| = %.3e, err=%s\n", e1, e2, cudaGetErrorString(cudaGetLastError()));
}
