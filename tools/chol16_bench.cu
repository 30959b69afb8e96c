// Latency of warp_chol16 / warp_trtri16 alone (one warp, thread 0 clock64)
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2204_04678_b200/csrc/potri.cuh"
using namespace pinla;

__global__ void k(const double* A, long long* out, int reps) {
  __shared__ double W[64 * kLDW];
  __shared__ double X[16 * kLDW];
  __shared__ double qd[64], rdiag[64], xc[16], tt[72];
  __shared__ int fail;
  for (int e = threadIdx.x; e < 4096; e += blockDim.x) W[(e >> 6) * kLDW + (e & 63)] = A[e];
  if (threadIdx.x < 64) qd[threadIdx.x] = A[threadIdx.x * 65];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    warp_chol16(W, kLDW, qd, 16, 1e-13, &fail, 0, rdiag, xc);
    W[0] = A[0];
  }
  long long t1 = clock64();
  for (int r = 0; r < reps; ++r) warp_trtri16(W, kLDW, X, kLDW, rdiag, tt);
  long long t2 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = (t1 - t0) / reps; out[1] = (t2 - t1) / reps; }
}

int main() {
  std::vector<double> A(4096);
  for (int i = 0; i < 64; ++i) for (int j = 0; j < 64; ++j) A[i * 64 + j] = (i == j ? 70.0 : 0.0) + 1.0 / (1.0 + std::abs(i - j));
  double* dA; long long* dO;
  cudaMalloc(&dA, 4096 * 8); cudaMalloc(&dO, 16 * 8);
  cudaMemcpy(dA, A.data(), 4096 * 8, cudaMemcpyHostToDevice);
  for (int blocks : {1, 148, 296}) {
    k<<<blocks, 128>>>(dA, dO, 100);
    long long o[2];
    cudaMemcpy(o, dO, 16, cudaMemcpyDeviceToHost);
    printf("blocks %d: chol16 %lld cycles, trtri16 %lld cycles  (%s)\n", blocks, o[0], o[1], cudaGetErrorString(cudaGetLastError()));
  }
}
