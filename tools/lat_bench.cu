// Single-thread dependent-chain latencies on B200.
#include <cstdio>
__global__ void k(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x * 1e-3 + 1.0, y = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x + 1.0);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = 1.0 / (x + 1.0);
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x + 1.0);
  long long t4 = clock64();
  float xf = (float)x;
  for (int i = 0; i < n; ++i) xf = fmaf(xf, (float)a, (float)b);
  long long t5 = clock64();
  double c0 = 0, c1 = 0;
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(x), "d"(y));
  long long t6 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31);
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; cyc[6] = t7 - t6;
  }
  out[threadIdx.x] = x + xf + c0 + c1;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024); cudaMalloc(&c, 64);
  int n = 4096;
  k<<<1, 32>>>(o, 1.0000001, 1e-9, n, c);
  k<<<1, 32>>>(o, 1.0000001, 1e-9, n, c);
  long long h[7]; cudaMemcpy(h, c, 56, cudaMemcpyDeviceToHost);
  const char* nm[7] = {"DFMA", "sqrt(f64)+add", "div(f64)+add", "rsqrt(f64)+add", "FFMA", "DMMA m8n8k4", "SHFL f64"};
  for (int i = 0; i < 7; ++i) printf("%-16s %.1f cycles/op\n", nm[i], (double)h[i] / n);
}
