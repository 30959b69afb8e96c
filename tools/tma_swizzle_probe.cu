// Empirical shared-memory image of a 2-D TMA box load (fp64, box 16 cols x 64 rows)
// for each swizzle mode: prints, per smem double index, the (row, col) it holds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/tma_swizzle_probe tools/tma_swizzle_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__global__ void probe(const __grid_constant__ CUtensorMap m, double* out, int x, int y, int nbytes) {
  extern __shared__ __align__(1024) double sm[];
  __shared__ unsigned long long bar;
  unsigned sb = (unsigned)__cvta_generic_to_shared(sm);
  unsigned pad = ((sb + 1023u) & ~1023u) - sb;
  double* box = sm + pad / 8;
  unsigned bb = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bb));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) box[i] = -1.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.proxy.async;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bb), "r"(nbytes));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            (unsigned)__cvta_generic_to_shared(box)),
        "l"(&m), "r"(x), "r"(y), "r"(bb)
        : "memory");
  }
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(bb)
      : "memory");
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) out[i] = box[i];
}
int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaFree(0);
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncFn enc = (EncFn)fp;
  const int R = 256, Cc = 64;
  std::vector<double> h(R * Cc);
  for (int r = 0; r < R; ++r) for (int c = 0; c < Cc; ++c) h[r * Cc + c] = r * 64 + c;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 2048 * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 20480);
  struct { CUtensorMapSwizzle s; const char* n; } modes[] = {
      {CU_TENSOR_MAP_SWIZZLE_NONE, "NONE"}, {CU_TENSOR_MAP_SWIZZLE_128B, "128B"},
      {CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, "128B_ATOM_32B"},
      {CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B_FLIP_8B, "128B_ATOM_32B_FLIP_8B"},
      {CU_TENSOR_MAP_SWIZZLE_128B_ATOM_64B, "128B_ATOM_64B"}, {CU_TENSOR_MAP_SWIZZLE_64B, "64B"}};
  for (auto& md : modes)
    for (int rows : {64, 24}) {
      CUtensorMap m;
      cuuint64_t gd[2] = {64, (cuuint64_t)R};
      cuuint64_t gs[1] = {512};
      cuuint32_t bx[2] = {16, (cuuint32_t)rows};
      if (md.s == CU_TENSOR_MAP_SWIZZLE_64B) bx[0] = 8;
      cuuint32_t es[2] = {1, 1};
      CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, gd, gs, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       md.s, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      printf("mode %s rows %d encode %d\n", md.n, rows, (int)r);
      if (r != CUDA_SUCCESS) continue;
      cudaMemset(o, 0, 2048 * 8);
      probe<<<1, 128, 20480>>>(m, o, 16, 64, bx[0] * rows * 8);
      cudaError_t e = cudaDeviceSynchronize();
      printf("  run: %s\n", cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
      std::vector<double> ho(2048);
      cudaMemcpy(ho.data(), o, 2048 * 8, cudaMemcpyDeviceToHost);
      // print rows 0..15 of the smem image: for each 128-byte smem row, the (row,col) pairs
      for (int sr = 0; sr < 16; ++sr) {
        printf("  smem row %2d:", sr);
        for (int k = 0; k < (int)bx[0]; ++k) {
          double v = ho[sr * bx[0] + k];
          if (v < 0) printf("   --  ");
          else printf(" %2d.%02d", ((int)v) / 64 - 64, ((int)v) % 64 - 16);
        }
        printf("\n");
      }
    }
  return 0;
}
