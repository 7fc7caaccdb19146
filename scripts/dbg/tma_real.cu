// Debug: load one halo plane tile through a complex-layout and a real-layout
// 5-D tensor map (as tem_b200.cu::make_tmap) and compare with the host.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <vector>
#include <stdlib.h>
__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int c0, int c1, int c2, int c3, int c4, int bytes, double* out) {
  extern __shared__ __align__(128) double sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                 ::"r"(su(sm)), "l"((uint64_t)&tm), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(su(&bar)) : "memory");
  }
  asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(su(&bar)));
  for (int i = threadIdx.x; i < bytes / 8; i += blockDim.x) out[i] = sm[i];
}
int main(int argc, char** argv) {
  const int nx1 = 33, ny1 = 33, nz1 = 33, S = 3, px = 34, ty = 12;
  const size_t Nn = (size_t)nx1 * ny1 * nz1;
  void* fn; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  double* buf; cudaMalloc(&buf, S * 3 * Nn * 16);
  std::vector<double> h(S * 3 * Nn * 2);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  cudaMemcpy(buf, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  double* out; cudaMalloc(&out, 1 << 20);
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  for (int real = 0; real < 2; ++real) {
    CUtensorMap tm;
    cuuint64_t dc[5] = {2 * (cuuint64_t)nx1, ny1, nz1, 3, S}, sc[4] = {16 * (cuuint64_t)nx1, 16 * (cuuint64_t)nx1 * ny1, 16 * Nn, 48 * Nn};
    cuuint64_t dr[5] = {(cuuint64_t)nx1, ny1, nz1, 3, S}, sr[4] = {8 * (cuuint64_t)px, 8 * (cuuint64_t)px * ny1, 8 * (cuuint64_t)px * ny1 * nz1, 48 * Nn};
    cuuint32_t box[5] = {(real ? 1u : 2u) * 34, (cuuint32_t)ty + 2, 1, 1, 1}, es[5] = {1, 1, 1, 1, 1};
    if (real && variant == 1) dr[0] = px;                        // no row padding in dims
    if (real && variant == 2) { box[0] = 32; }                   // box inner 256 B
    if (real && variant == 3) { sr[3] = 8 * (cuuint64_t)px * ny1 * nz1 * 3; }   // packed shifts
    if (real && variant == 4) { box[0] = 36; }                   // 288 B
    if (real && variant == 5) { dr[0] = px; box[0] = 32; }
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, buf, real ? dr : dc, real ? sr : sc, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int bytes = box[0] * box[1] * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    int c0r = argc > 2 ? atoi(argv[2]) : -1;
    k<<<1, 128, 16 * 1024>>>(tm, real ? c0r : -2, -1, 5, 1, 2, bytes, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("real=%d encode=%d launch=%s\n", real, (int)r, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
