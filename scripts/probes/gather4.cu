// Probe (development tool): semantics of TMA tile::gather4 on sm_100a.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/g4 scripts/probes/gather4.cu && /tmp/g4
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tm, const int *rows, double *out) {
  __shared__ alignas(128) double buf[4 * 16 * 2];
  __shared__ alignas(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(2 * 4 * 128) : "memory");
    for (int g = 0; g < 2; g++)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
          "%5, %6}], [%7];" ::"r"(sa(buf + g * 64)),
          "l"(&tm), "r"(0), "r"(rows[4 * g + 0]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3]),
          "r"(sa(&bar))
          : "memory");
  }
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok)
                 : "r"(sa(&bar)), "r"(0)
                 : "memory");
  } while (!ok);
  for (int i = threadIdx.x; i < 128; i += blockDim.x) out[i] = buf[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int n = 1000, W = 16;
  double *P, *out;
  int *rows;
  cudaMallocManaged(&P, sizeof(double) * n * W);
  cudaMallocManaged(&out, sizeof(double) * 128);
  cudaMallocManaged(&rows, sizeof(int) * 8);
  for (int i = 0; i < n; i++)
    for (int c = 0; c < W; c++) P[i * W + c] = i * 100 + c;
  int rr[8] = {5, 900, 3, 77, 999, 0, 5, 512};
  for (int i = 0; i < 8; i++) rows[i] = rr[i];
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)n};
  cuuint64_t strides[1] = {(cuuint64_t)W * 8};
  cuuint32_t box[2] = {(cuuint32_t)W, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P, dims, strides, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  k<<<1, 32>>>(tm, rows, out);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel %s\n", cudaGetErrorString(e));
  int bad = 0;
  for (int g = 0; g < 8; g++)
    for (int c = 0; c < W; c++)
      if (out[g * W + c] != rr[g] * 100 + c) bad++;
  printf("gather4 box{16,1}: %s (out[0..2]=%g %g %g, row1 c0=%g)\n", bad ? "MISMATCH" : "OK", out[0], out[1], out[2],
         out[16]);
  return bad != 0;
}
