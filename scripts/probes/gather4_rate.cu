// Probe (development tool): TMA throughput per SM for tile::gather4 (4 rows of 128 B
// per request) vs 2D tile loads of 32 rows (4 KB per request), rows from a 256 MB
// row-major fp64 array (n x 16), one block per SM, NW warps, each warp keeping one
// 32 KB batch in flight (64 gather4 or 8 tiles) per round.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/g4r scripts/probes/gather4_rate.cu && /tmp/g4r
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t *bar, uint32_t ph) {
  uint32_t ok = 0;
  do {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(sa(bar)), "r"(ph) : "memory");
  } while (!ok);
}

template <int MODE>  // 0 gather4 (lane issues 2), 1 tile 32 rows (lanes 0-7 issue 1)
__global__ void k(const __grid_constant__ CUtensorMap tg, const __grid_constant__ CUtensorMap tt, int n, int rounds,
                  int nw, double *out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  unsigned char *base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  double *buf = reinterpret_cast<double *>(base + (size_t)w * 32768);
  uint64_t *bar = reinterpret_cast<uint64_t *>(base + (size_t)nw * 32768) + w;
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t ph = 0;
  uint64_t x = 0x9E3779B97F4A7C15ULL * (blockIdx.x * 64 + w * 32 + lane + 1);
  double acc = 0;
  for (int r = 0; r < rounds; r++) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(32768) : "memory");
    __syncwarp();
    if (MODE == 0) {
      for (int g = 0; g < 2; g++) {
        int y[4];
        for (int q = 0; q < 4; q++) {
          x ^= x << 13; x ^= x >> 7; x ^= x << 17;
          y[q] = (int)(x % (uint64_t)n);
        }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4, %5, %6}], [%7];" ::"r"(sa(buf + (lane * 8 + g * 4) * 16)),
            "l"(&tg), "r"(0), "r"(y[0]), "r"(y[1]), "r"(y[2]), "r"(y[3]), "r"(sa(bar))
            : "memory");
      }
    } else if (lane < 8) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      int y0 = (int)(x % (uint64_t)(n - 32));
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
              sa(buf + lane * 512)),
          "l"(&tt), "r"(0), "r"(y0), "r"(sa(bar))
          : "memory");
    }
    wait(bar, ph);
    ph ^= 1;
    acc += buf[lane];
    __syncwarp();
  }
  if (acc == 1234.5) out[0] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
int main() {
  const int n = 2048383, W = 16;
  double *P, *out;
  cudaMalloc(&P, (size_t)n * W * 8);
  cudaMemset(P, 0, (size_t)n * W * 8);
  cudaMalloc(&out, 8);
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tg, tt;
  cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)n}, strides[1] = {(cuuint64_t)W * 8};
  cuuint32_t boxg[2] = {(cuuint32_t)W, 1}, boxt[2] = {(cuuint32_t)W, 32}, es[2] = {1, 1};
  ((EncodeFn)fn)(&tg, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P, dims, strides, boxg, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  ((EncodeFn)fn)(&tt, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, P, dims, strides, boxt, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int rounds = 200;
  for (int mode = 0; mode < 2; mode++)
    for (int nw : {1, 2, 4, 6}) {
      size_t smem = (size_t)nw * 32768 + 64 + 1024;
      auto kf = mode == 0 ? k<0> : k<1>;
      cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      kf<<<sms, nw * 32, smem>>>(tg, tt, n, 5, nw, out);
      cudaEventRecord(e0);
      kf<<<sms, nw * 32, smem>>>(tg, tt, n, rounds, nw, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double bytes = (double)sms * nw * rounds * 32768;
      printf("%s nw=%d: %.1f us, %.0f GB/s into smem, %.2f us per 32 KB round\n", mode ? "tile32" : "gather4", nw,
             ms * 1e3, bytes / (ms * 1e-3) / 1e9, ms * 1e3 / rounds);
    }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
