// Probe (development tool): cp.async.bulk issue/throughput per SM — W warps per block,
// each issuing C copies of B bytes (contiguous, L2-resident source) per round into its
// own buffer, R rounds; prints ns per copy per warp and aggregate GB/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/br scripts/probes/bulk_rate.cu && /tmp/br
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t sa(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const double *src, int64_t n_src, int copies, int bytes, int rounds, double *out) {
  extern __shared__ __align__(128) unsigned char sm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  unsigned char *buf = sm + (size_t)w * copies * bytes;
  uint64_t *bar = reinterpret_cast<uint64_t *>(sm + (size_t)nw * copies * bytes) + w;
  if (lane == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(1));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t ph = 0;
  const int64_t span = (n_src * 8 - bytes) / 256;
  uint64_t x = 0x9E3779B97F4A7C15ULL * (blockIdx.x * 64 + w + 1);
  for (int r = 0; r < rounds; r++) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(copies * bytes)
                   : "memory");
    __syncwarp();
    if (lane < copies) {
      x ^= x << 13; x ^= x >> 7; x ^= x << 17;
      const char *s = reinterpret_cast<const char *>(src) + (x % span) * 256;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(buf + lane * bytes)),
                   "l"(s), "r"(bytes), "r"(sa(bar))
                   : "memory");
    }
    uint32_t ok = 0;
    do {
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(sa(bar)), "r"(ph) : "memory");
    } while (!ok);
    ph ^= 1;
    __syncwarp();
  }
  if (lane == 0 && bar == nullptr) out[0] = 1;
}

int main() {
  const int64_t n_src = 4 << 20;  // 32 MB: L2-resident after the first touches
  double *src, *out;
  cudaMalloc(&src, n_src * 8);
  cudaMemset(src, 0, n_src * 8);
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int rounds = 200;
  for (int bytes : {512, 4096}) 
    for (int copies : {1, 8, 32})
      for (int nw : {1, 4, 8}) {
        size_t smem = (size_t)nw * copies * bytes + 8 * nw;
        if (smem > 200000) continue;
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k<<<sms, nw * 32, smem>>>(src, n_src, copies, bytes, 5, out);
        cudaEventRecord(e0);
        k<<<sms, nw * 32, smem>>>(src, n_src, copies, bytes, rounds, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double per_round_ns = ms * 1e6 / rounds;
        printf("bytes=%5d copies=%2d warps=%d: %7.0f ns/round  %6.1f ns/copy/warp  %7.0f GB/s\n", bytes, copies, nw,
               per_round_ns, per_round_ns / copies, (double)sms * nw * copies * bytes * rounds / (ms * 1e-3) / 1e9);
      }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
