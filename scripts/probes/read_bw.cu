// Probe: HBM bandwidth of a read-only stream vs a copy (read + write) on this GPU.
// MEASURED_PEAKS.json's hbm_gbs is a copy (torch copy_, read+write bytes); the SpMV
// (K1b) stream is ~97 % reads, so its achievable DRAM rate can exceed the copy figure.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rbw read_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void rd(const double2 *__restrict__ a, int64_t n2, double *out) {
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x) {
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a + i));
    s += v.x + v.y;
  }
  if (s == 12345.678) *out = s;  // keeps the loads
}
__global__ void cp(const double2 *__restrict__ a, double2 *__restrict__ b, int64_t n2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (int64_t)gridDim.x * blockDim.x)
    __stcs(b + i, __ldcs(a + i));
}

int main() {
  const int64_t bytes = 8ll << 30;  // 8 GiB read (copy: 4 GiB + 4 GiB)
  double2 *a, *b;
  double *o;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes / 2);
  cudaMalloc(&o, 8);
  cudaMemset(a, 0, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int bps : {4, 8, 16}) {
    float best_r = 1e9f, best_c = 1e9f;
    for (int r = 0; r < 8; r++) {
      float ms;
      cudaEventRecord(e0);
      rd<<<sms * bps, 256>>>(a, bytes / 16, o);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best_r) best_r = ms;
      cudaEventRecord(e0);
      cp<<<sms * bps, 256>>>(a, b, bytes / 32);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (r && ms < best_c) best_c = ms;
    }
    printf("blocks/SM %2d: read-only %.0f GB/s   copy (read+write bytes) %.0f GB/s\n", bps, bytes / (best_r * 1e-3) / 1e9,
           bytes / (best_c * 1e-3) / 1e9);
  }
  return 0;
}
