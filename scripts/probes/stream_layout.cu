// Probe (development tool): the K2-shaped streaming pass (r -= a q; z = d r; two dots)
// over an n x 16 block in column-major vs row-major layout, same bytes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sl scripts/probes/stream_layout.cu && /tmp/sl
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

constexpr int B = 256;
__global__ void colmajor(int64_t n, int64_t ld, const double *q, double *r, double *z, const double *d, double *out) {
  const int c = blockIdx.y;
  const double2 *q2 = (const double2 *)(q + c * ld), *d2 = (const double2 *)d;
  double2 *r2 = (double2 *)(r + c * ld), *z2 = (double2 *)(z + c * ld);
  double a0 = 0, a1 = 0;
  for (int64_t t = (int64_t)blockIdx.x * B + threadIdx.x; t < n / 2; t += (int64_t)gridDim.x * B) {
    double2 qq = __ldcs(q2 + t), dd = __ldg(d2 + t), rr = r2[t];
    rr.x = fma(-0.5, qq.x, rr.x);
    rr.y = fma(-0.5, qq.y, rr.y);
    double2 zz = make_double2(dd.x * rr.x, dd.y * rr.y);
    r2[t] = rr;
    z2[t] = zz;
    a0 = fma(rr.x, zz.x, a0);
    a1 = fma(rr.y, rr.y, a1);
  }
  if (a0 == 12345.0) out[0] = a1;
}
__global__ void rowmajor(int64_t n, int lkp, const double *q, double *r, double *z, const double *d, double *out) {
  const double2 *q2 = (const double2 *)q;
  double2 *r2 = (double2 *)r, *z2 = (double2 *)z;
  double a0 = 0, a1 = 0;
  const int sh = lkp - 1;
  for (int64_t t = (int64_t)blockIdx.x * B + threadIdx.x; t < (n << lkp) / 2; t += (int64_t)gridDim.x * B) {
    double2 qq = __ldcs(q2 + t), rr = r2[t];
    double dd = __ldg(d + (t >> sh));
    rr.x = fma(-0.5, qq.x, rr.x);
    rr.y = fma(-0.5, qq.y, rr.y);
    double2 zz = make_double2(dd * rr.x, dd * rr.y);
    r2[t] = rr;
    z2[t] = zz;
    a0 = fma(rr.x, zz.x, a0);
    a1 = fma(rr.y, rr.y, a1);
  }
  if (a0 == 12345.0) out[0] = a1;
}

__global__ void fill(double *p, int64_t m, uint64_t seed) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = seed + (i + 1) * 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    p[i] = (double)((z ^ (z >> 31)) >> 11) * (1.0 / 9007199254740992.0);
  }
}

int main() {
  const int64_t n = 2048383, k = 16, ld = (n + 31) / 32 * 32;
  double *q, *r, *z, *d, *out;
  cudaMalloc(&q, ld * k * 8);
  cudaMalloc(&r, ld * k * 8);
  cudaMalloc(&z, ld * k * 8);
  cudaMalloc(&d, ld * 8);
  cudaMalloc(&out, 8);
  fill<<<1024, 256>>>(q, ld * k, 1);
  fill<<<1024, 256>>>(r, ld * k, 2);
  fill<<<1024, 256>>>(z, ld * k, 3);
  fill<<<1024, 256>>>(d, ld, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = 40.0 * k * n;
  for (int rep = 0; rep < 2; rep++) {
    for (int g : {74, 148, 296}) {
      cudaEventRecord(e0);
      for (int i = 0; i < 10; i++) colmajor<<<dim3(g, k), B>>>(n, ld, q, r, z, d, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("colmajor gx=%d x 16: %.1f us  %.0f GB/s\n", g, ms * 100, bytes / (ms * 1e-4) / 1e9);
    }
    for (int g : {592, 1184, 2368, 4736}) {
      cudaEventRecord(e0);
      for (int i = 0; i < 10; i++) rowmajor<<<g, B>>>(n, 4, q, r, z, d, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("rowmajor g=%d: %.1f us  %.0f GB/s\n", g, ms * 100, bytes / (ms * 1e-4) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
