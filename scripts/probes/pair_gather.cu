// Probe (development tool): gather throughput of the C4 SpMM access pattern (7-point
// stencil on a 127^3 lattice, k = 16 columns) with the block vector column-major (one
// 8-B gather per (entry, column), the kernel in multi.cu) against pair-interleaved
// columns (one 16-B gather per (entry, column pair)).  Entries are computed from the
// row (no matrix stream), so the timing isolates the gathers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pair_gather pair_gather.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int M = 127, K = 16;
constexpr long N = (long)M * M * M;

__device__ __forceinline__ int nbr(long row, int u, bool &ok) {
  const int i = row % M, j = (row / M) % M, l = row / (M * M);
  const int di[7] = {0, 0, -1, 0, 1, 0, 0}, dj[7] = {0, -1, 0, 0, 0, 1, 0}, dl[7] = {-1, 0, 0, 0, 0, 0, 1};
  const int a = i + di[u], b = j + dj[u], c = l + dl[u];
  ok = a >= 0 && a < M && b >= 0 && b < M && c >= 0 && c < M;
  return ok ? a + M * (b + M * c) : (int)row;
}

__global__ void __launch_bounds__(256, 4) colmajor(const double *__restrict__ P, double *__restrict__ Q, long ld) {
  for (long row = (long)blockIdx.x * 256 + threadIdx.x; row < N; row += (long)gridDim.x * 256) {
    int j[7];
    bool ok[7];
#pragma unroll
    for (int u = 0; u < 7; u++) j[u] = nbr(row, u, ok[u]);
#pragma unroll 1
    for (int c = 0; c < K; c++) {
      const double *Pc = P + c * ld;
      double g[7], s = 0.0;
#pragma unroll
      for (int u = 0; u < 7; u++) g[u] = __ldg(Pc + j[u]);
#pragma unroll
      for (int u = 0; u < 7; u++) s = fma(ok[u] ? (u == 3 ? 6.0 : -1.0) : 0.0, g[u], s);
      Q[c * ld + row] = s;
    }
  }
}

__global__ void __launch_bounds__(256, 4) pairs(const double2 *__restrict__ P, double2 *__restrict__ Q, long ld) {
  for (long row = (long)blockIdx.x * 256 + threadIdx.x; row < N; row += (long)gridDim.x * 256) {
    int j[7];
    bool ok[7];
#pragma unroll
    for (int u = 0; u < 7; u++) j[u] = nbr(row, u, ok[u]);
#pragma unroll 1
    for (int c = 0; c < K / 2; c++) {
      const double2 *Pc = P + c * ld;
      double2 g[7];
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int u = 0; u < 7; u++) g[u] = __ldg(Pc + j[u]);
#pragma unroll
      for (int u = 0; u < 7; u++) {
        const double a = ok[u] ? (u == 3 ? 6.0 : -1.0) : 0.0;
        s0 = fma(a, g[u].x, s0);
        s1 = fma(a, g[u].y, s1);
      }
      Q[c * ld + row] = make_double2(s0, s1);
    }
  }
}

struct __align__(32) d4 { double x, y, z, w; };
__device__ __forceinline__ d4 ld4(const d4 *p) {
  d4 v;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
  return v;
}
__global__ void __launch_bounds__(256, 3) quads(const d4 *__restrict__ P, d4 *__restrict__ Q, long ld) {
  for (long row = (long)blockIdx.x * 256 + threadIdx.x; row < N; row += (long)gridDim.x * 256) {
    int j[7];
    bool ok[7];
#pragma unroll
    for (int u = 0; u < 7; u++) j[u] = nbr(row, u, ok[u]);
#pragma unroll 1
    for (int c = 0; c < K / 4; c++) {
      const d4 *Pc = P + c * ld;
      d4 g[7];
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int u = 0; u < 7; u++) g[u] = ld4(Pc + j[u]);
#pragma unroll
      for (int u = 0; u < 7; u++) {
        const double a = ok[u] ? (u == 3 ? 6.0 : -1.0) : 0.0;
        s0 = fma(a, g[u].x, s0);
        s1 = fma(a, g[u].y, s1);
        s2 = fma(a, g[u].z, s2);
        s3 = fma(a, g[u].w, s3);
      }
      d4 o = {s0, s1, s2, s3};
      Q[c * ld + row] = o;
    }
  }
}

int main() {
  const long ld = (N + 31) / 32 * 32;
  double *P, *Q;
  cudaMalloc(&P, sizeof(double) * ld * K);
  cudaMalloc(&Q, sizeof(double) * ld * K);
  cudaMemset(P, 0, sizeof(double) * ld * K);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; rep++) {
    float ms;
    colmajor<<<sms * 4, 256>>>(P, Q, ld);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; r++) colmajor<<<sms * 4, 256>>>(P, Q, ld);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("column-major: %.1f us per SpMM\n", ms * 100);
    pairs<<<sms * 4, 256>>>((const double2 *)P, (double2 *)Q, ld);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; r++) pairs<<<sms * 4, 256>>>((const double2 *)P, (double2 *)Q, ld);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("pair-interleaved: %.1f us per SpMM\n", ms * 100);
    quads<<<sms * 3, 256>>>((const d4 *)P, (d4 *)Q, ld);
    cudaEventRecord(e0);
    for (int r = 0; r < 10; r++) quads<<<sms * 3, 256>>>((const d4 *)P, (d4 *)Q, ld);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("quad-interleaved (v4.f64): %.1f us per SpMM\n", ms * 100);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
