// Probe: does the single-RHS SELL-32 SpMV at C5 scale gain from fewer, wider matrix
// loads?  7-point periodic lattice (every row 7 entries, like C5's interior), one warp
// per slice of 32 rows, y = A x, three layouts of the same entries:
//   scalar: [t][lane]                     8-B value + 4-B id loads per entry (the library's)
//   pair:   [t/2][lane][2] + tail [lane]  16-B value + 8-B id loads for t = 0..5, scalar t = 6
//   quad:   [lane][4] (t 0-3), [lane][2] (t 4-5), [lane] (t 6): 32-B / 16-B / 8-B loads
// Same sums (left to right), same bytes; only the number of load instructions per
// slice differs (scalar 14, pair 8, quad 6, + 7 gathers).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/svl sell_vector_loads.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

constexpr int T = 7;
constexpr int BLOCK = 256, WARPS = 8;

__device__ __forceinline__ void nbrs(int64_t i, int64_t N, int64_t n, int *c) {
  const int64_t o[7] = {-N * N, -N, -1, 0, 1, N, N * N};
  for (int t = 0; t < 7; t++) c[t] = (int)(((i + o[t]) % n + n) % n);
}
__device__ __forceinline__ double aval(int t) { return t == 3 ? 6.5 : -1.0 - 0.01 * t; }

__global__ void build(int64_t N, int64_t n, int layout, double *val, int *col) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t s = i >> 5;
  const int lane = i & 31;
  int c[7];
  nbrs(i, N, n, c);
  const int64_t base = s * 224;
  for (int t = 0; t < 7; t++) {
    int64_t e;
    if (layout == 0) e = base + t * 32 + lane;
    else if (layout == 1) e = t < 6 ? base + (t >> 1) * 64 + lane * 2 + (t & 1) : base + 192 + lane;
    else e = t < 4 ? base + lane * 4 + t : t < 6 ? base + 128 + lane * 2 + (t - 4) : base + 192 + lane;
    val[e] = aval(t);
    col[e] = c[t];
  }
}

__device__ __forceinline__ double ld1(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld1(const int *p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ double2 ld2(const double *p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ int2 ld2(const int *p) {
  int2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.s32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void ld4(const double *p, double *a) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a[0]), "=d"(a[1]), "=d"(a[2]), "=d"(a[3]) : "l"(p));
}
__device__ __forceinline__ int4 ld4(const int *p) {
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int LAYOUT>
__global__ void __launch_bounds__(BLOCK) spmv(int64_t n_slices, const double *__restrict__ val,
                                              const int *__restrict__ col, const double *__restrict__ x,
                                              double *__restrict__ y, int zero) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  for (int64_t s = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5); s < n_slices; s += nw) {
    const int64_t base = s * 224;
    double a[8];
    int j[8];
    if (LAYOUT == 0) {
#pragma unroll
      for (int t = 0; t < T; t++) j[t] = ld1(col + base + t * 32 + lane);
#pragma unroll
      for (int t = 0; t < T; t++) a[t] = ld1(val + base + t * 32 + lane);
    } else if (LAYOUT == 1) {
#pragma unroll
      for (int tp = 0; tp < 3; tp++) {
        const int2 c = ld2(col + base + tp * 64 + lane * 2);
        j[2 * tp] = c.x;
        j[2 * tp + 1] = c.y;
      }
      j[6] = ld1(col + base + 192 + lane);
#pragma unroll
      for (int tp = 0; tp < 3; tp++) {
        const double2 v = ld2(val + base + tp * 64 + lane * 2);
        a[2 * tp] = v.x;
        a[2 * tp + 1] = v.y;
      }
      a[6] = ld1(val + base + 192 + lane);
    } else {
      const int4 c = ld4(col + base + lane * 4);
      const int2 c2 = ld2(col + base + 128 + lane * 2);
      j[0] = c.x; j[1] = c.y; j[2] = c.z; j[3] = c.w; j[4] = c2.x; j[5] = c2.y;
      j[6] = ld1(col + base + 192 + lane);
      ld4(val + base + lane * 4, a);
      const double2 v2 = ld2(val + base + 128 + lane * 2);
      a[4] = v2.x; a[5] = v2.y;
      a[6] = ld1(val + base + 192 + lane);
    }
    const int xx = (j[0] ^ j[1] ^ j[2] ^ j[3] ^ j[4] ^ j[5] ^ j[6]) & zero;
    double g[8];
#pragma unroll
    for (int t = 0; t < T; t++) g[t] = __ldg(x + (j[t] | xx));
    double sum = 0.0;
#pragma unroll
    for (int t = 0; t < T; t++) sum = __fma_rn(a[t], g[t], sum);
    __stcs(y + s * 32 + lane, sum);
  }
}

int main(int argc, char **argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 512;
  const int64_t n = N * N * N;  // multiple of 32 for N even
  const int64_t ns = n / 32, nnz = n * 7;
  double *val, *x, *y, *flush;
  int *col;
  CK(cudaMalloc(&val, sizeof(double) * nnz));
  CK(cudaMalloc(&col, sizeof(int) * nnz));
  CK(cudaMalloc(&x, sizeof(double) * n));
  CK(cudaMalloc(&y, sizeof(double) * n));
  CK(cudaMalloc(&flush, 512 << 20));
  CK(cudaMemset(x, 0, sizeof(double) * n));
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const double bytes = 12.0 * nnz + 16.0 * n;
  printf("N=%lld n=%lld nnz=%lld bytes/SpMV=%.3f GB\n", (long long)N, (long long)n, (long long)nnz, bytes / 1e9);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int layout = 0; layout < 3; layout++) {
    build<<<(unsigned)((n + 255) / 256), 256>>>(N, n, layout, val, col);
    CK(cudaDeviceSynchronize());
    for (int bps : {2, 3, 4, 6, 8}) {
      const int grid = sms * bps;
      void (*k)(int64_t, const double *, const int *, const double *, double *, int) =
          layout == 0 ? spmv<0> : layout == 1 ? spmv<1> : spmv<2>;
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, BLOCK, 0);
      if (bps > occ) continue;
      float best = 1e30f, tot = 0;
      const int reps = 10;
      for (int r = 0; r < reps + 2; r++) {
        cudaMemsetAsync(flush, r, 512 << 20);
        cudaEventRecord(e0);
        k<<<grid, BLOCK>>>(ns, val, col, x, y, 0);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (r >= 2) {
          tot += ms;
          if (ms < best) best = ms;
        }
      }
      printf("layout %s blocks/SM %d (occ %d): mean %.1f us  best %.1f us  %.0f GB/s\n",
             layout == 0 ? "scalar" : layout == 1 ? "pair  " : "quad  ", bps, occ, tot / reps * 1e3, best * 1e3,
             bytes / (tot / reps * 1e-3) / 1e9);
    }
  }
  return 0;
}
