// fdcube.cu — on-device assembly of the paper's regular-grid systems (Table 1,
// P:104-110, reading R2): Laplace Δu = 0 on N^3 nodes
// of the unit cube, finite differences with w(i,j) = 1, node id
// i + N(j + N l) (x fastest); interior rows = the negated Laplacian row of P:79-88
// (6 on the diagonal, -1 per axis neighbour, columns ascending) with b = 0;
// boundary rows = identity with b = f(node) (Dirichlet u = f).
#include <cub/cub.cuh>

#include "fem_gen.h"
#include "matrix.cuh"

namespace pcgb {
namespace {

__device__ __forceinline__ bool on_boundary(int64_t id, int64_t N, int64_t *i, int64_t *j, int64_t *l) {
  *i = id % N;
  *j = (id / N) % N;
  *l = id / (N * N);
  return *i == 0 || *j == 0 || *l == 0 || *i == N - 1 || *j == N - 1 || *l == N - 1;
}

__global__ void fd_count_kernel(int64_t N, int64_t r0, int64_t r1, int64_t *len) {
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  int64_t i, j, l;
  len[r - r0] = on_boundary(r, N, &i, &j, &l) ? 1 : 7;
}

__global__ void fd_fill_kernel(int64_t N, int fkind, int64_t r0, int64_t r1, const int64_t *__restrict__ rp,
                               int64_t *__restrict__ col, double *__restrict__ val, double *__restrict__ b) {
  const int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= r1) return;
  int64_t i, j, l;
  int64_t k = rp[r - r0];
  if (on_boundary(r, N, &i, &j, &l)) {
    col[k] = r;
    val[k] = 1.0;
    if (b) {
      const double h = 1.0 / (double)(N - 1);
      const double x = (double)i * h, y = (double)j * h;
      b[r - r0] = fkind == FD_F_X2MY2 ? __dsub_rn(__dmul_rn(x, x), __dmul_rn(y, y)) : exp(M_PI * x) * sinpi(y);
    }
    return;
  }
  const int64_t nb[7] = {r - N * N, r - N, r - 1, r, r + 1, r + N, r + N * N};
#pragma unroll
  for (int q = 0; q < 7; q++) {
    col[k + q] = nb[q];
    val[k + q] = q == 3 ? 6.0 : -1.0;
  }
  if (b) b[r - r0] = 0.0;
}

}  // namespace
}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status fd_cube_count(int64_t N, int64_t r0, int64_t r1, int64_t *d_rp, int64_t *nnz_out, void *stream) {
  if (N < 3 || r0 < 0 || r1 < r0 || r1 > N * N * N || !d_rp || !nnz_out)
    return fail(PCG_ERR_INVALID_ARG, "fd_cube_count: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = r1 - r0;
  PCG_CUDA(cudaMemsetAsync(d_rp, 0, sizeof(int64_t) * (rows + 1), st));
  if (rows > 0) {
    fd_count_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(N, r0, r1, d_rp + 1);
    count_launch();
    size_t tb = 0;
    cub::DeviceScan::InclusiveSum(nullptr, tb, d_rp + 1, d_rp + 1, rows, st);
    void *tbuf;
    PCG_CUDA(cudaMallocAsync(&tbuf, tb, st));
    cub::DeviceScan::InclusiveSum(tbuf, tb, d_rp + 1, d_rp + 1, rows, st);
    PCG_CUDA(cudaFreeAsync(tbuf, st));
  }
  PCG_CUDA(cudaMemcpyAsync(nnz_out, d_rp + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}

extern "C" pcg_status fd_cube_assemble(int64_t N, int32_t fkind, int64_t r0, int64_t r1, const int64_t *d_rp,
                                       int64_t *d_col, double *d_val, double *d_b, void *stream) {
  if (N < 3 || r0 < 0 || r1 < r0 || r1 > N * N * N || !d_rp || !d_col || !d_val ||
      (fkind != FD_F_X2MY2 && fkind != FD_F_EXPSIN))
    return fail(PCG_ERR_INVALID_ARG, "fd_cube_assemble: bad argument");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = r1 - r0;
  if (rows > 0) {
    fd_fill_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(N, fkind, r0, r1, d_rp, d_col, d_val, d_b);
    count_launch();
    PCG_CUDA(cudaGetLastError());
  }
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}
