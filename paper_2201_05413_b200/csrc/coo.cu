// coo.cu — generic COO -> CSR on the device (include/fem_gen.h coo_to_csr;
// SURVEY.md §8(f) N1 "generic COO -> CSR (sort + segmented reduce)"; SPEC
// coo_to_csr S:50-57).  Restated: order the entries by (row, col); sum the values
// of each run of equal (row, col) left to right in input order from 0.0.
//
//   1. keys  : key = row * n_cols + col (range-checked), idx = input position
//   2. sort  : cub::DeviceRadixSort::SortPairs over the key bits in use — an LSD
//              radix sort is stable, so equal keys keep their input order
//   3. gather: v_sorted[j] = val[idx[j]] (coalesced writes, one random read each)
//   4. heads : flag[j] = (j == 0 || key[j] != key[j-1]); pos = exclusive scan
//   5. reduce: one thread per run sums v_sorted over the run (contiguous, in order)
//   6. row_ptr[r] = lower_bound(unique rows, r), one thread per r
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"
#include "fem_gen.h"

namespace pcgb {

__global__ void coo_keys_kernel(int64_t nnz, int64_t nr, int64_t nc, const int64_t *__restrict__ row,
                                const int64_t *__restrict__ col, uint64_t *__restrict__ key, int *__restrict__ idx,
                                int *err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = row[i], c = col[i];
    if (r < 0 || r >= nr || c < 0 || c >= nc) {
      atomicExch(err, 1);
      key[i] = 0;
    } else {
      key[i] = (uint64_t)r * (uint64_t)nc + (uint64_t)c;
    }
    idx[i] = (int)i;
  }
}

__global__ void coo_gather_kernel(int64_t nnz, const uint64_t *__restrict__ ks, const int *__restrict__ idx,
                                  const double *__restrict__ val, double *__restrict__ vs, int *__restrict__ flag) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
    vs[j] = val[idx[j]];
    flag[j] = j == 0 || ks[j] != ks[j - 1];
  }
}

__global__ void coo_reduce_kernel(int64_t nnz, int64_t nc, const uint64_t *__restrict__ ks,
                                  const int *__restrict__ flag, const int *__restrict__ pos,
                                  const double *__restrict__ vs, int64_t *__restrict__ col_out,
                                  double *__restrict__ val_out, int64_t *__restrict__ urow) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nnz; j += (int64_t)gridDim.x * blockDim.x) {
    if (!flag[j]) continue;
    double s = 0.0;
    int64_t e = j;
    do {
      s = __dadd_rn(s, vs[e]);
      e++;
    } while (e < nnz && !flag[e]);
    const int64_t u = pos[j];
    col_out[u] = (int64_t)(ks[j] % (uint64_t)nc);
    val_out[u] = s;
    urow[u] = (int64_t)(ks[j] / (uint64_t)nc);
  }
}

__global__ void coo_rowptr_kernel(int64_t nr, int64_t U, const int64_t *__restrict__ urow, int64_t *__restrict__ rp) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= nr; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = U;  // first unique entry with row >= r
    while (lo < hi) {
      const int64_t m = (lo + hi) >> 1;
      if (urow[m] < r) lo = m + 1;
      else hi = m;
    }
    rp[r] = lo;
  }
}

static unsigned coo_grid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 32)); }

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status coo_to_csr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t *row,
                                 const int64_t *col, const double *val, int64_t *row_ptr, int64_t *col_out,
                                 double *val_out, int64_t *nnz_out, void *stream) {
  const int64_t lim = int64_t(1) << 31;
  if (n_rows < 0 || n_cols < 0 || nnz < 0 || n_rows >= lim || n_cols >= lim || nnz >= lim || !row_ptr || !nnz_out ||
      (nnz > 0 && (!row || !col || !val || !col_out || !val_out)))
    return fail(PCG_ERR_INVALID_ARG, "coo_to_csr: null pointer or size out of range");
  cudaStream_t st = (cudaStream_t)stream;
  *nnz_out = 0;
  if (nnz == 0) {
    PCG_CUDA(cudaMemsetAsync(row_ptr, 0, sizeof(int64_t) * (n_rows + 1), st));
    PCG_CUDA(cudaStreamSynchronize(st));
    return PCG_OK;
  }
  // scratch: key[2][nnz] u64, idx[2][nnz] i32, flag, pos i32, urow i64, err, cub temp
  const uint64_t span = (uint64_t)n_rows * (uint64_t)n_cols;  // > 0 here unless indices are out of range
  int end_bit = 1;
  while (end_bit < 64 && (uint64_t(1) << end_bit) < span) end_bit++;
  size_t tmp_sort = 0, tmp_scan = 0;
  PCG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_sort, (uint64_t *)nullptr, (uint64_t *)nullptr,
                                           (int *)nullptr, (int *)nullptr, (int)nnz, 0, end_bit, st));
  PCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_scan, (int *)nullptr, (int *)nullptr, (int)nnz, st));
  const size_t n = (size_t)nnz, a256 = 256;
  auto up = [&](size_t b) { return (b + a256 - 1) / a256 * a256; };
  const size_t o_k0 = 0, o_k1 = o_k0 + up(8 * n), o_i0 = o_k1 + up(8 * n), o_i1 = o_i0 + up(4 * n),
               o_fl = o_i1 + up(4 * n), o_pos = o_fl + up(4 * n), o_ur = o_pos + up(4 * n), o_err = o_ur + up(8 * n),
               o_tmp = o_err + a256, total = o_tmp + up(std::max(tmp_sort, tmp_scan));
  char *buf = nullptr;
  PCG_CUDA(cudaMalloc(&buf, total));
  uint64_t *k0 = (uint64_t *)(buf + o_k0), *k1 = (uint64_t *)(buf + o_k1);
  int *i0 = (int *)(buf + o_i0), *i1 = (int *)(buf + o_i1), *flag = (int *)(buf + o_fl), *pos = (int *)(buf + o_pos);
  int64_t *urow = (int64_t *)(buf + o_ur);
  int *err = (int *)(buf + o_err);
  void *tmp = buf + o_tmp;
  double *vs = reinterpret_cast<double *>(k0);  // k0 is free after the sort
  pcg_status s = PCG_OK;
  int herr = 0, last_flag = 0, last_pos = 0;
  auto run = [&]() -> pcg_status {
    PCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
    coo_keys_kernel<<<coo_grid(nnz), 256, 0, st>>>(nnz, n_rows, n_cols, row, col, k0, i0, err);
    count_launch();
    PCG_CUDA(cudaGetLastError());
    PCG_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaStreamSynchronize(st));
    if (herr) return fail(PCG_ERR_INDEX_OUT_OF_RANGE, "coo_to_csr: an index is outside [0, n_rows) x [0, n_cols)");
    size_t ts = tmp_sort;
    PCG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, ts, k0, k1, i0, i1, (int)nnz, 0, end_bit, st));
    coo_gather_kernel<<<coo_grid(nnz), 256, 0, st>>>(nnz, k1, i1, val, vs, flag);
    count_launch();
    size_t tc = tmp_scan;
    PCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tc, flag, pos, (int)nnz, st));
    coo_reduce_kernel<<<coo_grid(nnz), 256, 0, st>>>(nnz, n_cols, k1, flag, pos, vs, col_out, val_out, urow);
    count_launch();
    PCG_CUDA(cudaMemcpyAsync(&last_flag, flag + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaMemcpyAsync(&last_pos, pos + nnz - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaStreamSynchronize(st));
    const int64_t U = (int64_t)last_pos + last_flag;
    coo_rowptr_kernel<<<coo_grid(n_rows + 1), 256, 0, st>>>(n_rows, U, urow, row_ptr);
    count_launch();
    PCG_CUDA(cudaGetLastError());
    PCG_CUDA(cudaStreamSynchronize(st));
    *nnz_out = U;
    return PCG_OK;
  };
  s = run();
  cudaFree(buf);
  return s;
}
