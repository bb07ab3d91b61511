// sigma.cu — SELL-C-sigma: rows sorted by length inside windows of sigma rows
// (BASELINE north_star "(a) a device sparse format: CSR plus a SELL-C-sigma
// variant, chosen per matrix from measured throughput").
//
// Natural-order SELL-32 pads every row of a slice to the slice's longest row.
// When row lengths alternate inside a slice (the P2 half-lattice of C3: vertex
// rows of 19 entries next to edge-midpoint rows of 9), up to a third of the
// entries streamed are padding.  Sorting the rows of each window of sigma
// consecutive rows by descending length makes slices nearly uniform.
//
// The sort is applied as a SYMMETRIC permutation of the whole system:
// A' = P A P^T, b' = P b, x = P^T x'.  Every kernel of the solver then runs
// unchanged on the permuted system (vectors in permuted order; dinv permuted),
// and the only cost is one gather of b/x0 on entry and one scatter of x on exit.
// Rows keep their entries in the caller's order (only column ids are renamed),
// so every row sum of A' x' is formed in exactly the order of the unpermuted
// SpMV: y' = P (A x) bitwise.  Inner products run over the permuted order (a
// different but fixed reduction order).  Rows move at most sigma - 1 places,
// which keeps the gathers of x local.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <utility>

#include "matrix.cuh"

namespace pcgb {

// one block per window: stable sort of (length desc, index asc) by a bitonic
// network over unique 64-bit keys in shared memory
template <int SIGMA>
__global__ void __launch_bounds__(256) sigma_sort_kernel(int64_t n, const int *__restrict__ rp, int *__restrict__ perm) {
  extern __shared__ unsigned long long key[];  // SIGMA keys (dynamic: up to 128 KB)
  const int64_t base = (int64_t)blockIdx.x * SIGMA;
  for (int t = threadIdx.x; t < SIGMA; t += blockDim.x) {
    const int64_t i = base + t;
    const unsigned int len = i < n ? (unsigned int)(rp[i + 1] - rp[i]) : 0u;
    // rows past n sort last (key high word 0xffffffff), real rows by descending length
    const unsigned int hi = i < n ? 0x7fffffffu - len : 0xffffffffu;
    key[t] = ((unsigned long long)hi << 32) | (unsigned int)t;
  }
  __syncthreads();
  for (int size = 2; size <= SIGMA; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int t = threadIdx.x; t < SIGMA; t += blockDim.x) {
        const int o = t ^ stride;
        if (o > t) {
          const bool up = (t & size) == 0;
          const unsigned long long a = key[t], b = key[o];
          if ((a > b) == up) {
            key[t] = b;
            key[o] = a;
          }
        }
      }
      __syncthreads();
    }
  for (int t = threadIdx.x; t < SIGMA; t += blockDim.x)
    if (base + t < n) perm[base + t] = (int)(base + (int64_t)(key[t] & 0xffffffffu));
}

__global__ void invert_perm_kernel(int64_t n, const int *__restrict__ perm, int *__restrict__ iperm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    iperm[perm[i]] = (int)i;
}

// p[i] = outer[p[i]]: a permutation of an already permuted system, in the caller's order
__global__ void compose_perm_kernel(int64_t n, const int *__restrict__ outer, int *__restrict__ p) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = outer[p[i]];
}

__global__ void perm_len_kernel(int64_t n, const int *__restrict__ perm, const int *__restrict__ rp,
                                const double *__restrict__ dinv, int *__restrict__ len2, double *__restrict__ dinv2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) {
      len2[n] = 0;
      continue;
    }
    const int src = perm[i];
    len2[i] = rp[src + 1] - rp[src];
    dinv2[i] = dinv[src];
  }
}

// one warp per permuted row: entries copied in their original order, columns renamed
__global__ void perm_fill_kernel(int64_t n, const int *__restrict__ perm, const int *__restrict__ iperm,
                                 const int *__restrict__ rp, const int *__restrict__ col,
                                 const double *__restrict__ val, const int *__restrict__ rp2, int *__restrict__ col2,
                                 double *__restrict__ val2) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int src = perm[r], s = rp[src], e = rp[src + 1], d = rp2[r];
    for (int k = lane; k < e - s; k += 32) {
      col2[d + k] = iperm[col[s + k]];
      val2[d + k] = val[s + k];
    }
  }
}

__global__ void gather_kernel(int64_t n, const int *__restrict__ perm, const double *__restrict__ src,
                              double *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[perm[i]];
}
__global__ void scatter_kernel(int64_t n, const int *__restrict__ perm, const double *__restrict__ src,
                               double *__restrict__ dst) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[perm[i]] = src[i];
}
// column blocks (grid.y = column): dst[:, c] = src[perm, c] / dst[perm, c] = src[:, c]
__global__ void gather_cols_kernel(int64_t n, const int *__restrict__ perm, const double *__restrict__ src, int64_t lds,
                                   double *__restrict__ dst, int64_t ldd) {
  const size_t os = (size_t)blockIdx.y * lds, od = (size_t)blockIdx.y * ldd;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[od + i] = src[os + perm[i]];
}
__global__ void scatter_cols_kernel(int64_t n, const int *__restrict__ perm, const double *__restrict__ src,
                                    int64_t lds, double *__restrict__ dst, int64_t ldd) {
  const size_t os = (size_t)blockIdx.y * lds, od = (size_t)blockIdx.y * ldd;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[od + perm[i]] = src[os + i];
}

static unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

int sigma_window() {
  static int s = [] {
    const char *e = getenv("PCG_SIGMA");
    int v = e ? atoi(e) : 4096;  // measured on C3: K1b 146 us at 256, 135 us at 4096
    int p = 64;
    while (p < v && p < 16384) p <<= 1;
    return p;
  }();
  return s;
}

// Build the permuted CSR (+ dinv, perm, iperm) of A's natural CSR into S.
pcg_status sigma_build(pcg_matrix *A, cudaStream_t st, SigmaSys *S) {
  const int64_t n = A->n, nnz = A->nnz;
  *S = SigmaSys();
  S->sigma = sigma_window();
  PCG_CUDA(cudaMalloc(&S->perm, sizeof(int) * std::max<int64_t>(n, 1)));
  PCG_CUDA(cudaMalloc(&S->iperm, sizeof(int) * std::max<int64_t>(n, 1)));
  PCG_CUDA(cudaMalloc(&S->row_ptr, sizeof(int) * (n + 1)));
  PCG_CUDA(cudaMalloc(&S->col, sizeof(int) * std::max<int64_t>(nnz, 1)));
  PCG_CUDA(cudaMalloc(&S->val, sizeof(double) * std::max<int64_t>(nnz, 1)));
  PCG_CUDA(cudaMalloc(&S->dinv, sizeof(double) * std::max<int64_t>(n, 1)));
  const unsigned nwin = (unsigned)((n + S->sigma - 1) / S->sigma);
  const size_t ksm = sizeof(unsigned long long) * (size_t)S->sigma;
#define SIGMA_SORT(W)                                                                                        \
  do {                                                                                                       \
    PCG_CUDA(cudaFuncSetAttribute(sigma_sort_kernel<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksm)); \
    sigma_sort_kernel<W><<<nwin, 256, ksm, st>>>(n, A->d_row_ptr, S->perm);                                  \
  } while (0)
  switch (S->sigma) {
    case 64: SIGMA_SORT(64); break;
    case 128: SIGMA_SORT(128); break;
    case 256: SIGMA_SORT(256); break;
    case 512: SIGMA_SORT(512); break;
    case 1024: SIGMA_SORT(1024); break;
    case 2048: SIGMA_SORT(2048); break;
    case 4096: SIGMA_SORT(4096); break;
    case 8192: SIGMA_SORT(8192); break;
    default: SIGMA_SORT(16384); break;
  }
#undef SIGMA_SORT
  invert_perm_kernel<<<grid_for(n), 256, 0, st>>>(n, S->perm, S->iperm);
  int *len2;
  PCG_CUDA(cudaMalloc(&len2, sizeof(int) * (n + 1)));
  perm_len_kernel<<<grid_for(n + 1), 256, 0, st>>>(n, S->perm, A->d_row_ptr, A->d_dinv, len2, S->dinv);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, len2, S->row_ptr, n + 1, st);
  void *tbuf;
  PCG_CUDA(cudaMalloc(&tbuf, tb));
  cub::DeviceScan::ExclusiveSum(tbuf, tb, len2, S->row_ptr, n + 1, st);
  perm_fill_kernel<<<grid_for(n * 32), 256, 0, st>>>(n, S->perm, S->iperm, A->d_row_ptr, A->d_col, A->d_val, S->row_ptr,
                                                      S->col, S->val);
  count_launch(5);
  if (A->d_perm) {  // A is already a permuted system (PCG_REORDER_RCM): compose to the caller's order
    compose_perm_kernel<<<grid_for(n), 256, 0, st>>>(n, A->d_perm, S->perm);
    invert_perm_kernel<<<grid_for(n), 256, 0, st>>>(n, S->perm, S->iperm);
    count_launch(2);
  }
  PCG_CUDA(cudaGetLastError());
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(tbuf);
  cudaFree(len2);
  return PCG_OK;
}

// A := P A P^T for a full permutation (perm[i'] = row of A placed at i', device, n
// ints; ownership passes to A).  Rows keep their entries in order, columns renamed
// (as above); A must not hold SELL arrays yet.  Used by PCG_REORDER_RCM (rcm.cu).
pcg_status apply_perm(pcg_matrix *A, int *perm, cudaStream_t st) {
  const int64_t n = A->n, nnz = A->nnz;
  int *iperm = nullptr, *rp2 = nullptr, *col2 = nullptr, *len2 = nullptr;
  double *val2 = nullptr, *dinv2 = nullptr;
  PCG_CUDA(cudaMalloc(&iperm, sizeof(int) * std::max<int64_t>(n, 1)));
  PCG_CUDA(cudaMalloc(&rp2, sizeof(int) * (n + 1)));
  PCG_CUDA(cudaMalloc(&len2, sizeof(int) * (n + 1)));
  PCG_CUDA(cudaMalloc(&col2, sizeof(int) * std::max<int64_t>(nnz, 1)));
  PCG_CUDA(cudaMalloc(&val2, sizeof(double) * std::max<int64_t>(nnz, 1)));
  PCG_CUDA(cudaMalloc(&dinv2, sizeof(double) * std::max<int64_t>(n, 1)));
  invert_perm_kernel<<<grid_for(n), 256, 0, st>>>(n, perm, iperm);
  perm_len_kernel<<<grid_for(n + 1), 256, 0, st>>>(n, perm, A->d_row_ptr, A->d_dinv, len2, dinv2);
  size_t tb = 0;
  PCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, len2, rp2, n + 1, st));
  void *tbuf;
  PCG_CUDA(cudaMalloc(&tbuf, tb));
  PCG_CUDA(cub::DeviceScan::ExclusiveSum(tbuf, tb, len2, rp2, n + 1, st));
  perm_fill_kernel<<<grid_for(n * 32), 256, 0, st>>>(n, perm, iperm, A->d_row_ptr, A->d_col, A->d_val, rp2, col2, val2);
  count_launch(4);
  PCG_CUDA(cudaGetLastError());
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(tbuf);
  cudaFree(len2);
  cudaFree(A->d_row_ptr);
  cudaFree(A->d_col);
  cudaFree(A->d_val);
  cudaFree(A->d_dinv);
  A->d_row_ptr = rp2;
  A->d_col = col2;
  A->d_val = val2;
  A->d_dinv = dinv2;
  A->d_perm = perm;
  A->d_iperm = iperm;
  return PCG_OK;
}

// exchange A's natural CSR/SELL arrays with S's permuted ones (SELL is rebuilt
// from whichever CSR A holds afterwards)
void sigma_swap(pcg_matrix *A, SigmaSys *S) {
  std::swap(A->d_row_ptr, S->row_ptr);
  std::swap(A->d_col, S->col);
  std::swap(A->d_val, S->val);
  std::swap(A->d_dinv, S->dinv);
  std::swap(A->d_slice_ptr, S->slice_ptr);
  std::swap(A->d_scol, S->scol);
  std::swap(A->d_sval, S->sval);
  std::swap(A->sell_entries, S->sell_entries);
  std::swap(A->d_perm, S->perm);
  std::swap(A->d_iperm, S->iperm);
  std::swap(A->sigma, S->sigma);
}

void sigma_free(SigmaSys *S) {
  for (void *p : {(void *)S->perm, (void *)S->iperm, (void *)S->row_ptr, (void *)S->col, (void *)S->val,
                  (void *)S->dinv, (void *)S->slice_ptr, (void *)S->scol, (void *)S->sval})
    if (p) cudaFree(p);
  *S = SigmaSys();
}

// vectors across the permutation boundary (no-ops when A is unpermuted)
pcg_status perm_in(pcg_matrix *A, const double *src_dev, double *dst, cudaStream_t st) {
  gather_kernel<<<grid_for(A->n), 256, 0, st>>>(A->n, A->d_perm, src_dev, dst);
  count_launch();
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}
pcg_status perm_out(pcg_matrix *A, const double *src, double *dst_dev, cudaStream_t st) {
  scatter_kernel<<<grid_for(A->n), 256, 0, st>>>(A->n, A->d_perm, src, dst_dev);
  count_launch();
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}
pcg_status perm_in_cols(pcg_matrix *A, int k, const double *src, int64_t lds, double *dst, int64_t ldd,
                        cudaStream_t st) {
  gather_cols_kernel<<<dim3(std::max(1u, grid_for(A->n) / 4), k), 256, 0, st>>>(A->n, A->d_perm, src, lds, dst, ldd);
  count_launch();
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}
pcg_status perm_out_cols(pcg_matrix *A, int k, const double *src, int64_t lds, double *dst, int64_t ldd,
                         cudaStream_t st) {
  scatter_cols_kernel<<<dim3(std::max(1u, grid_for(A->n) / 4), k), 256, 0, st>>>(A->n, A->d_perm, src, lds, dst, ldd);
  count_launch();
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

}  // namespace pcgb
