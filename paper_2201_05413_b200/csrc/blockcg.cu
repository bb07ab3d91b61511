// blockcg.cu — block conjugate gradients for k right-hand sides (SURVEY §8(f) N3:
// "block CG for C4 (shared Krylov space)"; reading R5; oracle orc_block_cg).
//
// The k columns share one block Krylov space: per step one SpMM Q = A P (the matrix
// streamed once for all columns), two k x k Gram matrices (P^T Q; R^T Z with the
// residual norms on its diagonal pass) and two k x k Cholesky solves, so every
// column converges in about as many steps as the fastest independent solve needs
// (C4: 366 instead of 549-578 products).  Data: column-major n x m blocks with
// ld = ceil(n/32)*32 (the pcg_solve_multi layout); m <= 32 active columns.
//
// Per iteration (all on the device; the host polls a done flag every 8 steps):
//   bcg_spmm      Q = A P                              12 nnz + 4(n+1) + 16 m n
//   bcg_gram      G = P^T Q   (fixed-order partials)   16 m n
//   bcg_small     alpha = G^-1 Gam (Cholesky, 32 threads)
//   bcg_update    X += P alpha, R -= Q alpha, Z = dinv R, Gam' = R^T Z, rr = diag R^T R
//                                                      56 m n + 8 n
//   bcg_small     stop test; beta = Gam^-1 Gam'
//   bcg_pupdate   P = Z + P beta                       24 m n
// Tiles of 32 rows x m columns are staged in shared memory for the m x m products.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <vector>

#include "matrix.cuh"
#include "rows.cuh"

namespace pcgb {

constexpr int BK = 32;   // widest block
constexpr int TR = 32;   // rows per shared-memory tile
constexpr int GT = 256;  // threads of the tile kernels

enum { BCG_RUNNING = 0, BCG_CHECK = 1, BCG_OK = 2, BCG_MAXIT = 3, BCG_BREAKDOWN = 4 };

struct BcgState {
  double G[BK * BK], Gam[BK * BK], Gn[BK * BK], al[BK * BK], be[BK * BK];
  double nb[BK], rr[BK], rec[BK];
  double tol;
  long long it, max_iter;
  int m, done;
};

// ---------------------------------------------------------------- Q = A P
__device__ __forceinline__ double bcg_long_row(const double *vp, const int *cp, int len, const double *__restrict__ Pc,
                                               int zero) {
  double sum = 0.0;
#pragma unroll 1
  for (int t = 0; t < len; t += 8) {
    double a[8], g[8];
    int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (t + u < len) {
        a[u] = __ldg(vp + (size_t)(t + u) * 32);
        j[u] = __ldg(cp + (size_t)(t + u) * 32);
      }
    cols_ready(j, zero);
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (t + u < len) g[u] = __ldg(Pc + j[u]);
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (t + u < len) sum = __fma_rn(a[u], g[u], sum);
  }
  return sum;
}

// one warp per SELL-32 slice: the slice's entries (<= 8 per row) stay in registers
// while the m columns are gathered one after another
__global__ void __launch_bounds__(BLOCK, 4) bcg_spmm_sell(SellView S, const double *__restrict__ P,
                                                          double *__restrict__ Q, int m, int64_t ld,
                                                          const BcgState *st) {
  if (st && st->done != BCG_RUNNING) return;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * WARPS;
  for (int64_t s = w0; s < S.n_slices; s += nw) {
    const int64_t base = __ldg(S.slice_ptr + s);
    const int len = (int)((__ldg(S.slice_ptr + s + 1) - base) >> 5);
    const int64_t row = s * 32 + lane;
    const bool ok = row < S.n;
    const double *vp = S.val + base + lane;
    const int *cp = S.col + base + lane;
    if (len <= 8) {
      double a[8];
      int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 8; u++) {
        a[u] = 0.0;
        if (u < len) {
          a[u] = ld_stream(vp + (size_t)u * 32);
          j[u] = ld_stream(cp + (size_t)u * 32);
        }
      }
      cols_ready(j, S.zero);
#pragma unroll 1
      for (int c = 0; c < m; c++) {
        const double *Pc = P + (size_t)c * ld;
        double g[8];
#pragma unroll
        for (int u = 0; u < 8; u++) g[u] = u < len ? __ldg(Pc + j[u]) : 0.0;
        double sum = 0.0;
#pragma unroll
        for (int u = 0; u < 8; u++) sum = __fma_rn(a[u], g[u], sum);
        if (ok) __stcs(Q + (size_t)c * ld + row, sum);
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < m; c++) {
        const double sum = bcg_long_row(vp, cp, len, P + (size_t)c * ld, S.zero);
        if (ok) __stcs(Q + (size_t)c * ld + row, sum);
      }
    }
  }
}

__global__ void __launch_bounds__(BLOCK) bcg_spmm_csr(CsrView C, const double *__restrict__ P, double *__restrict__ Q,
                                                      int m, int64_t ld, const BcgState *st) {
  if (st && st->done != BCG_RUNNING) return;
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < C.n; i += (int64_t)gridDim.x * BLOCK) {
    const int rs = C.row_ptr[i], re = C.row_ptr[i + 1];
#pragma unroll 1
    for (int c = 0; c < m; c++) {
      const double *Pc = P + (size_t)c * ld;
      double sum = 0.0;
      for (int k = rs; k < re; k++) sum = __fma_rn(__ldg(C.val + k), __ldg(Pc + __ldg(C.col + k)), sum);
      Q[(size_t)c * ld + i] = sum;
    }
  }
}

// ---------------------------------------------------------------- fixed-order reduction of the tile kernels' partials
// partials[e * nblk + block]; one block per entry e: strided per-thread sums, then a
// fixed tree (deterministic).  e < mm -> out[e]; e >= mm -> out2[e - mm]
template <int NV>
__device__ __forceinline__ void bcg_store_partials(const double (&acc)[NV], int count, double *partials) {
#pragma unroll
  for (int u = 0; u < NV; u++) {
    const int e = threadIdx.x + GT * u;
    if (e < count) partials[(size_t)e * gridDim.x + blockIdx.x] = acc[u];
  }
}
__global__ void __launch_bounds__(GT) bcg_reduce_kernel(const double *__restrict__ partials, int nblk, int mm,
                                                        double *out, double *out2, const BcgState *st) {
  if (st && st->done != BCG_RUNNING) return;
  __shared__ double sm[GT / 32];
  const int e = blockIdx.x;
  double t = 0.0;
  for (int b = threadIdx.x; b < nblk; b += GT) t += __ldcg(partials + (size_t)e * nblk + b);
  t = warp_sum(t);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double u = 0.0;
    for (int w = 0; w < GT / 32; w++) u += sm[w];
    if (e < mm) out[e] = u;
    else out2[e - mm] = u;
  }
}

// ---------------------------------------------------------------- G = P^T Q
__global__ void __launch_bounds__(GT) bcg_gram_kernel(int64_t n, int m, int64_t ld, const double *__restrict__ U,
                                                      const double *__restrict__ V, double *partials, BcgState *st) {
  if (st->done != BCG_RUNNING) return;
  __shared__ double su[BK][TR + 1], sv[BK][TR + 1];
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int mm = m * m;
  for (int64_t r0 = (int64_t)blockIdx.x * TR; r0 < n; r0 += (int64_t)gridDim.x * TR) {
    for (int idx = threadIdx.x; idx < m * TR; idx += GT) {
      const int c = idx / TR, r = idx % TR;
      const int64_t row = r0 + r;
      su[c][r] = row < n ? U[(size_t)c * ld + row] : 0.0;
      sv[c][r] = row < n ? V[(size_t)c * ld + row] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const int e = threadIdx.x + GT * u;
      if (e < mm) {
        const int a = e / m, b = e % m;
        double s = acc[u];
#pragma unroll 8
        for (int r = 0; r < TR; r++) s = __fma_rn(su[a][r], sv[b][r], s);
        acc[u] = s;
      }
    }
    __syncthreads();
  }
  bcg_store_partials<4>(acc, mm, partials);
}

// ---------------------------------------------------------------- X, R, Z (and P at a restart) + R^T Z, diag R^T R
// MODE 0 (restart / exit check): R = B - Q (Q = A X), Z = dinv R, P = Z
// MODE 1 (step):                  X += P alpha, R -= Q alpha, Z = dinv R
template <int MODE>
__global__ void __launch_bounds__(GT) bcg_update_kernel(int64_t n, int m, int64_t ld, double *__restrict__ X,
                                                        double *__restrict__ R, double *__restrict__ Z,
                                                        double *__restrict__ P, const double *__restrict__ Q,
                                                        const double *__restrict__ Bm, const double *__restrict__ dinv,
                                                        double *partials, BcgState *st) {
  if (MODE == 1 && st->done != BCG_RUNNING) return;
  __shared__ double sal[BK * BK];
  __shared__ double sp[MODE == 1 ? BK : 1][TR + 1], sq[MODE == 1 ? BK : 1][TR + 1];
  __shared__ double sr[BK][TR + 1], sz[BK][TR + 1];
  const int mm = m * m;
  if (MODE == 1)
    for (int e = threadIdx.x; e < mm; e += GT) sal[e] = st->al[e];
  double acc[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t r0 = (int64_t)blockIdx.x * TR; r0 < n; r0 += (int64_t)gridDim.x * TR) {
    if (MODE == 1) {
      for (int idx = threadIdx.x; idx < m * TR; idx += GT) {
        const int c = idx / TR, r = idx % TR;
        const int64_t row = r0 + r;
        sp[c][r] = row < n ? P[(size_t)c * ld + row] : 0.0;
        sq[c][r] = row < n ? Q[(size_t)c * ld + row] : 0.0;
      }
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * TR; idx += GT) {
      const int c = idx / TR, r = idx % TR;
      const int64_t row = r0 + r;
      double rv = 0.0, zv = 0.0;
      if (row < n) {
        const size_t e = (size_t)c * ld + row;
        if (MODE == 0) {
          rv = Bm[e] - Q[e];
        } else {
          double x = X[e];
          rv = R[e];
          for (int b = 0; b < m; b++) {
            const double ab = sal[b * m + c];
            x = __fma_rn(sp[b][r], ab, x);
            rv = __fma_rn(-sq[b][r], ab, rv);
          }
          X[e] = x;
        }
        zv = dinv[row] * rv;
        R[e] = rv;
        Z[e] = zv;
        if (MODE == 0) P[e] = zv;
      }
      sr[c][r] = rv;
      sz[c][r] = zv;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 5; u++) {
      const int e = threadIdx.x + GT * u;
      if (e < mm) {
        const int a = e / m, b = e % m;
        double s = acc[u];
#pragma unroll 8
        for (int r = 0; r < TR; r++) s = __fma_rn(sr[a][r], sz[b][r], s);
        acc[u] = s;
      } else if (e < mm + m) {
        const int a = e - mm;
        double s = acc[u];
#pragma unroll 8
        for (int r = 0; r < TR; r++) s = __fma_rn(sr[a][r], sr[a][r], s);
        acc[u] = s;
      }
    }
    __syncthreads();
  }
  bcg_store_partials<5>(acc, mm + m, partials);
}

// ---------------------------------------------------------------- P = Z + P beta
__global__ void __launch_bounds__(GT) bcg_pupdate_kernel(int64_t n, int m, int64_t ld, double *__restrict__ P,
                                                         const double *__restrict__ Z, const BcgState *st) {
  if (st->done != BCG_RUNNING) return;
  __shared__ double sbe[BK * BK];
  __shared__ double sp[BK][TR + 1];
  for (int e = threadIdx.x; e < m * m; e += GT) sbe[e] = st->be[e];
  for (int64_t r0 = (int64_t)blockIdx.x * TR; r0 < n; r0 += (int64_t)gridDim.x * TR) {
    for (int idx = threadIdx.x; idx < m * TR; idx += GT) {
      const int c = idx / TR, r = idx % TR;
      const int64_t row = r0 + r;
      sp[c][r] = row < n ? P[(size_t)c * ld + row] : 0.0;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * TR; idx += GT) {
      const int c = idx / TR, r = idx % TR;
      const int64_t row = r0 + r;
      if (row < n) {
        const size_t e = (size_t)c * ld + row;
        double v = Z[e];
        for (int b = 0; b < m; b++) v = __fma_rn(sp[b][r], sbe[b * m + c], v);
        P[e] = v;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- k x k solves (one warp)
// Y = G^-1 C by Cholesky G = L L^T (as oracle.c chol_solve); false on a non-positive pivot
__device__ bool bcg_chol_solve(int m, const double *G, const double *Cm, double *Y) {
  __shared__ double L[BK * BK];
  __shared__ int s_fail;
  const int t = threadIdx.x;
  if (t == 0) s_fail = 0;
  __syncwarp();
  for (int j = 0; j < m; j++) {
    if (t == 0) {
      double d = G[j * m + j];
      for (int s = 0; s < j; s++) d -= L[j * m + s] * L[j * m + s];
      if (!(d > 0.0)) s_fail = 1;
      L[j * m + j] = sqrt(d);
    }
    __syncwarp();
    if (s_fail) return false;
    if (t > j && t < m) {
      double s = G[t * m + j];
      for (int q = 0; q < j; q++) s -= L[t * m + q] * L[j * m + q];
      L[t * m + j] = s / L[j * m + j];
    }
    __syncwarp();
  }
  if (t < m) {
    const int c = t;
    for (int i = 0; i < m; i++) {
      double s = Cm[i * m + c];
      for (int q = 0; q < i; q++) s -= L[i * m + q] * Y[q * m + c];
      Y[i * m + c] = s / L[i * m + i];
    }
    for (int i = m - 1; i >= 0; i--) {
      double s = Y[i * m + c];
      for (int q = i + 1; q < m; q++) s -= L[q * m + i] * Y[q * m + c];
      Y[i * m + c] = s / L[i * m + i];
    }
  }
  __syncwarp();
  return true;
}

enum { BS_INIT = 0, BS_ALPHA = 1, BS_BETA = 2 };

// <<<1, 32>>>
__global__ void bcg_small_kernel(BcgState *st, int mode) {
  const int t = threadIdx.x, m = st->m, mm = m * m;
  if (mode == BS_INIT) {  // after a restart pass: Gam = R^T Z; every true residual small -> done
    for (int e = t; e < mm; e += 32) st->Gam[e] = st->Gn[e];
    __syncwarp();
    if (t == 0) {
      bool all = true;
      for (int a = 0; a < m; a++) all = all && sqrt(st->rr[a]) <= st->tol * st->nb[a];
      st->done = all ? BCG_OK : BCG_RUNNING;
    }
    return;
  }
  if (st->done != BCG_RUNNING) return;
  if (mode == BS_ALPHA) {
    if (t == 0) st->it++;
    if (!bcg_chol_solve(m, st->G, st->Gam, st->al) && t == 0) st->done = BCG_BREAKDOWN;
    return;
  }
  // BS_BETA: recurrence stop test, then beta
  __shared__ int s_state;
  if (t == 0) {
    bool all = true;
    for (int a = 0; a < m; a++) {
      st->rec[a] = sqrt(st->rr[a]) / st->nb[a];
      all = all && sqrt(st->rr[a]) <= st->tol * st->nb[a];
    }
    s_state = all ? BCG_CHECK : (st->it >= st->max_iter ? BCG_MAXIT : BCG_RUNNING);
    st->done = s_state;
  }
  __syncwarp();
  if (s_state != BCG_RUNNING) return;
  if (!bcg_chol_solve(m, st->Gam, st->Gn, st->be)) {
    if (t == 0) st->done = BCG_BREAKDOWN;
    return;
  }
  for (int e = t; e < mm; e += 32) st->Gam[e] = st->Gn[e];
}

// column norms ||b_c|| (one block per column, fixed order)
__global__ void __launch_bounds__(GT) bcg_norms_kernel(int64_t n, int64_t ld, const double *__restrict__ B,
                                                       double *__restrict__ nb) {
  __shared__ double sm[GT / 32];
  const double *Bc = B + (size_t)blockIdx.x * ld;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += GT) s = __fma_rn(Bc[i], Bc[i], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < GT / 32; w++) t += sm[w];
    nb[blockIdx.x] = sqrt(t);
  }
}

// ---------------------------------------------------------------- host side
namespace {
struct BcgBufs {
  double *X, *R, *Z, *P, *Q, *Bm;
};

int tile_grid(int64_t n, int sms) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + TR - 1) / TR, (int64_t)sms * 4));
}
}  // namespace

static pcg_status bcg_spmm(pcg_matrix *A, const double *P, double *Q, int m, int64_t ld, const BcgState *st,
                           cudaStream_t s) {
  const int sms = num_sms(A->device);
  if (A->format == PCG_FORMAT_CSR) {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((A->n + BLOCK - 1) / BLOCK, (int64_t)sms * 8));
    bcg_spmm_csr<<<g, BLOCK, 0, s>>>(A->csr(), P, Q, m, ld, st);
  } else {
    const unsigned g =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>((A->n_slices + WARPS - 1) / WARPS, (int64_t)sms * 4));
    bcg_spmm_sell<<<g, BLOCK, 0, s>>>(A->sell(), P, Q, m, ld, st);
  }
  count_launch();
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

// restart / exit check: R = B - A X, Z = dinv R, P = Z, Gam = R^T Z, rr; done = OK iff all small
static pcg_status bcg_restart(pcg_matrix *A, const BcgBufs &b, int m, int64_t ld, BcgState *st, double *part, int gt,
                              cudaStream_t s) {
  PCG_TRY(bcg_spmm(A, b.X, b.Q, m, ld, nullptr, s));
  bcg_update_kernel<0><<<gt, GT, 0, s>>>(A->n, m, ld, b.X, b.R, b.Z, b.P, b.Q, b.Bm, A->d_dinv, part, st);
  bcg_reduce_kernel<<<m * m + m, GT, 0, s>>>(part, gt, m * m, st->Gn, st->rr, nullptr);
  bcg_small_kernel<<<1, 32, 0, s>>>(st, BS_INIT);
  count_launch(3);
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

static pcg_status bcg_step(pcg_matrix *A, const BcgBufs &b, int m, int64_t ld, BcgState *st, double *part, int gt,
                           cudaStream_t s) {
  PCG_TRY(bcg_spmm(A, b.P, b.Q, m, ld, st, s));
  bcg_gram_kernel<<<gt, GT, 0, s>>>(A->n, m, ld, b.P, b.Q, part, st);
  bcg_reduce_kernel<<<m * m, GT, 0, s>>>(part, gt, m * m, st->G, nullptr, st);
  bcg_small_kernel<<<1, 32, 0, s>>>(st, BS_ALPHA);
  bcg_update_kernel<1><<<gt, GT, 0, s>>>(A->n, m, ld, b.X, b.R, b.Z, b.P, b.Q, b.Bm, A->d_dinv, part, st);
  bcg_reduce_kernel<<<m * m + m, GT, 0, s>>>(part, gt, m * m, st->Gn, st->rr, st);
  bcg_small_kernel<<<1, 32, 0, s>>>(st, BS_BETA);
  bcg_pupdate_kernel<<<gt, GT, 0, s>>>(A->n, m, ld, b.P, b.Z, st);
  count_launch(7);
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

static pcg_status block_cg_impl(pcg_matrix *A, int k, const double *B, int64_t ldb, double *X, int64_t ldx, double tol,
                                int64_t max_iter, cudaStream_t s, pcg_info *infos) {
  const int64_t n = A->n, ld = (n + 31) / 32 * 32;
  SolveWork &w = A->work;
  const size_t blk = (size_t)ld * k;
  if (w.bcg_cap < (int64_t)(6 * blk)) {
    if (w.bcg) cudaFree(w.bcg);
    w.bcg = nullptr;
    w.bcg_cap = 0;
    PCG_CUDA(cudaMalloc(&w.bcg, sizeof(double) * 6 * blk));
    w.bcg_cap = (int64_t)(6 * blk);
  }
  if (!w.bcg_st) {
    PCG_CUDA(cudaMalloc(&w.bcg_st, sizeof(BcgState)));
    PCG_CUDA(cudaMallocHost(&w.bcg_hst, sizeof(BcgState)));
  }
  const int sms = num_sms(A->device);
  const int gt = tile_grid(n, sms);
  const size_t npart = (size_t)gt * (BK * BK + BK);
  if (w.bcg_part_cap < (int64_t)npart) {
    if (w.bcg_part) cudaFree(w.bcg_part);
    w.bcg_part = nullptr;
    PCG_CUDA(cudaMalloc(&w.bcg_part, sizeof(double) * npart));
    w.bcg_part_cap = (int64_t)npart;
  }
  BcgState *st = (BcgState *)w.bcg_st, *hst = (BcgState *)w.bcg_hst;
  double *part = w.bcg_part;
  BcgBufs b{w.bcg, w.bcg + blk, w.bcg + 2 * blk, w.bcg + 3 * blk, w.bcg + 4 * blk, w.bcg + 5 * blk};
  // stage B and X0 (caller layout, host or device) into the compact blocks; the
  // permuted system (SELL-C-sigma / RCM) gathers them
  for (int c = 0; c < k; c++) {
    double *bd = A->d_perm ? b.R : b.Bm + (size_t)c * ld;  // (R, Z: scratch before the solve)
    double *xd = A->d_perm ? b.Z : b.X + (size_t)c * ld;
    PCG_CUDA(cudaMemcpyAsync(bd, B + (size_t)c * ldb, sizeof(double) * n, cudaMemcpyDefault, s));
    PCG_CUDA(cudaMemcpyAsync(xd, X + (size_t)c * ldx, sizeof(double) * n, cudaMemcpyDefault, s));
    if (A->d_perm) {
      PCG_TRY(perm_in(A, bd, b.Bm + (size_t)c * ld, s));
      PCG_TRY(perm_in(A, xd, b.X + (size_t)c * ld, s));
    }
  }
  // ||b_c||; columns with b_c = 0 leave the block (x_c = 0)
  double *d_nb = part;
  bcg_norms_kernel<<<k, GT, 0, s>>>(n, ld, b.Bm, d_nb);
  count_launch();
  std::vector<double> nb(k);
  PCG_CUDA(cudaMemcpyAsync(nb.data(), d_nb, sizeof(double) * k, cudaMemcpyDeviceToHost, s));
  PCG_CUDA(cudaStreamSynchronize(s));
  std::vector<int> cols;
  for (int c = 0; c < k; c++)
    if (nb[c] != 0.0) cols.push_back(c);
  const int m = (int)cols.size();
  for (int a = 0; a < m; a++)
    if (cols[a] != a) {  // compact (cols is increasing: a <= cols[a], no overlap issues)
      PCG_CUDA(cudaMemcpyAsync(b.Bm + (size_t)a * ld, b.Bm + (size_t)cols[a] * ld, sizeof(double) * n,
                               cudaMemcpyDeviceToDevice, s));
      PCG_CUDA(cudaMemcpyAsync(b.X + (size_t)a * ld, b.X + (size_t)cols[a] * ld, sizeof(double) * n,
                               cudaMemcpyDeviceToDevice, s));
    }
  memset(hst, 0, sizeof(BcgState));
  hst->m = m;
  hst->tol = tol;
  hst->max_iter = max_iter;
  for (int a = 0; a < m; a++) hst->nb[a] = nb[cols[a]];
  PCG_CUDA(cudaMemcpyAsync(st, hst, sizeof(BcgState), cudaMemcpyHostToDevice, s));
  cudaEvent_t e0, e1;
  PCG_CUDA(cudaEventCreate(&e0));
  PCG_CUDA(cudaEventCreate(&e1));
  PCG_CUDA(cudaEventRecord(e0, s));
  int64_t replacements = 0;
  int done = BCG_OK;
  if (m > 0) {
    PCG_TRY(bcg_restart(A, b, m, ld, st, part, gt, s));
    for (;;) {
      PCG_CUDA(cudaMemcpyAsync(&hst->done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, s));
      PCG_CUDA(cudaStreamSynchronize(s));
      done = hst->done;
      if (done == BCG_RUNNING) {
        for (int u = 0; u < 8; u++) PCG_TRY(bcg_step(A, b, m, ld, st, part, gt, s));
        continue;
      }
      if (done == BCG_CHECK) {  // exit check on the true residuals (restart if it fails)
        PCG_TRY(bcg_restart(A, b, m, ld, st, part, gt, s));
        PCG_CUDA(cudaMemcpyAsync(&hst->done, &st->done, sizeof(int), cudaMemcpyDeviceToHost, s));
        PCG_CUDA(cudaStreamSynchronize(s));
        if (hst->done == BCG_OK) {
          done = BCG_OK;
          break;
        }
        replacements++;
        continue;
      }
      break;  // OK at the first restart, MAXIT, BREAKDOWN
    }
    if (done != BCG_OK) {  // true residuals of the last iterate for the report
      PCG_TRY(bcg_restart(A, b, m, ld, st, part, gt, s));
    }
  }
  PCG_CUDA(cudaEventRecord(e1, s));
  // X out: active columns from the block, the others 0
  for (int c = k - 1, a = m - 1; c >= 0; c--) {
    const bool act = a >= 0 && cols[a] == c;
    double *dst = X + (size_t)c * ldx;
    if (act) {
      const double *src = b.X + (size_t)a * ld;
      if (A->d_perm) {
        PCG_TRY(perm_out(A, src, b.Q, s));
        src = b.Q;
      }
      PCG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDefault, s));
      a--;
    } else {
      PCG_CUDA(cudaMemsetAsync(b.Q, 0, sizeof(double) * n, s));
      PCG_CUDA(cudaMemcpyAsync(dst, b.Q, sizeof(double) * n, cudaMemcpyDefault, s));
    }
    PCG_CUDA(cudaStreamSynchronize(s));  // b.Q is reused per column
  }
  PCG_CUDA(cudaMemcpyAsync(hst, st, sizeof(BcgState), cudaMemcpyDeviceToHost, s));
  PCG_CUDA(cudaStreamSynchronize(s));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const pcg_status status = done == BCG_OK      ? PCG_OK
                            : done == BCG_MAXIT ? PCG_NOT_CONVERGED
                                                : PCG_ERR_NOT_SPD;
  if (done == BCG_BREAKDOWN) fail(PCG_ERR_NOT_SPD, "pcg_solve_block: breakdown (a k x k Gram matrix lost definiteness)");
  const double it = (double)hst->it;
  const double bytes = it * (12.0 * (double)A->nnz + 4.0 * (double)(n + 1) + 112.0 * m * (double)n + 8.0 * (double)n);
  for (int c = 0, a = 0; c < k && infos; c++) {
    pcg_info &f = infos[c];
    memset(&f, 0, sizeof(f));
    f.iterations = hst->it;
    f.replacements = replacements;
    f.t_solve_s = ms * 1e-3;
    if (a < m && cols[a] == c) {
      f.relres_true = sqrt(hst->rr[a]) / hst->nb[a];
      f.relres_recurrence = hst->rec[a];
      f.converged = f.relres_true <= tol;
      f.status = status == PCG_OK && !f.converged ? PCG_NOT_CONVERGED : status;
      f.bytes_algorithmic = m > 0 ? bytes / m : 0.0;
      f.flops = it * (2.0 * (double)A->nnz + 10.0 * m * (double)n);
      a++;
    } else {
      f.converged = 1;
      f.status = PCG_OK;
    }
  }
  return status;
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_solve_block(pcg_matrix_t A, int32_t k, const double *B, int64_t ldb, double *X, int64_t ldx,
                                      double tol, int64_t max_iter, void *stream, pcg_info *infos) {
  if (!A || !B || !X) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_block: null argument");
  if (k < 1 || k > BK) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_block: 1 <= k <= 32");
  if (ldb < A->n || ldx < A->n) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_block: ld < n");
  if (!(tol > 0.0) || max_iter < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_block: tol > 0, max_iter >= 1");
  if (A->comm) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_block: one-GPU handles only");
  if (A->n == 0) {
    for (int c = 0; c < k && infos; c++) {
      memset(&infos[c], 0, sizeof(pcg_info));
      infos[c].converged = 1;
    }
    return PCG_OK;
  }
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  return block_cg_impl(A, k, B, ldb, X, ldx, tol, max_iter, (cudaStream_t)stream, infos);
}
