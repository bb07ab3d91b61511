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
// The Gram matrices run on the fp64 tensor cores (mma.sync m8n8k4 over 32-row tiles
// staged per warp in shared memory); the k x k mixing (X, R, P updates) is one thread
// per row with its m entries in registers and alpha/beta broadcast from shared memory.
#include <atomic>
#include <algorithm>
#include <cstdlib>
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

// ---------------------------------------------------------------- tall-skinny products on the fp64 tensor cores
// The m x m Gram matrices are dense contractions over n: each warp stages a 32-row tile
// (row-major [row][col], columns >= m zero) in shared memory and accumulates
// U^T V with mma.sync m8n8k4 f64 (A = U^T: a(i,k) = U[k][i]; B = V: b(k,j) = V[k][j]).
constexpr int TW = 4;  // warps per block of the tile kernels

__device__ __forceinline__ void dmma(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int MB>
__device__ __forceinline__ void warp_gram(const double *tu, const double *tv, double (&acc)[MB / 8][MB / 8][2]) {
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
#pragma unroll
  for (int s = 0; s < 8; s++) {
    const int kk = 4 * s + q;
    double av[MB / 8], bv[MB / 8];
#pragma unroll
    for (int I = 0; I < MB / 8; I++) {
      av[I] = tu[kk * (MB + 1) + 8 * I + g];
      bv[I] = tv[kk * (MB + 1) + 8 * I + g];
    }
#pragma unroll
    for (int I = 0; I < MB / 8; I++)
#pragma unroll
      for (int J = 0; J < MB / 8; J++) dmma(acc[I][J][0], acc[I][J][1], av[I], bv[J]);
  }
}

// block-wide fixed-order sum of the warps' fragments -> partials[e * gridDim.x + block]
// (e = a * m + b for a, b < m; then `extra` per-column values at e = m*m + a)
template <int MB>
__device__ __forceinline__ void block_store(const double (&acc)[MB / 8][MB / 8][2], const double *extra, int m,
                                            double *red, double *partials) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  for (int t = threadIdx.x; t < MB * MB + MB; t += blockDim.x) red[t] = 0.0;
  __syncthreads();
  for (int w = 0; w < TW; w++) {
    if (wid == w) {
#pragma unroll
      for (int I = 0; I < MB / 8; I++)
#pragma unroll
        for (int J = 0; J < MB / 8; J++) {
          red[(8 * I + g) * MB + 8 * J + 2 * q] += acc[I][J][0];
          red[(8 * I + g) * MB + 8 * J + 2 * q + 1] += acc[I][J][1];
        }
      if (extra && lane < MB) red[MB * MB + lane] += extra[lane];
    }
    __syncthreads();
  }
  const int mm = m * m;
  for (int e = threadIdx.x; e < mm + (extra ? m : 0); e += blockDim.x) {
    const double v = e < mm ? red[(e / m) * MB + e % m] : red[MB * MB + e - mm];
    partials[(size_t)e * gridDim.x + blockIdx.x] = v;
  }
}

// G = P^T Q
template <int MB>
__global__ void __launch_bounds__(TW * 32) bcg_gram_kernel(int64_t n, int m, int64_t ld, const double *__restrict__ U,
                                                           const double *__restrict__ V, double *partials,
                                                           const BcgState *st) {
  if (st->done != BCG_RUNNING) return;
  extern __shared__ double dsm[];
  __shared__ double red[MB * MB + MB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double *tu = dsm + (size_t)wid * 2 * 32 * (MB + 1), *tv = tu + 32 * (MB + 1);
  for (int c = 0; c < MB; c++) tu[lane * (MB + 1) + c] = tv[lane * (MB + 1) + c] = 0.0;
  double acc[MB / 8][MB / 8][2] = {};
  const int64_t ntile = (n + 31) / 32, w0 = (int64_t)blockIdx.x * TW + wid, nw = (int64_t)gridDim.x * TW;
  for (int64_t t = w0; t < ntile; t += nw) {
    const int64_t row = t * 32 + lane;
    const bool ok = row < n;
    double uv[MB], vv[MB];  // all 2m loads of the row in flight at once
#pragma unroll
    for (int c = 0; c < MB; c++) {
      uv[c] = ok && c < m ? U[(size_t)c * ld + row] : 0.0;
      vv[c] = ok && c < m ? V[(size_t)c * ld + row] : 0.0;
    }
#pragma unroll
    for (int c = 0; c < MB; c++) {
      tu[lane * (MB + 1) + c] = uv[c];
      tv[lane * (MB + 1) + c] = vv[c];
    }
    __syncwarp();
    warp_gram<MB>(tu, tv, acc);
    __syncwarp();
  }
  block_store<MB>(acc, nullptr, m, red, partials);
}

// ---------------------------------------------------------------- X, R, Z (and P at a restart) + R^T Z, diag R^T R
// MODE 0 (restart / exit check): R = B - Q (Q = A X), Z = dinv R, P = Z
// MODE 1 (step): X += P alpha, R -= Q alpha on the tensor cores: per warp a 32-row
//   tile, the (32 x m) . (m x m) products as m8n8k4 mma with the accumulators
//   initialised from X and R (fragment rows 8I + g, columns 8J + 2q + {0, 1}); then
//   Z = dinv R in the fragments.  R and Z go to shared-memory tiles for R^T Z.
template <int MB, int MODE>
__global__ void __launch_bounds__(TW * 32, 4) bcg_update_kernel(int64_t n, int m, int64_t ld, double *__restrict__ X,
                                                             double *__restrict__ R, double *__restrict__ Z,
                                                             double *__restrict__ P, const double *__restrict__ Q,
                                                             const double *__restrict__ Bm,
                                                             const double *__restrict__ dinv, double *partials,
                                                             const BcgState *st) {
  if (MODE == 1 && st->done != BCG_RUNNING) return;
  extern __shared__ double dsm[];
  __shared__ double sal[MB * MB];
  __shared__ double red[MB * MB + MB];
  __shared__ double wex[TW][MB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  for (int e = threadIdx.x; e < MB * MB; e += blockDim.x) sal[e] = 0.0;
  __syncthreads();
  if (MODE == 1)
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) sal[(e / m) * MB + e % m] = st->al[e];
  // per warp two tiles: P, Q of the step, then (once every mma of the tile is done) R, Z
  // for the Gram in the same space
  double *tp = dsm + (size_t)wid * 2 * 32 * (MB + 1), *tq = tp + 32 * (MB + 1);
  double *tr = tp, *tz = tq;
  for (int c = 0; c < MB; c++) tp[lane * (MB + 1) + c] = tq[lane * (MB + 1) + c] = 0.0;
  __syncthreads();
  double acc[MB / 8][MB / 8][2] = {};
  double rr[MB / 8][2] = {};  // this lane's columns 8J + 2q + e
  const int64_t ntile = (n + 31) / 32, w0 = (int64_t)blockIdx.x * TW + wid, nw = (int64_t)gridDim.x * TW;
  for (int64_t t = w0; t < ntile; t += nw) {
    const int64_t r0 = t * 32;
    if (MODE == 1) {
      const int64_t row = r0 + lane;
      const bool ok = row < n;
#pragma unroll
      for (int c0 = 0; c0 < MB; c0 += 8) {  // 16 loads in flight, few registers
        double pv[8], qv[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          pv[u] = ok && c0 + u < m ? P[(size_t)(c0 + u) * ld + row] : 0.0;
          qv[u] = ok && c0 + u < m ? Q[(size_t)(c0 + u) * ld + row] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          tp[lane * (MB + 1) + c0 + u] = pv[u];
          tq[lane * (MB + 1) + c0 + u] = qv[u];
        }
      }
      __syncwarp();
    }
    // per pair of 8-row blocks: all fragment loads (X, R or B - Q; dinv), the mma, then
    // the stores and the R, Z tile (rows of other pairs are not touched meanwhile)
#pragma unroll
    for (int I0 = 0; I0 < 4; I0 += 2) {
      double xf[2][MB / 8][2], rf[2][MB / 8][2], dv[2];
#pragma unroll
      for (int i = 0; i < 2; i++) {
        const int64_t row = r0 + 8 * (I0 + i) + g;
        const bool rok = row < n;
        dv[i] = rok ? dinv[row] : 0.0;
#pragma unroll
        for (int J = 0; J < MB / 8; J++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int cc = 8 * J + 2 * q + e;
            xf[i][J][e] = rf[i][J][e] = 0.0;
            if (rok && cc < m) {
              const size_t ix = (size_t)cc * ld + row;
              if (MODE == 0) {
                rf[i][J][e] = Bm[ix] - Q[ix];
              } else {
                xf[i][J][e] = X[ix];
                rf[i][J][e] = R[ix];
              }
            }
          }
      }
      if (MODE == 1) {
#pragma unroll
        for (int i = 0; i < 2; i++) {
          const int rl = 8 * (I0 + i) + g;
#pragma unroll
          for (int J = 0; J < MB / 8; J++)
#pragma unroll
            for (int s4 = 0; s4 < MB / 4; s4++) {
              const double bal = sal[(4 * s4 + q) * MB + 8 * J + g];
              dmma(xf[i][J][0], xf[i][J][1], tp[rl * (MB + 1) + 4 * s4 + q], bal);
              dmma(rf[i][J][0], rf[i][J][1], -tq[rl * (MB + 1) + 4 * s4 + q], bal);
            }
        }
        __syncwarp();  // these rows of the P, Q tiles are dead: R, Z take their place
      }
#pragma unroll
      for (int i = 0; i < 2; i++) {
        const int rl = 8 * (I0 + i) + g;
        const int64_t row = r0 + rl;
        const bool rok = row < n;
#pragma unroll
        for (int J = 0; J < MB / 8; J++)
#pragma unroll
          for (int e = 0; e < 2; e++) {
            const int cc = 8 * J + 2 * q + e;
            const bool ok = rok && cc < m;
            const double rv = rf[i][J][e], zv = dv[i] * rv;
            if (ok) {
              const size_t ix = (size_t)cc * ld + row;
              if (MODE == 1) X[ix] = xf[i][J][e];
              R[ix] = rv;
              Z[ix] = zv;
              if (MODE == 0) P[ix] = zv;
            }
            tr[rl * (MB + 1) + cc] = ok ? rv : 0.0;
            tz[rl * (MB + 1) + cc] = ok ? zv : 0.0;
            rr[J][e] = __fma_rn(ok ? rv : 0.0, ok ? rv : 0.0, rr[J][e]);
          }
      }
    }
    __syncwarp();
    warp_gram<MB>(tr, tz, acc);
    __syncwarp();
  }
  // diag R^T R: lanes with the same q hold the same columns; fold over g (fixed xor tree)
#pragma unroll
  for (int J = 0; J < MB / 8; J++)
#pragma unroll
    for (int e = 0; e < 2; e++) {
      double v = rr[J][e];
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 16);
      if (g == 0) wex[wid][8 * J + 2 * q + e] = v;
    }
  __syncthreads();
  block_store<MB>(acc, wex[wid], m, red, partials);
}

// ---------------------------------------------------------------- P = Z + P beta (tensor cores, as the step update)
template <int MB>
__global__ void __launch_bounds__(TW * 32) bcg_pupdate_kernel(int64_t n, int m, int64_t ld, double *__restrict__ P,
                                                              const double *__restrict__ Z, const BcgState *st) {
  if (st->done != BCG_RUNNING) return;
  extern __shared__ double dsm[];
  __shared__ double sbe[MB * MB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, q = lane & 3;
  for (int e = threadIdx.x; e < MB * MB; e += blockDim.x) sbe[e] = 0.0;
  __syncthreads();
  for (int e = threadIdx.x; e < m * m; e += blockDim.x) sbe[(e / m) * MB + e % m] = st->be[e];
  double *tp = dsm + (size_t)wid * 32 * (MB + 1);
  for (int c = 0; c < MB; c++) tp[lane * (MB + 1) + c] = 0.0;
  __syncthreads();
  const int64_t ntile = (n + 31) / 32, w0 = (int64_t)blockIdx.x * TW + wid, nw = (int64_t)gridDim.x * TW;
  for (int64_t t = w0; t < ntile; t += nw) {
    const int64_t r0 = t * 32;
    {
      const int64_t row = r0 + lane;
      const bool ok = row < n;
      double pv[MB];
#pragma unroll
      for (int c = 0; c < MB; c++) pv[c] = ok && c < m ? P[(size_t)c * ld + row] : 0.0;
#pragma unroll
      for (int c = 0; c < MB; c++) tp[lane * (MB + 1) + c] = pv[c];
    }
    __syncwarp();
#pragma unroll
    for (int I = 0; I < 4; I++) {
      const int rl = 8 * I + g;
      const int64_t row = r0 + rl;
      const bool rok = row < n;
#pragma unroll
      for (int J = 0; J < MB / 8; J++) {
        double v[2] = {0.0, 0.0};
        int cc[2];
#pragma unroll
        for (int e = 0; e < 2; e++) {
          cc[e] = 8 * J + 2 * q + e;
          if (rok && cc[e] < m) v[e] = Z[(size_t)cc[e] * ld + row];
        }
#pragma unroll
        for (int s4 = 0; s4 < MB / 4; s4++)
          dmma(v[0], v[1], tp[rl * (MB + 1) + 4 * s4 + q], sbe[(4 * s4 + q) * MB + 8 * J + g]);
#pragma unroll
        for (int e = 0; e < 2; e++)
          if (rok && cc[e] < m) P[(size_t)cc[e] * ld + row] = v[e];
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- k x k solves (one warp)
// Y = G^-1 C by Cholesky G = L L^T (as oracle.c chol_solve); false on a non-positive pivot
__device__ bool bcg_chol_solve(int m, const double *G, const double *Cm, double *Y) {
  __shared__ double L[BK * BK], sC[BK * BK], sY[BK * BK];
  __shared__ int s_fail;
  const int t = threadIdx.x;
  for (int e = t; e < m * m; e += 32) {
    L[e] = G[e];  // lower triangle overwritten by the factor
    sC[e] = Cm[e];
  }
  if (t == 0) s_fail = 0;
  __syncwarp();
  for (int j = 0; j < m; j++) {
    if (t == 0) {
      double d = L[j * m + j];
      for (int s = 0; s < j; s++) d -= L[j * m + s] * L[j * m + s];
      if (!(d > 0.0)) s_fail = 1;
      L[j * m + j] = sqrt(d);
    }
    __syncwarp();
    if (s_fail) return false;
    if (t > j && t < m) {
      double s = L[t * m + j];
      for (int q = 0; q < j; q++) s -= L[t * m + q] * L[j * m + q];
      L[t * m + j] = s / L[j * m + j];
    }
    __syncwarp();
  }
  if (t < m) {
    const int c = t;
    for (int i = 0; i < m; i++) {
      double s = sC[i * m + c];
      for (int q = 0; q < i; q++) s -= L[i * m + q] * sY[q * m + c];
      sY[i * m + c] = s / L[i * m + i];
    }
    for (int i = m - 1; i >= 0; i--) {
      double s = sY[i * m + c];
      for (int q = i + 1; q < m; q++) s -= L[q * m + i] * sY[q * m + c];
      sY[i * m + c] = s / L[i * m + i];
    }
  }
  __syncwarp();
  for (int e = t; e < m * m; e += 32) Y[e] = sY[e];
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
      st->done = all ? BCG_OK : (st->it >= st->max_iter ? BCG_MAXIT : BCG_RUNNING);  // orc_block_cg's order
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

int tile_grid(int64_t n, int sms) {  // blocks of TW warps, one 32-row tile per warp at a time
  return (int)std::max<int64_t>(1, std::min<int64_t>(((n + 31) / 32 + TW - 1) / TW, (int64_t)sms * 8));
}
}  // namespace

static pcg_status bcg_spmm(pcg_matrix *A, const double *P, double *Q, int m, int64_t ld, const BcgState *st,
                           cudaStream_t s) {
  const int sms = num_sms(A->device);
  if (A->format == PCG_FORMAT_CSR) {
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>((A->n + BLOCK - 1) / BLOCK, (int64_t)sms * 8));
    bcg_spmm_csr<<<g, BLOCK, 0, s>>>(A->csr(), P, Q, m, ld, st);
  } else if (getenv("PCG_BCG_OWN_SPMM")) {  // A/B knob: this file's simpler SpMM
    const unsigned g =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>((A->n_slices + WARPS - 1) / WARPS, (int64_t)sms * 4));
    bcg_spmm_sell<<<g, BLOCK, 0, s>>>(A->sell(), P, Q, m, ld, st);
  } else {  // the multi-RHS SpMM (L2 first-touch prefetch), gated on the block state
    return block_spmm(A, P, Q, m, ld, st ? &st->done : nullptr, s);
  }
  count_launch();
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

// restart / exit check: R = B - A X, Z = dinv R, P = Z, Gam = R^T Z, rr; done = OK iff all small
template <int MB>
static size_t bcg_dyn_smem(int tiles = 2) { return (size_t)TW * tiles * 32 * (MB + 1) * sizeof(double); }

// The dynamic shared-memory opt-in is a per-device function attribute: recorded per
// device (a second GPU in the same process needs its own), set idempotently (two
// threads racing here both set the same value).
template <int MB>
static pcg_status bcg_prepare() {
  static std::atomic<bool> done[64];
  int dev = 0;
  PCG_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && done[dev].load(std::memory_order_acquire)) return PCG_OK;
  const int sm = (int)bcg_dyn_smem<MB>(), sm4 = (int)bcg_dyn_smem<MB>(2), sm1 = (int)bcg_dyn_smem<MB>(1);
  PCG_CUDA(cudaFuncSetAttribute(bcg_gram_kernel<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
  PCG_CUDA(cudaFuncSetAttribute(bcg_update_kernel<MB, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
  PCG_CUDA(cudaFuncSetAttribute(bcg_update_kernel<MB, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm4));
  PCG_CUDA(cudaFuncSetAttribute(bcg_pupdate_kernel<MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1));
  if (dev >= 0 && dev < 64) done[dev].store(true, std::memory_order_release);
  return PCG_OK;
}

// restart / exit check: R = B - A X, Z = dinv R, P = Z, Gam = R^T Z, rr; done = OK iff all small
template <int MB>
static pcg_status bcg_restart_mb(pcg_matrix *A, const BcgBufs &b, int m, int64_t ld, BcgState *st, double *part,
                                 int gt, cudaStream_t s) {
  PCG_TRY(bcg_prepare<MB>());
  PCG_TRY(bcg_spmm(A, b.X, b.Q, m, ld, nullptr, s));
  bcg_update_kernel<MB, 0><<<gt, TW * 32, bcg_dyn_smem<MB>(2), s>>>(A->n, m, ld, b.X, b.R, b.Z, b.P, b.Q, b.Bm,
                                                                   A->d_dinv, part, st);
  bcg_reduce_kernel<<<m * m + m, GT, 0, s>>>(part, gt, m * m, st->Gn, st->rr, nullptr);
  bcg_small_kernel<<<1, 32, 0, s>>>(st, BS_INIT);
  count_launch(3);
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

template <int MB>
static pcg_status bcg_step_mb(pcg_matrix *A, const BcgBufs &b, int m, int64_t ld, BcgState *st, double *part, int gt,
                              cudaStream_t s) {
  PCG_TRY(bcg_prepare<MB>());
  PCG_TRY(bcg_spmm(A, b.P, b.Q, m, ld, st, s));
  bcg_gram_kernel<MB><<<gt, TW * 32, bcg_dyn_smem<MB>(), s>>>(A->n, m, ld, b.P, b.Q, part, st);
  bcg_reduce_kernel<<<m * m, GT, 0, s>>>(part, gt, m * m, st->G, nullptr, st);
  bcg_small_kernel<<<1, 32, 0, s>>>(st, BS_ALPHA);
  bcg_update_kernel<MB, 1><<<gt, TW * 32, bcg_dyn_smem<MB>(2), s>>>(A->n, m, ld, b.X, b.R, b.Z, b.P, b.Q, b.Bm,
                                                                   A->d_dinv, part, st);
  bcg_reduce_kernel<<<m * m + m, GT, 0, s>>>(part, gt, m * m, st->Gn, st->rr, st);
  bcg_small_kernel<<<1, 32, 0, s>>>(st, BS_BETA);
  bcg_pupdate_kernel<MB><<<gt, TW * 32, bcg_dyn_smem<MB>(1), s>>>(A->n, m, ld, b.P, b.Z, st);
  count_launch(7);
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

static pcg_status bcg_restart(pcg_matrix *A, const BcgBufs &b, int m, int64_t ld, BcgState *st, double *part, int gt,
                              cudaStream_t s) {
  if (m <= 8) return bcg_restart_mb<8>(A, b, m, ld, st, part, gt, s);
  if (m <= 16) return bcg_restart_mb<16>(A, b, m, ld, st, part, gt, s);
  return bcg_restart_mb<32>(A, b, m, ld, st, part, gt, s);
}
static pcg_status bcg_step(pcg_matrix *A, const BcgBufs &b, int m, int64_t ld, BcgState *st, double *part, int gt,
                           cudaStream_t s) {
  if (m <= 8) return bcg_step_mb<8>(A, b, m, ld, st, part, gt, s);
  if (m <= 16) return bcg_step_mb<16>(A, b, m, ld, st, part, gt, s);
  return bcg_step_mb<32>(A, b, m, ld, st, part, gt, s);
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
  pcgb::NvtxRange nvtx_("pcg:pcg_solve_block");
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
