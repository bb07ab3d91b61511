// multi.cu — Jacobi-PCG for k right-hand sides.
//
// The paper's "block of r.h.s. terms" A X = B (Eq. MRH-TERMS) solved
// by an iterative method that "solve[s] a new linear system for every
// right-hand side term": column c runs the single-RHS recurrence of
// solver.cu independently and freezes at its own stopping test.
//
// Device layout: every block vector (R, Z, Q, P, X, B, W) is column-major
// n x k with a leading dimension ld = n rounded up to 32 (256-B aligned
// columns), the ABI's own layout, so B and X move with one 2D copy each.
//
// Three passes per block iteration (the single-RHS schedule 3 of solver.cu):
//   K1a (streaming, grid = row chunks x columns)  X_c += xpend_c P_c ; P_c = Z_c + beta_c P_c
//   K1b (SpMM over SELL-32 slices)                Q_c = A P_c ; sigma_c = P_c . Q_c -> alpha_c
//   K2  (streaming, grid = row chunks x columns)  R_c -= alpha_c Q_c ; Z_c = dinv R_c ;
//                                                 rho'_c, gamma_c -> stop test, beta_c
// = 12 nnz + 4(n+1) + 96 k n bytes per block iteration (88 k n: the 2-pass ideal).
// In K1b each warp loads its slice's matrix entries ONCE into registers and then
// runs k SpMV gather rounds from them (one per active column): the matrix is
// read from HBM once per iteration for all k columns, and every gather round is
// coalesced across the 32 rows of the slice exactly like the single-RHS SpMV.
// Frozen columns cost nothing: their blocks of K1a/K2 return at entry and K1b
// skips their gather round.  Column c's SpMM sum is formed left to right over
// the row with one fma per entry: bitwise the single-RHS SELL SpMV of column c.
#include <climits>
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "matrix.cuh"
#include "rows.cuh"
#include "staged.cuh"

namespace pcgb {

#ifndef PCG_MXDEFER_M  // default cycle of the k-column loop's deferred X update
#define PCG_MXDEFER_M 4
#endif

struct MVecs {
  double *R, *Z, *Q, *P, *X, *W;
  double *P1, *P2, *P3;  // deferred x update: the direction blocks hold passes write (P2, P3: 4-cycle)
  const double *Bm;  // right-hand sides (column-major, ld)
  const double *dinv;
  int64_t ld;        // leading dimension (n rounded up to 32)
};

enum { MS_SPMM = 0, MS_RESID = 1 };

__device__ __forceinline__ void mstop(int use_cond, cudaGraphConditionalHandle h) {
  if (use_cond) cudaGraphSetConditional(h, 0);
}

__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// ---------------------------------------------------------------- reductions
// Block partials are published as partials[(i * KMAX + c) * nb + b] for the NV
// values i of column c from block b (nb = blocks per column); the last block to
// arrive sums them per (i, c) in a fixed order (8 strands of a fixed stride, then
// the strands in order) into out[i][c].  Deterministic for a fixed grid.
__device__ __forceinline__ bool mlast_block(unsigned int *counter) {
  __shared__ bool s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x * gridDim.y - 1);
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

template <int NV>
__device__ void mcols_reduce(const double *partials, int nb, int k, double (*out)[KMAX], double (*sm)[KMAX]) {
  constexpr int STRANDS = BLOCK / KMAX;  // 8
  const int c = threadIdx.x % KMAX, strand = threadIdx.x / KMAX;
  for (int i = 0; i < NV; i++) {
    double acc = 0.0;
    if (c < k) {
#pragma unroll 4
      for (int b = strand; b < nb; b += STRANDS) acc += __ldcg(partials + ((size_t)i * KMAX + c) * nb + b);
    }
    sm[strand][c] = acc;
    __syncthreads();
    if (threadIdx.x < KMAX) {
      double t = 0.0;
#pragma unroll
      for (int s = 0; s < STRANDS; s++) t += sm[s][threadIdx.x];
      out[i][threadIdx.x] = t;
    }
    __syncthreads();
  }
}

// mcols_reduce for blocks with more than BLOCK threads (the windowed SpMM): the first
// BLOCK threads form the strands, the others only take part in the barriers
template <int NV>
__device__ void mcols_reduce_n(const double *partials, int nb, int k, double (*out)[KMAX], double (*sm)[KMAX]) {
  constexpr int STRANDS = BLOCK / KMAX;  // 8
  const int c = threadIdx.x % KMAX, strand = threadIdx.x / KMAX;
  for (int i = 0; i < NV; i++) {
    if (threadIdx.x < BLOCK) {
      double acc = 0.0;
      if (c < k) {
#pragma unroll 4
        for (int b = strand; b < nb; b += STRANDS) acc += __ldcg(partials + ((size_t)i * KMAX + c) * nb + b);
      }
      sm[strand][c] = acc;
    }
    __syncthreads();
    if (threadIdx.x < KMAX) {
      double t = 0.0;
#pragma unroll
      for (int s = 0; s < STRANDS; s++) t += sm[s][threadIdx.x];
      out[i][threadIdx.x] = t;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- finishers (thread 0 of the last block)
// pass: 0 = X updated every iteration; else the deferred X update's (M << 4) | j, pass
// j of an M-cycle (M = 2 or 4, mk1a_kernel): j < M-1 holds (the owed alpha of the direction
// in P[j] stays owed, the new direction is in P[j+1]), j = M-1 applies
__device__ void mk1b_finish(const double *sig, MultiScalars *sc, int use_cond, cudaGraphConditionalHandle h,
                            int pass) {
  const int xm = pass >> 4, xj = pass & 15;
  const bool hold = xm && xj < xm - 1;
  sc->cnt_a = 0;
  int na = 0;
  for (int c = 0; c < sc->kcols; c++) {
    if (!sc->active[c]) {
      sc->xpend[c] = 0.0;  // an owed x update was applied by this iteration's K1a
      sc->nheld[c] = 0;
      continue;
    }
    const double sigma = sig[c];
    sc->sigma[c] = sigma;
    const double owed = sc->xpend[c];  // alpha of the direction this iteration's K1a read
    if (!(sigma > 0.0)) {  // p^T A p <= 0: breakdown, A not SPD
      sc->done[c] = DONE_BREAKDOWN;
      sc->active[c] = 0;
      sc->xpend[c] = 0.0;
      if (hold) {  // a hold pass left alpha_{k-1} p_{k-1} (in P[j]) owed
        sc->ahold[xj][c] = owed;
        sc->nheld[c] = xj + 1;
        sc->lbuf[c] = xj + 1;
      } else {
        sc->nheld[c] = 0;
        sc->lbuf[c] = 0;
      }
    } else {
      sc->alpha[c] = sc->rho[c] / sigma;
      sc->xpend[c] = sc->alpha[c];  // x += alpha p is deferred to the next K1a / the tail
      if (hold) {
        sc->ahold[xj][c] = owed;
        sc->nheld[c] = xj + 1;
        sc->lbuf[c] = xj + 1;
      } else if (xm) {
        sc->nheld[c] = 0;
        sc->lbuf[c] = 0;
      }
      sc->k[c] += 1;
      na++;
    }
  }
  sc->n_active = na;
  sc->graph_launches += use_cond;
  if (na == 0) mstop(use_cond, h);
}

__device__ void mk2_finish(const double (*t)[KMAX], MultiScalars *sc, int use_cond, cudaGraphConditionalHandle h) {
  sc->cnt_b = 0;
  int na = 0;
  for (int c = 0; c < sc->kcols; c++) {
    if (!sc->active[c]) continue;
    const double rho_new = t[0][c], gamma = t[1][c];
    sc->gamma[c] = gamma;
    const double rr = sqrt(gamma);
    sc->relres_rec[c] = rr / sc->nb[c];
    if (rr <= sc->tol * sc->nb[c]) {
      sc->done[c] = DONE_CONVERGED;  // frozen; xpend = alpha_k still owed to x
      sc->active[c] = 0;
    } else if (!(gamma == gamma)) {
      sc->done[c] = DONE_NONFINITE;
      sc->active[c] = 0;
      sc->xpend[c] = 0.0;
    } else if (sc->k[c] >= sc->max_iter) {
      sc->done[c] = DONE_MAXIT;
      sc->active[c] = 0;
    } else {
      sc->beta[c] = rho_new / sc->rho[c];
      sc->rho[c] = rho_new;
      na++;
    }
  }
  sc->n_active = na;
  sc->graph_launches += use_cond;
  if (na == 0) mstop(use_cond, h);
}

// ---------------------------------------------------------------- K1a: X_c += xpend_c P_c ; P_c = Z_c + beta_c P_c
// grid (gx, k): blockIdx.y = column.  Just-frozen columns only receive their owed
// x update; settled frozen columns return at entry.
// Deferred X update (as the single-RHS k1a_hold / k1a_apply, per column): hold pass j
// writes P[j+1]_c = Z_c + beta_c P[j]_c and leaves X_c alone; the apply pass applies the
// held directions oldest first and then the latest, X_c = fma(xpend_c, P[M-1]_c,
// fma(ahold[M-2]_c, P[M-2]_c, ... X_c)), and writes P[0]_c = Z_c + beta_c P[M-1]_c — the
// fused multiply-adds of the every-iteration update in the same order (bitwise the same
// X).  A just-frozen column applies what it owes (held, then latest: P[lbuf_c]).
__host__ __device__ __forceinline__ double *mbuf(const MVecs &v, int b) {
  return b == 0 ? v.P : b == 1 ? v.P1 : b == 2 ? v.P2 : v.P3;
}

template <int M>
__device__ __forceinline__ void mk1a_apply(int64_t n, const MVecs &v, const volatile MultiScalars *vs, int c,
                                           double xp, double beta) {
  const size_t o = (size_t)c * v.ld;
  double ah[M - 1];
#pragma unroll
  for (int h = 0; h < M - 1; h++) ah[h] = vs->ahold[h][c];
  const double2 *hb[M - 1];
#pragma unroll
  for (int h = 0; h < M - 1; h++) hb[h] = reinterpret_cast<const double2 *>(mbuf(v, h) + o);
  const double *Pl = mbuf(v, M - 1) + o;
  const double2 *__restrict__ L2 = reinterpret_cast<const double2 *>(Pl);
  double2 *__restrict__ A2 = reinterpret_cast<double2 *>(v.P + o);
  double2 *__restrict__ X2 = reinterpret_cast<double2 *>(v.X + o);
  const double2 *__restrict__ Z2 = reinterpret_cast<const double2 *>(v.Z + o);
  const int64_t npair = n >> 1;
  const int64_t t0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x, ts = (int64_t)gridDim.x * BLOCK;
  for (int64_t t = t0; t < npair; t += ts) {
    const double2 pk = L2[t], zz = __ldcs(Z2 + t);
    double2 pm[M - 1];
#pragma unroll
    for (int h = 0; h < M - 1; h++) pm[h] = __ldcs(hb[h] + t);
    double2 xx = __ldcs(X2 + t);
#pragma unroll
    for (int h = 0; h < M - 1; h++) {
      xx.x = __fma_rn(ah[h], pm[h].x, xx.x);
      xx.y = __fma_rn(ah[h], pm[h].y, xx.y);
    }
    xx.x = __fma_rn(xp, pk.x, xx.x);
    xx.y = __fma_rn(xp, pk.y, xx.y);
    __stcs(X2 + t, xx);
    A2[t] = make_double2(__fma_rn(beta, pk.x, zz.x), __fma_rn(beta, pk.y, zz.y));
  }
  if ((n & 1) && t0 == 0) {
    const int64_t i = n - 1;
    double xi = v.X[o + i];
#pragma unroll
    for (int h = 0; h < M - 1; h++) xi = __fma_rn(ah[h], mbuf(v, h)[o + i], xi);
    v.X[o + i] = __fma_rn(xp, Pl[i], xi);
    v.P[o + i] = __fma_rn(beta, Pl[i], v.Z[o + i]);
  }
}

__device__ __forceinline__ void mk1a_deferred(int64_t n, const MVecs &v, const volatile MultiScalars *vs, int c,
                                              int pass) {
  const int xm = pass >> 4, xj = pass & 15;
  const double xp = vs->xpend[c], beta = vs->beta[c];
  const int act = vs->active[c], nh = vs->nheld[c];
  if (!act && xp == 0.0 && nh == 0) return;
  const size_t o = (size_t)c * v.ld;
  const int64_t t0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x, ts = (int64_t)gridDim.x * BLOCK;
  if (!act) {  // just frozen: the owed updates, held directions first
    const double *Pl = mbuf(v, vs->lbuf[c]) + o;
    double ah[3];
    for (int h = 0; h < 3; h++) ah[h] = vs->ahold[h][c];
    double *X = v.X + o;
    for (int64_t i = t0; i < n; i += ts) {
      double x = X[i];
      for (int h = 0; h < nh; h++)
        if (ah[h] != 0.0) x = __fma_rn(ah[h], mbuf(v, h)[o + i], x);
      if (xp != 0.0) x = __fma_rn(xp, Pl[i], x);
      X[i] = x;
    }
    return;
  }
  if (xj < xm - 1) {  // hold: P[j+1] = Z + beta P[j]
    const double *src = mbuf(v, xj) + o;
    double *dst = mbuf(v, xj + 1) + o;
    const double *Z = v.Z + o;
    const int64_t npair = n >> 1;
    const double2 *__restrict__ A2 = reinterpret_cast<const double2 *>(src);
    double2 *__restrict__ B2 = reinterpret_cast<double2 *>(dst);
    const double2 *__restrict__ Z2 = reinterpret_cast<const double2 *>(Z);
    for (int64_t t = t0; t < npair; t += ts) {
      const double2 po = __ldcs(A2 + t), zz = __ldcs(Z2 + t);
      B2[t] = make_double2(__fma_rn(beta, po.x, zz.x), __fma_rn(beta, po.y, zz.y));
    }
    if ((n & 1) && t0 == 0) dst[n - 1] = __fma_rn(beta, src[n - 1], Z[n - 1]);
  } else if (xm == 4) {
    mk1a_apply<4>(n, v, vs, c, xp, beta);
  } else {
    mk1a_apply<2>(n, v, vs, c, xp, beta);
  }
}

__global__ void __launch_bounds__(BLOCK, 4) mk1a_kernel(int64_t n, MVecs v, MultiScalars *sc, int use_cond,
                                                     cudaGraphConditionalHandle h, int pass) {
  const volatile MultiScalars *vs = sc;
  if (vs->n_active == 0) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) mstop(use_cond, h);
    return;
  }
  const int c = blockIdx.y;
  if (pass) {
    mk1a_deferred(n, v, vs, c, pass);
    return;
  }
  const double xp = vs->xpend[c], beta = vs->beta[c];
  const int act = vs->active[c];
  if (!act && xp == 0.0) return;
  double *__restrict__ P = v.P + (size_t)c * v.ld;
  double *__restrict__ X = v.X + (size_t)c * v.ld;
  const double *__restrict__ Z = v.Z + (size_t)c * v.ld;
  const int64_t npair = n >> 1;
  double2 *__restrict__ P2 = reinterpret_cast<double2 *>(P);
  double2 *__restrict__ X2 = reinterpret_cast<double2 *>(X);
  const double2 *__restrict__ Z2 = reinterpret_cast<const double2 *>(Z);
  const int64_t t0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x, ts = (int64_t)gridDim.x * BLOCK;
  if (act) {
    for (int64_t t = t0; t < npair; t += ts) {
      const double2 po = P2[t], zz = __ldcs(Z2 + t);
      if (xp != 0.0) {
        double2 xx = __ldcs(X2 + t);
        xx.x = __fma_rn(xp, po.x, xx.x);
        xx.y = __fma_rn(xp, po.y, xx.y);
        __stcs(X2 + t, xx);
      }
      P2[t] = make_double2(__fma_rn(beta, po.x, zz.x), __fma_rn(beta, po.y, zz.y));
    }
  } else {
    for (int64_t t = t0; t < npair; t += ts) {
      const double2 po = __ldcs(P2 + t);
      double2 xx = __ldcs(X2 + t);
      xx.x = __fma_rn(xp, po.x, xx.x);
      xx.y = __fma_rn(xp, po.y, xx.y);
      __stcs(X2 + t, xx);
    }
  }
  if ((n & 1) && t0 == 0) {
    const int64_t i = n - 1;
    const double po = P[i];
    if (xp != 0.0) X[i] = __fma_rn(xp, po, X[i]);
    if (act) P[i] = __fma_rn(beta, po, Z[i]);
  }
}

// rows longer than 8 entries (slow path, kept out of line so the fast path keeps
// its registers): entries re-read per column in chunks of 8 (L1/L2 hits)
__device__ __forceinline__ double long_row_sum(const double *vp, const int *cp, int len, const double *__restrict__ Gc,
                                            int zero) {
  double sum = 0.0;
#pragma unroll 1
  for (int t = 0; t < len; t += 8) {
    double aa[8], g[8];
    int jj[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (t + u < len) {
        aa[u] = __ldg(vp + (size_t)(t + u) * 32);
        jj[u] = __ldg(cp + (size_t)(t + u) * 32);
      }
    cols_ready(jj, zero);
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (t + u < len) g[u] = __ldg(Gc + jj[u]);
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (t + u < len) sum = __fma_rn(aa[u], g[u], sum);
  }
  return sum;
}

// ---------------------------------------------------------------- K1b: SpMM (and the residual pass)
// One warp per SELL-32 slice (lane = row).  The slice's entries are loaded once
// (8 at a time, all column loads before the first gather: rows.cuh cols_ready)
// and reused by one gather round per column.  Slices with more than 8 entries per
// row re-read their entries per column (L1/L2 hits) in chunks of 8; that path is
// compiled only into the LONG instantiation, used when max row length > 8.
//   MS_SPMM : Q_c = A P_c, block partial sigma_c = Σ P_c Q_c           (active columns)
//   MS_RESID: W_c = B_c - A X_c, block partials (W.W, W.(dinv W), B.B)   (all k columns)
// Per (slice, column) the row values meet in a fixed xor tree and lane 0 adds
// them to the warp's accumulator in slice order; warps are combined in order.
#ifndef PCG_SPMM_PAT  // A/B knob: the SpMM reads shared value-free slice patterns
#define PCG_SPMM_PAT 1
#endif
template <int MODE, bool LONG>
__global__ void __launch_bounds__(BLOCK, LONG ? 1 : 4) mspmm_kernel(SellViewDia S, MVecs v, MultiScalars *sc, double *partials, int k,
                                                      int pf, int use_cond, cudaGraphConditionalHandle h,
                                                      int pass) {
  constexpr int NV = MODE == MS_SPMM ? 1 : 3;
  __shared__ int s_act[KMAX];
  __shared__ double s_red[NV][WARPS][KMAX];
  __shared__ double s_sm[BLOCK / KMAX][KMAX];
  __shared__ double s_out[NV][KMAX];
  const volatile MultiScalars *vs = sc;
  if (MODE == MS_SPMM && vs->n_active == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) mstop(use_cond, h);
    return;
  }
  if (threadIdx.x < KMAX) s_act[threadIdx.x] = threadIdx.x < k && (MODE == MS_RESID || vs->active[threadIdx.x]);

  for (int t = threadIdx.x; t < NV * WARPS * KMAX; t += BLOCK) (&s_red[0][0][0])[t] = 0.0;
  extern __shared__ double s_acc[];  // MS_SPMM: [k][BLOCK] per-thread sigma partials
  // MS_SPMM with k <= 16: per-thread sigma partials in shared memory (no per-slice warp
  // reduction); larger k would cost occupancy, so those reduce per slice instead
  const bool acc_smem = MODE == MS_SPMM && k <= 16;
  if (acc_smem)
    for (int t = threadIdx.x; t < k * BLOCK; t += BLOCK) s_acc[t] = 0.0;
  // the matrix's value-free slice patterns (common.cuh SellViewDia::dpat): such a slice's
  // entries come from shared memory instead of the value/id streams
  __shared__ DiaPat s_pat[DIA_MAXPAT];
  __shared__ int s_plen[DIA_MAXPAT];
  const bool pats = PCG_SPMM_PAT && S.dpat != nullptr && S.npat > 0;
  if (pats) {
    for (int t = threadIdx.x; t < S.npat * 12; t += BLOCK)
      reinterpret_cast<double *>(s_pat)[t] = reinterpret_cast<const double *>(S.ptab)[t];
    for (int t = threadIdx.x; t < S.npat; t += BLOCK) s_plen[t] = S.plen[t];
  }
  __syncthreads();
  unsigned int act = 0;  // active columns as a register mask (s_act costs a shared load per use)
  for (int c = 0; c < k; c++) act |= (unsigned int)s_act[c] << c;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // grid-stride slice map: at any time the whole grid works on one window of rows, so
  // gathered lines shared with other SMs (the far stencil neighbours) meet in L2.  (A
  // contiguous chunk per block, for L1 reuse, measured 316 vs 229 us on C4.)
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + wid, nw = (int64_t)gridDim.x * WARPS;
  const double *__restrict__ G = MODE == MS_SPMM ? v.P : v.X;  // gathered block vector
  // the next slice's pattern index is fetched one slice ahead (indexed by slice)
  unsigned pid_n = pats && w0 < S.n_slices ? (unsigned)S.dpat[w0] : (unsigned)DIA_NOPAT;
  for (int64_t s = w0; s < S.n_slices; s += nw) {
    const unsigned pid = pid_n;
    pid_n = pats && s + nw < S.n_slices ? (unsigned)S.dpat[s + nw] : (unsigned)DIA_NOPAT;
    int64_t base = 0;
    int len;
    if (pid != DIA_NOPAT) {
      len = s_plen[pid];
    } else {
      base = __ldg(S.slice_ptr + s);
      len = (int)((__ldg(S.slice_ptr + s + 1) - base) >> 5);
    }
    const int64_t row = s * 32 + lane;
    const bool ok = row < S.n;
    const double *vp = S.val + base + lane;
    const int *cp = S.col + base + lane;
    // epilogue of column c for this slice (row sum -> output + reduction values)
    auto finish_col = [&](int c, double sum) {
      double r[NV];
#pragma unroll
      for (int i = 0; i < NV; i++) r[i] = 0.0;
      if (ok) {
        const size_t e = (size_t)c * v.ld + row;
        if (MODE == MS_SPMM) {
          __stcs(v.Q + e, sum);
          r[0] = __ldg(v.P + e) * sum;  // (reusing the diagonal's gather measured slower)
        } else {
          const double bi = v.Bm[e];
          const double w = bi - sum;
          v.W[e] = w;
          const double z = v.dinv[row] * w;
          r[0] = w * w;
          r[NV > 1 ? 1 : 0] = w * z;
          r[NV - 1] = bi * bi;
        }
      }
      if (MODE == MS_SPMM && acc_smem) {  // per-thread running sum; lanes meet once, at the end
        s_acc[c * BLOCK + threadIdx.x] += r[0];
      } else {
#pragma unroll
        for (int i = 0; i < NV; i++) {
          r[i] = warp_sum(r[i]);
          if (lane == 0) s_red[i][wid][c] += r[i];
        }
      }
    };
    if (!LONG || len <= 8) {  // fast path: the slice's entries stay in registers for all columns
      double a[8];
      int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (pid != DIA_NOPAT) {  // the pattern's offsets and values (the slice's own, bitwise)
        const DiaPat &P = s_pat[pid];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          a[u] = u < len ? P.val[u] : 0.0;
          j[u] = u < len ? (int)row + P.off[u] : 0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; u++) {
          a[u] = 0.0;
          if (u < len) {
            a[u] = ld_stream(vp + (size_t)u * 32);
            j[u] = ld_stream(cp + (size_t)u * 32);
          }
        }
        cols_ready(j, S.zero);
      }
      if (pf) {  // first touch of a gathered line is (mostly) its largest column: start every
                 // column's fetch now so only the first gather round waits on HBM (padding
                 // entries are column 0; a select of j[len - 1] went to local memory)
        int jl = j[0];
#pragma unroll
        for (int u = 1; u < 8; u++) jl = max(jl, j[u]);
#pragma unroll 1
        for (int c = 0; c < k; c++)
          if (act >> c & 1) prefetch_l2(G + (size_t)c * v.ld + jl);
      }
      unsigned int off[8];  // byte offsets of the gathered entries (columns < 2^29)
#pragma unroll
      for (int u = 0; u < 8; u++) off[u] = (unsigned int)j[u] << 3;
      const int64_t ld = v.ld;
      const char *Gb = reinterpret_cast<const char *>(G);
#pragma unroll 1
      for (int c = 0; c < k; c++, Gb += ld * 8) {
        if (!(act >> c & 1)) continue;
        double g[8];
#pragma unroll
        for (int u = 0; u < 8; u++) g[u] = u < len ? __ldg(reinterpret_cast<const double *>(Gb + off[u])) : 0.0;
        // entries past the row's length are a = g = 0: fma(0, 0, s) == s exactly (s is never -0),
        // so the unpredicated chain is bitwise the left-to-right sum over the row
        double sum = 0.0;
#pragma unroll
        for (int u = 0; u < 8; u++) sum = __fma_rn(a[u], g[u], sum);
        finish_col(c, sum);
      }
    } else {
#pragma unroll 1
      for (int c = 0; c < k; c++) {
        if (!(act >> c & 1)) continue;
        finish_col(c, long_row_sum(vp, cp, len, G + (size_t)c * v.ld, S.zero));
      }
    }
  }
  if (acc_smem) {  // each warp folds its lanes' running sums (fixed xor tree)
    for (int c = 0; c < k; c++) {
      const double t = warp_sum(s_acc[c * BLOCK + threadIdx.x]);
      if (lane == 0) s_red[0][wid][c] = t;
    }
  }
  __syncthreads();
  if (threadIdx.x < KMAX) {
#pragma unroll
    for (int i = 0; i < NV; i++) {
      double t = 0.0;
#pragma unroll
      for (int w = 0; w < WARPS; w++) t += s_red[i][w][threadIdx.x];
      partials[((size_t)i * KMAX + threadIdx.x) * gridDim.x + blockIdx.x] = t;
    }
  }
  unsigned int *cnt = MODE == MS_SPMM ? &sc->cnt_a : &sc->cnt_c;
  if (!mlast_block(cnt)) return;
  mcols_reduce<NV>(partials, gridDim.x, k, s_out, s_sm);
  if (threadIdx.x == 0) {
    if (MODE == MS_SPMM) {
      mk1b_finish(s_out[0], sc, use_cond, h, pass);
    } else {
      sc->cnt_c = 0;
      for (int c = 0; c < KMAX; c++)
        for (int i = 0; i < NV; i++) sc->part[i][c] = c < k ? s_out[i][c] : 0.0;
    }
  }
}

// ---------------------------------------------------------------- K2: R_c -= alpha_c Q_c ; Z_c = dinv R_c ; rho'_c, gamma_c
// grid (gx, k): blockIdx.y = column; frozen columns publish zero partials.
__global__ void __launch_bounds__(BLOCK) mk2_kernel(int64_t n, MVecs v, MultiScalars *sc, double *partials,
                                                    int use_cond, cudaGraphConditionalHandle h,
                                                    const double *__restrict__ dsl) {
  __shared__ double sm2[2][WARPS];
  __shared__ double s_sm[BLOCK / KMAX][KMAX];
  __shared__ double s_out[2][KMAX];
  const volatile MultiScalars *vs = sc;
  if (vs->n_active == 0) {
    if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) mstop(use_cond, h);
    return;
  }
  const int c = blockIdx.y;
  const int act = vs->active[c];
  const double alpha = vs->alpha[c];
  double a0 = 0.0, a1 = 0.0;
  if (act) {
    double *__restrict__ R = v.R + (size_t)c * v.ld;
    double *__restrict__ Z = v.Z + (size_t)c * v.ld;
    const double *__restrict__ Q = v.Q + (size_t)c * v.ld;
    const int64_t npair = n >> 1;
    const double2 *__restrict__ q2 = reinterpret_cast<const double2 *>(Q);
    const double2 *__restrict__ d2 = reinterpret_cast<const double2 *>(v.dinv);
    double2 *__restrict__ r2 = reinterpret_cast<double2 *>(R);
    double2 *__restrict__ z2 = reinterpret_cast<double2 *>(Z);
    const int64_t t0 = (int64_t)blockIdx.x * BLOCK + threadIdx.x, ts = (int64_t)gridDim.x * BLOCK;
    for (int64_t t = t0; t < npair; t += ts) {
      const double2 qq = __ldcs(q2 + t);
      double2 rr = r2[t];
      // one dinv per 32-row slice where the slice shares one (SolveWork::dslice; same values)
      const double du = dsl ? __ldg(dsl + (t >> 4)) : __longlong_as_double(0x7ff8000000000000ll);
      const double2 dd = du == du ? make_double2(du, du) : __ldg(d2 + t);
      rr.x = __fma_rn(-alpha, qq.x, rr.x);
      rr.y = __fma_rn(-alpha, qq.y, rr.y);
      const double2 zz = make_double2(dd.x * rr.x, dd.y * rr.y);
      r2[t] = rr;
      z2[t] = zz;
      a0 = __fma_rn(rr.x, zz.x, a0);
      a0 = __fma_rn(rr.y, zz.y, a0);
      a1 = __fma_rn(rr.x, rr.x, a1);
      a1 = __fma_rn(rr.y, rr.y, a1);
    }
    if ((n & 1) && t0 == 0) {
      const int64_t i = n - 1;
      const double ri = __fma_rn(-alpha, Q[i], R[i]);
      const double zi = v.dinv[i] * ri;
      R[i] = ri;
      Z[i] = zi;
      a0 = __fma_rn(ri, zi, a0);
      a1 = __fma_rn(ri, ri, a1);
    }
  }
  double red[2] = {a0, a1};
  block_sum<2>(red, sm2);
  if (threadIdx.x == 0) {  // partials per column: [i][c][bx]
    partials[((size_t)0 * KMAX + c) * gridDim.x + blockIdx.x] = red[0];
    partials[((size_t)1 * KMAX + c) * gridDim.x + blockIdx.x] = red[1];
  }
  if (!mlast_block(&sc->cnt_b)) return;
  mcols_reduce<2>(partials, gridDim.x, gridDim.y, s_out, s_sm);
  if (threadIdx.x == 0) mk2_finish(s_out, sc, use_cond, h);
}

// ---------------------------------------------------------------- init / exit scalar logic (after mspmm<RESID>)
__global__ void mresid_finish_kernel(MultiScalars *sc, int mode) {
  int na = 0;
  for (int c = 0; c < KMAX; c++) {
    sc->replace[c] = 0;
    if (c >= sc->kcols) {
      sc->active[c] = 0;
      sc->done[c] = DONE_ZERO_RHS;
      continue;
    }
    const double ww = sc->part[0][c], wz = sc->part[1][c], bb = sc->part[2][c];
    if (mode == 0) {  // init
      sc->k[c] = 0;
      sc->nrep[c] = 0;
      sc->xpend[c] = 0.0;
      sc->alpha[c] = sc->beta[c] = 0.0;
      sc->relres_true[c] = 0.0;
      sc->active[c] = 0;
      if (!isfinite(bb) || !isfinite(ww)) {
        sc->done[c] = DONE_NONFINITE;
        continue;
      }
      sc->nb[c] = sqrt(bb);
      if (sc->nb[c] == 0.0) {
        sc->done[c] = DONE_ZERO_RHS;
        continue;
      }
      const double rr = sqrt(ww);
      sc->relres_rec[c] = rr / sc->nb[c];
      if (rr <= sc->tol * sc->nb[c]) {
        sc->done[c] = DONE_CONVERGED;
        continue;
      }
      sc->done[c] = DONE_RUNNING;
      sc->active[c] = 1;
      sc->replace[c] = 1;
      sc->rho[c] = wz;
      na++;
    } else {  // exit check
      if (sc->done[c] == DONE_ZERO_RHS || sc->done[c] == DONE_NONFINITE) continue;
      sc->relres_true[c] = sqrt(ww) / sc->nb[c];
      if (sc->done[c] == DONE_CONVERGED && !(sc->relres_true[c] <= sc->tol)) {
        if (sc->k[c] >= sc->max_iter) {
          sc->done[c] = DONE_MAXIT;
        } else {  // residual replacement for this column
          sc->done[c] = DONE_RUNNING;
          sc->active[c] = 1;
          sc->replace[c] = 1;
          sc->nrep[c] += 1;
          sc->rho[c] = wz;
          sc->beta[c] = 0.0;
          sc->xpend[c] = 0.0;
          na++;
        }
      }
    }
  }
  sc->n_active = na;
}

// R_c = W_c, Z_c = dinv W_c, P_c = 0 for columns being (re)started; grid (gx, k)
__global__ void mreplace_kernel(int64_t n, MVecs v, const MultiScalars *sc) {
  const int c = blockIdx.y;
  if (!sc->replace[c]) return;
  const size_t o = (size_t)c * v.ld;
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    const double w = v.W[o + i];
    v.R[o + i] = w;
    v.Z[o + i] = v.dinv[i] * w;
    v.P[o + i] = 0.0;
  }
}

// deferred X_c += xpend_c P_c after the loop stops; grid (gx, k)
// (deferred x update: the held directions first, then the latest one in P[lbuf])
__global__ void mtail_kernel(int64_t n, MVecs v, const MultiScalars *sc) {
  const int c = blockIdx.y;
  const double xp = sc->xpend[c];
  const int nh = sc->nheld[c];
  if (xp == 0.0 && nh == 0) return;
  const size_t o = (size_t)c * v.ld;
  const double *Pl = mbuf(v, sc->lbuf[c]) + o;
  double ah[3];
  for (int h = 0; h < 3; h++) ah[h] = sc->ahold[h][c];
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    double x = v.X[o + i];
    for (int h = 0; h < nh; h++)
      if (ah[h] != 0.0) x = __fma_rn(ah[h], mbuf(v, h)[o + i], x);
    if (xp != 0.0) x = __fma_rn(xp, Pl[i], x);
    v.X[o + i] = x;
  }
}
__global__ void mclear_xpend_kernel(MultiScalars *sc) {
  for (int c = 0; c < KMAX; c++) {
    sc->xpend[c] = 0.0;
    for (int h = 0; h < 3; h++) sc->ahold[h][c] = 0.0;
    sc->nheld[c] = 0;
    sc->lbuf[c] = 0;
  }
}
// x = 0 for b = 0 columns; grid (gx, k)
__global__ void mzero_rhs_kernel(int64_t n, MVecs v, const MultiScalars *sc) {
  const int c = blockIdx.y;
  if (sc->done[c] != DONE_ZERO_RHS) return;
  const size_t o = (size_t)c * v.ld;
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) v.X[o + i] = 0.0;
}

// ---------------------------------------------------------------- host side
static int64_t mld(int64_t n) { return ((n > 0 ? n : 1) + 31) / 32 * 32; }

pcg_status ensure_multi_work(pcg_matrix *A, int k) {
  SolveWork &w = A->work;
  if (w.kcap >= k && w.msc) return PCG_OK;
  for (double *p : {w.mr, w.mz, w.mq, w.mp[0], w.mp[1], w.mp23[0], w.mp23[1], w.mx, w.mb, w.mw})
    if (p) cudaFree(p);
  w.mr = w.mz = w.mq = w.mp[0] = w.mp[1] = w.mp23[0] = w.mp23[1] = w.mx = w.mb = w.mw = nullptr;
  if (w.mloop_exec) cudaGraphExecDestroy(w.mloop_exec);
  if (w.mloop_graph) cudaGraphDestroy(w.mloop_graph);
  w.mloop_exec = nullptr;
  w.mloop_graph = nullptr;
  w.mgraph_k = 0;
  w.kcap = 0;
  const size_t nk = sizeof(double) * (size_t)mld(A->n) * k;
  PCG_CUDA(cudaMalloc(&w.mr, nk));
  PCG_CUDA(cudaMalloc(&w.mz, nk));
  PCG_CUDA(cudaMalloc(&w.mq, nk));
  PCG_CUDA(cudaMalloc(&w.mp[0], nk));
  PCG_CUDA(cudaMalloc(&w.mp[1], nk));
  PCG_CUDA(cudaMemset(w.mp[1], 0, nk));
  PCG_CUDA(cudaMalloc(&w.mx, nk));
  PCG_CUDA(cudaMalloc(&w.mb, nk));
  PCG_CUDA(cudaMalloc(&w.mw, nk));
  PCG_CUDA(cudaMemset(w.mp[0], 0, nk));
  PCG_CUDA(cudaMemset(w.mz, 0, nk));
  PCG_CUDA(cudaMemset(w.mx, 0, nk));
  // partials: 3 x KMAX x (SpMM grid <= 8 per SM) + 2 x KMAX x (vector grid x <= 8 per SM)
  if (!w.mpart) PCG_CUDA(cudaMalloc(&w.mpart, sizeof(double) * 5 * KMAX * (size_t)num_sms(A->device) * 8));
  if (!w.msc) {
    PCG_CUDA(cudaMalloc(&w.msc, sizeof(MultiScalars)));
    PCG_CUDA(cudaMemset(w.msc, 0, sizeof(MultiScalars)));
    PCG_CUDA(cudaMallocHost(&w.h_msc, sizeof(MultiScalars)));
  }
  w.kcap = k;
  return PCG_OK;
}

static MVecs mvecs_of(pcg_matrix *A) {
  SolveWork &w = A->work;
  return MVecs{w.mr, w.mz, w.mq, w.mp[0], w.mx, w.mw, w.mp[1], w.mp23[0], w.mp23[1], w.mb, A->d_dinv, mld(A->n)};
}

// streaming passes: grid (gx, k) with gx * k ~ 8 blocks per SM
static dim3 mgrid_vec(pcg_matrix *A, int k) {
  const int64_t need = std::max<int64_t>(1, (A->n / 2 + BLOCK - 1) / BLOCK);
  const int64_t g = std::max<int64_t>(1, (int64_t)num_sms(A->device) * 8 / k);
  return dim3((unsigned)std::min(g, need), (unsigned)k, 1);
}

// SpMM pass: persistent grid of SMs x resident blocks (<= 8 per SM: the partials capacity)
static int mgrid_spmm(pcg_matrix *A, int k) {
  // up to 32 KB of per-thread sigma partials (k <= 16): a per-device function attribute,
  // set on every call (cheap, idempotent) so a second GPU in the process gets it too
  cudaFuncSetAttribute(mspmm_kernel<MS_SPMM, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * BLOCK * 16);
  cudaFuncSetAttribute(mspmm_kernel<MS_SPMM, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * BLOCK * 16);
  int b = 0;
  const size_t smem = k <= 16 ? sizeof(double) * BLOCK * k : 0;
  cudaError_t e = A->max_row_len > 8
                      ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, mspmm_kernel<MS_SPMM, true>, BLOCK, smem)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, mspmm_kernel<MS_SPMM, false>, BLOCK, smem);
  if (e != cudaSuccess) {
    cudaGetLastError();
    b = 4;
  }
  b = std::max(1, std::min(8, b));
  const int64_t need = std::max<int64_t>(1, (A->n_slices + WARPS - 1) / WARPS);
  return (int)std::min<int64_t>((int64_t)num_sms(A->device) * b, need);
}

// ---------------------------------------------------------------- windowed SpMM (K1b for k right-hand sides)
// The register-gather SpMM above moves every gathered P entry from L2 to the SM
// (7 gathers per row and column for the 7-point stencil: ~1.8 GB per SpMM at C4, k =
// 16, against 0.7 GB of HBM traffic), which makes the L2 -> SM path, not HBM, its
// bound.  Here the column windows a tile of rows references are copied ONCE per
// (tile, column) into shared memory by the TMA bulk-copy engine and every gather is a
// shared-memory load:
//   * tile = WT_SLICES SELL slices (512 rows); its referenced columns, sorted, split
//     into at most W_NWIN contiguous windows where consecutive columns are more than
//     W_GAP apart (the 7-point stencil: the -m^2 band, the [-m, +m] band, the +m^2
//     band); the windows total at most W_CAP entries;
//   * per SELL entry, its 16-bit offset in the concatenated windows (the "plan",
//     built once per matrix on the device, win_plan_kernel);
//   * one producer thread per CTA issues, per (tile, active column), one
//     cp.async.bulk per window into a ring of W_STAGES shared-memory stages (full /
//     empty mbarriers, expect_tx bytes); W_CW consumer warps, 2 slices each, hold their
//     slices' entries in registers for all columns of the tile and form each row sum
//     left to right with one fma per entry (bitwise the SpMV's sum), write Q_c and
//     their sigma_c partial (P_c at the row is in the window that holds the tile's
//     own rows).
// L2 -> SM bytes per row and column: the windows' (3 T + 2 m) / T x 8 B ~ 28 B
// instead of ~57 B.  Matrices with rows longer than 8, or whose tiles need more
// windows or space, keep the register-gather kernel (multi.cu mspmm_kernel).
constexpr int WT_SLICES = 16, WT_ROWS = WT_SLICES * 32, W_NWIN = 4, W_CAP = 2048, W_STAGES = 4, W_CW = 8;
constexpr int W_THREADS = (W_CW + 1) * 32, W_GAP = 64, W_KEYS = WT_ROWS * 8;

struct WinDesc {
  int nwin, self_off, start[W_NWIN], len[W_NWIN], off[W_NWIN], pad[2];
};
static_assert(sizeof(WinDesc) == 64, "WinDesc is one 64-B record");

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// one CTA (512 threads) per tile: sort the tile's referenced columns (bitonic, in shared
// memory), cut them into windows, write the descriptor and every entry's window offset
__global__ void __launch_bounds__(512) win_plan_kernel(SellView S, int64_t n_tiles, WinDesc *__restrict__ desc,
                                                       uint16_t *__restrict__ lidx, int *__restrict__ fail) {
  __shared__ int keys[W_KEYS];
  __shared__ WinDesc d;
  __shared__ int s_bad;
  const int64_t t = blockIdx.x;
  const int64_t s0 = t * WT_SLICES, s1 = (s0 + WT_SLICES < S.n_slices) ? s0 + WT_SLICES : S.n_slices;
  const int64_t e0 = S.slice_ptr[s0], e1 = S.slice_ptr[s1];
  const int cnt = (int)(e1 - e0);
  if (threadIdx.x == 0) s_bad = cnt > W_KEYS;
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) atomicAdd(fail, 1);
    return;
  }
  // entry e lies in slice s(e): its row is s*32 + lane; rows >= n are padding of the last slice
  for (int i = threadIdx.x; i < W_KEYS; i += blockDim.x) {
    int key = INT_MAX;
    if (i < cnt) {
      const int64_t e = e0 + i;
      int64_t s = s0;
      while (S.slice_ptr[s + 1] <= e) s++;
      const int64_t row = s * 32 + (e & 31);
      if (row < S.n) key = S.col[e];
    }
    keys[i] = key;
  }
  __syncthreads();
  for (int k = 2; k <= W_KEYS; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < W_KEYS; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const int a = keys[i], b = keys[l];
          if ((a > b) == up) {
            keys[i] = b;
            keys[l] = a;
          }
        }
      }
      __syncthreads();
    }
  if (threadIdx.x == 0) {
    int nw = 0, bad = 0;
    int st[W_NWIN + 1], en[W_NWIN + 1];
    int prev = keys[0];
    if (prev != INT_MAX) {
      st[0] = prev;
      nw = 1;
      for (int i = 1; i < W_KEYS && keys[i] != INT_MAX; i++) {
        const int c = keys[i];
        if (c == prev) continue;
        if (c - prev > W_GAP) {
          en[nw - 1] = prev + 1;
          if (nw == W_NWIN) {
            bad = 1;
            break;
          }
          st[nw++] = c;
        }
        prev = c;
      }
      if (!bad) en[nw - 1] = prev + 1;
    }
    int tot = 0;
    d.nwin = bad ? 0 : nw;
    for (int w = 0; w < W_NWIN; w++) {
      d.start[w] = d.len[w] = d.off[w] = 0;
      if (!bad && w < nw) {
        const int a = st[w] & ~1, b = (en[w] + 1) & ~1;  // 16-B aligned copies
        d.start[w] = a;
        d.len[w] = b - a;
        d.off[w] = tot;
        tot += b - a;
      }
    }
    if (tot > W_CAP) bad = 1;
    const int64_t r0 = s0 * 32, r1 = (s1 * 32 < S.n) ? s1 * 32 : S.n;
    d.self_off = -1;
    for (int w = 0; w < nw && !bad; w++)
      if (d.start[w] <= r0 && r1 <= d.start[w] + d.len[w]) d.self_off = d.off[w] + (int)(r0 - d.start[w]);
    if (d.self_off < 0) bad = 1;
    d.pad[0] = d.pad[1] = 0;
    s_bad = bad;
    if (bad) atomicAdd(fail, 1);
    desc[t] = d;
  }
  __syncthreads();
  if (s_bad) return;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int64_t e = e0 + i;
    int64_t s = s0;
    while (S.slice_ptr[s + 1] <= e) s++;
    const int64_t row = s * 32 + (e & 31);
    int o = 0;  // padding rows (>= n): any in-window offset (a = 0, result unused)
    if (row < S.n) {
      const int c = S.col[e];
      for (int w = 0; w < d.nwin; w++)
        if (c >= d.start[w] && c < d.start[w] + d.len[w]) o = d.off[w] + c - d.start[w];
    }
    lidx[e] = (uint16_t)o;
  }
}

// Q_c = A P_c and sigma_c = P_c . Q_c for the active columns, windows staged by TMA.
__global__ void __launch_bounds__(W_THREADS, 3)
    mspmm_win_kernel(SellView S, const WinDesc *__restrict__ desc, const uint16_t *__restrict__ lidx, MVecs v,
                     MultiScalars *sc, double *partials, int k, int use_cond, cudaGraphConditionalHandle h) {
  extern __shared__ __align__(128) unsigned char smem[];
  double *ring = reinterpret_cast<double *>(smem);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)W_STAGES * W_CAP * 8);
  uint64_t *empty = full + W_STAGES;
  __shared__ double s_red[W_CW][KMAX];
  __shared__ double s_sm[BLOCK / KMAX][KMAX];
  __shared__ double s_out[1][KMAX];
  const volatile MultiScalars *vs = sc;
  if (vs->n_active == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) mstop(use_cond, h);
    return;
  }
  unsigned int act = 0;
  for (int c = 0; c < k; c++) act |= (unsigned int)(vs->active[c] != 0) << c;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t n_tiles = (S.n_slices + WT_SLICES - 1) / WT_SLICES;
  const int64_t ld = v.ld;
  if (threadIdx.x == 0) {
    for (int s = 0; s < W_STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], W_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < W_CW * KMAX; i += blockDim.x) (&s_red[0][0])[i] = 0.0;
  __syncthreads();
  if (warp == W_CW) {  // ---- producer: one elected thread issues the window copies
    if (lane == 0) {
      int q = 0;
      for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const WinDesc d = desc[t];
        const int64_t tn = t + gridDim.x;  // the next tile's matrix entries, toward L2
        if (tn < n_tiles) {
          const int64_t a = __ldg(S.slice_ptr + tn * WT_SLICES);
          const int64_t b = __ldg(S.slice_ptr + ((tn + 1) * WT_SLICES < S.n_slices ? (tn + 1) * WT_SLICES : S.n_slices));
          if (b > a) {
            bulk_prefetch_l2(S.val + a, (uint32_t)((b - a) * 8));
            bulk_prefetch_l2(lidx + a, (uint32_t)(((b - a) * 2 + 15) & ~15));
          }
        }
        uint32_t bytes = 0;
        for (int w = 0; w < d.nwin; w++) bytes += (uint32_t)d.len[w] * 8;
        for (int c = 0; c < k; c++) {
          if (!(act >> c & 1)) continue;
          const int st = q % W_STAGES;
          if (q >= W_STAGES) mbar_wait(&empty[st], (uint32_t)((q / W_STAGES - 1) & 1));
          mbar_expect_tx(&full[st], bytes);
          const double *Pc = v.P + (size_t)c * ld;
          for (int w = 0; w < d.nwin; w++)
            bulk_g2s(ring + (size_t)st * W_CAP + d.off[w], Pc + d.start[w], (uint32_t)d.len[w] * 8, &full[st]);
          q++;
        }
      }
    }
  } else {  // ---- consumers: 2 slices per warp
    int q = 0;
    for (int64_t t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      const int self_off = __ldg(&desc[t].self_off);
      const int64_t r0 = t * WT_ROWS;
      double a[2][8];
      int li[2][8];
      bool has[2];
#pragma unroll
      for (int j = 0; j < 2; j++) {
        const int64_t s = t * WT_SLICES + warp * 2 + j;
        has[j] = s < S.n_slices;
        int len = 0;
        int64_t base = 0;
        if (has[j]) {
          base = __ldg(S.slice_ptr + s);
          len = (int)((__ldg(S.slice_ptr + s + 1) - base) >> 5);
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          a[j][u] = 0.0;
          li[j][u] = 0;  // beyond the row: a = 0 times the (written) first window entry
          if (u < len) {
            a[j][u] = ld_stream(S.val + base + (size_t)u * 32 + lane);
            li[j][u] = (int)__ldg(lidx + base + (size_t)u * 32 + lane);
          }
        }
      }
      for (int c = 0; c < k; c++) {
        if (!(act >> c & 1)) continue;
        const int st = q % W_STAGES;
        mbar_wait(&full[st], (uint32_t)((q / W_STAGES) & 1));
        const double *buf = ring + (size_t)st * W_CAP;
        double acc = 0.0;
#pragma unroll
        for (int j = 0; j < 2; j++) {
          if (!has[j]) continue;
          double sum = 0.0;
#pragma unroll
          for (int u = 0; u < 8; u++) sum = __fma_rn(a[j][u], buf[li[j][u]], sum);
          const int64_t row = (t * WT_SLICES + warp * 2 + j) * 32 + lane;
          if (row < S.n) {
            __stcs(v.Q + (size_t)c * ld + row, sum);
            acc = __fma_rn(buf[self_off + (int)(row - r0)], sum, acc);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        acc = warp_sum(acc);
        if (lane == 0) s_red[warp][c] += acc;
        q++;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < KMAX) {
    double tsum = 0.0;
#pragma unroll
    for (int w = 0; w < W_CW; w++) tsum += s_red[w][threadIdx.x];
    partials[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = tsum;
  }
  if (!mlast_block(&sc->cnt_a)) return;
  mcols_reduce_n<1>(partials, gridDim.x, k, s_out, s_sm);
  if (threadIdx.x == 0) mk1b_finish(s_out[0], sc, use_cond, h, 0);  // (the deferred x update is off here)
}

static size_t win_smem() { return (size_t)W_STAGES * W_CAP * 8 + 2 * W_STAGES * 8; }

static int win_grid(pcg_matrix *A) {
  cudaFuncSetAttribute(mspmm_win_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem());
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, mspmm_win_kernel, W_THREADS, win_smem()) != cudaSuccess) {
    cudaGetLastError();
    b = 1;
  }
  b = std::max(1, std::min(8, b));
  const int64_t n_tiles = (A->n_slices + WT_SLICES - 1) / WT_SLICES;
  return (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms(A->device) * b, n_tiles));
}

// build the window plan once per matrix (SELL-32 with rows of at most 8 entries)
static pcg_status win_plan(pcg_matrix *A, cudaStream_t st) {
  if (A->wplan != 0) return PCG_OK;
  // opt-in (PCG_SPMM_WIN=1): measured as fast as the register-gather SpMM, not faster
  // (the SM's load pipe, not L2, bounds both)
  const char *e = getenv("PCG_SPMM_WIN");
  if (!(e && atoi(e) == 1) || A->max_row_len > 8 || A->n_slices == 0 || A->comm || A->n + 2 > (int64_t(1) << 31)) {
    A->wplan = -1;
    return PCG_OK;
  }
  const int64_t n_tiles = (A->n_slices + WT_SLICES - 1) / WT_SLICES;
  PCG_CUDA(cudaMalloc(&A->d_wdesc, sizeof(WinDesc) * n_tiles));
  PCG_CUDA(cudaMalloc(&A->d_wlidx, sizeof(uint16_t) * std::max<int64_t>(A->sell_entries, 8)));
  int *d_fail;
  PCG_CUDA(cudaMalloc(&d_fail, sizeof(int)));
  PCG_CUDA(cudaMemsetAsync(d_fail, 0, sizeof(int), st));
  win_plan_kernel<<<(unsigned)n_tiles, 512, 0, st>>>(A->sell(), n_tiles, (WinDesc *)A->d_wdesc, A->d_wlidx, d_fail);
  count_launch();
  int fails = 0;
  PCG_CUDA(cudaMemcpyAsync(&fails, d_fail, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_fail);
  if (fails) {
    cudaFree(A->d_wdesc);
    cudaFree(A->d_wlidx);
    A->d_wdesc = nullptr;
    A->d_wlidx = nullptr;
    A->wplan = -1;
  } else {
    A->wplan = 1;
  }
  return PCG_OK;
}

// tuning knob PCG_SPMM_PF (default 1): L2 prefetch of each slice's first-touch lines
static int spmm_prefetch() {
  static int v = [] {
    const char *e = getenv("PCG_SPMM_PF");
    return e ? atoi(e) : 1;
  }();
  return v;
}

template <int MODE>
static void launch_mspmm(pcg_matrix *A, int k, cudaStream_t st, int use_cond, cudaGraphConditionalHandle h,
                         int pass = 0) {
  SolveWork &w = A->work;
  if (MODE == MS_SPMM && A->wplan == 1) {
    mspmm_win_kernel<<<win_grid(A), W_THREADS, win_smem(), st>>>(A->sell(), (const WinDesc *)A->d_wdesc, A->d_wlidx,
                                                                 mvecs_of(A), w.msc, w.mpart, k, use_cond, h);
    return;
  }
  const int g = mgrid_spmm(A, k);
  const SellViewDia S = A->sell_dia();
  MVecs v = mvecs_of(A);
  if (pass) {  // the block this pass's K1a wrote: P[j+1] after a hold, P[0] after the apply
    const int xm = pass >> 4, xj = pass & 15;
    v.P = mbuf(v, xj < xm - 1 ? xj + 1 : 0);
  }
  const size_t smem = MODE == MS_SPMM && k <= 16 ? sizeof(double) * BLOCK * k : 0;
  if (A->max_row_len > 8)
    mspmm_kernel<MODE, true><<<g, BLOCK, smem, st>>>(S, v, w.msc, w.mpart, k, spmm_prefetch(), use_cond, h, pass);
  else
    mspmm_kernel<MODE, false><<<g, BLOCK, smem, st>>>(S, v, w.msc, w.mpart, k, spmm_prefetch(), use_cond, h, pass);
}

// ---------------------------------------------------------------- the SpMM alone, for block CG (blockcg.cu)
// Q = A P over SELL-32 for k <= 32 column-major columns (ld), through mspmm_kernel on
// a scratch MultiScalars re-armed before every launch (all k columns active; none if
// *d_done != 0, so finished block solves skip it).  Its sigma side results stay in
// the scratch state.
__global__ void bspmm_arm_kernel(MultiScalars *sc, int k, const int *d_done) {
  const int t = threadIdx.x;
  if (t < KMAX) {
    sc->active[t] = t < k;
    sc->done[t] = 0;
    sc->rho[t] = 1.0;
  }
  if (t == 0) {
    sc->n_active = (d_done && *d_done != 0) ? 0 : k;
    sc->kcols = k;
    sc->cnt_a = 0;
  }
}

pcg_status block_spmm(pcg_matrix *A, const double *P, double *Q, int k, int64_t ld, const int *d_done,
                      cudaStream_t st) {
  SolveWork &w = A->work;
  if (!w.bspmm_sc) {
    PCG_CUDA(cudaMalloc(&w.bspmm_sc, sizeof(MultiScalars)));
    PCG_CUDA(cudaMemset(w.bspmm_sc, 0, sizeof(MultiScalars)));
    PCG_CUDA(cudaMalloc(&w.bspmm_part, sizeof(double) * 3 * KMAX * (size_t)num_sms(A->device) * 8));
  }
  MultiScalars *sc = (MultiScalars *)w.bspmm_sc;
  bspmm_arm_kernel<<<1, 32, 0, st>>>(sc, k, d_done);
  const int g = mgrid_spmm(A, k);
  MVecs v{};
  v.P = const_cast<double *>(P);
  v.Q = Q;
  v.ld = ld;
  const size_t smem = k <= 16 ? sizeof(double) * BLOCK * k : 0;
  if (A->max_row_len > 8)
    mspmm_kernel<MS_SPMM, true><<<g, BLOCK, smem, st>>>(A->sell_dia(), v, sc, w.bspmm_part, k, spmm_prefetch(), 0, 0, 0);
  else
    mspmm_kernel<MS_SPMM, false><<<g, BLOCK, smem, st>>>(A->sell_dia(), v, sc, w.bspmm_part, k, spmm_prefetch(), 0, 0, 0);
  count_launch(2);
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

static double *mpart_rz(pcg_matrix *A) { return A->work.mpart + (size_t)3 * KMAX * num_sms(A->device) * 8; }

// deferred x update for the k-column loop (mk1a_deferred): not with the windowed SpMM
// (opt-in); PCG_XDEFER=0 turns it off
static int mxdefer(const pcg_matrix *A) {  // the cycle M (0: off); PCG_XDEFER as solver.cu
  if (A->wplan == 1) return 0;
  const char *e = getenv("PCG_XDEFER");
  const int m = e ? atoi(e) : PCG_MXDEFER_M;
  return m == 2 || m == 4 ? m : (m == 0 ? 0 : PCG_MXDEFER_M);
}
static int mxd_arg(int m, int u) { return m ? (m << 4) | (u % m) : 0; }

// the 4-cycle's direction blocks P[2], P[3] (once per workspace)
static pcg_status ensure_mdir(pcg_matrix *A, int k, int m) {
  SolveWork &w = A->work;
  if (m != 4 || w.mp23[0]) return PCG_OK;
  const size_t nk = sizeof(double) * (size_t)mld(A->n) * (size_t)w.kcap;
  for (double *&q : w.mp23) {
    PCG_CUDA(cudaMalloc(&q, nk));
    PCG_CUDA(cudaMemset(q, 0, nk));
  }
  (void)k;
  return PCG_OK;
}

static pcg_status mlaunch_iteration(pcg_matrix *A, int k, cudaStream_t st, int use_cond, cudaGraphConditionalHandle h,
                                    int pass) {
  SolveWork &w = A->work;
  MVecs v = mvecs_of(A);
  const dim3 gv = mgrid_vec(A, k);
  mk1a_kernel<<<gv, BLOCK, 0, st>>>(A->n, v, w.msc, use_cond, h, pass);
  launch_mspmm<MS_SPMM>(A, k, st, use_cond, h, pass);
  mk2_kernel<<<gv, BLOCK, 0, st>>>(A->n, v, w.msc, mpart_rz(A), use_cond, h, w.dslice);
  count_launch(3);
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

static pcg_status mbuild_graph(pcg_matrix *A, int k) {
  SolveWork &w = A->work;
  PCG_TRY(ensure_mdir(A, k, mxdefer(A)));
  if (w.mgraph_k == k && w.mloop_exec) return PCG_OK;
  if (w.mloop_exec) cudaGraphExecDestroy(w.mloop_exec);
  if (w.mloop_graph) cudaGraphDestroy(w.mloop_graph);
  w.mloop_exec = nullptr;
  w.mloop_graph = nullptr;
  cudaStream_t cap;
  PCG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t g;
  PCG_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  PCG_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  alignas(cudaGraphNodeParams) unsigned char npbuf[sizeof(cudaGraphNodeParams)] = {};
  cudaGraphNodeParams &np = *reinterpret_cast<cudaGraphNodeParams *>(npbuf);
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t node;
  PCG_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  PCG_CUDA(cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  pcg_status s = PCG_OK;
  const int xm = mxdefer(A);
  const int nbody = xm == 4 ? 4 : 2;  // body = one deferral cycle
  for (int u = 0; u < nbody && s == PCG_OK; u++) s = mlaunch_iteration(A, k, cap, 1, h, mxd_arg(xm, u));
  cudaGraph_t out;
  cudaError_t e = cudaStreamEndCapture(cap, &out);
  if (s != PCG_OK) return s;
  PCG_CUDA(e);
  PCG_CUDA(cudaGraphInstantiate(&w.mloop_exec, g, 0));
  w.mloop_graph = g;
  w.mgraph_k = k;
  cudaStreamDestroy(cap);
  return PCG_OK;
}

// residual pass + scalar logic (+ restart of the columns that need it)
static pcg_status mresid(pcg_matrix *A, int k, int mode, cudaStream_t st) {
  SolveWork &w = A->work;
  MVecs v = mvecs_of(A);
  launch_mspmm<MS_RESID>(A, k, st, 0, 0);
  mresid_finish_kernel<<<1, 1, 0, st>>>(w.msc, mode);
  mreplace_kernel<<<mgrid_vec(A, k), BLOCK, 0, st>>>(A->n, v, w.msc);
  count_launch(3);
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

static pcg_status multi_prepare(pcg_matrix *A, int k, cudaStream_t st) {
  PCG_TRY(ensure_work(A));
  PCG_TRY(build_sell(A, st));  // the SpMM runs over SELL-32 slices whatever format SpMV uses
  PCG_TRY(ensure_multi_work(A, k));
  PCG_TRY(win_plan(A, st));
  return PCG_OK;
}

static pcg_status solve_multi_chunk(pcg_matrix *A, int k, const double *B, int64_t ldb, double *X, int64_t ldx,
                                    double tol, int64_t max_iter, cudaStream_t st, pcg_info *infos) {
  PCG_TRY(multi_prepare(A, k, st));
  PCG_TRY(mbuild_graph(A, k));
  SolveWork &w = A->work;
  const int64_t n = A->n, ld = mld(n);
  const bool bd = is_device_ptr(B), xd = is_device_ptr(X);
  // SELL-C-sigma handles hold P A P^T: columns enter as P B, P X0 (through W as staging)
  double *bdst = A->d_perm ? w.mw : w.mb, *xdst = A->d_perm ? w.mw : w.mx;
  PCG_CUDA(cudaMemcpy2DAsync(bdst, sizeof(double) * ld, B, sizeof(double) * ldb, sizeof(double) * n, k,
                             bd ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  if (A->d_perm) PCG_TRY(perm_in_cols(A, k, w.mw, ld, w.mb, ld, st));
  PCG_CUDA(cudaMemcpy2DAsync(xdst, sizeof(double) * ld, X, sizeof(double) * ldx, sizeof(double) * n, k,
                             xd ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  if (A->d_perm) PCG_TRY(perm_in_cols(A, k, w.mw, ld, w.mx, ld, st));
  MultiScalars *h = w.h_msc;
  memset(h, 0, sizeof(MultiScalars));
  h->tol = tol;
  h->max_iter = max_iter;
  h->kcols = k;
  PCG_CUDA(cudaMemcpyAsync(w.msc, h, sizeof(MultiScalars), cudaMemcpyHostToDevice, st));
  MVecs v = mvecs_of(A);
  const dim3 gv = mgrid_vec(A, k);
  cudaEvent_t e0, e1;
  PCG_CUDA(cudaEventCreate(&e0));
  PCG_CUDA(cudaEventCreate(&e1));
  PCG_CUDA(cudaEventRecord(e0, st));
  int mode = 0;
  for (;;) {
    PCG_TRY(mresid(A, k, mode, st));
    if (mode == 1) {
      PCG_CUDA(cudaMemcpyAsync(h, w.msc, sizeof(MultiScalars), cudaMemcpyDeviceToHost, st));
      PCG_CUDA(cudaStreamSynchronize(st));
      if (h->n_active == 0) break;
    }
    PCG_CUDA(cudaGraphLaunch(w.mloop_exec, st));
    mtail_kernel<<<gv, BLOCK, 0, st>>>(n, v, w.msc);
    mclear_xpend_kernel<<<1, 1, 0, st>>>(w.msc);
    count_launch(2);
    PCG_CUDA(cudaGetLastError());
    mode = 1;
  }
  PCG_CUDA(cudaEventRecord(e1, st));
  mzero_rhs_kernel<<<gv, BLOCK, 0, st>>>(n, v, w.msc);
  count_launch();
  const double *xsrc = w.mx;
  if (A->d_perm) {  // X = P^T X'
    PCG_TRY(perm_out_cols(A, k, w.mx, ld, w.mw, ld, st));
    xsrc = w.mw;
  }
  PCG_CUDA(cudaMemcpy2DAsync(X, sizeof(double) * ldx, xsrc, sizeof(double) * ld, sizeof(double) * n, k,
                             xd ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  g_host_launches += (int64_t)h->graph_launches;
  pcg_status worst = PCG_OK;
  long long kmax = 0;
  for (int c = 0; c < k; c++) kmax = std::max(kmax, h->k[c]);
  for (int c = 0; c < k; c++) {
    pcg_status s;
    switch (h->done[c]) {
      case DONE_CONVERGED: s = h->relres_true[c] <= tol ? PCG_OK : PCG_NOT_CONVERGED; break;
      case DONE_ZERO_RHS: s = PCG_OK; break;
      case DONE_BREAKDOWN: s = PCG_ERR_NOT_SPD; break;
      case DONE_NONFINITE: s = PCG_ERR_NONFINITE; break;
      default: s = PCG_NOT_CONVERGED; break;
    }
    if (s > worst) worst = s;
    if (infos) {
      pcg_info &I = infos[c];
      memset(&I, 0, sizeof(I));
      I.iterations = h->k[c];
      I.replacements = h->nrep[c];
      I.relres_recurrence = h->relres_rec[c];
      I.relres_true = h->done[c] == DONE_ZERO_RHS ? 0.0 : h->relres_true[c];
      I.converged = s == PCG_OK;
      I.status = s;
      I.t_solve_s = ms * 1e-3;
      const double nn = (double)n, nz = (double)A->nnz;
      // the matrix pass is shared: per block iteration 12 nnz + 4(n+1), attributed 1/k per
      // column, plus 96 n per column iteration (SURVEY §8(d), 3-pass schedule)
      I.bytes_algorithmic = (double)kmax * (12.0 * nz + 4.0 * (nn + 1)) / k + (double)h->k[c] * (96.0 - (mxdefer(A) == 4 ? 6.0 : mxdefer(A) == 2 ? 4.0 : 0.0)) * nn;
      I.flops = (double)h->k[c] * (2.0 * nz + 13.0 * nn);
    }
  }
  if (worst != PCG_OK) set_error(std::string("pcg_solve_multi: worst column status ") + pcg_status_string(worst));
  return worst;
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_profile_multi(pcg_matrix_t A, int32_t k, const double *B, int64_t ldb, int32_t reps,
                                        void *stream, double *us, int32_t *reps_done) {
  if (!A || !B || !us || reps < 1 || k < 1 || k > KMAX || ldb < A->n)
    return fail(PCG_ERR_INVALID_ARG, "pcg_profile_multi: bad argument");
  if (A->comm) return fail(PCG_ERR_INVALID_ARG, "pcg_profile_multi: single-GPU handles only");
  if (!is_device_ptr(B)) return fail(PCG_ERR_INVALID_ARG, "pcg_profile_multi: B must be a device pointer");
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  cudaStream_t st = (cudaStream_t)stream;
  PCG_TRY(multi_prepare(A, k, st));
  PCG_TRY(ensure_mdir(A, k, mxdefer(A)));
  SolveWork &w = A->work;
  const int64_t n = A->n, ld = mld(n);
  PCG_CUDA(cudaMemcpy2DAsync(A->d_perm ? w.mw : w.mb, sizeof(double) * ld, B, sizeof(double) * ldb,
                             sizeof(double) * n, k, cudaMemcpyDeviceToDevice, st));
  if (A->d_perm) PCG_TRY(perm_in_cols(A, k, w.mw, ld, w.mb, ld, st));
  PCG_CUDA(cudaMemsetAsync(w.mx, 0, sizeof(double) * ld * k, st));
  MultiScalars *h = w.h_msc;
  memset(h, 0, sizeof(MultiScalars));
  h->tol = 1e-300;  // never stops on the residual inside the profiled window
  h->max_iter = (long long)reps + 1;
  h->kcols = k;
  PCG_CUDA(cudaMemcpyAsync(w.msc, h, sizeof(MultiScalars), cudaMemcpyHostToDevice, st));
  PCG_TRY(mresid(A, k, 0, st));
  MVecs v = mvecs_of(A);
  const dim3 gv = mgrid_vec(A, k);
  std::vector<cudaEvent_t> ev(3 * (size_t)reps + 1);
  for (auto &e : ev) PCG_CUDA(cudaEventCreate(&e));
  PCG_CUDA(cudaEventRecord(ev[0], st));
  for (int r = 0; r < reps; r++) {
    const int pass = mxd_arg(mxdefer(A), r);
    mk1a_kernel<<<gv, BLOCK, 0, st>>>(n, v, w.msc, 0, 0, pass);
    PCG_CUDA(cudaEventRecord(ev[3 * r + 1], st));
    launch_mspmm<MS_SPMM>(A, k, st, 0, 0, pass);
    PCG_CUDA(cudaEventRecord(ev[3 * r + 2], st));
    mk2_kernel<<<gv, BLOCK, 0, st>>>(n, v, w.msc, mpart_rz(A), 0, 0, w.dslice);
    PCG_CUDA(cudaEventRecord(ev[3 * r + 3], st));
    count_launch(3);
  }
  PCG_CUDA(cudaStreamSynchronize(st));
  PCG_CUDA(cudaGetLastError());
  PCG_CUDA(cudaMemcpy(h, w.msc, sizeof(MultiScalars), cudaMemcpyDeviceToHost));
  long long kmin = reps;
  for (int c = 0; c < k; c++) kmin = std::min(kmin, h->k[c]);
  const int done = (int)kmin;
  double t[3] = {0, 0, 0};
  for (int r = 0; r < done; r++)
    for (int q = 0; q < 3; q++) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[3 * r + q], ev[3 * r + q + 1]);
      t[q] += ms;
    }
  for (auto &e : ev) cudaEventDestroy(e);
  for (int q = 0; q < 3; q++) us[q] = done ? t[q] * 1e3 / done : 0.0;
  if (reps_done) *reps_done = done;
  return PCG_OK;
}

extern "C" pcg_status pcg_solve_multi(pcg_matrix_t A, int32_t k, const double *B, int64_t ldb, double *X,
                                      int64_t ldx, double tol, int64_t max_iter, void *stream, pcg_info *infos) {
  pcgb::NvtxRange nvtx_("pcg:pcg_solve_multi");
  if (!A || !B || !X) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: null argument");
  if (k < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: k must be >= 1");
  if (ldb < A->n || ldx < A->n) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: ld < n");
  if (!(tol > 0.0) || max_iter < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: tol > 0, max_iter >= 1");
  if (A->comm) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: distributed handles take one RHS per solve");
  if (A->n == 0) {
    for (int c = 0; c < k && infos; c++) {
      memset(&infos[c], 0, sizeof(pcg_info));
      infos[c].converged = 1;
    }
    return PCG_OK;
  }
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  pcg_status worst = PCG_OK;
  for (int c0 = 0; c0 < k; c0 += KMAX) {
    const int kc = std::min(KMAX, k - c0);
    pcg_status s = solve_multi_chunk(A, kc, B + (size_t)c0 * ldb, ldb, X + (size_t)c0 * ldx, ldx, tol, max_iter,
                                     (cudaStream_t)stream, infos ? infos + c0 : nullptr);
    if (s >= PCG_ERR_INVALID_ARG) return s;
    if (s > worst) worst = s;
  }
  return worst;
}
