// solver.cu — fused Jacobi-PCG kernels and the single-RHS driver.
//
// The recurrence is SURVEY §8(c).8 (the reading of P:69-75 + P:132-135 listed
// in DESIGN.md §3).  It runs as TWO fused passes per iteration (the "2-kernel
// schedule"), each ending in a deterministic last-block
// grid reduction that also evaluates the scalar recurrence on the device:
//
//   K1 (pass A, after beta_{k-1} is known), per row i:
//        p_k[i]  = z[i] + beta_{k-1} p_{k-1}[i]        (own row, written)
//        q[i]    = Σ_j a_ij (z[j] + beta_{k-1} p_{k-1}[j])   (p_k recomputed at gather time)
//        x[i]   += alpha_{k-1} p_{k-1}[i]              (deferred x update)
//        sigma  += p_k[i] q[i]            -> finisher: alpha_k = rho/sigma, k++
//   K2 (pass B, after alpha_k is known), per row i:
//        r[i] -= alpha_k q[i];  z[i] = dinv[i] r[i]
//        rho' += r z;  gamma += r r       -> finisher: stop test sqrt(gamma) <= tol*||b||,
//                                            beta = rho'/rho
//
// HBM bytes per iteration: matrix once + 48n (K1: z, p, x in; p, q, x out) +
// 40n (K2: r, q, dinv in; r, z out) = 12 nnz + 4(n+1) + 88 n.
// The loop runs inside ONE CUDA graph launch: a conditional WHILE node whose
// body is {K1, K2}; the finishers clear the condition when the solve stops.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <vector>

#include "matrix.cuh"
#include "rows.cuh"
#include "staged.cuh"

namespace pcgb {

enum { MODE_INIT = 0, MODE_EXIT = 1 };


__device__ __forceinline__ void stop_loop(int use_cond, cudaGraphConditionalHandle h) {
  if (use_cond) cudaGraphSetConditional(h, 0);
}

// ---------------------------------------------------------------- finishers
// xd (deferred x update, k1a_kernel): 0 = off, else (M << 4) | j — pass j of an
// M-cycle (M = 2 or 4): passes 0..M-2 "hold" (their K1a wrote p_k to p[j+1] and left
// the owed alpha p of the direction in p[j] to x), pass M-1 "applies" (x current up to
// alpha_{k-1}, p_k in p[0]).  Scalars: ahold[0..xhold-1] the held alphas (directions
// p[0..xhold-1]), parity the buffer of the latest direction.
__device__ __forceinline__ int xd_m(int xd) { return xd >> 4; }
__device__ __forceinline__ int xd_j(int xd) { return xd & 15; }

__device__ void finish_alpha(Scalars *sc, double sigma, int use_cond, cudaGraphConditionalHandle h, int flip = 1,
                             int xd = 0) {
  const int xm = xd_m(xd), xj = xd_j(xd);
  const bool hold = xm && xj < xm - 1;
  sc->sigma = sigma;
  if (!(sigma > 0.0)) {  // p^T A p <= 0 (or NaN): CG breakdown, A not SPD
    sc->done = DONE_BREAKDOWN;
    stop_loop(use_cond, h);
    if (hold) {  // alpha_{k-1} p_{k-1} (in p[j]) is still owed: the tail applies it
      sc->ahold[xj] = sc->alpha;  // pass j holds direction j (xhold == j before)
      sc->xhold = xj + 1;
      sc->alpha = 0.0;
      sc->parity = xj + 1;
    } else if (xm) {  // an apply pass: this iteration's K1a applied everything owed
      sc->xhold = 0;
    }
  } else {
    if (hold) {
      sc->ahold[xj] = sc->alpha;
      sc->xhold = xj + 1;
      sc->parity = xj + 1;
    } else if (xm) {
      sc->xhold = 0;
      sc->parity = 0;
    }
    sc->alpha = sc->rho / sigma;
    sc->k += 1;
    sc->parity ^= flip;
  }
  sc->graph_launches += use_cond;
}

__device__ void finish_beta(Scalars *sc, double rho_new, double gamma, int use_cond,
                            cudaGraphConditionalHandle h) {
  sc->gamma = gamma;
  const double rr = sqrt(gamma);
  sc->relres_rec = rr / sc->nb;
  if (rr <= sc->tol * sc->nb) {
    sc->done = DONE_CONVERGED;
    stop_loop(use_cond, h);
  } else if (!(gamma == gamma)) {
    sc->done = DONE_NONFINITE;
    stop_loop(use_cond, h);
  } else if (sc->k >= sc->max_iter) {
    sc->done = DONE_MAXIT;
    stop_loop(use_cond, h);
  } else {
    sc->beta = rho_new / sc->rho;
    sc->rho = rho_new;
  }
  sc->graph_launches += use_cond;
}

// ---------------------------------------------------------------- K1: SpMV + p update + x update + sigma
// (SELL-32 row engine k1_sell_rows: rows.cuh)
template <int FMT, int L, int CH = 8>
__global__ void __launch_bounds__(BLOCK) k1_kernel(SellView S, CsrView C, int64_t n_ghost, Vecs v,
                                                   Scalars *sc, double *partials, int dist,
                                                   int use_cond, cudaGraphConditionalHandle h) {
  __shared__ double sm[1][WARPS];
  const volatile Scalars *vs = sc;
  if (vs->done != DONE_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) stop_loop(use_cond, h);
    return;
  }
  const double beta = vs->beta, alpha_prev = vs->alpha;
  const int par = vs->parity;
  const double *__restrict__ pold = par ? v.p1 : v.p0;
  double *__restrict__ pnew = par ? v.p0 : v.p1;
  const double *__restrict__ z = v.z;
  double *__restrict__ x = v.x;
  double *__restrict__ q = v.q;
  double acc = 0.0;
  if (FMT == FMT_SELL_TMA) {
    struct Own {
      double po, zi;
    };
    StageIO<1, 2> io;
    io.own[0] = x;
    io.pf[0] = pold;
    io.pf[1] = z;
    io.pf_len = S.n + n_ghost;
    auto pre = [&](int64_t i) { return Own{__ldg(pold + i), __ldg(z + i)}; };
    auto gather = [&](int j) { return __fma_rn(beta, __ldg(pold + j), __ldg(z + j)); };
    auto epi = [&](int64_t i, double s, const Own &o, const double *own) {
      const double pi = __fma_rn(beta, o.po, o.zi);
      __stcs(pnew + i, pi);
      __stcs(q + i, s);
      __stcs(x + i, __fma_rn(alpha_prev, o.po, own[0]));
      acc = __fma_rn(pi, s, acc);
    };
    sell_staged_rows<CH>(S, io, pre, gather, epi);
  } else if (FMT == PCG_FORMAT_SELL) {
    k1_sell_rows<CH>(S, beta, alpha_prev, pold, pnew, z, x, q, acc);
  } else {
    auto gather = [&](int j) { return __fma_rn(beta, __ldg(pold + j), __ldg(z + j)); };
    auto epi = [&](int64_t i, double s) {
      const double po = pold[i];
      const double pi = __fma_rn(beta, po, z[i]);
      pnew[i] = pi;
      q[i] = s;
      x[i] = __fma_rn(alpha_prev, po, x[i]);
      acc = __fma_rn(pi, s, acc);
    };
    csr_rows<L>(C, gather, epi);
  }
  // ghost copies of p advance by the same recurrence (bitwise equal to the owner's)
  if (n_ghost) {
    const int64_t n = FMT != PCG_FORMAT_CSR ? S.n : C.n;
    for (int64_t g = (int64_t)blockIdx.x * BLOCK + threadIdx.x; g < n_ghost; g += (int64_t)gridDim.x * BLOCK)
      pnew[n + g] = __fma_rn(beta, pold[n + g], z[n + g]);
  }
  double red[1] = {acc};
  block_sum<1>(red, sm);
  if (publish_and_arrive<1>(red, partials, &sc->cnt_a)) {
    double tot[1];
    reduce_partials<1>(partials, tot, sm);
    if (threadIdx.x == 0) {
      sc->cnt_a = 0;
      if (dist) {
        sc->sigma = tot[0];  // local partial; allreduce + finish_alpha_kernel follow
        sc->graph_launches += use_cond;
      } else {
        finish_alpha(sc, tot[0], use_cond, h);
      }
    }
  }
}

// ---------------------------------------------------------------- K2: r, z updates + rho', gamma
#ifndef PCG_K2_UNROLL  // element pairs per thread and trip in K2 (A/B knob: 1 or 2)
#define PCG_K2_UNROLL 1
#endif
__global__ void __launch_bounds__(BLOCK) k2_kernel(int64_t n, Vecs v, Scalars *sc, double *partials,
                                                   int dist, int use_cond, cudaGraphConditionalHandle h,
                                                   const double *__restrict__ dsl, int zlazy) {
  __shared__ double sm[2][WARPS];
  const volatile Scalars *vs = sc;
  if (vs->done != DONE_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) stop_loop(use_cond, h);
    return;
  }
  const double alpha = vs->alpha;
  double a0 = 0.0, a1 = 0.0;
  const int64_t npair = n >> 1;
  const double2 *__restrict__ q2 = reinterpret_cast<const double2 *>(v.q);
  const double2 *__restrict__ d2 = reinterpret_cast<const double2 *>(v.dinv);
  double2 *__restrict__ r2 = reinterpret_cast<double2 *>(v.r);
  double2 *__restrict__ z2 = reinterpret_cast<double2 *>(v.z);
  // a slice with one common dinv (SolveWork::dslice): 8 bytes per 32 rows, the same values
  auto dinv2 = [&](int64_t i, double du) { return du == du ? make_double2(du, du) : __ldg(d2 + i); };
  auto step = [&](double2 qq, double2 rr, double2 dd, int64_t i) {
    rr.x = __fma_rn(-alpha, qq.x, rr.x);
    rr.y = __fma_rn(-alpha, qq.y, rr.y);
    const double2 zz = make_double2(dd.x * rr.x, dd.y * rr.y);
    r2[i] = rr;
    if (!zlazy) z2[i] = zz;  // (lazy: K1a forms z from r; the odd tail row below stores it)
    a0 = __fma_rn(rr.x, zz.x, a0);
    a0 = __fma_rn(rr.y, zz.y, a0);
    a1 = __fma_rn(rr.x, rr.x, a1);
    a1 = __fma_rn(rr.y, rr.y, a1);
  };
  const double nan = __longlong_as_double(0x7ff8000000000000ll);
  const int64_t st = (int64_t)gridDim.x * BLOCK;
  int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  // PCG_K2_UNROLL pairs per trip, every load issued first (the same element order per
  // thread, so the same sums)
  for (; PCG_K2_UNROLL == 2 && i + st < npair; i += 2 * st) {
    const double2 qa = __ldcs(q2 + i), qb = __ldcs(q2 + i + st);
    const double2 ra = r2[i], rb = r2[i + st];
    const double ua = dsl ? __ldg(dsl + (i >> 4)) : nan, ub = dsl ? __ldg(dsl + ((i + st) >> 4)) : nan;
    const double2 da = dinv2(i, ua), db = dinv2(i + st, ub);
    step(qa, ra, da, i);
    step(qb, rb, db, i + st);
  }
  for (; i < npair; i += st) {
    const double2 qq = __ldcs(q2 + i), rr = r2[i];
    const double du = dsl ? __ldg(dsl + (i >> 4)) : nan;
    step(qq, rr, dinv2(i, du), i);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t i = n - 1;
    const double ri = __fma_rn(-alpha, v.q[i], v.r[i]);
    const double zi = v.dinv[i] * ri;
    v.r[i] = ri;
    v.z[i] = zi;
    a0 = __fma_rn(ri, zi, a0);
    a1 = __fma_rn(ri, ri, a1);
  }
  double red[2] = {a0, a1};
  block_sum<2>(red, sm);
  if (publish_and_arrive<2>(red, partials, &sc->cnt_b)) {
    double tot[2];
    reduce_partials<2>(partials, tot, sm);
    if (threadIdx.x == 0) {
      sc->cnt_b = 0;
      if (dist) {
        sc->rho_part[0] = tot[0];
        sc->rho_part[1] = tot[1];
        sc->graph_launches += use_cond;
      } else {
        finish_beta(sc, tot[0], tot[1], use_cond, h);
      }
    }
  }
}

// ---------------------------------------------------------------- 3-pass schedule
// K1a (streaming): p = z + beta p ; x += alpha_prev p_old   (reads z, p, x; writes p, x: 40n B)
// K1b (SpMV):      q = A p ; sigma = p.q -> alpha           (matrix + 16n B)
// K2  (as above):  r, z updates + rho', gamma -> beta       (40n B)
// 96n + matrix bytes per iteration, every pass a plain streaming or SpMV pass.
//
// Deferred x update (the graph loops; SURVEY §8(d) bytes): x is needed only at the exit
// check, so over a cycle of M iterations (M = 2 or 4) K1a runs M - 1 "hold" passes
//   pass j < M-1:  p[j+1] = z + beta p[j]; x untouched               (reads z, p: 24n B)
// and one "apply" pass
//   pass M-1:      x = fma(alpha_k, p[M-1], fma(alpha_h[M-2], p[M-2], ... fma(alpha_h[0], p[0], x)))
//                  p[0] = z + beta p[M-1]                  (reads z, M directions, x: 8(M+2)n B)
// M = 2: 36n, M = 4: 34n per iteration instead of 40n, and the SAME fused multiply-adds
// in the same order as the every-iteration update (oldest direction first), so x is
// bitwise the same.  The tail applies what a stop leaves owed (Scalars::xhold, ahold).
__device__ __forceinline__ double *dir_buf(const Vecs &v, int b) {
  return b == 0 ? v.p0 : b == 1 ? v.p1 : b == 2 ? v.p2 : v.p3;
}

// z = dinv r of the pair i.  Where every slice shares one dinv (SolveWork::dslice_all,
// one GPU, 3-pass schedule: `zl` non-null) K2 stores no z and K1a forms it from r and the
// slice's dinv — the same product, so bitwise the stored z.
template <bool LAZY>
__device__ __forceinline__ double2 z_pair(const Vecs &v, const double *__restrict__ zl, int64_t i) {
  if (LAZY) {
    const double du = __ldg(zl + (i >> 4));
    const double2 rr = __ldcs(reinterpret_cast<const double2 *>(v.r) + i);
    return make_double2(du * rr.x, du * rr.y);
  }
  return __ldcs(reinterpret_cast<const double2 *>(v.z) + i);
}

template <int M, bool LAZY>
__device__ __forceinline__ void k1a_apply(int64_t n, int64_t n_ghost, const Vecs &v, double beta, double alpha,
                                          const volatile double *ahold, const double *__restrict__ zl) {
  const int64_t npair = n >> 1;
  const int64_t t = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nt = (int64_t)gridDim.x * BLOCK;
  double ah[M - 1];
#pragma unroll
  for (int h = 0; h < M - 1; h++) ah[h] = ahold[h];
  const double2 *__restrict__ z2 = reinterpret_cast<const double2 *>(v.z);
  const double2 *hb[M - 1];
#pragma unroll
  for (int h = 0; h < M - 1; h++) hb[h] = reinterpret_cast<const double2 *>(dir_buf(v, h));
  const double2 *__restrict__ l2 = reinterpret_cast<const double2 *>(dir_buf(v, M - 1));
  double2 *__restrict__ a2 = reinterpret_cast<double2 *>(v.p0);
  double2 *__restrict__ x2 = reinterpret_cast<double2 *>(v.x);
  for (int64_t i = t; i < npair; i += nt) {
    const double2 zz = z_pair<LAZY>(v, zl, i), pk = l2[i];
    double2 pm[M - 1];
#pragma unroll
    for (int h = 0; h < M - 1; h++) pm[h] = __ldcs(hb[h] + i);
    double2 xx = __ldcs(x2 + i);
#pragma unroll
    for (int h = 0; h < M - 1; h++) {
      xx.x = __fma_rn(ah[h], pm[h].x, xx.x);
      xx.y = __fma_rn(ah[h], pm[h].y, xx.y);
    }
    xx.x = __fma_rn(alpha, pk.x, xx.x);
    xx.y = __fma_rn(alpha, pk.y, xx.y);
    a2[i] = make_double2(__fma_rn(beta, pk.x, zz.x), __fma_rn(beta, pk.y, zz.y));
    __stcs(x2 + i, xx);
  }
  const double *pl = dir_buf(v, M - 1);
  if ((n & 1) && t == 0) {
    const int64_t i = n - 1;
    double xi = v.x[i];
#pragma unroll
    for (int h = 0; h < M - 1; h++) xi = __fma_rn(ah[h], dir_buf(v, h)[i], xi);
    v.x[i] = __fma_rn(alpha, pl[i], xi);
    v.p0[i] = __fma_rn(beta, pl[i], v.z[i]);
  }
  for (int64_t g = t; g < n_ghost; g += nt) v.p0[n + g] = __fma_rn(beta, pl[n + g], v.z[n + g]);
}

template <bool LAZY>
__device__ __forceinline__ void k1a_hold(int64_t n, int64_t n_ghost, const Vecs &v, double beta, int j,
                                         const double *__restrict__ zl) {
  const int64_t npair = n >> 1;
  const int64_t t = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nt = (int64_t)gridDim.x * BLOCK;
  const double *src = dir_buf(v, j);
  double *dst = dir_buf(v, j + 1);
  const double2 *__restrict__ z2 = reinterpret_cast<const double2 *>(v.z);
  const double2 *__restrict__ a2 = reinterpret_cast<const double2 *>(src);
  double2 *__restrict__ b2 = reinterpret_cast<double2 *>(dst);
  for (int64_t i = t; i < npair; i += nt) {
    const double2 zz = z_pair<LAZY>(v, zl, i), po = __ldcs(a2 + i);
    b2[i] = make_double2(__fma_rn(beta, po.x, zz.x), __fma_rn(beta, po.y, zz.y));
  }
  if ((n & 1) && t == 0) dst[n - 1] = __fma_rn(beta, src[n - 1], v.z[n - 1]);
  for (int64_t g = t; g < n_ghost; g += nt) dst[n + g] = __fma_rn(beta, src[n + g], v.z[n + g]);
}

template <bool LAZY>
__global__ void __launch_bounds__(BLOCK, 4) k1a_kernel(int64_t n, int64_t n_ghost, Vecs v, Scalars *sc, int use_cond,
                                                    cudaGraphConditionalHandle h, int xd,
                                                    const double *__restrict__ zl = nullptr) {
  const volatile Scalars *vs = sc;
  if (vs->done != DONE_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) stop_loop(use_cond, h);
    return;
  }
  const double beta = vs->beta, alpha_prev = vs->alpha;
  if (xd) {
    const int xm = xd_m(xd), xj = xd_j(xd);
    if (xj < xm - 1) k1a_hold<LAZY>(n, n_ghost, v, beta, xj, zl);
    else if (xm == 4) k1a_apply<4, LAZY>(n, n_ghost, v, beta, alpha_prev, vs->ahold, zl);
    else k1a_apply<2, LAZY>(n, n_ghost, v, beta, alpha_prev, vs->ahold, zl);
    return;
  }
  double *__restrict__ p = v.p0;
  const int64_t npair = n >> 1;
  const double2 *__restrict__ z2 = reinterpret_cast<const double2 *>(v.z);
  double2 *__restrict__ p2 = reinterpret_cast<double2 *>(p);
  double2 *__restrict__ x2 = reinterpret_cast<double2 *>(v.x);
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < npair; i += (int64_t)gridDim.x * BLOCK) {
    const double2 zz = z_pair<LAZY>(v, zl, i), po = p2[i];
    double2 xx = __ldcs(x2 + i);
    xx.x = __fma_rn(alpha_prev, po.x, xx.x);
    xx.y = __fma_rn(alpha_prev, po.y, xx.y);
    p2[i] = make_double2(__fma_rn(beta, po.x, zz.x), __fma_rn(beta, po.y, zz.y));
    __stcs(x2 + i, xx);
  }
  const int64_t t = (int64_t)blockIdx.x * BLOCK + threadIdx.x;
  if ((n & 1) && t == 0) {
    const double po = p[n - 1];
    v.x[n - 1] = __fma_rn(alpha_prev, po, v.x[n - 1]);
    p[n - 1] = __fma_rn(beta, po, v.z[n - 1]);
  }
  for (int64_t g = t; g < n_ghost; g += (int64_t)gridDim.x * BLOCK) p[n + g] = __fma_rn(beta, p[n + g], v.z[n + g]);
}

template <int FMT, int L>
// row0/phase: the distributed overlap runs K1b over row ranges (views offset by row0);
// phase 1 starts p.q (sigma_acc = local), 3 adds to it, 2 completes it (sigma = acc + local)
__global__ void __launch_bounds__(BLOCK, D16_MINB(FMT)) k1b_kernel(SellViewDia S, CsrView C, int64_t n_ghost, Vecs v, Scalars *sc,
                                                    double *partials, int dist, int use_cond,
                                                    cudaGraphConditionalHandle h, int64_t row0, int phase,
                                                    int xdefer) {
  __shared__ double sm[1][WARPS];
  const volatile Scalars *vs = sc;
  if (vs->done != DONE_RUNNING) {
    if (blockIdx.x == 0 && threadIdx.x == 0) stop_loop(use_cond, h);
    return;
  }
  const double *__restrict__ p = v.p0;
  double *__restrict__ q = v.q + row0;
  const double *__restrict__ pr = v.p0 + row0;
  double acc = 0.0;
  auto gather = [&](int j) { return __ldg(p + j); };
  auto epi = [&](int64_t i, double s) {
    __stcs(q + i, s);
    acc = __fma_rn(__ldg(pr + i), s, acc);
  };
  if (FMT == FMT_SELL_TMA) {
    StageIO<0, 1> io;
    io.pf[0] = p;
    io.pf_len = S.n + n_ghost;
    auto pre = [&](int64_t) { return 0; };
    auto epi2 = [&](int64_t i, double s, int, const double *) { epi(i, s); };
    sell_staged_rows<8>(S, io, pre, gather, epi2);
  } else if (FMT == PCG_FORMAT_SELL) {
    sell_rows(S, gather, epi);
  } else if (FMT == FMT_SELL_D16) {
    sell_rows_d16(S, gather, epi);
  } else if (FMT == FMT_SELL_SHORT) {
    sell_rows_short(S, gather, epi);
  } else if (FMT == FMT_SELL_DIA) {
    sell_rows_dia(S, gather, epi);
  } else {
    csr_rows<L>(C, gather, epi);
  }
  double red[1] = {acc};
  block_sum<1>(red, sm);
  if (publish_and_arrive<1>(red, partials, &sc->cnt_a)) {
    double tot[1];
    reduce_partials<1>(partials, tot, sm);
    if (threadIdx.x == 0) {
      sc->cnt_a = 0;
      if (phase == 1) {
        sc->sigma_acc = tot[0];
      } else if (phase == 3) {
        sc->sigma_acc += tot[0];
      } else if (phase == 2) {
        sc->sigma = sc->sigma_acc + tot[0];
      } else if (dist) {
        sc->sigma = tot[0];
        sc->graph_launches += use_cond;
      } else {
        finish_alpha(sc, tot[0], use_cond, h, 0, xdefer);
      }
    }
  }
}

// distributed overlap: ghost copies of p advance once the z halo has arrived
// (deferred x update: a hold iteration advances p[0] -> p[1], an apply iteration p[1] -> p[0])
__global__ void __launch_bounds__(BLOCK) ghost_p_kernel(int64_t n, int64_t n_ghost, Vecs v, const Scalars *sc,
                                                        int xd) {
  const volatile Scalars *vs = sc;
  if (vs->done != DONE_RUNNING) return;
  const double beta = vs->beta;
  const int xm = xd_m(xd), xj = xd_j(xd);
  const double *src = !xm ? v.p0 : dir_buf(v, xj < xm - 1 ? xj : xm - 1);
  double *dst = !xm ? v.p0 : dir_buf(v, xj < xm - 1 ? xj + 1 : 0);
  for (int64_t g = (int64_t)blockIdx.x * BLOCK + threadIdx.x; g < n_ghost; g += (int64_t)gridDim.x * BLOCK)
    dst[n + g] = __fma_rn(beta, src[n + g], v.z[n + g]);
}

// distributed finishers (after the NCCL allreduce of the partials)
__global__ void finish_alpha_kernel(Scalars *sc, int use_cond, cudaGraphConditionalHandle h, int flip, int xdefer) {
  if (sc->done != DONE_RUNNING) return;
  finish_alpha(sc, sc->sigma, use_cond, h, flip, xdefer);
}
__global__ void finish_beta_kernel(Scalars *sc, int use_cond, cudaGraphConditionalHandle h) {
  if (sc->done != DONE_RUNNING) return;
  finish_beta(sc, sc->rho_part[0], sc->rho_part[1], use_cond, h);
}

// ---------------------------------------------------------------- residual (init / exit check / replacement)
// w = b - A x; r = w; z = dinv w; p[parity] = 0; partial sums (w.w, w.z, b.b).
template <int FMT, int L>
__global__ void __launch_bounds__(BLOCK, D16_MINB(FMT)) resid_kernel(SellViewDia S, CsrView C, int64_t n_ghost,
                                                      const double *__restrict__ b, Vecs v, Scalars *sc,
                                                      double *partials, int mode, int dist) {
  __shared__ double sm[3][WARPS];
  const int par = sc->parity;
  double *__restrict__ pz = par ? v.p1 : v.p0;
  const double *__restrict__ x = v.x;
  double ww = 0.0, wz = 0.0, bb = 0.0;
  auto gather = [&](int j) { return __ldg(x + j); };
  auto epi = [&](int64_t i, double s) {
    const double bi = b[i];
    const double wi = bi - s;
    const double zi = v.dinv[i] * wi;
    v.r[i] = wi;
    v.z[i] = zi;
    pz[i] = 0.0;
    ww = __fma_rn(wi, wi, ww);
    wz = __fma_rn(wi, zi, wz);
    bb = __fma_rn(bi, bi, bb);
  };
  if (FMT == FMT_SELL_TMA) {
    StageIO<0, 1> io;
    io.pf[0] = x;
    io.pf_len = S.n + n_ghost;
    auto pre = [&](int64_t i) { return b[i]; };
    auto epi2 = [&](int64_t i, double s, double, const double *) { epi(i, s); };
    sell_staged_rows<8>(S, io, pre, gather, epi2);
  } else if (FMT == PCG_FORMAT_SELL) {
    sell_rows(S, gather, epi);
  } else if (FMT == FMT_SELL_D16) {
    sell_rows_d16(S, gather, epi);
  } else if (FMT == FMT_SELL_SHORT) {
    sell_rows_short(S, gather, epi);
  } else if (FMT == FMT_SELL_DIA) {
    sell_rows_dia(S, gather, epi);
  } else {
    csr_rows<L>(C, gather, epi);
  }
  if (n_ghost) {
    const int64_t n = FMT != PCG_FORMAT_CSR ? S.n : C.n;
    for (int64_t g = (int64_t)blockIdx.x * BLOCK + threadIdx.x; g < n_ghost; g += (int64_t)gridDim.x * BLOCK)
      pz[n + g] = 0.0;
  }
  double red[3] = {ww, wz, bb};
  block_sum<3>(red, sm);
  if (publish_and_arrive<3>(red, partials, &sc->cnt_c)) {
    double tot[3];
    reduce_partials<3>(partials, tot, sm);
    if (threadIdx.x == 0) {
      sc->cnt_c = 0;
      sc->res_part[0] = tot[0];
      sc->res_part[1] = tot[1];
      sc->res_part[2] = tot[2];
    }
  }
}

// scalar logic of init / exit (after any allreduce of res_part)
__global__ void resid_finish_kernel(Scalars *sc, int mode) {
  const double ww = sc->res_part[0], wz = sc->res_part[1], bb = sc->res_part[2];
  if (mode == MODE_INIT) {
    sc->k = 0;
    sc->replacements = 0;
    sc->alpha = 0.0;
    sc->beta = 0.0;
    sc->relres_true = 0.0;
    if (!isfinite(bb) || !isfinite(ww)) {
      sc->done = DONE_NONFINITE;
      return;
    }
    sc->nb = sqrt(bb);
    if (sc->nb == 0.0) {
      sc->done = DONE_ZERO_RHS;
      return;
    }
    const double rr = sqrt(ww);
    sc->relres_rec = rr / sc->nb;
    if (rr <= sc->tol * sc->nb) {
      sc->done = DONE_CONVERGED;
    } else {
      sc->done = DONE_RUNNING;
      sc->rho = wz;
    }
  } else {
    sc->relres_true = sqrt(ww) / sc->nb;
    if (sc->done == DONE_CONVERGED && !(sc->relres_true <= sc->tol)) {
      if (sc->k >= sc->max_iter) {
        sc->done = DONE_MAXIT;
      } else {  // residual replacement: r = b - Ax, z = dinv r, p = z (beta = 0), rho = r.z
        sc->done = DONE_RUNNING;
        sc->rho = wz;
        sc->alpha = 0.0;
        sc->beta = 0.0;
        sc->replacements += 1;
      }
    }
  }
}

// deferred x += alpha_k p_k after the loop stops on the recurrence or max_iter
// x += alpha_k p_k still owed at a stop (converged / max_iter), after the held
// directions of the deferred update (oldest first), in the order the loop applies them
__global__ void tail_kernel(int64_t n, Vecs v, const Scalars *sc) {
  const int done = sc->done;
  const double alpha = sc->alpha;
  const bool last = (done == DONE_CONVERGED || done == DONE_MAXIT) && alpha != 0.0;
  const int nh = sc->xhold;
  if (!last && nh == 0) return;
  double ah[3];
  for (int h = 0; h < 3; h++) ah[h] = sc->ahold[h];
  const double *p = dir_buf(v, sc->parity);
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    double xi = v.x[i];
    for (int h = 0; h < nh; h++) xi = __fma_rn(ah[h], dir_buf(v, h)[i], xi);
    if (last) xi = __fma_rn(alpha, p[i], xi);
    v.x[i] = xi;
  }
}
// after the tail: nothing owed; the deferred loop restarts (replacement) with p in p[0]
__global__ void clear_alpha_kernel(Scalars *sc, int xdefer) {
  sc->alpha = 0.0;
  for (int h = 0; h < 3; h++) sc->ahold[h] = 0.0;
  sc->xhold = 0;
  if (xdefer) sc->parity = 0;
}

// ---------------------------------------------------------------- standalone SpMV  y = A x
template <int FMT, int L>
__global__ void __launch_bounds__(BLOCK, D16_MINB(FMT)) spmv_kernel(SellViewDia S, CsrView C, const double *__restrict__ x,
                                                     double *__restrict__ y, int64_t x_len) {
  auto gather = [&](int j) { return __ldg(x + j); };
  auto epi = [&](int64_t i, double s) { __stcs(y + i, s); };
  if (FMT == FMT_SELL_TMA) {
    StageIO<0, 1> io;
    io.pf[0] = x;
    io.pf_len = x_len;
    auto pre = [&](int64_t) { return 0; };
    auto epi2 = [&](int64_t i, double s, int, const double *) { __stcs(y + i, s); };
    sell_staged_rows<8>(S, io, pre, gather, epi2);
  } else if (FMT == PCG_FORMAT_SELL) {
    sell_rows(S, gather, epi);
  } else if (FMT == FMT_SELL_D16) {
    sell_rows_d16(S, gather, epi);
  } else if (FMT == FMT_SELL_SHORT) {
    sell_rows_short(S, gather, epi);
  } else if (FMT == FMT_SELL_DIA) {
    sell_rows_dia(S, gather, epi);
  } else {
    csr_rows<L>(C, gather, epi);
  }
}

// ---------------------------------------------------------------- launch helpers
template <template <int, int> class K>
struct Dispatch;

#define PCG_DISPATCH(FMTV, LANES, KERNEL, ...)                                   \
  do {                                                                           \
    if ((FMTV) == PCG_FORMAT_SELL) KERNEL<PCG_FORMAT_SELL, 1>__VA_ARGS__;        \
    else if ((FMTV) == FMT_SELL_TMA) KERNEL<FMT_SELL_TMA, 1>__VA_ARGS__;         \
    else switch (LANES) {                                                        \
        case 1: KERNEL<PCG_FORMAT_CSR, 1>__VA_ARGS__; break;                     \
        case 2: KERNEL<PCG_FORMAT_CSR, 2>__VA_ARGS__; break;                     \
        case 4: KERNEL<PCG_FORMAT_CSR, 4>__VA_ARGS__; break;                     \
        case 8: KERNEL<PCG_FORMAT_CSR, 8>__VA_ARGS__; break;                     \
        case 16: KERNEL<PCG_FORMAT_CSR, 16>__VA_ARGS__; break;                   \
        default: KERNEL<PCG_FORMAT_CSR, 32>__VA_ARGS__; break;                   \
      }                                                                          \
  } while (0)

// SELL-32 handles with 16-bit delta column ids run the D16 engine in the passes below
#define PCG_DISPATCH_D16(FMTV, LANES, KERNEL, ...)                          \
  do {                                                                      \
    if ((FMTV) == FMT_SELL_D16) KERNEL<FMT_SELL_D16, 1>__VA_ARGS__;         \
    else if ((FMTV) == FMT_SELL_SHORT) KERNEL<FMT_SELL_SHORT, 1>__VA_ARGS__; \
    else if ((FMTV) == FMT_SELL_DIA) KERNEL<FMT_SELL_DIA, 1>__VA_ARGS__;     \
    else PCG_DISPATCH(FMTV, LANES, KERNEL, __VA_ARGS__);                    \
  } while (0)

// the SELL row engine of a handle: 16-bit ids (opt-in), the one-chunk engine (rows of
// at most 8 entries), else the general chunked engine
static int fmt_d16(const pcg_matrix *A, int fmt) {
  if (fmt != PCG_FORMAT_SELL) return fmt;
  if (A->d_sdcol) return FMT_SELL_D16;
  return A->short_rows ? (A->d_sdoff ? FMT_SELL_DIA : FMT_SELL_SHORT) : fmt;
}

static Vecs vecs_of(pcg_matrix *A) {
  SolveWork &w = A->work;
  return Vecs{w.r, w.z, w.q, w.p[0], w.p[1], w.x, A->d_dinv, w.p23[0], w.p23[1]};
}

pcg_status launch_spmv_fmt(pcg_matrix *A, int fmt, const double *x, double *y, cudaStream_t st) {
  PCG_DISPATCH_D16(fmt_d16(A, fmt), A->csr_lanes, spmv_kernel,
                   <<<A->grid_spmv, BLOCK, A->dyn_smem, st>>>(A->sell_dia(), A->csr(), x, y, A->n + A->n_ghost));
  count_launch();
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

pcg_status launch_spmv(pcg_matrix *A, const double *x, double *y, cudaStream_t st) {
  return launch_spmv_fmt(A, A->format, x, y, st);
}

static int k1_chunk() {  // tuning knob (PCG_K1_CHUNK=4|8), default 8
  static int c = [] {
    const char *e = getenv("PCG_K1_CHUNK");
    return (e && atoi(e) == 4) ? 4 : 8;
  }();
  return c;
}

// the buffer holding the direction K1b multiplies in deferral pass xd (host side)
static double *k1b_dir(const Vecs &v, int xd) {
  const int m = xd >> 4, j = xd & 15;
  const int b = j < m - 1 ? j + 1 : 0;
  return b == 0 ? v.p0 : b == 1 ? v.p1 : b == 2 ? v.p2 : v.p3;
}

// K2 stores no z and K1a forms it from r where every slice shares one dinv (one GPU, the
// 3-pass schedule: no z halo, no gather of z; PCG_ZLAZY=0: off)
static int zlazy(const pcg_matrix *A) {
  static const int off = [] {
    const char *e = getenv("PCG_ZLAZY");
    return e && atoi(e) == 0;
  }();
  return !off && !A->comm && A->schedule == 3 && A->work.dslice && A->work.dslice_all ? 1 : 0;
}

static pcg_status launch_k1(pcg_matrix *A, cudaStream_t st, int use_cond, cudaGraphConditionalHandle h,
                            int xdefer = 0) {
  Vecs v = vecs_of(A);
  SolveWork &w = A->work;
  if (A->schedule == 3 && A->comm && A->ov) {
    // K1a (owned rows) + K1b over the interior rows on the side stream || the z halo on
    // the main stream (every NCCL call stays on one stream, in one order on all ranks);
    // after the join the ghost p update and K1b over the boundary rows (head, tail)
    PCG_CUDA(cudaEventRecord(A->ov_fork, st));
    PCG_CUDA(cudaStreamWaitEvent(A->ov_side, A->ov_fork, 0));
    k1a_kernel<false><<<A->grid_vec, BLOCK, 0, A->ov_side>>>(A->n, 0, v, w.sc, use_cond, h, xdefer);
    count_launch();
    Vecs vb = v;
    if (xdefer) vb.p0 = k1b_dir(v, xdefer);  // the direction this pass's K1a wrote
    struct Range {
      int64_t r0, r1;
    } rs[3] = {{A->ov_ia, A->ov_ib}, {0, A->ov_ia}, {A->ov_ib, A->n}};
    int last = rs[2].r1 > rs[2].r0 ? 2 : 1;
    for (int t = 0; t <= last; t++) {
      const Range R = rs[t];
      if (t == 1) {  // boundary rows need the ghosts: halo, join, advance ghost p
        PCG_CUDA(cudaEventRecord(A->ov_join, A->ov_side));
        PCG_TRY(halo_exchange(A, w.z, 1, st));
        PCG_CUDA(cudaStreamWaitEvent(st, A->ov_join, 0));
        ghost_p_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((A->n_ghost + BLOCK - 1) / BLOCK, 1184)),
                         BLOCK, 0, st>>>(A->n, A->n_ghost, v, w.sc, xdefer);
        count_launch();
      }
      if (R.r1 <= R.r0) continue;
      const int phase = t == 0 ? 1 : (t == last ? 2 : 3);
      SellViewDia S = A->sell_dia();
      CsrView Cv = A->csr();
      const int64_t s0 = R.r0 / 32, s1 = R.r1 == A->n ? A->n_slices : R.r1 / 32;
      S.slice_ptr += s0;
      S.row0 = s0 * 32;
      S.n_slices = s1 - s0;
      S.n = R.r1 - R.r0;
      Cv.row_ptr += R.r0;
      Cv.n = R.r1 - R.r0;
      const int64_t need = A->format == PCG_FORMAT_SELL ? (S.n_slices + WARPS - 1) / WARPS
                                                       : (Cv.n * A->csr_lanes + BLOCK - 1) / BLOCK;
      const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(A->grid_spmv, need));
      cudaStream_t ks = t == 0 ? A->ov_side : st;
      PCG_DISPATCH_D16(fmt_d16(A, A->format), A->csr_lanes, k1b_kernel,
                       <<<g, BLOCK, A->dyn_smem, ks>>>(S, Cv, A->n_ghost, vb, w.sc, w.partials, 1, use_cond, h, R.r0,
                                                      phase, 0));
      count_launch();
    }
    PCG_CUDA(cudaGetLastError());
    PCG_TRY(allreduce_sum(A, &w.sc->sigma, 1, st));
    finish_alpha_kernel<<<1, 1, 0, st>>>(w.sc, use_cond, h, 0, xdefer);
    count_launch();
    return PCG_OK;
  }
  if (A->schedule == 3) {  // K1a (streaming p/x update) + K1b (SpMV + sigma)
    if (zlazy(A))
      k1a_kernel<true><<<A->grid_vec, BLOCK, 0, st>>>(A->n, A->n_ghost, v, w.sc, use_cond, h, xdefer, w.dslice);
    else
      k1a_kernel<false><<<A->grid_vec, BLOCK, 0, st>>>(A->n, A->n_ghost, v, w.sc, use_cond, h, xdefer);
    count_launch();
    Vecs vb = v;
    if (xdefer) vb.p0 = k1b_dir(v, xdefer);  // the direction this pass's K1a wrote
    PCG_DISPATCH_D16(fmt_d16(A, A->format), A->csr_lanes, k1b_kernel,
                     <<<A->grid_spmv, BLOCK, A->dyn_smem, st>>>(A->sell_dia(), A->csr(), A->n_ghost, vb, w.sc, w.partials,
                                                                A->comm ? 1 : 0, use_cond, h, 0, 0, xdefer));
    count_launch();
    PCG_CUDA(cudaGetLastError());
    if (A->comm) {
      PCG_TRY(allreduce_sum(A, &w.sc->sigma, 1, st));
      finish_alpha_kernel<<<1, 1, 0, st>>>(w.sc, use_cond, h, 0, xdefer);
      count_launch();
    }
    return PCG_OK;
  }
  if (A->format == PCG_FORMAT_SELL && k1_chunk() == 4)
    k1_kernel<PCG_FORMAT_SELL, 1, 4><<<A->grid_spmv, BLOCK, A->dyn_smem, st>>>(A->sell(), A->csr(), A->n_ghost, v, w.sc,
                                                                     w.partials, A->comm ? 1 : 0, use_cond, h);
  else
    PCG_DISPATCH(A->format, A->csr_lanes, k1_kernel,
                 <<<A->grid_spmv, BLOCK, A->dyn_smem, st>>>(A->sell(), A->csr(), A->n_ghost, v, w.sc, w.partials,
                                                  A->comm ? 1 : 0, use_cond, h));
  count_launch();
  PCG_CUDA(cudaGetLastError());
  if (A->comm) {
    PCG_TRY(allreduce_sum(A, &w.sc->sigma, 1, st));
    finish_alpha_kernel<<<1, 1, 0, st>>>(w.sc, use_cond, h, 1, 0);
    count_launch();
  }
  return PCG_OK;
}

static pcg_status launch_k2(pcg_matrix *A, cudaStream_t st, int use_cond, cudaGraphConditionalHandle h) {
  Vecs v = vecs_of(A);
  SolveWork &w = A->work;
  k2_kernel<<<A->grid_vec, BLOCK, 0, st>>>(A->n, v, w.sc, w.partials + 2 * (size_t)A->grid_spmv, A->comm ? 1 : 0,
                                           use_cond, h, w.dslice, zlazy(A));
  count_launch();
  PCG_CUDA(cudaGetLastError());
  if (A->comm) {
    PCG_TRY(allreduce_sum(A, w.sc->rho_part, 2, st));
    finish_beta_kernel<<<1, 1, 0, st>>>(w.sc, use_cond, h);
    count_launch();
    // ghosts of z for the next K1 (z is final after K2); the overlapped K1 exchanges them itself
    if (!(A->ov && A->schedule == 3)) PCG_TRY(halo_exchange(A, w.z, 1, st));
  }
  return PCG_OK;
}

static pcg_status launch_resid(pcg_matrix *A, const double *b, int mode, cudaStream_t st) {
  Vecs v = vecs_of(A);
  SolveWork &w = A->work;
  if (A->comm) PCG_TRY(halo_exchange(A, w.x, 1, st));
  PCG_DISPATCH_D16(fmt_d16(A, A->format), A->csr_lanes, resid_kernel,
               <<<A->grid_spmv, BLOCK, A->dyn_smem, st>>>(A->sell_dia(), A->csr(), A->n_ghost, b, v, w.sc, w.partials,
                                                mode, A->comm ? 1 : 0));
  count_launch();
  PCG_CUDA(cudaGetLastError());
  if (A->comm) PCG_TRY(allreduce_sum(A, w.sc->res_part, 3, st));
  resid_finish_kernel<<<1, 1, 0, st>>>(w.sc, mode);
  count_launch();
  if (A->comm) PCG_TRY(halo_exchange(A, w.z, 1, st));
  PCG_CUDA(cudaGetLastError());
  return PCG_OK;
}

// deferred x update (k1a_hold / k1a_apply): 3-pass schedule (one GPU or distributed);
// the cycle M: PCG_XDEFER=0 (off: x every iteration), 2 or 4 (default XDEFER_M)
#ifndef PCG_XDEFER_M  // default cycle: measured C5 3.200 (off) / 3.125 (2) / 3.091 s (4)
#define PCG_XDEFER_M 4
#endif
static int xdefer_m(const pcg_matrix *A) {
  if (A->schedule != 3) return 0;
  const char *xd = getenv("PCG_XDEFER");
  const int m = xd ? atoi(xd) : PCG_XDEFER_M;
  return m == 2 || m == 4 ? m : (m == 0 ? 0 : PCG_XDEFER_M);
}
// the 4-cycle's direction buffers p[2], p[3] (allocated once per handle)
static pcg_status ensure_dir_bufs(pcg_matrix *A, int m) {
  SolveWork &w = A->work;
  if (m != 4 || w.p23[0]) return PCG_OK;
  const size_t ngb = sizeof(double) * ((size_t)(A->n + A->n_ghost) + 64);
  for (double *&q : w.p23) {
    PCG_CUDA(cudaMalloc(&q, ngb));
    PCG_CUDA(cudaMemset(q, 0, ngb));
  }
  A->device_bytes += 2.0 * ngb;
  return PCG_OK;
}
// kernel argument of pass u of the loop (0: off)
static int xd_arg(int m, int u) { return m ? (m << 4) | (u % m) : 0; }

// Build the loop graph once per handle: WHILE(cond) { K1; K2 } (1 GPU), or an
// unrolled chunk of U iterations polled from the host (distributed: NCCL calls
// are kept out of conditional bodies).
static pcg_status build_loop_graph(pcg_matrix *A) {
  SolveWork &w = A->work;
  if (w.graph_ready) return PCG_OK;
  // host-callback communicator, or PCG_NO_GRAPH=1 (profilers that do not descend into
  // conditional graph bodies): the same iterations as direct launches, host-polled
  w.xdefer = xdefer_m(A);
  PCG_TRY(ensure_dir_bufs(A, w.xdefer));
  if ((A->comm && !comm_uses_graphs(A->comm)) || getenv("PCG_NO_GRAPH")) {
    w.graph_kind = 3;
    w.unroll = 8;  // a multiple of the deferral cycle
    w.graph_ready = true;
    return PCG_OK;
  }
  cudaStream_t cap;
  PCG_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  cudaGraph_t g;
  PCG_CUDA(cudaGraphCreate(&g, 0));
  pcg_status st = PCG_OK;
  if (!A->comm) {
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
    const int nbody = w.xdefer == 4 ? 4 : 2;  // iterations per conditional body: one deferral cycle
    for (int u = 0; u < nbody && st == PCG_OK; u++) {
      st = launch_k1(A, cap, 1, h, xd_arg(w.xdefer, u));
      if (st == PCG_OK) st = launch_k2(A, cap, 1, h);
    }
    cudaGraph_t out;
    cudaError_t e = cudaStreamEndCapture(cap, &out);
    if (st != PCG_OK) return st;
    PCG_CUDA(e);
    w.graph_kind = 1;
    w.unroll = nbody;
  } else {
    const int U = 8;
    PCG_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
    for (int u = 0; u < U && st == PCG_OK; u++) {  // U a multiple of the deferral cycle
      st = launch_k1(A, cap, 0, 0, xd_arg(w.xdefer, u));
      if (st == PCG_OK) st = launch_k2(A, cap, 0, 0);
    }
    cudaGraph_t out;
    cudaError_t e = cudaStreamEndCapture(cap, &out);
    if (st != PCG_OK) return st;
    PCG_CUDA(e);
    cudaGraphDestroy(g);
    g = out;
    w.graph_kind = 2;
    w.unroll = U;
  }
  PCG_CUDA(cudaGraphInstantiate(&w.loop_exec, g, 0));
  w.loop_graph = g;
  w.graph_ready = true;
  cudaStreamDestroy(cap);
  return PCG_OK;
}

static pcg_status status_of_done(int done, double relres_true, double tol) {
  switch (done) {
    case DONE_CONVERGED: return relres_true <= tol ? PCG_OK : PCG_NOT_CONVERGED;
    case DONE_ZERO_RHS: return PCG_OK;
    case DONE_MAXIT: return PCG_NOT_CONVERGED;
    case DONE_BREAKDOWN: return PCG_ERR_NOT_SPD;
    case DONE_NONFINITE: return PCG_ERR_NONFINITE;
    default: return PCG_NOT_CONVERGED;
  }
}

bool is_device_ptr(const void *p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static pcg_status solve_impl(pcg_matrix *A, const double *b, double *x, double tol, int64_t max_iter,
                             cudaStream_t st, pcg_info *info) {
  PCG_TRY(ensure_work(A));
  const bool persist = persist_wanted(A);
  if (!persist) PCG_TRY(build_loop_graph(A));
  SolveWork &w = A->work;
  const int64_t n = A->n;
  const bool b_dev = is_device_ptr(b), x_dev = is_device_ptr(x);
  const double *db = b;
  if (A->d_perm) {  // SELL-C-sigma: the device system is P A P^T; b' = P b, x0' = P x0
    const double *bs = b, *xs = x;
    if (!b_dev) {
      PCG_CUDA(cudaMemcpyAsync(w.w, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      bs = w.w;
    }
    PCG_TRY(perm_in(A, bs, w.stage_b, st));
    db = w.stage_b;
    if (!x_dev) {
      PCG_CUDA(cudaMemcpyAsync(w.q, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      xs = w.q;
    }
    PCG_TRY(perm_in(A, xs, w.x, st));
  } else {
    if (!b_dev) {
      PCG_CUDA(cudaMemcpyAsync(w.stage_b, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      db = w.stage_b;
    }
    PCG_CUDA(cudaMemcpyAsync(w.x, x, sizeof(double) * n, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  }
  // scalars
  Scalars *h = w.h_sc;
  memset(h, 0, sizeof(Scalars));
  h->tol = tol;
  h->max_iter = max_iter;
  h->done = DONE_RUNNING;
  PCG_CUDA(cudaMemcpyAsync(w.sc, h, sizeof(Scalars), cudaMemcpyHostToDevice, st));
  cudaEvent_t e0, e1;
  PCG_CUDA(cudaEventCreate(&e0));
  PCG_CUDA(cudaEventCreate(&e1));
  PCG_CUDA(cudaEventRecord(e0, st));
  {
    NvtxRange r_("pcg:init");
    PCG_TRY(launch_resid(A, db, MODE_INIT, st));
  }
  for (int round = 0;; round++) {
    NvtxRange r_("pcg:iterate+exit_check");
    if (persist) {
      PCG_TRY(persist_launch(A, vecs_of(A), st));
    } else if (w.graph_kind == 1) {
      PCG_CUDA(cudaGraphLaunch(w.loop_exec, st));
    } else {
      for (;;) {  // unrolled chunks, host-polled
        PCG_CUDA(cudaMemcpyAsync(h, w.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
        PCG_TRY(comm_wait(A->comm, st));
        if (h->done != DONE_RUNNING) break;
        if (w.graph_kind == 2) {
          PCG_CUDA(cudaGraphLaunch(w.loop_exec, st));
        } else {  // 3: the same iterations launched directly (collectives through host callbacks)
          for (int u = 0; u < w.unroll; u++) {
            PCG_TRY(launch_k1(A, st, 0, 0, xd_arg(w.xdefer, u)));
            PCG_TRY(launch_k2(A, st, 0, 0));
          }
        }
      }
    }
    tail_kernel<<<A->grid_vec, BLOCK, 0, st>>>(n, vecs_of(A), w.sc);
    clear_alpha_kernel<<<1, 1, 0, st>>>(w.sc, !persist && w.xdefer);
    count_launch(2);
    PCG_TRY(launch_resid(A, db, MODE_EXIT, st));
    PCG_CUDA(cudaMemcpyAsync(h, w.sc, sizeof(Scalars), cudaMemcpyDeviceToHost, st));
    PCG_TRY(comm_wait(A->comm, st));
    if (h->done != DONE_RUNNING) break;  // else: residual replacement, run the loop again
  }
  PCG_CUDA(cudaEventRecord(e1, st));
  if (h->done == DONE_ZERO_RHS) PCG_CUDA(cudaMemsetAsync(w.x, 0, sizeof(double) * n, st));
  if (A->d_perm) {  // x = P^T x'
    if (x_dev) {
      PCG_TRY(perm_out(A, w.x, x, st));
    } else {
      PCG_TRY(perm_out(A, w.x, w.w, st));
      PCG_CUDA(cudaMemcpyAsync(x, w.w, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    }
  } else {
    PCG_CUDA(cudaMemcpyAsync(x, w.x, sizeof(double) * n, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  }
  PCG_TRY(comm_wait(A->comm, st));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  g_host_launches += (int64_t)h->graph_launches;
  pcg_status s = status_of_done(h->done, h->relres_true, tol);
  if (info) {
    memset(info, 0, sizeof(*info));
    info->iterations = h->k;
    info->relres_recurrence = h->relres_rec;
    info->relres_true = h->done == DONE_ZERO_RHS ? 0.0 : h->relres_true;
    info->converged = (s == PCG_OK);
    info->status = s;
    info->replacements = h->replacements;
    info->t_solve_s = ms * 1e-3;
    const double nn = (double)A->n, nz = (double)A->nnz;
    const int sched = persist ? persist_schedule(A) : A->schedule;
    // K1a: 40n, 36n (x every 2nd iteration), 34n (every 4th)
    const double vb = sched == 3 ? (persist || !w.xdefer ? 96.0 : (w.xdefer == 4 ? 90.0 : 92.0)) : 88.0;
    info->bytes_algorithmic = (double)h->k * (12.0 * nz + 4.0 * (nn + 1) + vb * nn);
    info->flops = (double)h->k * (2.0 * nz + 13.0 * nn);
  }
  if (s == PCG_ERR_NOT_SPD) set_error("pcg_solve: p^T A p <= 0 (matrix not SPD)");
  if (s == PCG_ERR_NONFINITE) set_error("pcg_solve: non-finite right-hand side, x0 or iterate");
  if (s == PCG_NOT_CONVERGED) set_error("pcg_solve: not converged within max_iter");
  return s;
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_solve(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                                void *stream, pcg_info *info) {
  pcgb::NvtxRange nvtx_("pcg:pcg_solve");
  if (!A || ((!b || !x) && A->n > 0)) return fail(PCG_ERR_INVALID_ARG, "pcg_solve: null argument");
  if (!(tol > 0.0)) return fail(PCG_ERR_INVALID_ARG, "pcg_solve: tol must be > 0");
  if (max_iter < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_solve: max_iter must be >= 1");
  if (A->n == 0 && !A->comm) {  // empty system: b = 0, nothing to do
    if (info) {
      memset(info, 0, sizeof(*info));
      info->converged = 1;
    }
    return PCG_OK;
  }
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  return solve_impl(A, b, x, tol, max_iter, (cudaStream_t)stream, info);
}

extern "C" pcg_status pcg_spmv(pcg_matrix_t A, const double *x, double *y, void *stream) {
  if (!A || !x || !y) return fail(PCG_ERR_INVALID_ARG, "pcg_spmv: null argument");
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  PCG_TRY(ensure_work(A));
  cudaStream_t st = (cudaStream_t)stream;
  const bool xd = is_device_ptr(x), yd = is_device_ptr(y);
  if (A->d_perm) {  // y = P^T (P A P^T)(P x)
    const double *xs = x;
    if (!xd) {
      PCG_CUDA(cudaMemcpyAsync(A->work.stage_b, x, sizeof(double) * A->n, cudaMemcpyHostToDevice, st));
      xs = A->work.stage_b;
    }
    PCG_TRY(perm_in(A, xs, A->work.stage_x, st));
    PCG_TRY(launch_spmv(A, A->work.stage_x, A->work.w, st));
    if (yd) {
      PCG_TRY(perm_out(A, A->work.w, y, st));
    } else {
      PCG_TRY(perm_out(A, A->work.w, A->work.stage_b, st));
      PCG_CUDA(cudaMemcpyAsync(y, A->work.stage_b, sizeof(double) * A->n, cudaMemcpyDeviceToHost, st));
    }
    PCG_CUDA(cudaStreamSynchronize(st));
    return PCG_OK;
  }
  const double *dx = x;
  if (A->comm || !xd) {  // gathered vector needs n + n_ghost entries in device memory
    PCG_CUDA(cudaMemcpyAsync(A->work.stage_x, x, sizeof(double) * A->n,
                             xd ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    if (A->comm) PCG_TRY(halo_exchange(A, A->work.stage_x, 1, st));
    dx = A->work.stage_x;
  }
  double *dy = yd ? y : A->work.w;
  PCG_TRY(launch_spmv(A, dx, dy, st));
  if (!yd) PCG_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * A->n, cudaMemcpyDeviceToHost, st));
  PCG_TRY(comm_wait(A->comm, st));
  return PCG_OK;
}

namespace pcgb {
// TMA-staged kernels need their dynamic shared memory opted in (> 48 KB)
pcg_status prepare_staged(size_t smem) {
  const int v = (int)smem;
  PCG_CUDA(cudaFuncSetAttribute(k1_kernel<FMT_SELL_TMA, 1, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
  PCG_CUDA(cudaFuncSetAttribute(k1_kernel<FMT_SELL_TMA, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
  PCG_CUDA(cudaFuncSetAttribute(resid_kernel<FMT_SELL_TMA, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
  PCG_CUDA(cudaFuncSetAttribute(spmv_kernel<FMT_SELL_TMA, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
  PCG_CUDA(cudaFuncSetAttribute(k1b_kernel<FMT_SELL_TMA, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, v));
  return PCG_OK;
}

int k1_blocks_per_sm(int fmt, int lanes, size_t smem) {
  int b = 0;
  cudaError_t e;
  if (fmt == FMT_SELL_SHORT || fmt == FMT_SELL_DIA) {
    e = fmt == FMT_SELL_DIA ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1b_kernel<FMT_SELL_DIA, 1>, BLOCK, 0)
                            : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1b_kernel<FMT_SELL_SHORT, 1>, BLOCK, 0);
  } else if (fmt == FMT_SELL_TMA) {
    e = k1_chunk() == 4 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<FMT_SELL_TMA, 1, 4>, BLOCK, smem)
                        : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<FMT_SELL_TMA, 1, 8>, BLOCK, smem);
  } else if (fmt == PCG_FORMAT_SELL) {
    e = k1_chunk() == 4 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_SELL, 1, 4>, BLOCK, 0)
                        : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_SELL, 1, 8>, BLOCK, 0);
  } else {
    switch (lanes) {
      case 1: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_CSR, 1>, BLOCK, 0); break;
      case 2: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_CSR, 2>, BLOCK, 0); break;
      case 4: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_CSR, 4>, BLOCK, 0); break;
      case 8: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_CSR, 8>, BLOCK, 0); break;
      case 16: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_CSR, 16>, BLOCK, 0); break;
      default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k1_kernel<PCG_FORMAT_CSR, 32>, BLOCK, 0); break;
    }
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 4;
  }
  return b < 1 ? 1 : (b > 8 ? 8 : b);
}
}  // namespace pcgb

extern "C" pcg_status pcg_profile_kernels(pcg_matrix_t A, const double *b, int32_t reps, void *stream, double *us,
                                          int32_t *reps_done) {
  if (!A || !b || !us || reps < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_profile_kernels: bad argument");
  if (A->comm) return fail(PCG_ERR_INVALID_ARG, "pcg_profile_kernels: single-GPU handles only");
  if (!is_device_ptr(b)) return fail(PCG_ERR_INVALID_ARG, "pcg_profile_kernels: b must be a device pointer");
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  PCG_TRY(ensure_work(A));
  cudaStream_t st = (cudaStream_t)stream;
  SolveWork &w = A->work;
  PCG_CUDA(cudaMemsetAsync(w.x, 0, sizeof(double) * A->n, st));
  Scalars *h = w.h_sc;
  memset(h, 0, sizeof(Scalars));
  h->tol = 1e-300;  // never stops on the residual inside the profiled window
  h->max_iter = (long long)reps + 1;
  PCG_CUDA(cudaMemcpyAsync(w.sc, h, sizeof(Scalars), cudaMemcpyHostToDevice, st));
  if (A->d_perm) {
    PCG_TRY(perm_in(A, b, w.stage_b, st));
    b = w.stage_b;
  }
  PCG_TRY(launch_resid(A, b, MODE_INIT, st));
  const int xm = xdefer_m(A);  // the loop's K1a passes (hold / apply) when x is deferred
  PCG_TRY(ensure_dir_bufs(A, xm));
  Vecs v = vecs_of(A);
  std::vector<cudaEvent_t> ev(3 * (size_t)reps + 1);
  for (auto &e : ev) PCG_CUDA(cudaEventCreate(&e));
  PCG_CUDA(cudaEventRecord(ev[0], st));
  for (int r = 0; r < reps; r++) {
    if (A->schedule == 3) {  // the loop's kernels: hold / apply K1a pairs when x is deferred
      const int xd = xd_arg(xm, r);
      Vecs vb = v;
      if (xd) vb.p0 = k1b_dir(v, xd);
      if (zlazy(A))
        k1a_kernel<true><<<A->grid_vec, BLOCK, 0, st>>>(A->n, A->n_ghost, v, w.sc, 0, 0, xd, w.dslice);
      else
        k1a_kernel<false><<<A->grid_vec, BLOCK, 0, st>>>(A->n, A->n_ghost, v, w.sc, 0, 0, xd);
      PCG_CUDA(cudaEventRecord(ev[3 * r + 1], st));
      PCG_DISPATCH_D16(fmt_d16(A, A->format), A->csr_lanes, k1b_kernel,
                       <<<A->grid_spmv, BLOCK, A->dyn_smem, st>>>(A->sell_dia(), A->csr(), A->n_ghost, vb, w.sc,
                                                                  w.partials, 0, 0, 0, 0, 0, xd));
      count_launch(2);
    } else {
      PCG_CUDA(cudaEventRecord(ev[3 * r + 1], st));
      PCG_TRY(launch_k1(A, st, 0, 0));
    }
    PCG_CUDA(cudaEventRecord(ev[3 * r + 2], st));
    PCG_TRY(launch_k2(A, st, 0, 0));
    PCG_CUDA(cudaEventRecord(ev[3 * r + 3], st));
  }
  PCG_CUDA(cudaStreamSynchronize(st));
  PCG_CUDA(cudaMemcpy(h, w.sc, sizeof(Scalars), cudaMemcpyDeviceToHost));
  const int done = (int)std::min<long long>(h->k, reps);
  double t[3] = {0, 0, 0};
  for (int r = 0; r < done; r++)
    for (int k = 0; k < 3; k++) {
      float ms = 0;
      cudaEventElapsedTime(&ms, ev[3 * r + k], ev[3 * r + k + 1]);
      t[k] += ms;
    }
  for (auto &e : ev) cudaEventDestroy(e);
  for (int k = 0; k < 3; k++) us[k] = done ? t[k] * 1e3 / done : 0.0;
  if (reps_done) *reps_done = done;
  return PCG_OK;
}
