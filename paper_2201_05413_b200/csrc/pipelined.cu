// pipelined.cu — preconditioned pipelined CG (DESIGN.md reading
// R4; Ghysels & Vanroose 2014, Alg. 3) with the Jacobi preconditioner: ONE
// reduction phase per iteration instead of PCG's two, the SpMV on m = M^-1 w
// independent of it.  Restated:
//
//   (re)start: r = b - A x ; stop test on ||r|| ; u = M^-1 r ; w = A u
//   loop:  gamma = r.u ; delta = w.u ; rr = r.r             (one reduction)
//          stop test on sqrt(rr) (then the true residual of Eq. relativeError decides)
//          first step after a (re)start: beta = 0, alpha = gamma/delta
//          else beta = gamma/gamma_old, alpha = gamma/(delta - beta gamma/alpha_old)
//          n = A m   (m = M^-1 w, written by the previous pass)
//          z = n + beta z ; q = m + beta q ; s = w + beta s ; p = u + beta p
//          x += alpha p ; r -= alpha s ; u -= alpha q ; w -= alpha z ; m' = M^-1 w
//   alpha <= 0: on the first step after a (re)start A is not SPD; later the recurrences
//   have drifted (pipelined CG's known instability) and the solve restarts from x.
//
// The whole solve is one cooperative kernel: each iteration is ONE fused pass (the
// SpMV on m with every vector update, the next m and the next iteration's
// reduction partials in its epilogue) and ONE grid barrier (two alternating
// partial regions remove the write-after-read hazard); every block evaluates
// the scalars identically from the fixed-order block partials (coop.cuh).  m is
// double-buffered: the pass gathers m while writing m'.  Per-element arithmetic
// is rounded like the oracle's (orc_pcg_pipelined: a + b*c in two roundings).
// Bytes per iteration: 12 nnz + 4(n+1) + 160 n (m gathered once; z q s p u w x r
// dinv m read; z q s p x r u w m' written) — 64 n more than PCG's 3-pass
// schedule: on one GPU it pays where barriers and launches, not bytes, bound the
// iteration (small systems); across GPUs it removes one allreduce per iteration.
#include <cstring>

#include "coop.cuh"
#include "matrix.cuh"
#include "rows.cuh"

namespace pcgb {

struct PipeVecs {
  double *x, *r, *u, *w, *m0, *m1, *z, *q, *s, *p;
  const double *b, *dinv;
};

struct PipeState {
  double tol, nb, relres_rec, relres_true;
  long long k, max_iter, restarts;
  int done, pad;
};

enum { PD_RUNNING = 0, PD_CONVERGED = 1, PD_MAXIT = 2, PD_BREAKDOWN = 3, PD_ZERO_RHS = 4, PD_NONFINITE = 5 };

__device__ __forceinline__ double axpy_rn(double a, double b, double c) { return __dadd_rn(a, __dmul_rn(b, c)); }

// SpMV passes outside the loop: RESID r = b - A x (rr), U_TO_W w = A u (with m = dinv w and
// the first reduction's partials), TRUE t = b - A x (tt only)
enum { PP_RESID = 0, PP_W = 1, PP_TRUE = 2 };

template <int FMT, int L, int MODE>
__device__ __noinline__ void pipe_spmv(const SellView &S, const CsrView &C, const PipeVecs &v, double *m_out,
                                       double (&a)[3]) {  // (re)start / exit check only: kept out of the hot loop
  const double *__restrict__ G = MODE == PP_W ? v.u : v.x;
  auto gather = [&](int j) { return ld_weak(G + j); };  // inside the cooperative kernel
  auto epi = [&](int64_t i, double sv) {
    if (MODE == PP_W) {
      v.w[i] = sv;
      m_out[i] = __dmul_rn(v.dinv[i], sv);
      const double ri = v.r[i], ui = v.u[i];
      a[0] = __fma_rn(ri, ui, a[0]);
      a[1] = __fma_rn(sv, ui, a[1]);
      a[2] = __fma_rn(ri, ri, a[2]);
    } else {
      const double ri = __dsub_rn(v.b[i], sv);
      if (MODE == PP_RESID) v.r[i] = ri;
      a[0] = __fma_rn(ri, ri, a[0]);
    }
  };
  if (FMT == PCG_FORMAT_SELL) sell_rows(S, gather, epi);
  else csr_rows<L>(C, gather, epi);
}

template <int NV>
__device__ __forceinline__ void pipe_publish(const double (&a)[3], double *part, double (*sm)[WARPS]) {
  double red[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) red[i] = a[i];
  block_sum<NV>(red, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < NV; i++) part[(size_t)i * gridDim.x + blockIdx.x] = red[i];
}

// MINB: resident blocks per SM the kernel is compiled for — 1 (no spills: the
// latency-bound small systems) or 3 (more warps in flight: the larger ones)
template <int FMT, int L, int MINB>
__global__ void __launch_bounds__(BLOCK, MINB) pipe_kernel(SellView S_, CsrView C_, PipeVecs v_, PipeState *st,
                                                        double *part, GridBar *bar) {
  __shared__ double sm[3][WARPS];
  __shared__ double s_tot[3];
  __shared__ SellView S;
  __shared__ CsrView C;
  __shared__ PipeVecs v;
  if (threadIdx.x == 0) {
    S = S_;
    C = C_;
    v = v_;
  }
  __syncthreads();
  const int64_t n = FMT == PCG_FORMAT_SELL ? S.n : C.n;
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nth = (int64_t)gridDim.x * BLOCK;
  const double tol = st->tol;
  const long long max_iter = st->max_iter;
  long long k = st->k, restarts = 0;
  double relres_rec = 0.0, relres_true = 0.0;
  // ||b||
  double nb;
  {
    double a[3] = {0.0, 0.0, 0.0};
    for (int64_t i = tid; i < n; i += nth) a[0] = __fma_rn(v.b[i], v.b[i], a[0]);
    pipe_publish<1>(a, part, sm);
    grid_sync(bar);
    double t[1];
    all_blocks_sum<1>(part, t, sm, s_tot);
    nb = sqrt(t[0]);
  }
  int done = nb == 0.0 ? PD_ZERO_RHS : (!(nb == nb) ? PD_NONFINITE : PD_RUNNING);
  if (done != PD_RUNNING)
    for (int64_t i = tid; i < n; i += nth) v.x[i] = 0.0;
  bool restart = true, first = true;
  double gamma_old = 0.0, alpha_old = 0.0;
  double *mc = v.m0, *mn = v.m1;  // m of this iteration / of the next
  // two partial regions: the loop top reads prd while the fused pass publishes into
  // pwr, so one barrier per iteration orders both (a block can only overwrite prd
  // after the next barrier, which every reader of prd has passed)
  double *prd = part, *pwr = part + 3 * gridDim.x;
  while (done == PD_RUNNING) {
    if (restart) {
      double a[3] = {0.0, 0.0, 0.0};
      grid_sync(bar);  // every block is past its last use of x, r and the partials
      pipe_spmv<FMT, L, PP_RESID>(S, C, v, nullptr, a);
      pipe_publish<1>(a, prd, sm);
      grid_sync(bar);
      double t[1];
      all_blocks_sum<1>(prd, t, sm, s_tot);
      const double rr0 = sqrt(t[0]);
      relres_rec = rr0 / nb;
      if (rr0 <= tol * nb) {  // converged on entry: the true residual is this one
        relres_true = relres_rec;
        done = PD_CONVERGED;
        break;
      }
      for (int64_t i = tid; i < n; i += nth) v.u[i] = __dmul_rn(v.dinv[i], v.r[i]);
      grid_sync(bar);
      double b3[3] = {0.0, 0.0, 0.0};
      pipe_spmv<FMT, L, PP_W>(S, C, v, mc, b3);
      pipe_publish<3>(b3, pwr, sm);
      double *tp = prd;
      prd = pwr;
      pwr = tp;
      restart = false;
      first = true;
    }
    grid_sync(bar);
    double t[3];
    all_blocks_sum<3>(prd, t, sm, s_tot);
    const double gamma = t[0], delta = t[1], rr = sqrt(t[2]);
    relres_rec = rr / nb;
    if (!first && rr <= tol * nb) {  // exit check: the true residual decides
      double a[3] = {0.0, 0.0, 0.0};
      pipe_spmv<FMT, L, PP_TRUE>(S, C, v, nullptr, a);
      pipe_publish<1>(a, pwr, sm);
      grid_sync(bar);
      double tt[1];
      all_blocks_sum<1>(pwr, tt, sm, s_tot);
      relres_true = sqrt(tt[0]) / nb;
      if (relres_true <= tol) {
        done = PD_CONVERGED;
        break;
      }
      restart = true;
      restarts++;
      continue;
    }
    if (!(rr == rr)) {
      done = PD_NONFINITE;
      break;
    }
    if (k >= max_iter) {
      done = PD_MAXIT;
      break;
    }
    double alpha, beta;
    if (first) {
      beta = 0.0;
      alpha = __ddiv_rn(gamma, delta);
    } else {
      beta = __ddiv_rn(gamma, gamma_old);
      alpha = __ddiv_rn(gamma, __dsub_rn(delta, __ddiv_rn(__dmul_rn(beta, gamma), alpha_old)));
    }
    if (!(alpha > 0.0)) {  // reading R4: not SPD on a first step, drifted recurrences later
      if (first) {
        done = PD_BREAKDOWN;
        break;
      }
      restart = true;
      restarts++;
      continue;
    }
    // ---- the fused pass: n = A m, all updates, m' = M^-1 w, next partials
    {
      double a[3] = {0.0, 0.0, 0.0};
      const double *__restrict__ m = mc;
      double *__restrict__ m2 = mn;
      auto gather = [&](int j) { return ld_weak(m + j); };  // m is written by this kernel
      auto epi = [&](int64_t i, double nv) {
        const double zi = axpy_rn(nv, beta, v.z[i]);
        const double qi = axpy_rn(m[i], beta, v.q[i]);
        const double si = axpy_rn(v.w[i], beta, v.s[i]);
        const double pi = axpy_rn(v.u[i], beta, v.p[i]);
        const double xi = axpy_rn(v.x[i], alpha, pi);
        const double ri = __dsub_rn(v.r[i], __dmul_rn(alpha, si));
        const double ui = __dsub_rn(v.u[i], __dmul_rn(alpha, qi));
        const double wi = __dsub_rn(v.w[i], __dmul_rn(alpha, zi));
        v.z[i] = zi;
        v.q[i] = qi;
        v.s[i] = si;
        v.p[i] = pi;
        v.x[i] = xi;
        v.r[i] = ri;
        v.u[i] = ui;
        v.w[i] = wi;
        m2[i] = __dmul_rn(v.dinv[i], wi);
        a[0] = __fma_rn(ri, ui, a[0]);
        a[1] = __fma_rn(wi, ui, a[1]);
        a[2] = __fma_rn(ri, ri, a[2]);
      };
      if (FMT == PCG_FORMAT_SELL) sell_rows(S, gather, epi);
      else csr_rows<L>(C, gather, epi);
      pipe_publish<3>(a, pwr, sm);
    }
    double *tmp = mc;
    mc = mn;
    mn = tmp;
    tmp = prd;
    prd = pwr;
    pwr = tmp;
    gamma_old = gamma;
    alpha_old = alpha;
    first = false;
    k++;
  }
  if (done == PD_MAXIT || done == PD_BREAKDOWN || done == PD_NONFINITE) {  // final true residual
    double a[3] = {0.0, 0.0, 0.0};
    pipe_spmv<FMT, L, PP_TRUE>(S, C, v, nullptr, a);
    pipe_publish<1>(a, pwr, sm);
    grid_sync(bar);
    double tt[1];
    all_blocks_sum<1>(pwr, tt, sm, s_tot);
    relres_true = sqrt(tt[0]) / nb;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->nb = nb;
    st->relres_rec = relres_rec;
    st->relres_true = relres_true;
    st->k = k;
    st->restarts = restarts;
    st->done = done;
  }
}

// ---------------------------------------------------------------- distributed schedule
// Row-partitioned over GPUs (csr_create_dist handles): the same recurrence as
// separate kernels with the exchange steps between them, per iteration
//   fused pass (n = A m, all updates, m' own rows, partials)  ->  ONE allreduce of
//   (r.u, w.u, r.r)  ->  halo exchange of m'  ->  finisher (alpha, beta, stop test)
// — one collective phase per iteration where PCG needs two (sigma, then rho'/gamma).
// The host launches U iterations between polls; once a finisher sets `stop` the
// remaining kernels of the chunk return at entry (the collectives still run, so every
// rank issues the same sequence), and the host performs the exit check / restart.
struct PdState {
  double tol, nb, gamma_old, alpha_old, alpha, beta, relres_rec, relres_true;
  double part[3];  // local sums awaiting the allreduce
  long long k, max_iter, restarts;
  int done, stop, first, need_check, need_restart, pad;
  unsigned int cnt;
};

enum { PDR_RESID = 0, PDR_W = 1, PDR_TRUE = 2 };

template <int NV>
__device__ __forceinline__ void pd_reduce(double (&a)[3], PdState *sc, double *partials, double (*sm)[WARPS]) {
  double red[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) red[i] = a[i];
  block_sum<NV>(red, sm);
  if (publish_and_arrive<NV>(red, partials, &sc->cnt)) {
    double tot[NV];
    reduce_partials<NV>(partials, tot, sm);
    if (threadIdx.x == 0) {
      sc->cnt = 0;
#pragma unroll
      for (int i = 0; i < NV; i++) sc->part[i] = tot[i];
    }
  }
}

// RESID: r = b - A x (r.r, b.b); W: w = A u, m = M^-1 w (r.u, w.u, r.r); TRUE: (t.t)
template <int FMT, int L, int MODE>
__global__ void __launch_bounds__(BLOCK) pd_spmv_kernel(SellView S, CsrView C, PipeVecs v, double *m_out,
                                                        PdState *sc, double *partials) {
  __shared__ double sm[3][WARPS];
  double a[3] = {0.0, 0.0, 0.0};
  const double *__restrict__ G = MODE == PDR_W ? v.u : v.x;
  auto gather = [&](int j) { return __ldg(G + j); };
  auto epi = [&](int64_t i, double sv) {
    if (MODE == PDR_W) {
      v.w[i] = sv;
      m_out[i] = __dmul_rn(v.dinv[i], sv);
      const double ri = v.r[i], ui = v.u[i];
      a[0] = __fma_rn(ri, ui, a[0]);
      a[1] = __fma_rn(sv, ui, a[1]);
      a[2] = __fma_rn(ri, ri, a[2]);
    } else {
      const double bi = v.b[i];
      const double ri = __dsub_rn(bi, sv);
      a[0] = __fma_rn(ri, ri, a[0]);
      if (MODE == PDR_RESID) {
        v.r[i] = ri;
        a[1] = __fma_rn(bi, bi, a[1]);
      }
    }
  };
  if (FMT == PCG_FORMAT_SELL) sell_rows(S, gather, epi);
  else csr_rows<L>(C, gather, epi);
  if (MODE == PDR_W) pd_reduce<3>(a, sc, partials, sm);
  else pd_reduce<2>(a, sc, partials, sm);
}

__global__ void pd_u_kernel(int64_t n, PipeVecs v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    v.u[i] = __dmul_rn(v.dinv[i], v.r[i]);
}

template <int FMT, int L>
__global__ void __launch_bounds__(BLOCK) pd_fused_kernel(SellView S, CsrView C, PipeVecs v, const double *mc,
                                                         double *mn, PdState *sc, double *partials) {
  __shared__ double sm[3][WARPS];
  const volatile PdState *vs = sc;
  if (vs->stop) return;
  const double alpha = vs->alpha, beta = vs->beta;
  double a[3] = {0.0, 0.0, 0.0};
  const double *__restrict__ m = mc;
  double *__restrict__ m2 = mn;
  auto gather = [&](int j) { return __ldg(m + j); };
  auto epi = [&](int64_t i, double nv) {
    const double zi = axpy_rn(nv, beta, v.z[i]);
    const double qi = axpy_rn(m[i], beta, v.q[i]);
    const double si = axpy_rn(v.w[i], beta, v.s[i]);
    const double pi = axpy_rn(v.u[i], beta, v.p[i]);
    const double xi = axpy_rn(v.x[i], alpha, pi);
    const double ri = __dsub_rn(v.r[i], __dmul_rn(alpha, si));
    const double ui = __dsub_rn(v.u[i], __dmul_rn(alpha, qi));
    const double wi = __dsub_rn(v.w[i], __dmul_rn(alpha, zi));
    v.z[i] = zi;
    v.q[i] = qi;
    v.s[i] = si;
    v.p[i] = pi;
    v.x[i] = xi;
    v.r[i] = ri;
    v.u[i] = ui;
    v.w[i] = wi;
    m2[i] = __dmul_rn(v.dinv[i], wi);
    a[0] = __fma_rn(ri, ui, a[0]);
    a[1] = __fma_rn(wi, ui, a[1]);
    a[2] = __fma_rn(ri, ri, a[2]);
  };
  if (FMT == PCG_FORMAT_SELL) sell_rows(S, gather, epi);
  else csr_rows<L>(C, gather, epi);
  pd_reduce<3>(a, sc, partials, sm);
}

// after the allreduce of (r.u, w.u, r.r): stop test, alpha and beta for the next pass
__global__ void pd_finish_kernel(PdState *sc) {
  if (sc->stop) return;
  const double gamma = sc->part[0], delta = sc->part[1], rr = sqrt(sc->part[2]);
  sc->relres_rec = rr / sc->nb;
  if (!sc->first && rr <= sc->tol * sc->nb) {
    sc->stop = 1;
    sc->need_check = 1;
    return;
  }
  if (!(rr == rr)) {
    sc->done = PD_NONFINITE;
    sc->stop = 1;
    return;
  }
  if (sc->k >= sc->max_iter) {
    sc->done = PD_MAXIT;
    sc->stop = 1;
    return;
  }
  double alpha, beta;
  if (sc->first) {
    beta = 0.0;
    alpha = __ddiv_rn(gamma, delta);
  } else {
    beta = __ddiv_rn(gamma, sc->gamma_old);
    alpha = __ddiv_rn(gamma, __dsub_rn(delta, __ddiv_rn(__dmul_rn(beta, gamma), sc->alpha_old)));
  }
  if (!(alpha > 0.0)) {  // reading R4
    sc->stop = 1;
    if (sc->first) sc->done = PD_BREAKDOWN;
    else sc->need_restart = 1;
    return;
  }
  sc->alpha = alpha;
  sc->beta = beta;
  sc->gamma_old = gamma;
  sc->alpha_old = alpha;
  sc->first = 0;
  sc->k++;
}

// after RESID + allreduce: mode 0 = the solve's start (||b||), 1 = a restart
__global__ void pd_start_kernel(PdState *sc, int mode) {
  if (mode == 0) {
    sc->nb = sqrt(sc->part[1]);
    if (sc->nb == 0.0 || !(sc->nb == sc->nb)) {
      sc->done = sc->nb == 0.0 ? PD_ZERO_RHS : PD_NONFINITE;
      sc->stop = 1;
      return;
    }
  } else {
    sc->restarts++;
  }
  const double rr0 = sqrt(sc->part[0]);
  sc->relres_rec = rr0 / sc->nb;
  sc->stop = sc->need_check = sc->need_restart = 0;
  sc->first = 1;
  if (rr0 <= sc->tol * sc->nb) {
    sc->relres_true = sc->relres_rec;
    sc->done = PD_CONVERGED;
    sc->stop = 1;
  }
}

// after TRUE + allreduce: the exit check (mode 0) or the final true residual (mode 1)
__global__ void pd_check_kernel(PdState *sc, int mode) {
  sc->relres_true = sqrt(sc->part[0]) / sc->nb;
  if (mode == 0 && sc->relres_true <= sc->tol) sc->done = PD_CONVERGED;
}

// ---------------------------------------------------------------- host side
template <int MINB>
static void *pipe_fn_b(int fmt, int lanes) {
  if (fmt == PCG_FORMAT_SELL) return (void *)pipe_kernel<PCG_FORMAT_SELL, 1, MINB>;
  switch (lanes) {
    case 1: return (void *)pipe_kernel<PCG_FORMAT_CSR, 1, MINB>;
    case 2: return (void *)pipe_kernel<PCG_FORMAT_CSR, 2, MINB>;
    case 4: return (void *)pipe_kernel<PCG_FORMAT_CSR, 4, MINB>;
    case 8: return (void *)pipe_kernel<PCG_FORMAT_CSR, 8, MINB>;
    case 16: return (void *)pipe_kernel<PCG_FORMAT_CSR, 16, MINB>;
    default: return (void *)pipe_kernel<PCG_FORMAT_CSR, 32, MINB>;
  }
}

// measured (C1 / C4 / C6 solve seconds): 1 block/SM 0.54 ms / 0.105 / 0.142, 2 blocks
// 0.70 ms / 0.083 / 0.127, 3 blocks 0.72 ms / 0.080 / 0.124
static void *pipe_fn(int fmt, int lanes, int64_t n) {
  return n < (int64_t(1) << 18) ? pipe_fn_b<1>(fmt, lanes) : pipe_fn_b<3>(fmt, lanes);
}

// distributed launchers per (format, CSR lanes)
struct PdOps {
  void (*spmv)(int mode, pcg_matrix *, const PipeVecs &, double *, PdState *, cudaStream_t);
  void (*fused)(pcg_matrix *, const PipeVecs &, const double *, double *, PdState *, cudaStream_t);
};
template <int FMT, int L>
static void pd_spmv_l(int mode, pcg_matrix *A, const PipeVecs &v, double *m_out, PdState *sc, cudaStream_t st) {
  double *part = A->work.partials;
  if (mode == PDR_RESID)
    pd_spmv_kernel<FMT, L, PDR_RESID><<<A->grid_spmv, BLOCK, 0, st>>>(A->sell(), A->csr(), v, m_out, sc, part);
  else if (mode == PDR_W)
    pd_spmv_kernel<FMT, L, PDR_W><<<A->grid_spmv, BLOCK, 0, st>>>(A->sell(), A->csr(), v, m_out, sc, part);
  else
    pd_spmv_kernel<FMT, L, PDR_TRUE><<<A->grid_spmv, BLOCK, 0, st>>>(A->sell(), A->csr(), v, m_out, sc, part);
  count_launch();
}
template <int FMT, int L>
static void pd_fused_l(pcg_matrix *A, const PipeVecs &v, const double *mc, double *mn, PdState *sc, cudaStream_t st) {
  pd_fused_kernel<FMT, L><<<A->grid_spmv, BLOCK, 0, st>>>(A->sell(), A->csr(), v, mc, mn, sc, A->work.partials);
  count_launch();
}
template <int FMT, int L>
static PdOps pd_ops_t() {
  return {pd_spmv_l<FMT, L>, pd_fused_l<FMT, L>};
}
static PdOps pd_ops(int fmt, int lanes) {
  if (fmt == PCG_FORMAT_SELL) return pd_ops_t<PCG_FORMAT_SELL, 1>();
  switch (lanes) {
    case 1: return pd_ops_t<PCG_FORMAT_CSR, 1>();
    case 2: return pd_ops_t<PCG_FORMAT_CSR, 2>();
    case 4: return pd_ops_t<PCG_FORMAT_CSR, 4>();
    case 8: return pd_ops_t<PCG_FORMAT_CSR, 8>();
    case 16: return pd_ops_t<PCG_FORMAT_CSR, 16>();
    default: return pd_ops_t<PCG_FORMAT_CSR, 32>();
  }
}

// the distributed solve: every rank issues the same sequence (decisions come from
// allreduced values, identical on all ranks); fills the single-GPU state fields
static pcg_status pd_solve(pcg_matrix *A, const PipeVecs &v, double tol, int64_t max_iter, cudaStream_t st,
                           PipeState *out) {
  SolveWork &w = A->work;
  if (!w.pdsc) PCG_CUDA(cudaMalloc(&w.pdsc, sizeof(PdState)));
  PdState *sc = (PdState *)w.pdsc, h;
  memset(&h, 0, sizeof(h));
  h.tol = tol;
  h.max_iter = max_iter;
  PCG_CUDA(cudaMemcpyAsync(sc, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  const PdOps ops = pd_ops(A->format == FMT_SELL_TMA ? PCG_FORMAT_SELL : A->format, A->csr_lanes);
  auto read = [&]() -> pcg_status {
    PCG_CUDA(cudaGetLastError());
    PCG_CUDA(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
    PCG_TRY(comm_wait(A->comm, st));
    return PCG_OK;
  };
  auto residual = [&](int mode) -> pcg_status {  // r = b - A x (+ ||b||^2), allreduced, start / restart
    PCG_TRY(halo_exchange(A, v.x, 1, st));
    ops.spmv(PDR_RESID, A, v, nullptr, sc, st);
    PCG_TRY(allreduce_sum(A, sc->part, 2, st));
    pd_start_kernel<<<1, 1, 0, st>>>(sc, mode);
    count_launch();
    return read();
  };
  auto true_res = [&](int mode) -> pcg_status {
    PCG_TRY(halo_exchange(A, v.x, 1, st));
    ops.spmv(PDR_TRUE, A, v, nullptr, sc, st);
    PCG_TRY(allreduce_sum(A, sc->part, 1, st));
    pd_check_kernel<<<1, 1, 0, st>>>(sc, mode);
    count_launch();
    return read();
  };
  const int U = 8;
  PCG_TRY(residual(0));
  if (h.done == PD_ZERO_RHS || h.done == PD_NONFINITE) PCG_CUDA(cudaMemsetAsync(v.x, 0, sizeof(double) * A->n, st));
  double *mc = v.m0, *mn = v.m1;
  while (h.done == PD_RUNNING) {
    // (re)start from x: u = M^-1 r, w = A u, m = M^-1 w, first reduction, ghosts of m
    pd_u_kernel<<<A->grid_vec, BLOCK, 0, st>>>(A->n, v);
    count_launch();
    PCG_TRY(halo_exchange(A, v.u, 1, st));
    ops.spmv(PDR_W, A, v, mc, sc, st);
    PCG_TRY(allreduce_sum(A, sc->part, 3, st));
    PCG_TRY(halo_exchange(A, mc, 1, st));
    pd_finish_kernel<<<1, 1, 0, st>>>(sc);
    count_launch();
    PCG_TRY(read());
    while (!h.stop) {
      for (int u = 0; u < U; u++) {
        ops.fused(A, v, mc, mn, sc, st);
        PCG_TRY(allreduce_sum(A, sc->part, 3, st));
        PCG_TRY(halo_exchange(A, mn, 1, st));
        pd_finish_kernel<<<1, 1, 0, st>>>(sc);
        count_launch();
        std::swap(mc, mn);
      }
      PCG_TRY(read());
    }
    if (h.done != PD_RUNNING) break;
    if (h.need_check) {
      PCG_TRY(true_res(0));
      if (h.done != PD_RUNNING) break;
    }
    PCG_TRY(residual(1));  // failed exit check or drifted recurrences: restart from x
  }
  if (h.done == PD_MAXIT || h.done == PD_BREAKDOWN || h.done == PD_NONFINITE) PCG_TRY(true_res(1));
  out->nb = h.nb;
  out->relres_rec = h.relres_rec;
  out->relres_true = h.relres_true;
  out->k = h.k;
  out->restarts = h.restarts;
  out->done = h.done;
  return PCG_OK;
}

static pcg_status pipe_report(pcg_matrix *A, const PipeState &hs, double tol, float ms, pcg_info *info) {
  pcg_status s;
  switch (hs.done) {
    case PD_CONVERGED: s = hs.relres_true <= tol ? PCG_OK : PCG_NOT_CONVERGED; break;
    case PD_ZERO_RHS: s = PCG_OK; break;
    case PD_MAXIT: s = PCG_NOT_CONVERGED; break;
    case PD_BREAKDOWN: s = PCG_ERR_NOT_SPD; break;
    default: s = PCG_ERR_NONFINITE; break;
  }
  if (info) {
    memset(info, 0, sizeof(*info));
    info->iterations = hs.k;
    info->relres_recurrence = hs.relres_rec;
    info->relres_true = hs.done == PD_ZERO_RHS ? 0.0 : hs.relres_true;
    info->converged = s == PCG_OK;
    info->status = s;
    info->replacements = hs.restarts;
    info->t_solve_s = ms * 1e-3;
    const double nn = (double)A->n, nz = (double)A->nnz;
    info->bytes_algorithmic = (double)hs.k * (12.0 * nz + 4.0 * (nn + 1) + 160.0 * nn);
    info->flops = (double)hs.k * (2.0 * nz + 27.0 * nn);
  }
  if (s == PCG_ERR_NOT_SPD) set_error("pcg_solve_pipelined: alpha <= 0 (A not SPD or breakdown)");
  if (s == PCG_NOT_CONVERGED) set_error("pcg_solve_pipelined: not converged within max_iter");
  if (s == PCG_ERR_NONFINITE) set_error("pcg_solve_pipelined: non-finite right-hand side or iterate");
  return s;
}

static pcg_status pipe_impl(pcg_matrix *A, const double *b, double *x, double tol, int64_t max_iter, cudaStream_t st,
                            pcg_info *info) {
  PCG_TRY(ensure_work(A));
  SolveWork &w = A->work;
  const int64_t n = A->n, ldv = n + A->n_ghost + 64;  // gathered vectors carry ghost slots
  if (!w.pv) {
    PCG_CUDA(cudaMalloc(&w.pv, sizeof(double) * (size_t)ldv * 10));  // x r u w m0 m1 z q s p
    PCG_CUDA(cudaMalloc(&w.pstate, sizeof(PipeState)));
    PCG_CUDA(cudaMalloc(&w.ppbar, sizeof(GridBar)));
    PCG_CUDA(cudaMemsetAsync(w.ppbar, 0, sizeof(GridBar), st));
  }
  PipeVecs v;
  double *base = w.pv;
  v.x = base;
  v.r = base + ldv;
  v.u = base + 2 * ldv;
  v.w = base + 3 * ldv;
  v.m0 = base + 4 * ldv;
  v.m1 = base + 5 * ldv;
  v.z = base + 6 * ldv;
  v.q = base + 7 * ldv;
  v.s = base + 8 * ldv;
  v.p = base + 9 * ldv;
  v.dinv = A->d_dinv;
  PCG_CUDA(cudaMemsetAsync(v.z, 0, sizeof(double) * (size_t)ldv * 4, st));  // z q s p: beta = 0 multiplies them
  const bool b_dev = is_device_ptr(b), x_dev = is_device_ptr(x);
  if (A->d_perm) {  // SELL-C-sigma: the device system is P A P^T
    const double *bs = b, *xs = x;
    if (!b_dev) {
      PCG_CUDA(cudaMemcpyAsync(w.w, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      bs = w.w;
    }
    PCG_TRY(perm_in(A, bs, w.stage_b, st));
    if (!x_dev) {
      PCG_CUDA(cudaMemcpyAsync(w.q, x, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      xs = w.q;
    }
    PCG_TRY(perm_in(A, xs, v.x, st));
  } else {
    PCG_CUDA(cudaMemcpyAsync(w.stage_b, b, sizeof(double) * n, b_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                             st));
    PCG_CUDA(cudaMemcpyAsync(v.x, x, sizeof(double) * n, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  }
  v.b = w.stage_b;
  PipeState hs;
  memset(&hs, 0, sizeof(hs));
  hs.tol = tol;
  hs.max_iter = max_iter;
  PipeState *dst = (PipeState *)w.pstate;
  if (A->comm) {  // row-partitioned: kernels + collectives, host-polled
    cudaEvent_t f0, f1;
    PCG_CUDA(cudaEventCreate(&f0));
    PCG_CUDA(cudaEventCreate(&f1));
    PCG_CUDA(cudaEventRecord(f0, st));
    PCG_TRY(pd_solve(A, v, tol, max_iter, st, &hs));
    PCG_CUDA(cudaEventRecord(f1, st));
    PCG_CUDA(cudaMemcpyAsync(x, v.x, sizeof(double) * n, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    PCG_TRY(comm_wait(A->comm, st));
    float fms = 0;
    cudaEventElapsedTime(&fms, f0, f1);
    cudaEventDestroy(f0);
    cudaEventDestroy(f1);
    return pipe_report(A, hs, tol, fms, info);
  }
  PCG_CUDA(cudaMemcpyAsync(dst, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));
  void *fn = pipe_fn(A->format == FMT_SELL_TMA ? PCG_FORMAT_SELL : A->format, A->csr_lanes, n);
  if (w.ppgrid == 0) {
    int nbk = 0;
    PCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbk, fn, BLOCK, 0));
    w.ppgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms(A->device) * std::min(nbk, 8),
                                                          std::max<int64_t>(1, (n + BLOCK - 1) / BLOCK)));
  }
  SellView S = A->sell();
  CsrView Cv = A->csr();
  double *part = w.partials;  // 2 x 3 x grid (<= 8 x SMs; partials hold 6 x 32 x SMs)
  GridBar *bar = (GridBar *)w.ppbar;
  void *args[] = {&S, &Cv, &v, &dst, &part, &bar};
  cudaEvent_t e0, e1;
  PCG_CUDA(cudaEventCreate(&e0));
  PCG_CUDA(cudaEventCreate(&e1));
  PCG_CUDA(cudaEventRecord(e0, st));
  PCG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(w.ppgrid), dim3(BLOCK), args, 0, st));
  count_launch();
  PCG_CUDA(cudaEventRecord(e1, st));
  if (A->d_perm) {
    if (x_dev) {
      PCG_TRY(perm_out(A, v.x, x, st));
    } else {
      PCG_TRY(perm_out(A, v.x, w.w, st));
      PCG_CUDA(cudaMemcpyAsync(x, w.w, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    }
  } else {
    PCG_CUDA(cudaMemcpyAsync(x, v.x, sizeof(double) * n, x_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
  }
  PCG_CUDA(cudaMemcpyAsync(&hs, dst, sizeof(hs), cudaMemcpyDeviceToHost, st));
  PCG_TRY(comm_wait(A->comm, st));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return pipe_report(A, hs, tol, ms, info);
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_solve_pipelined(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                                          void *stream, pcg_info *info) {
  pcgb::NvtxRange nvtx_("pcg:pcg_solve_pipelined");
  if (!A || ((!b || !x) && A->n > 0)) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_pipelined: null argument");
  if (!(tol > 0.0) || max_iter < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_pipelined: tol > 0 and max_iter >= 1");
  if (A->n == 0) {
    if (info) {
      memset(info, 0, sizeof(*info));
      info->converged = 1;
    }
    return PCG_OK;
  }
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  return pipe_impl(A, b, x, tol, max_iter, (cudaStream_t)stream, info);
}
