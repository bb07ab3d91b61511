// persist.cu — the whole Jacobi-PCG loop of a single-GPU solve as ONE
// cooperative (co-resident, persistent) kernel.
//
// Same dataflow and bytes as the 3-pass schedule of solver.cu (K1a p/x update,
// K1b SpMV + sigma, K2 r/z update + rho', gamma; 12 nnz + 4(n+1) + 96 n bytes per
// iteration), but the three passes are separated by grid-wide barriers instead
// of kernel boundaries, and the scalar recurrence (alpha, beta, the stop test of
// SURVEY §8(c).8) is evaluated redundantly and identically by every block from
// the fixed-order block partials — so there is no finisher, no launch and no
// graph node per pass.  For systems whose passes take tens of microseconds
// (C1-C4) the kernel boundaries, not HBM, set the iteration time; for C5 the
// 3-pass graph is kept (the host picks by size, PCG_PERSIST overrides).
//
// Co-residency of all blocks is guaranteed by cudaLaunchCooperativeKernel with a
// grid of at most (resident blocks per SM) x SMs; the barrier is a sense counter
// in global memory.  One launch per solve (per residual replacement).
#include <cstdlib>

#include "matrix.cuh"
#include "rows.cuh"
#include "coop.cuh"

namespace pcgb {

// SCHED 3: K1a | K1b | K2, three barriers per iteration (96 n bytes); SCHED 2: K1 (SpMV
// with p = z + beta p recomputed at gather time, x += alpha_prev p_old) | K2, two
// barriers (88 n bytes, twice the gathers).
#ifndef PCG_PERSIST_MINB  // resident blocks per SM the persistent kernel is compiled for
#define PCG_PERSIST_MINB 3
#endif

template <int FMT, int L, int SCHED>
__global__ void __launch_bounds__(BLOCK, PCG_PERSIST_MINB) pcg_persist_kernel(SellView S, CsrView C, Vecs v, Scalars *sc, double *part,
                                                            GridBar *bar) {
  __shared__ double sm[2][WARPS];
  __shared__ double s_tot[2];
  const int64_t n = FMT == PCG_FORMAT_SELL ? S.n : C.n;
  // recurrence state: read once, then evolved identically by every block
  double rho = sc->rho, beta = sc->beta, alpha = sc->alpha;
  const double tol = sc->tol, nb = sc->nb;
  long long k = sc->k;
  const long long max_iter = sc->max_iter;
  int done = sc->done;
  double sigma = sc->sigma, gamma = sc->gamma, relres_rec = sc->relres_rec;
  double *__restrict__ p = v.p0;  // SCHED 3 (SCHED 2 tracks p[par])
  double *__restrict__ q = v.q;
  const int64_t npair = n >> 1;
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nth = (int64_t)gridDim.x * BLOCK;
  double *part_s = part, *part_rz = part + gridDim.x;  // sigma | (rho', gamma)
  int par = sc->parity;  // SCHED 2: p[par] is the current direction
  while (done == DONE_RUNNING) {
    if (SCHED == 2) {
      // ---- K1: p_new = z + beta p_old ; q = A p_new ; sigma ; x += alpha_prev p_old
      double acc = 0.0;
      const double *__restrict__ pold = par ? v.p1 : v.p0;
      double *__restrict__ pnew = par ? v.p0 : v.p1;
      if (FMT == PCG_FORMAT_SELL) {
        k1_sell_rows<8>(S, beta, alpha, pold, pnew, v.z, v.x, q, acc);
      } else {
        auto gather = [&](int j) { return __fma_rn(beta, ld_weak(pold + j), ld_weak(v.z + j)); };
        auto epi = [&](int64_t i, double s) {
          const double po = pold[i];
          const double pi = __fma_rn(beta, po, v.z[i]);
          pnew[i] = pi;
          q[i] = s;
          v.x[i] = __fma_rn(alpha, po, v.x[i]);
          acc = __fma_rn(pi, s, acc);
        };
        csr_rows<L>(C, gather, epi);
      }
      double red[1] = {acc};
      block_sum<1>(red, sm);
      if (threadIdx.x == 0) part_s[blockIdx.x] = red[0];
      par ^= 1;
      p = pnew;
    } else {
    // ---- K1a: p = z + beta p ; x += alpha_prev p_old
    {
      double2 *__restrict__ p2 = reinterpret_cast<double2 *>(p);
      double2 *__restrict__ x2 = reinterpret_cast<double2 *>(v.x);
      const double2 *__restrict__ z2 = reinterpret_cast<const double2 *>(v.z);
      for (int64_t i = tid; i < npair; i += nth) {
        const double2 zz = __ldcs(z2 + i), po = p2[i];
        double2 xx = __ldcs(x2 + i);
        xx.x = __fma_rn(alpha, po.x, xx.x);
        xx.y = __fma_rn(alpha, po.y, xx.y);
        p2[i] = make_double2(__fma_rn(beta, po.x, zz.x), __fma_rn(beta, po.y, zz.y));
        __stcs(x2 + i, xx);
      }
      if ((n & 1) && tid == 0) {
        const double po = p[n - 1];
        v.x[n - 1] = __fma_rn(alpha, po, v.x[n - 1]);
        p[n - 1] = __fma_rn(beta, po, v.z[n - 1]);
      }
    }
    grid_sync(bar);
    // ---- K1b: q = A p ; sigma = p.q
    {
      double acc = 0.0;
      auto gather = [&](int j) { return ld_weak(p + j); };
      auto epi = [&](int64_t i, double s) {
        __stcs(q + i, s);
        acc = __fma_rn(ld_weak(p + i), s, acc);
      };
      if (FMT == PCG_FORMAT_SELL) sell_rows(S, gather, epi);
      else csr_rows<L>(C, gather, epi);
      double red[1] = {acc};
      block_sum<1>(red, sm);
      if (threadIdx.x == 0) part_s[blockIdx.x] = red[0];
    }
    }
    grid_sync(bar);
    {
      double t[1];
      all_blocks_sum<1>(part_s, t, sm, s_tot);
      sigma = t[0];
    }
    if (!(sigma > 0.0)) {  // p^T A p <= 0: breakdown (x already holds every applied update)
      done = DONE_BREAKDOWN;
      break;
    }
    alpha = rho / sigma;
    k += 1;
    // ---- K2: r -= alpha q ; z = dinv r ; rho' = r.z ; gamma = r.r
    {
      double a0 = 0.0, a1 = 0.0;
      const double2 *__restrict__ q2 = reinterpret_cast<const double2 *>(q);
      const double2 *__restrict__ d2 = reinterpret_cast<const double2 *>(v.dinv);
      double2 *__restrict__ r2 = reinterpret_cast<double2 *>(v.r);
      double2 *__restrict__ z2 = reinterpret_cast<double2 *>(v.z);
      for (int64_t i = tid; i < npair; i += nth) {
        const double2 qq = __ldcs(q2 + i), dd = __ldg(d2 + i);
        double2 rr = r2[i];
        rr.x = __fma_rn(-alpha, qq.x, rr.x);
        rr.y = __fma_rn(-alpha, qq.y, rr.y);
        const double2 zz = make_double2(dd.x * rr.x, dd.y * rr.y);
        r2[i] = rr;
        z2[i] = zz;
        a0 = __fma_rn(rr.x, zz.x, a0);
        a0 = __fma_rn(rr.y, zz.y, a0);
        a1 = __fma_rn(rr.x, rr.x, a1);
        a1 = __fma_rn(rr.y, rr.y, a1);
      }
      if ((n & 1) && tid == 0) {
        const int64_t i = n - 1;
        const double ri = __fma_rn(-alpha, q[i], v.r[i]);
        const double zi = v.dinv[i] * ri;
        v.r[i] = ri;
        v.z[i] = zi;
        a0 = __fma_rn(ri, zi, a0);
        a1 = __fma_rn(ri, ri, a1);
      }
      double red[2] = {a0, a1};
      block_sum<2>(red, sm);
      if (threadIdx.x == 0) {
        part_rz[blockIdx.x] = red[0];
        part_rz[gridDim.x + blockIdx.x] = red[1];
      }
    }
    grid_sync(bar);
    double t[2];
    all_blocks_sum<2>(part_rz, t, sm, s_tot);
    gamma = t[1];
    const double rr = sqrt(gamma);
    relres_rec = rr / nb;
    if (rr <= tol * nb) {
      done = DONE_CONVERGED;  // alpha_k still owed to x (tail_kernel)
    } else if (!(gamma == gamma)) {
      done = DONE_NONFINITE;
    } else if (k >= max_iter) {
      done = DONE_MAXIT;
    } else {
      beta = t[0] / rho;
      rho = t[0];
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    sc->rho = rho;
    sc->beta = beta;
    sc->alpha = alpha;
    sc->sigma = sigma;
    sc->gamma = gamma;
    sc->relres_rec = relres_rec;
    sc->k = k;
    sc->done = done;
    sc->parity = SCHED == 2 ? par : 0;
    sc->graph_launches += 1;
  }
}

// ---------------------------------------------------------------- host side
template <int SCHED>
static void *persist_fn_s(int fmt, int lanes) {
  if (fmt == PCG_FORMAT_SELL) return (void *)pcg_persist_kernel<PCG_FORMAT_SELL, 1, SCHED>;
  switch (lanes) {
    case 1: return (void *)pcg_persist_kernel<PCG_FORMAT_CSR, 1, SCHED>;
    case 2: return (void *)pcg_persist_kernel<PCG_FORMAT_CSR, 2, SCHED>;
    case 4: return (void *)pcg_persist_kernel<PCG_FORMAT_CSR, 4, SCHED>;
    case 8: return (void *)pcg_persist_kernel<PCG_FORMAT_CSR, 8, SCHED>;
    case 16: return (void *)pcg_persist_kernel<PCG_FORMAT_CSR, 16, SCHED>;
    default: return (void *)pcg_persist_kernel<PCG_FORMAT_CSR, 32, SCHED>;
  }
}

static void *persist_fn(int fmt, int lanes, int sched) {
  return sched == 2 ? persist_fn_s<2>(fmt, lanes) : persist_fn_s<3>(fmt, lanes);
}

// Schedule inside the persistent kernel: 2 passes (two barriers, twice the gathers) for
// the smallest, barrier-bound systems, else 3 (measured: C1 0.85 vs 1.00 ms; C2 0.182 vs
// 0.160 s, C4 0.044 vs 0.036 s, C3 1.20 vs 0.90 s); PCG_SCHEDULE forces either.
int persist_schedule(const pcg_matrix *A) {
  return getenv("PCG_SCHEDULE") ? A->schedule : (A->n < (int64_t(1) << 16) ? 2 : 3);
}

// Whether the handle solves with the persistent kernel: one GPU, SELL or CSR, and a
// system small enough that kernel boundaries matter (PCG_PERSIST=0/1 forces it).
bool persist_wanted(const pcg_matrix *A) {
  if (A->comm || (A->format != PCG_FORMAT_SELL && A->format != PCG_FORMAT_CSR)) return false;
  if (getenv("PCG_NO_GRAPH")) return false;  // profiling: one launch per pass
  const char *e = getenv("PCG_PERSIST");
  if (e) return atoi(e) != 0;
  // measured crossover (µs per iteration, persistent -> graph): rows of <= 8 entries run the
  // graph loop's one-chunk SpMV at 4 blocks/SM and its x deferral, and win from ~4M rows
  // (C1 4.2M 121.6 -> 113.3, C2 4.2M 132.0 -> 131.3, C5 construction 16.6M 498 -> 461;
  // 2M rows: C4 62 -> 73); longer rows keep the persistent kernel up to 32M (C3 4.2M
  // 177 -> 192, C6 16.6M 754 -> 763)
  return A->n <= (A->short_rows ? int64_t(3) << 20 : int64_t(32) << 20);
}

pcg_status persist_launch(pcg_matrix *A, Vecs v, cudaStream_t st) {
  SolveWork &w = A->work;
  void *fn = persist_fn(A->format, A->csr_lanes, persist_schedule(A));
  if (!w.pbar) {
    PCG_CUDA(cudaMalloc(&w.pbar, sizeof(GridBar)));
    PCG_CUDA(cudaMemset(w.pbar, 0, sizeof(GridBar)));
    int b = 0;
    PCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fn, BLOCK, 0));
    const int64_t need = A->format == PCG_FORMAT_SELL ? (A->n_slices + WARPS - 1) / WARPS
                                                     : (A->n * A->csr_lanes + BLOCK - 1) / BLOCK;
    w.pgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms(A->device) * std::min(b, 8),
                                                        std::max<int64_t>(need, 1)));
  }
  SellView S = A->sell();
  CsrView C = A->csr();
  Scalars *sc = w.sc;
  double *part = w.partials;  // 3 x grid (<= 8 x SMs; partials hold 6 x 32 x SMs)
  GridBar *bar = (GridBar *)w.pbar;
  void *args[] = {&S, &C, &v, &sc, &part, &bar};
  PCG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(w.pgrid), dim3(BLOCK), args, 0, st));
  count_launch();
  return PCG_OK;
}

}  // namespace pcgb
