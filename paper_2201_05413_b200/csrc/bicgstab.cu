// bicgstab.cu — right-preconditioned BiCGSTAB with (Block-)Jacobi: the Krylov
// solver the paper selects (Block-Jacobi P:194), for the
// nonsymmetric systems CG cannot take (the Table 1 identity-row grids).
// SURVEY §8(f) N2; the algorithm and every reading are DESIGN.md R2, restated:
//
//   r = b - A x ; r^ = fixed pseudo-random vector ; rho_old = alpha = omega = 1 ; p = v = 0
//   loop:  rho = r^.r ;  beta = (rho/rho_old)(alpha/omega)
//          p = r + beta (p - omega v) ; p^ = M^-1 p ; v = A p^ ; alpha = rho / (r^.v)
//          s = r - alpha v ;  stop if ||s|| <= tol ||b||  (x += alpha p^)
//          s^ = M^-1 s ; t = A s^ ; omega = (t.s)/(t.t)
//          x += alpha p^ + omega s^ ; r = s - omega t ; stop if ||r|| <= tol ||b||
//   stop -> true residual ||b - A x||/||b|| (Eq. relativeError) decides; else
//   restart from x (same r^), iterations keep counting.
//
// Two device schedules of the same five passes per iteration — two SpMVs
// (sell_rows / csr_rows of rows.cuh) and three streaming passes:
//  * graph (default): five kernels per iteration in a CUDA-graph conditional WHILE
//    loop; last-block finishers evaluate the scalars on the device;
//  * persist (PCG_BICG=persist): the whole solve (init, iterations, exit check,
//    restarts) as ONE cooperative kernel, passes separated by grid barriers, every
//    block evaluating the scalars identically from fixed-order block partials.
// Block-Jacobi applies the LU factors (partial pivoting) of each bs x bs diagonal
// block, computed at setup, one thread per block — bitwise the oracle's M^-1.
#include <cstring>

#include "coop.cuh"
#include "matrix.cuh"
#include "rows.cuh"

namespace pcgb {

struct BicgVecs {
  double *x, *r, *rh, *p, *ph, *v, *sh, *t;
  const double *b;
  const double *dinv;  // bs = 1
  const double *lu;    // bs > 1: [block][bs][bs] LU factors of the diagonal blocks (unit L, U)
  const int *piv;      // bs > 1: [block][bs] row permutation of the partial pivoting
  const int *iperm;    // SELL-C-sigma handles: device row of original row o (else null)
};

struct BicgState {
  double tol, nb, relres_rec, relres_true;
  long long k, max_iter, restarts;
  int done, pad;
};

__device__ __forceinline__ uint64_t bicg_mix(uint64_t seed, uint64_t idx) {
  uint64_t z = seed + (idx + 1) * 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// r^_i = 2 u(5413, i) - 1 on the ORIGINAL row index (perm maps SELL-C-sigma rows back)
// (distributed handles: row0 = the rank's first global row)
__global__ void shadow_kernel(int64_t n, const int *__restrict__ perm, int64_t row0, double *__restrict__ rh) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t g = perm ? (uint64_t)perm[i] : (uint64_t)(row0 + i);
    const double u = (double)(bicg_mix(5413ULL, g) >> 11) * (1.0 / 9007199254740992.0);
    rh[i] = __dsub_rn(__dmul_rn(2.0, u), 1.0);
  }
}

// LU factors (partial pivoting, Doolittle, in place) of the bs x bs diagonal blocks
// (rows/cols [blk*bs, +m)), one thread per block.  Written with explicitly rounded
// operations in the order of the oracle's bj_setup (oracle.c), so the factors —
// and with bj_apply below every application of M^-1 — are bitwise the oracle's.
// Output: lu[blk][bs][bs] (unit L below, U on and above the diagonal), piv[blk][bs].
// On a SELL-C-sigma handle (device system P A P^T) the blocks are still consecutive
// rows of the CALLER's numbering: original row o lives at device row iperm[o], and a
// device column c is original column perm[c].
template <int BS>
__global__ void bj_lu_kernel(int64_t n, const int *__restrict__ rp, const int *__restrict__ col,
                             const double *__restrict__ val, const int *__restrict__ perm,
                             const int *__restrict__ iperm, double *__restrict__ lu, int *__restrict__ piv, int *err) {
  const int64_t blk = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nblk = (n + BS - 1) / BS;
  if (blk >= nblk) return;
  const int64_t r0 = blk * BS;
  const int m = (int)((r0 + BS <= n) ? BS : n - r0);
  double *D = lu + blk * BS * BS;
  int *pv = piv + blk * BS;
  for (int a = 0; a < BS * BS; a++) D[a] = 0.0;
  for (int a = 0; a < m; a++) {
    const int64_t dr = iperm ? iperm[r0 + a] : r0 + a;
    for (int k = rp[dr]; k < rp[dr + 1]; k++) {
      const int64_t c = (perm ? perm[col[k]] : col[k]) - r0;
      if (c >= 0 && c < m) D[a * BS + c] = val[k];
    }
  }
  for (int a = 0; a < BS; a++) pv[a] = a;
  for (int c = 0; c < m; c++) {
    int p = c;
    for (int a = c + 1; a < m; a++)
      if (fabs(D[a * BS + c]) > fabs(D[p * BS + c])) p = a;
    if (D[p * BS + c] == 0.0) {
      atomicExch(err, 1);
      return;
    }
    if (p != c) {
      for (int q = 0; q < m; q++) {
        const double t = D[c * BS + q];
        D[c * BS + q] = D[p * BS + q];
        D[p * BS + q] = t;
      }
      const int t = pv[c];
      pv[c] = pv[p];
      pv[p] = t;
    }
    for (int a = c + 1; a < m; a++) {
      const double f = __ddiv_rn(D[a * BS + c], D[c * BS + c]);
      D[a * BS + c] = f;
      for (int q = c + 1; q < m; q++) D[a * BS + q] = __dsub_rn(D[a * BS + q], __dmul_rn(f, D[c * BS + q]));
    }
  }
}

// bs code of the ILU(0) Block-Jacobi preconditioner (its block size lives in the plan)
constexpr int BS_ILU = -1;

enum { BD_RUNNING = 0, BD_CONVERGED = 1, BD_MAXIT = 2, BD_BREAKDOWN = 3, BD_ZERO_RHS = 4, BD_NONFINITE = 5 };

// Block-uniform scalar state lives in shared memory (thread 0 writes after the
// fixed-order reductions, a barrier publishes), not in registers across the
// passes; each pass is its own non-inlined function, so the SpMV passes get a
// register allocation of their own (no spills in the gather loops).
struct BicgShared {
  double rho, rho_old, alpha, omega, beta, nb, relres_rec, relres_true;
  long long k, restarts;
  int done, need_resid, half;
};

enum { SP_RESID = 0, SP_AV = 1, SP_AT = 2, SP_FINAL = 3 };

// the SpMV passes: RESID w = b - A x (r = w, p = v = 0; sums w.w, r^.w, b.b),
// AV v = A p^ (r^.v), AT t = A s^ (t.s, t.t), FINAL w = b - A x (w.w)
template <int FMT, int L, int MODE>
__device__ __forceinline__ void spmv_body(const SellViewDia &S, const CsrView &C, const BicgVecs &v, double &a0,
                                          double &a1, double &a2) {
  const double *__restrict__ G = MODE == SP_AV ? v.ph : (MODE == SP_AT ? v.sh : v.x);
  auto gather = [&](int j) { return ld_weak(G + j); };  // also inside the cooperative kernel
  auto epi = [&](int64_t i, double sv) {
    if (MODE == SP_RESID || MODE == SP_FINAL) {
      const double bi = v.b[i];
      const double w = bi - sv;
      a0 = __fma_rn(w, w, a0);
      if (MODE == SP_RESID) {
        v.r[i] = w;
        v.p[i] = 0.0;
        v.v[i] = 0.0;
        a1 = __fma_rn(v.rh[i], w, a1);
        a2 = __fma_rn(bi, bi, a2);
      }
    } else if (MODE == SP_AV) {
      v.v[i] = sv;
      a0 = __fma_rn(v.rh[i], sv, a0);
    } else {
      v.t[i] = sv;
      a0 = __fma_rn(sv, v.r[i], a0);
      a1 = __fma_rn(sv, sv, a1);
    }
  };
  if (FMT == PCG_FORMAT_SELL) sell_rows(S, gather, epi);
  else if (FMT == FMT_SELL_SHORT) sell_rows_short(S, gather, epi);  // rows of <= 8 entries (graph schedule)
  else if (FMT == FMT_SELL_DIA) sell_rows_dia(S, gather, epi);
  else csr_rows<L>(C, gather, epi);
}

template <int FMT, int L, int MODE>
__device__ __noinline__ void bicg_spmv_pass(const SellViewDia &S, const CsrView &C, const BicgVecs &v, double *out,
                                            double (*sm)[WARPS]) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  spmv_body<FMT, L, MODE>(S, C, v, a0, a1, a2);
  double red[2] = {a0, a1};
  block_sum<2>(red, sm);
  if (threadIdx.x == 0) {
    out[blockIdx.x] = red[0];
    out[gridDim.x + blockIdx.x] = red[1];
  }
}

// y = M^-1 u on block blk: BS = 1 dinv * u; else P, L, U substitution (oracle bj_apply order)
template <int BS>
__device__ __forceinline__ void bj_apply(const BicgVecs &v, int64_t n, int64_t blk, const double (&u)[BS],
                                         double (&y)[BS]) {
  if (BS == 1) {
    y[0] = __dmul_rn(v.dinv[blk], u[0]);
  } else {
    const double *D = v.lu + blk * BS * BS;
    const int *pv = v.piv + blk * BS;
    const int m = (int)((blk * BS + BS <= n) ? BS : n - blk * BS);
#pragma unroll
    for (int a = 0; a < BS; a++) {  // L z = P u
      double sacc = 0.0;
      const int pr = pv[a];
#pragma unroll
      for (int c = 0; c < BS; c++)
        if (c == pr) sacc = u[c];
#pragma unroll
      for (int c = 0; c < a; c++) sacc = __dsub_rn(sacc, __dmul_rn(D[a * BS + c], y[c]));
      y[a] = sacc;
    }
#pragma unroll
    for (int a = BS - 1; a >= 0; a--) {  // U y = z
      if (a >= m) continue;
      double sacc = y[a];
#pragma unroll
      for (int c = a + 1; c < BS; c++)
        if (c < m) sacc = __dsub_rn(sacc, __dmul_rn(D[a * BS + c], y[c]));
      y[a] = __ddiv_rn(sacc, D[a * BS + a]);
    }
  }
}

// P1 (STAGE 0): p = r + beta (p - omega v) ; p^ = M^-1 p
// P3 (STAGE 1): s = r - alpha v (kept in r) ; s^ = M^-1 s ; partial s.s
template <int BS, int STAGE>
__device__ __forceinline__ void precond_body(const BicgVecs &v, int64_t n, double c1, double c2, double &a0) {
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nth = (int64_t)gridDim.x * BLOCK;
  const int64_t nblk = (n + BS - 1) / BS;
  for (int64_t blk = tid; blk < nblk; blk += nth) {
    double u[BS], y[BS];
    int64_t pos[BS];
#pragma unroll
    for (int a = 0; a < BS; a++) {
      const int64_t o = blk * BS + a;
      pos[a] = (BS > 1 && v.iperm && o < n) ? v.iperm[o] : o;
      const int64_t i = pos[a];
      u[a] = 0.0;
      if (o < n) {
        if (STAGE == 0) {  // c1 = beta, c2 = omega
          u[a] = __fma_rn(c1, __fma_rn(-c2, v.v[i], v.p[i]), v.r[i]);
          v.p[i] = u[a];
        } else {  // c1 = alpha
          u[a] = __fma_rn(-c1, v.v[i], v.r[i]);
          v.r[i] = u[a];
          a0 = __fma_rn(u[a], u[a], a0);
        }
      }
    }
    bj_apply<BS>(v, n, blk, u, y);
    double *dst = STAGE == 0 ? v.ph : v.sh;
#pragma unroll
    for (int a = 0; a < BS; a++)
      if (blk * BS + a < n) dst[pos[a]] = y[a];
  }
}

// Block-Jacobi (BS > 1) on natural row order, one lane per ROW: the BS lanes of a
// block hold its BS rows (vectors and LU rows load coalesced) and meet through
// width-BS shuffles.  Forward substitution: at step c lane c's value is final and is
// broadcast; every lane a > c subtracts L[a][c] y_c — so lane a subtracts its terms
// in the order c = 0, 1, ..., a-1, the oracle's order.  Back substitution from the
// last row up: lane a, once every y_c (c > a) is known, forms its sum over
// c = a+1, a+2, ... ascending and divides by U[a][a].  Explicitly rounded like
// bj_apply, so M^-1 u is bitwise the thread-per-block path (and the oracle's).
template <int BS, int STAGE>
__device__ __forceinline__ void precond_rows(const BicgVecs &v, int64_t n, double c1, double c2, double &a0) {
  const int lane = threadIdx.x & 31, a = lane % BS;
  const int64_t stride = (int64_t)gridDim.x * BLOCK, nr = (n + 31) & ~(int64_t)31;
  for (int64_t i = (int64_t)blockIdx.x * BLOCK + threadIdx.x; i < nr; i += stride) {
    const bool live = i < n;
    const int64_t blk = i / BS;
    const int m = (int)((blk * BS + BS <= n) ? BS : n - blk * BS);
    double u = 0.0;
    if (live) {
      if (STAGE == 0) {  // c1 = beta, c2 = omega
        u = __fma_rn(c1, __fma_rn(-c2, v.v[i], v.p[i]), v.r[i]);
        v.p[i] = u;
      } else {  // c1 = alpha
        u = __fma_rn(-c1, v.v[i], v.r[i]);
        v.r[i] = u;
        a0 = __fma_rn(u, u, a0);
      }
    }
    double D[BS];
    int pr = a;
    if (live) {
      const double2 *row2 = reinterpret_cast<const double2 *>(v.lu + blk * BS * BS + a * BS);
#pragma unroll
      for (int q = 0; q < BS / 2; q++) {
        const double2 d2 = __ldg(row2 + q);
        D[2 * q] = d2.x;
        D[2 * q + 1] = d2.y;
      }
      pr = __ldg(v.piv + blk * BS + a);
    } else {
#pragma unroll
      for (int q = 0; q < BS; q++) D[q] = 0.0;
    }
    // L z = P u
    double sacc = __shfl_sync(0xffffffffu, u, pr, BS);
    double y[BS];
#pragma unroll
    for (int c = 0; c < BS; c++) {
      y[c] = __shfl_sync(0xffffffffu, sacc, c, BS);  // lane c is final at step c
      if (a > c) sacc = __dsub_rn(sacc, __dmul_rn(D[c], y[c]));
    }
    // U y = z, bottom up
#pragma unroll
    for (int k = BS - 1; k >= 0; k--) {
      double t = 0.0;
      if (a == k && k < m) {
        t = y[k];
#pragma unroll
        for (int c = k + 1; c < BS; c++)
          if (c < m) t = __dsub_rn(t, __dmul_rn(D[c], y[c]));
        t = __ddiv_rn(t, D[k]);
      }
      y[k] = __shfl_sync(0xffffffffu, t, k, BS);
    }
    if (live) (STAGE == 0 ? v.ph : v.sh)[i] = y[a];
  }
}

template <int BS, int STAGE>
__device__ __noinline__ void bicg_precond_pass(const BicgVecs &v, int64_t n, double c1, double c2, double *out,
                                               double (*sm)[WARPS]) {
  double a0 = 0.0;
  precond_body<BS, STAGE>(v, n, c1, c2, a0);
  if (STAGE == 1) {
    double red[1] = {a0};
    block_sum<1>(red, sm);
    if (threadIdx.x == 0) out[blockIdx.x] = red[0];
  }
}

// P5: x += alpha p^ + omega s^ ; r = s - omega t ; partials r.r, r^.r
__device__ __forceinline__ void update_body(const BicgVecs &v, int64_t n, double alpha, double omega, double &a0,
                                            double &a1) {
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nth = (int64_t)gridDim.x * BLOCK;
  for (int64_t i = tid; i < n; i += nth) {
    v.x[i] = __fma_rn(omega, v.sh[i], __fma_rn(alpha, v.ph[i], v.x[i]));
    const double ri = __fma_rn(-omega, v.t[i], v.r[i]);
    v.r[i] = ri;
    a0 = __fma_rn(ri, ri, a0);
    a1 = __fma_rn(v.rh[i], ri, a1);
  }
}

__device__ __noinline__ void bicg_update_pass(const BicgVecs &v, int64_t n, double alpha, double omega, double *out,
                                              double (*sm)[WARPS]) {
  double a0 = 0.0, a1 = 0.0;
  update_body(v, n, alpha, omega, a0, a1);
  double red[2] = {a0, a1};
  block_sum<2>(red, sm);
  if (threadIdx.x == 0) {
    out[blockIdx.x] = red[0];
    out[gridDim.x + blockIdx.x] = red[1];
  }
}

template <int FMT, int L, int BS>
__global__ void __launch_bounds__(BLOCK, 3) bicg_kernel(SellViewDia S_, CsrView C_, BicgVecs v_, BicgState *st,
                                                        double *part, GridBar *bar) {
  __shared__ double sm[2][WARPS];
  __shared__ double s_tot[2];
  __shared__ BicgShared q;
  __shared__ SellViewDia S;
  __shared__ CsrView C;
  __shared__ BicgVecs v;
  if (threadIdx.x == 0) {
    S = S_;
    C = C_;
    v = v_;
  }
  __syncthreads();
  const int64_t n = FMT == PCG_FORMAT_SELL ? S.n : C.n;
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nth = (int64_t)gridDim.x * BLOCK;
  double *pa = part, *pb = part + 2 * gridDim.x;  // two alternating partial regions
  // ---- ||b||
  {
    double a0 = 0.0;
    for (int64_t i = tid; i < n; i += nth) a0 = __fma_rn(v.b[i], v.b[i], a0);
    double red[1] = {a0};
    block_sum<1>(red, sm);
    if (threadIdx.x == 0) pa[blockIdx.x] = red[0];
    grid_sync(bar);
    double t[1];
    all_blocks_sum<1>(pa, t, sm, s_tot);
    if (threadIdx.x == 0) {
      q.nb = sqrt(t[0]);
      q.k = st->k;
      q.restarts = 0;
      q.relres_rec = q.relres_true = 0.0;
      q.rho = q.rho_old = q.alpha = q.omega = 1.0;
      q.done = q.nb == 0.0 ? BD_ZERO_RHS : (!(q.nb == q.nb) ? BD_NONFINITE : BD_RUNNING);
      q.need_resid = 1;
    }
    __syncthreads();
  }
  if (q.done != BD_RUNNING)
    for (int64_t i = tid; i < n; i += nth) v.x[i] = 0.0;
  const double tol = st->tol;
  const long long max_iter = st->max_iter;
  while (q.done == BD_RUNNING) {
    if (q.need_resid) {  // (re)start / exit check
      bicg_spmv_pass<FMT, L, SP_RESID>(S, C, v, pb, sm);
      grid_sync(bar);
      double t[2];
      all_blocks_sum<2>(pb, t, sm, s_tot);
      if (threadIdx.x == 0) {
        const double rr = sqrt(t[0]);
        q.relres_rec = rr / q.nb;
        if (q.k > 0 || q.restarts > 0) q.relres_true = q.relres_rec;  // this pass was an exit check
        if (rr <= tol * q.nb) {
          q.relres_true = q.relres_rec;
          q.done = BD_CONVERGED;
        } else {
          if (q.k > 0) q.restarts++;
          q.rho = t[1];
          q.rho_old = q.alpha = q.omega = 1.0;
          q.need_resid = 0;
        }
      }
      __syncthreads();
      if (q.done != BD_RUNNING) break;
    }
    if (threadIdx.x == 0) {
      if (q.k >= max_iter) q.done = BD_MAXIT;
      else if (q.rho == 0.0 || !(q.rho == q.rho)) q.done = q.rho == 0.0 ? BD_BREAKDOWN : BD_NONFINITE;
      else q.beta = (q.rho / q.rho_old) * (q.alpha / q.omega);
    }
    __syncthreads();
    if (q.done != BD_RUNNING) break;
    bicg_precond_pass<BS, 0>(v, n, q.beta, q.omega, nullptr, sm);  // P1
    grid_sync(bar);
    bicg_spmv_pass<FMT, L, SP_AV>(S, C, v, pa, sm);  // P2
    grid_sync(bar);
    {
      double t[2];
      all_blocks_sum<2>(pa, t, sm, s_tot);
      if (threadIdx.x == 0) {
        if (t[0] == 0.0 || !(t[0] == t[0])) {
          q.done = t[0] == 0.0 ? BD_BREAKDOWN : BD_NONFINITE;
        } else {
          q.alpha = q.rho / t[0];
          q.k++;
        }
      }
      __syncthreads();
      if (q.done != BD_RUNNING) break;
    }
    bicg_precond_pass<BS, 1>(v, n, q.alpha, 0.0, pb, sm);  // P3
    grid_sync(bar);
    {
      double t[1];
      all_blocks_sum<1>(pb, t, sm, s_tot);
      if (threadIdx.x == 0) {
        const double ss = sqrt(t[0]);
        q.half = ss <= tol * q.nb;
        if (q.half) q.relres_rec = ss / q.nb;
      }
      __syncthreads();
      if (q.half) {  // converged at the half step: x += alpha p^, then the exit check
        const double alpha = q.alpha;
        for (int64_t i = tid; i < n; i += nth) v.x[i] = __fma_rn(alpha, v.ph[i], v.x[i]);
        grid_sync(bar);
        if (threadIdx.x == 0) q.need_resid = 1;
        __syncthreads();
        continue;
      }
    }
    bicg_spmv_pass<FMT, L, SP_AT>(S, C, v, pa, sm);  // P4
    grid_sync(bar);
    {
      double t[2];
      all_blocks_sum<2>(pa, t, sm, s_tot);
      if (threadIdx.x == 0) q.omega = t[1] > 0.0 ? t[0] / t[1] : 0.0;
      __syncthreads();
    }
    bicg_update_pass(v, n, q.alpha, q.omega, pb, sm);  // P5
    grid_sync(bar);
    {
      double t[2];
      all_blocks_sum<2>(pb, t, sm, s_tot);
      if (threadIdx.x == 0) {
        const double rr = sqrt(t[0]);
        q.relres_rec = rr / q.nb;
        if (rr <= tol * q.nb) {
          q.need_resid = 1;  // exit check (and restart if it fails)
        } else if (q.omega == 0.0) {
          q.done = BD_BREAKDOWN;
        } else {
          q.rho_old = q.rho;
          q.rho = t[1];
        }
      }
      __syncthreads();
    }
  }
  if (q.done == BD_MAXIT || q.done == BD_BREAKDOWN || q.done == BD_NONFINITE) {  // final true residual
    grid_sync(bar);
    bicg_spmv_pass<FMT, L, SP_FINAL>(S, C, v, pa, sm);
    grid_sync(bar);
    double t[1];
    all_blocks_sum<1>(pa, t, sm, s_tot);
    if (threadIdx.x == 0) q.relres_true = sqrt(t[0]) / q.nb;
    __syncthreads();
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->nb = q.nb;
    st->relres_rec = q.relres_rec;
    st->relres_true = q.relres_true;
    st->k = q.k;
    st->restarts = q.restarts;
    st->done = q.done;
  }
}

// ---------------------------------------------------------------- graph schedule
// The same iteration as five kernels per iteration inside a CUDA-graph conditional
// WHILE loop (body = two iterations), for systems whose passes are long enough
// that kernel boundaries cost less than one kernel holding every pass (register
// pressure, spills).  Scalars live in BgScalars on the device; each reducing
// kernel's last block (publish_and_arrive: fixed-order partials) evaluates the
// recurrence exactly as the persistent kernel's thread 0 does.  Any finisher that
// ends the loop sets `stop` (and the graph condition); later kernels of the body
// see `stop` and return.  The exit check / restart (resid pass) runs between
// graph launches, host-driven, as in the CG solver.
struct BgScalars {
  double tol, nb, rho, rho_old, alpha, omega, beta, relres_rec, relres_true;
  double part[3];  // distributed handles: this rank's sums awaiting the allreduce
  long long k, max_iter, restarts;
  int done, half, need_resid, stop;
  unsigned int cnt[4];
};

enum { BR_INIT = 0, BR_CHECK = 1, BR_FINAL = 2 };

__device__ __forceinline__ void bg_stop(BgScalars *sc, int use_cond, cudaGraphConditionalHandle h) {
  sc->stop = 1;
  if (use_cond) cudaGraphSetConditional(h, 0);
}

// loop-top tests of the persistent kernel (max_iter, rho breakdown) and beta
__device__ __forceinline__ void bg_loop_top(BgScalars *sc, int use_cond, cudaGraphConditionalHandle h) {
  if (sc->k >= sc->max_iter) {
    sc->done = BD_MAXIT;
    bg_stop(sc, use_cond, h);
  } else if (sc->rho == 0.0 || !(sc->rho == sc->rho)) {
    sc->done = sc->rho == 0.0 ? BD_BREAKDOWN : BD_NONFINITE;
    bg_stop(sc, use_cond, h);
  } else {
    sc->beta = (sc->rho / sc->rho_old) * (sc->alpha / sc->omega);
  }
}

#define BG_ENTRY()                                                        \
  const volatile BgScalars *vs = sc;                                      \
  if (vs->stop) {                                                         \
    if (use_cond && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, 0); \
    return;                                                               \
  }

// finishers (thread 0 of the last block, or a 1-thread kernel after the allreduce on
// distributed handles) — the persistent kernel's scalar logic
template <int MODE>
__device__ void bg_fin_spmv(BgScalars *sc, const double *t, int rmode, int use_cond, cudaGraphConditionalHandle h) {
  if (MODE == SP_RESID) {
    if (rmode == BR_INIT) {
      sc->nb = sqrt(t[2]);
      sc->k = 0;
      sc->restarts = 0;
      sc->relres_rec = sc->relres_true = 0.0;
      sc->stop = sc->half = sc->need_resid = 0;
      if (sc->nb == 0.0 || !(sc->nb == sc->nb)) {
        sc->done = sc->nb == 0.0 ? BD_ZERO_RHS : BD_NONFINITE;
        return;
      }
      sc->done = BD_RUNNING;
    }
    const double rr = sqrt(t[0]);
    sc->relres_rec = rr / sc->nb;
    if (rmode == BR_CHECK) sc->relres_true = sc->relres_rec;
    if (rr <= sc->tol * sc->nb) {
      sc->relres_true = sc->relres_rec;
      sc->done = BD_CONVERGED;
    } else {
      if (rmode == BR_CHECK) sc->restarts++;
      sc->rho = t[1];
      sc->rho_old = sc->alpha = sc->omega = 1.0;
      sc->stop = sc->half = sc->need_resid = 0;
      bg_loop_top(sc, 0, h);
    }
  } else if (MODE == SP_FINAL) {
    sc->relres_true = sqrt(t[0]) / sc->nb;
  } else if (MODE == SP_AV) {
    if (t[0] == 0.0 || !(t[0] == t[0])) {
      sc->done = t[0] == 0.0 ? BD_BREAKDOWN : BD_NONFINITE;
      bg_stop(sc, use_cond, h);
    } else {
      sc->alpha = sc->rho / t[0];
      sc->k++;
    }
  } else {  // SP_AT
    sc->omega = t[1] > 0.0 ? t[0] / t[1] : 0.0;
  }
}

__device__ void bg_fin_p3(BgScalars *sc, const double *t) {
  const double ss = sqrt(t[0]);
  if (ss <= sc->tol * sc->nb) {
    sc->half = 1;
    sc->relres_rec = ss / sc->nb;
  }
}

__device__ void bg_fin_update(BgScalars *sc, const double *t, int half, int use_cond, cudaGraphConditionalHandle h) {
  if (half) {
    sc->half = 0;
    sc->need_resid = 1;
    bg_stop(sc, use_cond, h);
    return;
  }
  const double rr = sqrt(t[0]);
  sc->relres_rec = rr / sc->nb;
  if (rr <= sc->tol * sc->nb) {
    sc->need_resid = 1;
    bg_stop(sc, use_cond, h);
  } else if (sc->omega == 0.0) {
    sc->done = BD_BREAKDOWN;
    bg_stop(sc, use_cond, h);
  } else {
    sc->rho_old = sc->rho;
    sc->rho = t[1];
    bg_loop_top(sc, use_cond, h);
  }
}

// last block: the finisher (one GPU) or this rank's sums into sc->part (distributed)
template <int NV>
__device__ __forceinline__ bool bg_last(double (&red)[NV], double *part, unsigned int *cnt, BgScalars *sc, int dist,
                                        double (*sm)[WARPS], double (&t)[NV]) {
  block_sum<NV>(red, sm);
  if (!publish_and_arrive<NV>(red, part, cnt)) return false;
  reduce_partials<NV>(part, t, sm);
  if (threadIdx.x != 0) return false;
  *cnt = 0;
  if (dist) {
#pragma unroll
    for (int i = 0; i < NV; i++) sc->part[i] = t[i];
    return false;
  }
  return true;
}

// SpMV kernels: RESID (rmode BR_INIT / BR_CHECK), AV, AT, FINAL (rmode BR_FINAL)
template <int FMT, int L, int MODE>
__global__ void __launch_bounds__(BLOCK, D16_MINB(FMT)) bg_spmv_kernel(SellViewDia S, CsrView C, BicgVecs v, BgScalars *sc,
                                                        double *part, int rmode, int dist, int use_cond,
                                                        cudaGraphConditionalHandle h) {
  __shared__ double sm[3][WARPS];
  if (MODE == SP_AV || MODE == SP_AT) {
    BG_ENTRY();
    if (MODE == SP_AT && vs->half) return;  // converged at the half step: no t this iteration
  }
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  spmv_body<FMT, L, MODE>(S, C, v, a0, a1, a2);
  double red[3] = {a0, a1, a2}, t[3];
  if (bg_last<3>(red, part, &sc->cnt[0], sc, dist, sm, t)) bg_fin_spmv<MODE>(sc, t, rmode, use_cond, h);
}

// P1 / P3 (precond_body); P3's last block takes the half-step test
template <int BS, int STAGE>
__global__ void __launch_bounds__(BLOCK) bg_precond_kernel(int64_t n, BicgVecs v, BgScalars *sc, double *part,
                                                           int dist, int use_cond, cudaGraphConditionalHandle h) {
  __shared__ double sm[1][WARPS];
  BG_ENTRY();
  double a0 = 0.0;
  const bool rows = BS > 1 && v.iperm == nullptr;  // lane-per-row path (natural order)
  if (STAGE == 0) {
    if (rows) precond_rows<BS, 0>(v, n, vs->beta, vs->omega, a0);
    else precond_body<BS, 0>(v, n, vs->beta, vs->omega, a0);
    return;
  }
  if (rows) precond_rows<BS, 1>(v, n, vs->alpha, 0.0, a0);
  else precond_body<BS, 1>(v, n, vs->alpha, 0.0, a0);
  double red[1] = {a0}, t[1];
  if (bg_last<1>(red, part, &sc->cnt[1], sc, dist, sm, t)) bg_fin_p3(sc, t);
}

// P5; at a half-step convergence only x += alpha p^, then the loop ends for the exit check
__global__ void __launch_bounds__(BLOCK) bg_update_kernel(int64_t n, BicgVecs v, BgScalars *sc, double *part,
                                                          int dist, int use_cond, cudaGraphConditionalHandle h) {
  __shared__ double sm[2][WARPS];
  BG_ENTRY();
  const int half = vs->half;
  const double alpha = vs->alpha, omega = vs->omega;
  double a0 = 0.0, a1 = 0.0;
  if (half) {
    const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nth = (int64_t)gridDim.x * BLOCK;
    for (int64_t i = tid; i < n; i += nth) v.x[i] = __fma_rn(alpha, v.ph[i], v.x[i]);
  } else {
    update_body(v, n, alpha, omega, a0, a1);
  }
  double red[2] = {a0, a1}, t[2];
  if (bg_last<2>(red, part, &sc->cnt[2], sc, dist, sm, t)) bg_fin_update(sc, t, half, use_cond, h);
}

// ILU(0) Block-Jacobi (ilu.cu): P1 / P3 without the preconditioner, which runs as its
// own level-scheduled kernel after them.  STAGE 0: p = r + beta (p - omega v);
// STAGE 1: s = r - alpha v (into r) and the partial ||s||^2 (half-step test).
template <int STAGE>
__global__ void __launch_bounds__(BLOCK) bg_vec_kernel(int64_t n, BicgVecs v, BgScalars *sc, double *part,
                                                       int use_cond, cudaGraphConditionalHandle h) {
  __shared__ double sm[1][WARPS];
  BG_ENTRY();
  const int64_t tid = (int64_t)blockIdx.x * BLOCK + threadIdx.x, nth = (int64_t)gridDim.x * BLOCK;
  double a0 = 0.0;
  if (STAGE == 0) {
    const double beta = vs->beta, omega = vs->omega;
    for (int64_t i = tid; i < n; i += nth) v.p[i] = __fma_rn(beta, __fma_rn(-omega, v.v[i], v.p[i]), v.r[i]);
    return;
  }
  const double alpha = vs->alpha;
  for (int64_t i = tid; i < n; i += nth) {
    const double u = __fma_rn(-alpha, v.v[i], v.r[i]);
    v.r[i] = u;
    a0 = __fma_rn(u, u, a0);
  }
  double red[1] = {a0}, t[1];
  if (bg_last<1>(red, part, &sc->cnt[1], sc, 0, sm, t)) bg_fin_p3(sc, t);
}

// distributed handles: the finisher after the allreduce of sc->part
enum { BF_RESID = 0, BF_AV = 1, BF_P3 = 2, BF_AT = 3, BF_UPDATE = 4, BF_FINAL = 5 };
__global__ void bg_finish_kernel(BgScalars *sc, int which, int rmode) {
  const double t[3] = {sc->part[0], sc->part[1], sc->part[2]};
  if (which == BF_RESID) return bg_fin_spmv<SP_RESID>(sc, t, rmode, 0, 0);
  if (which == BF_FINAL) return bg_fin_spmv<SP_FINAL>(sc, t, rmode, 0, 0);
  if (sc->stop) return;  // a finisher earlier in this chunk ended the loop
  if (which == BF_AV) return bg_fin_spmv<SP_AV>(sc, t, 0, 0, 0);
  if (which == BF_P3) return bg_fin_p3(sc, t);
  if (which == BF_AT) {
    if (!sc->half) bg_fin_spmv<SP_AT>(sc, t, 0, 0, 0);
    return;
  }
  bg_fin_update(sc, t, sc->half, 0, 0);
}

// ---------------------------------------------------------------- host side
template <int BS>
static void *bicg_fn(int fmt, int lanes) {
  if (fmt == PCG_FORMAT_SELL) return (void *)bicg_kernel<PCG_FORMAT_SELL, 1, BS>;
  switch (lanes) {
    case 1: return (void *)bicg_kernel<PCG_FORMAT_CSR, 1, BS>;
    case 2: return (void *)bicg_kernel<PCG_FORMAT_CSR, 2, BS>;
    case 4: return (void *)bicg_kernel<PCG_FORMAT_CSR, 4, BS>;
    case 8: return (void *)bicg_kernel<PCG_FORMAT_CSR, 8, BS>;
    case 16: return (void *)bicg_kernel<PCG_FORMAT_CSR, 16, BS>;
    default: return (void *)bicg_kernel<PCG_FORMAT_CSR, 32, BS>;
  }
}

static void *bicg_select(int fmt, int lanes, int bs) {
  switch (bs) {
    case 1: return bicg_fn<1>(fmt, lanes);
    case 2: return bicg_fn<2>(fmt, lanes);
    case 4: return bicg_fn<4>(fmt, lanes);
    default: return bicg_fn<8>(fmt, lanes);
  }
}

// graph schedule: launchers per (format, CSR lanes, block size)
struct BgOps {
  void (*iter)(pcg_matrix *, const BicgVecs &, BgScalars *, double *, cudaStream_t, int, cudaGraphConditionalHandle);
  void (*resid)(pcg_matrix *, const BicgVecs &, BgScalars *, double *, int, cudaStream_t);
};

template <int FMT, int L, int BS>
static void bg_iteration(pcg_matrix *A, const BicgVecs &v, BgScalars *sc, double *part, cudaStream_t st, int use_cond,
                         cudaGraphConditionalHandle h) {
  const SellViewDia S = A->sell_dia();
  const CsrView C = A->csr();
  const int gs = A->grid_spmv, gv = A->grid_vec;
  bg_precond_kernel<BS, 0><<<gv, BLOCK, 0, st>>>(A->n, v, sc, part, 0, use_cond, h);
  bg_spmv_kernel<FMT, L, SP_AV><<<gs, BLOCK, 0, st>>>(S, C, v, sc, part, 0, 0, use_cond, h);
  bg_precond_kernel<BS, 1><<<gv, BLOCK, 0, st>>>(A->n, v, sc, part, 0, use_cond, h);
  bg_spmv_kernel<FMT, L, SP_AT><<<gs, BLOCK, 0, st>>>(S, C, v, sc, part, 0, 0, use_cond, h);
  bg_update_kernel<<<gv, BLOCK, 0, st>>>(A->n, v, sc, part, 0, use_cond, h);
  count_launch(5);
}

template <int FMT, int L>
static void bg_iteration_ilu(pcg_matrix *A, const BicgVecs &v, BgScalars *sc, double *part, cudaStream_t st,
                             int use_cond, cudaGraphConditionalHandle h) {
  const SellViewDia S = A->sell_dia();
  const CsrView C = A->csr();
  const int gs = A->grid_spmv, gv = A->grid_vec;
  bg_vec_kernel<0><<<gv, BLOCK, 0, st>>>(A->n, v, sc, part, use_cond, h);
  ilu_launch(A->work.ilu, v.p, v.ph, &sc->stop, nullptr, st);
  bg_spmv_kernel<FMT, L, SP_AV><<<gs, BLOCK, 0, st>>>(S, C, v, sc, part, 0, 0, use_cond, h);
  bg_vec_kernel<1><<<gv, BLOCK, 0, st>>>(A->n, v, sc, part, use_cond, h);
  ilu_launch(A->work.ilu, v.r, v.sh, &sc->stop, &sc->half, st);
  bg_spmv_kernel<FMT, L, SP_AT><<<gs, BLOCK, 0, st>>>(S, C, v, sc, part, 0, 0, use_cond, h);
  bg_update_kernel<<<gv, BLOCK, 0, st>>>(A->n, v, sc, part, 0, use_cond, h);
  count_launch(5);
}

template <int FMT, int L, int BS>
static void bg_resid(pcg_matrix *A, const BicgVecs &v, BgScalars *sc, double *part, int rmode, cudaStream_t st) {
  if (rmode == BR_FINAL)
    bg_spmv_kernel<FMT, L, SP_FINAL><<<A->grid_spmv, BLOCK, 0, st>>>(A->sell_dia(), A->csr(), v, sc, part, rmode, 0, 0, 0);
  else
    bg_spmv_kernel<FMT, L, SP_RESID><<<A->grid_spmv, BLOCK, 0, st>>>(A->sell_dia(), A->csr(), v, sc, part, rmode, 0, 0, 0);
  count_launch();
}

template <int FMT, int L, int BS>
static BgOps bg_ops_t() {
  return {bg_iteration<FMT, L, BS>, bg_resid<FMT, L, BS>};
}

template <int BS>
static BgOps bg_ops_bs(int fmt, int lanes) {
  if (fmt == FMT_SELL_SHORT) return bg_ops_t<FMT_SELL_SHORT, 1, BS>();
  if (fmt == FMT_SELL_DIA) return bg_ops_t<FMT_SELL_DIA, 1, BS>();
  if (fmt == PCG_FORMAT_SELL) return bg_ops_t<PCG_FORMAT_SELL, 1, BS>();
  switch (lanes) {
    case 1: return bg_ops_t<PCG_FORMAT_CSR, 1, BS>();
    case 2: return bg_ops_t<PCG_FORMAT_CSR, 2, BS>();
    case 4: return bg_ops_t<PCG_FORMAT_CSR, 4, BS>();
    case 8: return bg_ops_t<PCG_FORMAT_CSR, 8, BS>();
    case 16: return bg_ops_t<PCG_FORMAT_CSR, 16, BS>();
    default: return bg_ops_t<PCG_FORMAT_CSR, 32, BS>();
  }
}

template <int FMT, int L>
static BgOps bg_ops_ilu_t() {
  return {bg_iteration_ilu<FMT, L>, bg_resid<FMT, L, 1>};
}

// the SpMV engine of the graph / distributed schedules: SELL (TMA handles too), the
// one-chunk engine where every row has <= 8 entries (pcg_matrix::short_rows), or CSR
static int bg_fmt(const pcg_matrix *A) {
  const int f = A->format == FMT_SELL_TMA ? PCG_FORMAT_SELL : A->format;
  return f == PCG_FORMAT_SELL && A->short_rows ? (A->d_sdoff ? FMT_SELL_DIA : FMT_SELL_SHORT) : f;
}

static BgOps bg_ops(int fmt, int lanes, int bs) {
  if (bs == BS_ILU) {
    if (fmt == FMT_SELL_SHORT) return bg_ops_ilu_t<FMT_SELL_SHORT, 1>();
    if (fmt == FMT_SELL_DIA) return bg_ops_ilu_t<FMT_SELL_DIA, 1>();
    if (fmt == PCG_FORMAT_SELL) return bg_ops_ilu_t<PCG_FORMAT_SELL, 1>();
    switch (lanes) {
      case 1: return bg_ops_ilu_t<PCG_FORMAT_CSR, 1>();
      case 2: return bg_ops_ilu_t<PCG_FORMAT_CSR, 2>();
      case 4: return bg_ops_ilu_t<PCG_FORMAT_CSR, 4>();
      case 8: return bg_ops_ilu_t<PCG_FORMAT_CSR, 8>();
      case 16: return bg_ops_ilu_t<PCG_FORMAT_CSR, 16>();
      default: return bg_ops_ilu_t<PCG_FORMAT_CSR, 32>();
    }
  }
  switch (bs) {
    case 1: return bg_ops_bs<1>(fmt, lanes);
    case 2: return bg_ops_bs<2>(fmt, lanes);
    case 4: return bg_ops_bs<4>(fmt, lanes);
    default: return bg_ops_bs<8>(fmt, lanes);
  }
}

// default: the graph schedule (measured faster on both Table 1 grids);
// PCG_BICG=persist selects the single cooperative kernel
static int bicg_use_graph(const pcg_matrix *) {
  const char *e = getenv("PCG_BICG");
  return !(e && !strcmp(e, "persist"));
}

static pcg_status bg_build(pcg_matrix *A, const BgOps &ops, const BicgVecs &v, int bs) {
  SolveWork &w = A->work;
  const int key = bs == BS_ILU ? -(int)std::min<int64_t>(ilu_block_rows(w.ilu), 1 << 30) : bs;
  if (w.bg_exec && w.bg_bs == key) return PCG_OK;
  if (w.bg_exec) cudaGraphExecDestroy(w.bg_exec);
  if (w.bg_graph) cudaGraphDestroy(w.bg_graph);
  w.bg_exec = nullptr;
  w.bg_graph = nullptr;
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
  PCG_CUDA(cudaStreamBeginCaptureToGraph(cap, np.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                         cudaStreamCaptureModeThreadLocal));
  BgScalars *sc = (BgScalars *)w.bgsc;
  for (int u = 0; u < 2; u++) ops.iter(A, v, sc, w.partials, cap, 1, h);  // body = two iterations
  cudaGraph_t out;
  cudaError_t e = cudaStreamEndCapture(cap, &out);
  cudaStreamDestroy(cap);
  PCG_CUDA(e);
  PCG_CUDA(cudaGraphInstantiate(&w.bg_exec, g, 0));
  w.bg_graph = g;
  w.bg_bs = key;
  return PCG_OK;
}

// graph-scheduled solve; fills the persistent kernel's BicgState fields
static pcg_status bg_solve(pcg_matrix *A, const BicgVecs &v, int bs, double tol, int64_t max_iter, cudaStream_t st,
                           BicgState *hs) {
  SolveWork &w = A->work;
  if (!w.bgsc) PCG_CUDA(cudaMalloc(&w.bgsc, sizeof(BgScalars)));
  const BgOps ops = bg_ops(bg_fmt(A), A->csr_lanes, bs);
  PCG_TRY(bg_build(A, ops, v, bs));
  BgScalars *sc = (BgScalars *)w.bgsc, h;
  memset(&h, 0, sizeof(h));
  h.tol = tol;
  h.max_iter = max_iter;
  PCG_CUDA(cudaMemcpyAsync(sc, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  auto read = [&]() -> pcg_status {
    PCG_CUDA(cudaGetLastError());
    PCG_CUDA(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
    PCG_TRY(comm_wait(A->comm, st));
    return PCG_OK;
  };
  ops.resid(A, v, sc, w.partials, BR_INIT, st);
  PCG_TRY(read());
  if (h.done == BD_ZERO_RHS || h.done == BD_NONFINITE) PCG_CUDA(cudaMemsetAsync(v.x, 0, sizeof(double) * A->n, st));
  const bool direct = getenv("PCG_NO_GRAPH") != nullptr;  // profilers: the same kernels, launched directly
  while (h.done == BD_RUNNING) {
    if (direct) {
      for (int u = 0; u < 8; u++) ops.iter(A, v, sc, w.partials, st, 0, 0);
    } else {
      PCG_CUDA(cudaGraphLaunch(w.bg_exec, st));
      count_launch();
    }
    PCG_TRY(read());
    if (direct && h.stop == 0 && h.done == BD_RUNNING) continue;
    if (h.done != BD_RUNNING) break;
    ops.resid(A, v, sc, w.partials, BR_CHECK, st);  // exit check (need_resid), restart if it fails
    PCG_TRY(read());
  }
  if (h.done == BD_MAXIT || h.done == BD_BREAKDOWN || h.done == BD_NONFINITE) {
    ops.resid(A, v, sc, w.partials, BR_FINAL, st);
    PCG_TRY(read());
  }
  hs->nb = h.nb;
  hs->relres_rec = h.relres_rec;
  hs->relres_true = h.relres_true;
  hs->k = h.k;
  hs->restarts = h.restarts;
  hs->done = h.done;
  return PCG_OK;
}

// distributed handles (csr_create_dist; point Jacobi): the same five passes as
// direct launches with the exchanges between them — halo of p^ before v = A p^ and
// of s^ before t = A s^; an allreduce of this rank's sums before every finisher (four
// per iteration: r^.v | s.s | t.s, t.t | r.r, r^.r).  U iterations per host poll;
// the exit check / restart between polls, as on one GPU.
template <int FMT, int L>
struct BgdOps {
  static void spmv(pcg_matrix *A, const BicgVecs &v, BgScalars *sc, int mode, int rmode, cudaStream_t st) {
    double *part = A->work.partials;
    const SellViewDia S = A->sell_dia();
    const CsrView C = A->csr();
    switch (mode) {
      case SP_RESID: bg_spmv_kernel<FMT, L, SP_RESID><<<A->grid_spmv, BLOCK, 0, st>>>(S, C, v, sc, part, rmode, 1, 0, 0); break;
      case SP_AV: bg_spmv_kernel<FMT, L, SP_AV><<<A->grid_spmv, BLOCK, 0, st>>>(S, C, v, sc, part, 0, 1, 0, 0); break;
      case SP_AT: bg_spmv_kernel<FMT, L, SP_AT><<<A->grid_spmv, BLOCK, 0, st>>>(S, C, v, sc, part, 0, 1, 0, 0); break;
      default: bg_spmv_kernel<FMT, L, SP_FINAL><<<A->grid_spmv, BLOCK, 0, st>>>(S, C, v, sc, part, rmode, 1, 0, 0); break;
    }
    count_launch();
  }
};
using BgdSpmv = void (*)(pcg_matrix *, const BicgVecs &, BgScalars *, int, int, cudaStream_t);
static BgdSpmv bgd_spmv_fn(int fmt, int lanes) {
  if (fmt == FMT_SELL_SHORT) return BgdOps<FMT_SELL_SHORT, 1>::spmv;
  if (fmt == FMT_SELL_DIA) return BgdOps<FMT_SELL_DIA, 1>::spmv;
  if (fmt == PCG_FORMAT_SELL) return BgdOps<PCG_FORMAT_SELL, 1>::spmv;
  switch (lanes) {
    case 1: return BgdOps<PCG_FORMAT_CSR, 1>::spmv;
    case 2: return BgdOps<PCG_FORMAT_CSR, 2>::spmv;
    case 4: return BgdOps<PCG_FORMAT_CSR, 4>::spmv;
    case 8: return BgdOps<PCG_FORMAT_CSR, 8>::spmv;
    case 16: return BgdOps<PCG_FORMAT_CSR, 16>::spmv;
    default: return BgdOps<PCG_FORMAT_CSR, 32>::spmv;
  }
}

static pcg_status bgd_solve(pcg_matrix *A, const BicgVecs &v, double tol, int64_t max_iter, cudaStream_t st,
                            BicgState *hs) {
  SolveWork &w = A->work;
  if (!w.bgsc) PCG_CUDA(cudaMalloc(&w.bgsc, sizeof(BgScalars)));
  BgScalars *sc = (BgScalars *)w.bgsc, h;
  memset(&h, 0, sizeof(h));
  h.tol = tol;
  h.max_iter = max_iter;
  PCG_CUDA(cudaMemcpyAsync(sc, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  const BgdSpmv spmv = bgd_spmv_fn(bg_fmt(A), A->csr_lanes);
  double *part = w.partials;
  auto read = [&]() -> pcg_status {
    PCG_CUDA(cudaGetLastError());
    PCG_CUDA(cudaMemcpyAsync(&h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
    PCG_TRY(comm_wait(A->comm, st));
    return PCG_OK;
  };
  auto finish = [&](int which, int rmode, int count) -> pcg_status {
    PCG_TRY(allreduce_sum(A, sc->part, count, st));
    bg_finish_kernel<<<1, 1, 0, st>>>(sc, which, rmode);
    count_launch();
    return PCG_OK;
  };
  auto resid = [&](int rmode) -> pcg_status {  // the (re)start / exit check / final residual
    PCG_TRY(halo_exchange(A, v.x, 1, st));
    spmv(A, v, sc, rmode == BR_FINAL ? SP_FINAL : SP_RESID, rmode, st);
    PCG_TRY(finish(rmode == BR_FINAL ? BF_FINAL : BF_RESID, rmode, rmode == BR_FINAL ? 1 : 3));
    return read();
  };
  const int U = 8;
  PCG_TRY(resid(BR_INIT));
  if (h.done == BD_ZERO_RHS || h.done == BD_NONFINITE) PCG_CUDA(cudaMemsetAsync(v.x, 0, sizeof(double) * A->n, st));
  while (h.done == BD_RUNNING) {
    for (int u = 0; u < U; u++) {
      bg_precond_kernel<1, 0><<<A->grid_vec, BLOCK, 0, st>>>(A->n, v, sc, part, 1, 0, 0);  // p, p^
      count_launch();
      PCG_TRY(halo_exchange(A, v.ph, 1, st));
      spmv(A, v, sc, SP_AV, 0, st);  // v = A p^
      PCG_TRY(finish(BF_AV, 0, 1));
      bg_precond_kernel<1, 1><<<A->grid_vec, BLOCK, 0, st>>>(A->n, v, sc, part, 1, 0, 0);  // s, s^
      count_launch();
      PCG_TRY(finish(BF_P3, 0, 1));
      PCG_TRY(halo_exchange(A, v.sh, 1, st));
      spmv(A, v, sc, SP_AT, 0, st);  // t = A s^
      PCG_TRY(finish(BF_AT, 0, 2));
      bg_update_kernel<<<A->grid_vec, BLOCK, 0, st>>>(A->n, v, sc, part, 1, 0, 0);
      count_launch();
      PCG_TRY(finish(BF_UPDATE, 0, 2));
    }
    PCG_TRY(read());
    if (h.done != BD_RUNNING) break;
    if (h.stop) PCG_TRY(resid(BR_CHECK));  // exit check (need_resid), restart if it fails
  }
  if (h.done == BD_MAXIT || h.done == BD_BREAKDOWN || h.done == BD_NONFINITE) PCG_TRY(resid(BR_FINAL));
  hs->nb = h.nb;
  hs->relres_rec = h.relres_rec;
  hs->relres_true = h.relres_true;
  hs->k = h.k;
  hs->restarts = h.restarts;
  hs->done = h.done;
  return PCG_OK;
}

static pcg_status bicg_setup(pcg_matrix *A, int bs, int64_t ilu_rows, cudaStream_t st) {
  SolveWork &w = A->work;
  if (bs == BS_ILU) {
    int64_t want = ilu_rows;
    if (want < 1) want = std::max<int64_t>(1, (A->n + num_sms(A->device) - 1) / num_sms(A->device));
    if (want > A->n) want = A->n;
    if (!w.ilu || ilu_block_rows(w.ilu) != want) {
      if (w.ilu) ilu_free(w.ilu);
      w.ilu = nullptr;
      PCG_TRY(ilu_setup(A, want, st, &w.ilu));
    }
  }
  if (!w.bv) {
    const size_t nb = sizeof(double) * ((size_t)(A->n + A->n_ghost) + 64);  // ghost slots for x, p^, s^
    PCG_CUDA(cudaMalloc(&w.bv, nb * 8));  // x r rh p ph v sh t
    PCG_CUDA(cudaMemsetAsync(w.bv, 0, nb * 8, st));
    PCG_CUDA(cudaMalloc(&w.bstate, sizeof(BicgState)));
    PCG_CUDA(cudaMalloc(&w.bbar, sizeof(GridBar)));
    PCG_CUDA(cudaMemsetAsync(w.bbar, 0, sizeof(GridBar), st));
    shadow_kernel<<<(unsigned)std::min<int64_t>((A->n + 255) / 256, 148 * 16), 256, 0, st>>>(
        A->n, A->d_perm, A->row_begin, w.bv + 2 * (A->n + A->n_ghost + 64));
    count_launch();
    PCG_CUDA(cudaGetLastError());
  }
  if (bs > 1 && w.bminv_bs != bs) {
    if (w.bminv) cudaFree(w.bminv);
    w.bminv = nullptr;
    const int64_t nblk = (A->n + bs - 1) / bs;
    // LU factors then pivots in one allocation
    PCG_CUDA(cudaMalloc(&w.bminv, sizeof(double) * (size_t)nblk * bs * bs + sizeof(int) * (size_t)nblk * bs + 64));
    double *lu = w.bminv;
    int *piv = reinterpret_cast<int *>(w.bminv + (size_t)nblk * bs * bs);
    int *err;
    PCG_CUDA(cudaMalloc(&err, sizeof(int)));
    PCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
    const unsigned g = (unsigned)((nblk + 127) / 128);
    switch (bs) {
      case 2: bj_lu_kernel<2><<<g, 128, 0, st>>>(A->n, A->d_row_ptr, A->d_col, A->d_val, A->d_perm, A->d_iperm, lu, piv, err); break;
      case 4: bj_lu_kernel<4><<<g, 128, 0, st>>>(A->n, A->d_row_ptr, A->d_col, A->d_val, A->d_perm, A->d_iperm, lu, piv, err); break;
      default: bj_lu_kernel<8><<<g, 128, 0, st>>>(A->n, A->d_row_ptr, A->d_col, A->d_val, A->d_perm, A->d_iperm, lu, piv, err); break;
    }
    count_launch();
    int h = 0;
    PCG_CUDA(cudaMemcpyAsync(&h, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    PCG_TRY(comm_wait(A->comm, st));
    cudaFree(err);
    if (h) return fail(PCG_ERR_ZERO_DIAGONAL, "pcg_bicgstab: a Block-Jacobi diagonal block is singular");
    w.bminv_bs = bs;
  }
  return PCG_OK;
}

static pcg_status bicg_impl(pcg_matrix *A, const double *b, double *x, double tol, int64_t max_iter, int bs,
                            int64_t ilu_rows, cudaStream_t st, pcg_info *info) {
  PCG_TRY(ensure_work(A));
  PCG_TRY(bicg_setup(A, bs, ilu_rows, st));
  SolveWork &w = A->work;
  const int64_t n = A->n, ldv = n + A->n_ghost + 64;
  BicgVecs v;
  v.x = w.bv;
  v.r = w.bv + ldv;
  v.rh = w.bv + 2 * ldv;
  v.p = w.bv + 3 * ldv;
  v.ph = w.bv + 4 * ldv;
  v.v = w.bv + 5 * ldv;
  v.sh = w.bv + 6 * ldv;
  v.t = w.bv + 7 * ldv;
  v.dinv = A->d_dinv;
  v.lu = w.bminv;
  v.piv = bs > 1 ? reinterpret_cast<const int *>(w.bminv + (size_t)((n + bs - 1) / bs) * bs * bs) : nullptr;
  v.iperm = A->d_iperm;
  const bool b_dev = is_device_ptr(b), x_dev = is_device_ptr(x);
  // b -> stage_b, x0 -> v.x (through the SELL-C-sigma permutation when the handle has one)
  if (A->d_perm) {
    const double *bs_ = b, *xs = x;
    if (!b_dev) {
      PCG_CUDA(cudaMemcpyAsync(w.w, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
      bs_ = w.w;
    }
    PCG_TRY(perm_in(A, bs_, w.stage_b, st));
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
  BicgState hs;
  memset(&hs, 0, sizeof(hs));
  hs.tol = tol;
  hs.max_iter = max_iter;
  cudaEvent_t e0, e1;
  PCG_CUDA(cudaEventCreate(&e0));
  PCG_CUDA(cudaEventCreate(&e1));
  if (A->comm) {
    PCG_CUDA(cudaEventRecord(e0, st));
    const pcg_status gs = bgd_solve(A, v, tol, max_iter, st, &hs);
    PCG_CUDA(cudaEventRecord(e1, st));
    if (gs != PCG_OK) return gs;
  } else if (bs == BS_ILU || bicg_use_graph(A)) {
    PCG_CUDA(cudaEventRecord(e0, st));
    const pcg_status gs = bg_solve(A, v, bs, tol, max_iter, st, &hs);
    PCG_CUDA(cudaEventRecord(e1, st));
    if (gs != PCG_OK) return gs;
  } else {
    BicgState *dst = (BicgState *)w.bstate;
    PCG_CUDA(cudaMemcpyAsync(dst, &hs, sizeof(hs), cudaMemcpyHostToDevice, st));
    void *fn = bicg_select(A->format == FMT_SELL_TMA ? PCG_FORMAT_SELL : A->format, A->csr_lanes, bs);
    if (w.bgrid == 0 || w.bgrid_bs != bs) {
      int nbk = 0;
      PCG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nbk, fn, BLOCK, 0));
      w.bgrid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)num_sms(A->device) * std::min(nbk, 8),
                                                           std::max<int64_t>(1, (n + BLOCK - 1) / BLOCK)));
      w.bgrid_bs = bs;
    }
    SellViewDia S = A->sell_dia();
    CsrView Cv = A->csr();
    double *part = w.partials;  // 4 x grid (<= 8 x SMs; partials hold 6 x 32 x SMs)
    GridBar *bar = (GridBar *)w.bbar;
    void *args[] = {&S, &Cv, &v, &dst, &part, &bar};
    PCG_CUDA(cudaEventRecord(e0, st));
    PCG_CUDA(cudaLaunchCooperativeKernel(fn, dim3(w.bgrid), dim3(BLOCK), args, 0, st));
    count_launch();
    PCG_CUDA(cudaEventRecord(e1, st));
    PCG_CUDA(cudaMemcpyAsync(&hs, dst, sizeof(hs), cudaMemcpyDeviceToHost, st));
  }
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
  PCG_TRY(comm_wait(A->comm, st));
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  pcg_status s;
  switch (hs.done) {
    case BD_CONVERGED: s = hs.relres_true <= tol ? PCG_OK : PCG_NOT_CONVERGED; break;
    case BD_ZERO_RHS: s = PCG_OK; break;
    case BD_MAXIT: s = PCG_NOT_CONVERGED; break;
    case BD_BREAKDOWN: s = PCG_ERR_BREAKDOWN; break;
    default: s = PCG_ERR_NONFINITE; break;
  }
  if (info) {
    memset(info, 0, sizeof(*info));
    info->iterations = hs.k;
    info->relres_recurrence = hs.relres_rec;
    info->relres_true = hs.done == BD_ZERO_RHS ? 0.0 : hs.relres_true;
    info->converged = s == PCG_OK;
    info->status = s;
    info->replacements = hs.restarts;
    info->t_solve_s = ms * 1e-3;
    const double nn = (double)n, nz = (double)A->nnz;
    // per iteration: 2 SpMVs (12 nnz + 4(n+1) + gather 8n + write 8n + r^ 8n each) + 3 streaming passes
    // P1 (r,p,v in; p,p^ out: 40n + M^-1 8 bs n), P3 (r,v in; r,s^ out: 32n + 8 bs n), P5 (x,p^,s^,r,t,r^ in; x,r out: 64n)
    info->bytes_algorithmic =
        bs == BS_ILU
            // 2 SpMVs + P1 (r, p, v in; p out) + P3 (r, v in; r out) + P5 (64 n) + 2 ILU(0) applications
            ? (double)hs.k * (2 * (12.0 * nz + 4.0 * (nn + 1) + 24.0 * nn) + 120.0 * nn + 2 * ilu_bytes_per_apply(A->work.ilu))
            : (double)hs.k * (2 * (12.0 * nz + 4.0 * (nn + 1) + 24.0 * nn) + 136.0 * nn + 16.0 * bs * nn);
    info->flops = (double)hs.k * (4.0 * nz + 30.0 * nn);
  }
  if (s == PCG_ERR_BREAKDOWN) set_error("pcg_bicgstab: breakdown (rho, r^.v or omega = 0)");
  if (s == PCG_NOT_CONVERGED) set_error("pcg_bicgstab: not converged within max_iter");
  if (s == PCG_ERR_NONFINITE) set_error("pcg_bicgstab: non-finite right-hand side or iterate");
  return s;
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_bicgstab(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                                   int32_t block_size, void *stream, pcg_info *info) {
  pcgb::NvtxRange nvtx_("pcg:pcg_bicgstab");
  if (!A || ((!b || !x) && A->n > 0)) return fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab: null argument");
  if (!(tol > 0.0) || max_iter < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab: tol > 0 and max_iter >= 1");
  if (block_size != 1 && block_size != 2 && block_size != 4 && block_size != 8)
    return fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab: block_size must be 1, 2, 4 or 8");
  if (A->comm && block_size != 1)
    return fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab: distributed handles take point Jacobi (block_size 1)");
  if (A->n == 0) {
    if (info) {
      memset(info, 0, sizeof(*info));
      info->converged = 1;
    }
    return PCG_OK;
  }
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  return bicg_impl(A, b, x, tol, max_iter, block_size, 0, (cudaStream_t)stream, info);
}

extern "C" pcg_status pcg_bicgstab_ilu(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                                       int64_t block_rows, void *stream, pcg_info *info) {
  pcgb::NvtxRange nvtx_("pcg:pcg_bicgstab_ilu");
  if (!A || ((!b || !x) && A->n > 0)) return fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab_ilu: null argument");
  if (!(tol > 0.0) || max_iter < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab_ilu: tol > 0 and max_iter >= 1");
  if (A->comm) return fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab_ilu: one-GPU handles only");
  if (A->d_perm)
    return fail(PCG_ERR_INVALID_ARG,
                "pcg_bicgstab_ilu: the handle holds a permuted system (SELL-C-sigma / RCM); create it with "
                "PCG_FMT_CSR or PCG_FMT_SELL");
  if (A->n == 0) {
    if (info) {
      memset(info, 0, sizeof(*info));
      info->converged = 1;
    }
    return PCG_OK;
  }
  std::lock_guard<std::mutex> lk(A->mu);
  PCG_CUDA(cudaSetDevice(A->device));
  return bicg_impl(A, b, x, tol, max_iter, BS_ILU, block_rows, (cudaStream_t)stream, info);
}
