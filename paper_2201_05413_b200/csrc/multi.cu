// multi.cu — Jacobi-PCG for k right-hand sides.
//
// The paper's "block of r.h.s. terms" A X = B (Eq. MRH-TERMS) solved
// by an iterative method that "solve[s] a new linear system for every
// right-hand side term": column j runs the single-RHS recurrence of
// solver.cu independently and freezes at its own stopping test.  On the device
// the k columns share ONE pass over the matrix per iteration: vectors are
// row-major n x K (K = k rounded up to a power of two <= 32), K lanes work on
// one row, every lane gathers its own column, and each (a_ij, j) is loaded once
// for all K columns (the SpMM of SURVEY §8(a) a7).  Column sums are formed in
// the same left-to-right order as the single-RHS kernels, so column j of the
// SpMM equals the SpMV of column j bitwise.
//
// Bytes per iteration: 12 nnz + 4(n+1) + 88 k n  (K1: Z, P, X in, P, Q, X out;
// K2: R, Q, dinv(shared) in, R, Z out).
#include <cmath>
#include <cstring>

#include "matrix.cuh"
#include "rows.cuh"

namespace pcgb {

struct MVecs {
  double *R, *Z, *Q, *P0, *P1, *X, *W;
  const double *Bm;  // row-major n x K right-hand sides
  const double *dinv;
};

template <int K>
__device__ __forceinline__ void col_block_sum(double v, double *sm /*[WARPS][K]*/, double *out /*[K] in t<K*/) {
#pragma unroll
  for (int o = 16; o >= K; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane < K) sm[w * K + lane] = v;
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < WARPS; j++) s += sm[j * K + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// NV values per column: publish block partials (layout [i][block][c], coalesced),
// the last block reduces them in a fixed order into stot[i][c] (shared memory).
template <int K, int NV>
__device__ bool multi_reduce(double (&v)[NV], double *partials, unsigned int *counter, double (*stot)[K],
                             double *sm /*[BLOCK]*/) {
  __shared__ double blk[NV][K];
  __shared__ bool s_last;
#pragma unroll
  for (int i = 0; i < NV; i++) {
    col_block_sum<K>(v[i], sm, blk[i]);
    __syncthreads();
  }
  if (threadIdx.x < K)
#pragma unroll
    for (int i = 0; i < NV; i++) partials[((size_t)i * gridDim.x + blockIdx.x) * K + threadIdx.x] = blk[i][threadIdx.x];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  constexpr int S = BLOCK / K;
  const int c = threadIdx.x % K, sl = threadIdx.x / K;
  for (int i = 0; i < NV; i++) {
    double acc = 0.0;
    for (unsigned int b = sl; b < gridDim.x; b += S) acc += __ldcg(partials + ((size_t)i * gridDim.x + b) * K + c);
    sm[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < K) {
      double t = 0.0;
      for (int s2 = 0; s2 < S; s2++) t += sm[s2 * K + threadIdx.x];
      stot[i][threadIdx.x] = t;
    }
    __syncthreads();
  }
  return true;
}

__device__ __forceinline__ void mstop(int use_cond, cudaGraphConditionalHandle h) {
  if (use_cond) cudaGraphSetConditional(h, 0);
}

// ---------------------------------------------------------------- K1: SpMM + P, X updates + sigma_c
template <int K>
__global__ void __launch_bounds__(BLOCK) mk1_kernel(CsrView A, MVecs v, MultiScalars *sc, double *partials,
                                                    int use_cond, cudaGraphConditionalHandle h) {
  __shared__ double s_beta[K], s_xp[K];
  __shared__ int s_act[K];
  __shared__ double sm[BLOCK];
  __shared__ double t2[1][K];
  volatile MultiScalars *vs = sc;
  if (vs->n_active == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) mstop(use_cond, h);
    return;
  }
  if (threadIdx.x < K) {
    s_beta[threadIdx.x] = vs->beta[threadIdx.x];
    s_xp[threadIdx.x] = vs->xpend[threadIdx.x];
    s_act[threadIdx.x] = vs->active[threadIdx.x];
  }
  __syncthreads();
  const int par = vs->parity;
  const double *__restrict__ Po = par ? v.P1 : v.P0;
  double *__restrict__ Pn = par ? v.P0 : v.P1;
  const double *__restrict__ Z = v.Z;
  const int c = threadIdx.x & (K - 1);
  const double beta = s_beta[c], xp = s_xp[c];
  const int act = s_act[c];
  double acc = 0.0;
  const int64_t g0 = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) / K, ng = (int64_t)gridDim.x * BLOCK / K;
  for (int64_t row = g0; row < A.n; row += ng) {
    const int64_t e = row * K + c;
    if (!act) {  // frozen column: only the owed x update (once, right after freezing)
      if (xp != 0.0) v.X[e] = __fma_rn(xp, Po[e], v.X[e]);
      continue;
    }
    const double po = Po[e];
    if (xp != 0.0) v.X[e] = __fma_rn(xp, po, v.X[e]);
    const int rs = A.row_ptr[row], re = A.row_ptr[row + 1];
    double sum = 0.0;
    for (int k0 = rs; k0 < re; k0 += 8) {  // all 8 (val, col) loads before the first gather
      double a[8], g[8];
      int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (k0 + u < re) {
          a[u] = __ldg(A.val + k0 + u);
          j[u] = __ldg(A.col + k0 + u);
        }
      cols_ready(j, A.zero);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (k0 + u < re) {
          const int64_t jj = (int64_t)j[u] * K + c;
          g[u] = __fma_rn(beta, __ldg(Po + jj), __ldg(Z + jj));
        }
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (k0 + u < re) sum = __fma_rn(a[u], g[u], sum);
    }
    const double pi = __fma_rn(beta, po, Z[e]);
    Pn[e] = pi;
    v.Q[e] = sum;
    acc = __fma_rn(pi, sum, acc);
  }
  double red[1] = {acc};
  if (multi_reduce<K, 1>(red, partials, &sc->cnt_a, t2, sm) && threadIdx.x == 0) {
    sc->cnt_a = 0;
    int na = 0;
    for (int cc = 0; cc < K; cc++) {
      if (!sc->active[cc]) {
        sc->xpend[cc] = 0.0;
        continue;
      }
      const double sigma = t2[0][cc];
      sc->sigma[cc] = sigma;
      if (!(sigma > 0.0)) {
        sc->done[cc] = DONE_BREAKDOWN;
        sc->active[cc] = 0;
        sc->xpend[cc] = 0.0;
      } else {
        sc->alpha[cc] = sc->rho[cc] / sigma;
        sc->xpend[cc] = sc->alpha[cc];
        sc->k[cc] += 1;
        na++;
      }
    }
    sc->parity ^= 1;
    sc->n_active = na;
    sc->graph_launches += use_cond;
    if (na == 0) mstop(use_cond, h);
  }
}

// ---------------------------------------------------------------- K2: R, Z updates + rho'_c, gamma_c
template <int K>
__global__ void __launch_bounds__(BLOCK) mk2_kernel(int64_t n, MVecs v, MultiScalars *sc, double *partials,
                                                    int use_cond, cudaGraphConditionalHandle h) {
  __shared__ double s_alpha[K];
  __shared__ int s_act[K];
  __shared__ double sm[BLOCK];
  __shared__ double t2[2][K];
  volatile MultiScalars *vs = sc;
  if (vs->n_active == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) mstop(use_cond, h);
    return;
  }
  if (threadIdx.x < K) {
    s_alpha[threadIdx.x] = vs->alpha[threadIdx.x];
    s_act[threadIdx.x] = vs->active[threadIdx.x];
  }
  __syncthreads();
  const int c = threadIdx.x & (K - 1);
  const double alpha = s_alpha[c];
  const int act = s_act[c];
  double a0 = 0.0, a1 = 0.0;
  const int64_t g0 = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) / K, ng = (int64_t)gridDim.x * BLOCK / K;
  if (act) {
    for (int64_t row = g0; row < n; row += ng) {
      const int64_t e = row * K + c;
      const double r = __fma_rn(-alpha, __ldcs(v.Q + e), v.R[e]);
      const double z = __ldg(v.dinv + row) * r;
      v.R[e] = r;
      v.Z[e] = z;
      a0 = __fma_rn(r, z, a0);
      a1 = __fma_rn(r, r, a1);
    }
  }
  double red[2] = {a0, a1};
  if (multi_reduce<K, 2>(red, partials, &sc->cnt_b, t2, sm) && threadIdx.x == 0) {
    sc->cnt_b = 0;
    int na = 0;
    for (int cc = 0; cc < K; cc++) {
      if (!sc->active[cc]) continue;
      const double rho_new = t2[0][cc], gamma = t2[1][cc];
      sc->gamma[cc] = gamma;
      const double rr = sqrt(gamma);
      sc->relres_rec[cc] = rr / sc->nb[cc];
      if (rr <= sc->tol * sc->nb[cc]) {
        sc->done[cc] = DONE_CONVERGED;  // frozen; xpend = alpha_k still owed to x
        sc->active[cc] = 0;
      } else if (!(gamma == gamma)) {
        sc->done[cc] = DONE_NONFINITE;
        sc->active[cc] = 0;
        sc->xpend[cc] = 0.0;
      } else if (sc->k[cc] >= sc->max_iter) {
        sc->done[cc] = DONE_MAXIT;
        sc->active[cc] = 0;
      } else {
        sc->beta[cc] = rho_new / sc->rho[cc];
        sc->rho[cc] = rho_new;
        na++;
      }
    }
    sc->n_active = na;
    sc->graph_launches += use_cond;
    if (na == 0) mstop(use_cond, h);
  }
}

// ---------------------------------------------------------------- residual W = B - A X and its norms
template <int K>
__global__ void __launch_bounds__(BLOCK) mresid_kernel(CsrView A, MVecs v, MultiScalars *sc, double *partials) {
  __shared__ double sm[BLOCK];
  __shared__ double t3[3][K];
  const int c = threadIdx.x & (K - 1);
  double ww = 0.0, wz = 0.0, bb = 0.0;
  const int64_t g0 = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) / K, ng = (int64_t)gridDim.x * BLOCK / K;
  for (int64_t row = g0; row < A.n; row += ng) {
    const int rs = A.row_ptr[row], re = A.row_ptr[row + 1];
    double sum = 0.0;
    for (int k0 = rs; k0 < re; k0 += 8) {
      double a[8], g[8];
      int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (k0 + u < re) {
          a[u] = __ldg(A.val + k0 + u);
          j[u] = __ldg(A.col + k0 + u);
        }
      cols_ready(j, A.zero);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (k0 + u < re) g[u] = __ldg(v.X + (int64_t)j[u] * K + c);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (k0 + u < re) sum = __fma_rn(a[u], g[u], sum);
    }
    const int64_t e = row * K + c;
    const double bi = v.Bm[e];
    const double w = bi - sum;
    v.W[e] = w;
    const double z = v.dinv[row] * w;
    ww = __fma_rn(w, w, ww);
    wz = __fma_rn(w, z, wz);
    bb = __fma_rn(bi, bi, bb);
  }
  double red[3] = {ww, wz, bb};
  if (multi_reduce<K, 3>(red, partials, &sc->cnt_c, t3, sm) && threadIdx.x == 0) {
    sc->cnt_c = 0;
    for (int cc = 0; cc < K; cc++)
      for (int i = 0; i < 3; i++) sc->part[i][cc] = t3[i][cc];
  }
}

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

// R = W, Z = dinv W, P[parity] = 0 for columns being (re)started
template <int K>
__global__ void mreplace_kernel(int64_t n, MVecs v, const MultiScalars *sc) {
  const int c = threadIdx.x & (K - 1);
  if (!sc->replace[c]) return;
  double *P = sc->parity ? v.P1 : v.P0;
  const int64_t g0 = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) / K, ng = (int64_t)gridDim.x * BLOCK / K;
  for (int64_t row = g0; row < n; row += ng) {
    const int64_t e = row * K + c;
    const double w = v.W[e];
    v.R[e] = w;
    v.Z[e] = v.dinv[row] * w;
    P[e] = 0.0;
  }
}

template <int K>
__global__ void mtail_kernel(int64_t n, MVecs v, const MultiScalars *sc) {
  const int c = threadIdx.x & (K - 1);
  const double xp = sc->xpend[c];
  if (xp == 0.0) return;
  const double *P = sc->parity ? v.P1 : v.P0;
  const int64_t g0 = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) / K, ng = (int64_t)gridDim.x * BLOCK / K;
  for (int64_t row = g0; row < n; row += ng) {
    const int64_t e = row * K + c;
    v.X[e] = __fma_rn(xp, P[e], v.X[e]);
  }
}
__global__ void mclear_xpend_kernel(MultiScalars *sc) {
  for (int c = 0; c < KMAX; c++) sc->xpend[c] = 0.0;
}

// column-major (ld) <-> row-major n x K; zero rows for padded / zero-RHS columns
__global__ void to_rowmajor_kernel(int64_t n, int k, int K, const double *__restrict__ cm, int64_t ld,
                                   double *__restrict__ rm) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * K; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / K;
    const int c = (int)(e % K);
    rm[e] = c < k ? cm[row + (int64_t)c * ld] : 0.0;
  }
}
__global__ void to_colmajor_kernel(int64_t n, int k, int K, const double *__restrict__ rm, double *__restrict__ cm,
                                   int64_t ld, const MultiScalars *sc) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n * k; e += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(e / n);
    const int64_t row = e % n;
    cm[row + (int64_t)c * ld] = sc->done[c] == DONE_ZERO_RHS ? 0.0 : rm[row * K + c];
  }
}

// ---------------------------------------------------------------- host side
pcg_status ensure_multi_work(pcg_matrix *A, int K) {
  SolveWork &w = A->work;
  if (w.kcap == K && w.msc) return PCG_OK;
  for (double *p : {w.mr, w.mz, w.mq, w.mp[0], w.mp[1], w.mx, w.mb, w.mw})
    if (p) cudaFree(p);
  if (w.mloop_exec) cudaGraphExecDestroy(w.mloop_exec);
  if (w.mloop_graph) cudaGraphDestroy(w.mloop_graph);
  w.mloop_exec = nullptr;
  w.mloop_graph = nullptr;
  w.mgraph_k = 0;
  const size_t nk = sizeof(double) * (size_t)(A->n > 0 ? A->n : 1) * K;
  PCG_CUDA(cudaMalloc(&w.mr, nk));
  PCG_CUDA(cudaMalloc(&w.mz, nk));
  PCG_CUDA(cudaMalloc(&w.mq, nk));
  PCG_CUDA(cudaMalloc(&w.mp[0], nk));
  PCG_CUDA(cudaMalloc(&w.mp[1], nk));
  PCG_CUDA(cudaMalloc(&w.mx, nk));
  PCG_CUDA(cudaMalloc(&w.mb, nk));
  PCG_CUDA(cudaMalloc(&w.mw, nk));
  PCG_CUDA(cudaMemset(w.mp[0], 0, nk));
  PCG_CUDA(cudaMemset(w.mp[1], 0, nk));
  PCG_CUDA(cudaMemset(w.mz, 0, nk));
  if (!w.mpart) PCG_CUDA(cudaMalloc(&w.mpart, sizeof(double) * 3 * KMAX * (size_t)num_sms(A->device) * 8));
  if (!w.msc) {
    PCG_CUDA(cudaMalloc(&w.msc, sizeof(MultiScalars)));
    PCG_CUDA(cudaMemset(w.msc, 0, sizeof(MultiScalars)));
    PCG_CUDA(cudaMallocHost(&w.h_msc, sizeof(MultiScalars)));
  }
  w.kcap = K;
  return PCG_OK;
}

static MVecs mvecs_of(pcg_matrix *A) {
  SolveWork &w = A->work;
  return MVecs{w.mr, w.mz, w.mq, w.mp[0], w.mp[1], w.mx, w.mw, w.mb, A->d_dinv};
}

static int mgrid(pcg_matrix *A, int K) {
  const int64_t need = (A->n * K + BLOCK - 1) / BLOCK;
  const int64_t g = (int64_t)num_sms(A->device) * 8;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, need));
}

#define MK_DISPATCH(K, EXPR)                    \
  switch (K) {                                  \
    case 1: { constexpr int KK = 1; EXPR; } break;   \
    case 2: { constexpr int KK = 2; EXPR; } break;   \
    case 4: { constexpr int KK = 4; EXPR; } break;   \
    case 8: { constexpr int KK = 8; EXPR; } break;   \
    case 16: { constexpr int KK = 16; EXPR; } break; \
    default: { constexpr int KK = 32; EXPR; } break; \
  }

static pcg_status mbuild_graph(pcg_matrix *A, int K) {
  SolveWork &w = A->work;
  if (w.mgraph_k == K && w.mloop_exec) return PCG_OK;
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
  const int grid = mgrid(A, K);
  MVecs v = mvecs_of(A);
  double *part = w.mpart;
  MK_DISPATCH(K, (mk1_kernel<KK><<<grid, BLOCK, 0, cap>>>(A->csr(), v, w.msc, part, 1, h),
                  mk2_kernel<KK><<<grid, BLOCK, 0, cap>>>(A->n, v, w.msc, part + (size_t)KMAX * grid, 1, h)));
  cudaGraph_t out;
  PCG_CUDA(cudaStreamEndCapture(cap, &out));
  PCG_CUDA(cudaGetLastError());
  PCG_CUDA(cudaGraphInstantiate(&w.mloop_exec, g, 0));
  w.mloop_graph = g;
  w.mgraph_k = K;
  cudaStreamDestroy(cap);
  return PCG_OK;
}

static pcg_status solve_multi_chunk(pcg_matrix *A, int k, const double *B, int64_t ldb, double *X, int64_t ldx,
                                    double tol, int64_t max_iter, cudaStream_t st, pcg_info *infos) {
  int K = 1;
  while (K < k) K <<= 1;
  PCG_TRY(ensure_work(A));
  PCG_TRY(ensure_multi_work(A, K));
  const int grid = mgrid(A, K);  // <= 8 * SMs: mpart holds 3 x KMAX x grid
  PCG_TRY(mbuild_graph(A, K));
  SolveWork &w = A->work;
  const int64_t n = A->n;
  const bool bd = is_device_ptr(B), xd = is_device_ptr(X);
  // stage column-major inputs through mw (n x k, ld n), then to row-major
  double *cm = w.mw;  // scratch (n*K >= n*k)
  PCG_CUDA(cudaMemcpy2DAsync(cm, sizeof(double) * n, B, sizeof(double) * ldb, sizeof(double) * n, k,
                             bd ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  to_rowmajor_kernel<<<1184, 256, 0, st>>>(n, k, K, cm, n, w.mb);
  PCG_CUDA(cudaMemcpy2DAsync(cm, sizeof(double) * n, X, sizeof(double) * ldx, sizeof(double) * n, k,
                             xd ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  to_rowmajor_kernel<<<1184, 256, 0, st>>>(n, k, K, cm, n, w.mx);
  count_launch(2);
  MultiScalars *h = w.h_msc;
  memset(h, 0, sizeof(MultiScalars));
  h->tol = tol;
  h->max_iter = max_iter;
  h->kcols = k;
  PCG_CUDA(cudaMemcpyAsync(w.msc, h, sizeof(MultiScalars), cudaMemcpyHostToDevice, st));
  MVecs v = mvecs_of(A);
  cudaEvent_t e0, e1;
  PCG_CUDA(cudaEventCreate(&e0));
  PCG_CUDA(cudaEventCreate(&e1));
  PCG_CUDA(cudaEventRecord(e0, st));
  int mode = 0;
  for (;;) {
    MK_DISPATCH(K, (mresid_kernel<KK><<<grid, BLOCK, 0, st>>>(A->csr(), v, w.msc, w.mpart)));
    mresid_finish_kernel<<<1, 1, 0, st>>>(w.msc, mode);
    MK_DISPATCH(K, (mreplace_kernel<KK><<<grid, BLOCK, 0, st>>>(n, v, w.msc)));
    count_launch(3);
    if (mode == 1) {
      PCG_CUDA(cudaMemcpyAsync(h, w.msc, sizeof(MultiScalars), cudaMemcpyDeviceToHost, st));
      PCG_CUDA(cudaStreamSynchronize(st));
      if (h->n_active == 0) break;
    }
    PCG_CUDA(cudaGraphLaunch(w.mloop_exec, st));
    MK_DISPATCH(K, (mtail_kernel<KK><<<grid, BLOCK, 0, st>>>(n, v, w.msc)));
    mclear_xpend_kernel<<<1, 1, 0, st>>>(w.msc);
    count_launch(2);
    PCG_CUDA(cudaGetLastError());
    mode = 1;
  }
  PCG_CUDA(cudaEventRecord(e1, st));
  to_colmajor_kernel<<<1184, 256, 0, st>>>(n, k, K, w.mx, cm, n, w.msc);
  count_launch();
  PCG_CUDA(cudaMemcpy2DAsync(X, sizeof(double) * ldx, cm, sizeof(double) * n, sizeof(double) * n, k,
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
      I.relres_recurrence = h->relres_rec[c];
      I.relres_true = h->done[c] == DONE_ZERO_RHS ? 0.0 : h->relres_true[c];
      I.converged = s == PCG_OK;
      I.status = s;
      I.t_solve_s = ms * 1e-3;
      const double nn = (double)n, nz = (double)A->nnz;
      // shared matrix pass: per block-iteration 12 nnz + 4(n+1) + 88 k n, attributed per column
      I.bytes_algorithmic = (double)kmax * (12.0 * nz + 4.0 * (nn + 1)) / k + (double)h->k[c] * 88.0 * nn;
      I.flops = (double)h->k[c] * (2.0 * nz + 13.0 * nn);
    }
  }
  if (worst != PCG_OK) set_error(std::string("pcg_solve_multi: worst column status ") + pcg_status_string(worst));
  return worst;
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_solve_multi(pcg_matrix_t A, int32_t k, const double *B, int64_t ldb, double *X,
                                      int64_t ldx, double tol, int64_t max_iter, void *stream, pcg_info *infos) {
  if (!A || !B || !X) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: null argument");
  if (k < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: k must be >= 1");
  if (ldb < A->n || ldx < A->n) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: ld < n");
  if (!(tol > 0.0) || max_iter < 1) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: tol > 0, max_iter >= 1");
  if (A->comm) return fail(PCG_ERR_INVALID_ARG, "pcg_solve_multi: distributed handles take one RHS per solve");
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
