// ilu.cu — Block-Jacobi with ILU(0) blocks, the preconditioner of the paper's own
// iterative solver (PETSc BiCGSTAB + Block-Jacobi, whose default sub-solver is ILU(0):
// P:194), for pcg_bicgstab_ilu.  SURVEY §8(f) N2; reading R6.
//
// M = blockdiag(L_b U_b): blocks of `bs` consecutive rows; in each block the incomplete
// LU with zero fill of Saad, Alg. 10.4 (IKJ), written with explicitly rounded
// operations in the oracle's order (oracle.c ilu0_setup / ilu0_apply), so the factors
// and every application of M^-1 are bitwise the oracle's.
//
// Triangular solves are level-scheduled.  Row i of a block depends (forward, L) on
// the rows k < i of its block that it references, and (backward, U) on the rows j > i;
// its level is one more than the largest level it depends on, and the rows of one
// level are independent.  One CTA per block walks the levels in order with a block
// barrier between them; the block's vector lives in shared memory when it fits (bs
// <= 22K rows), so a level costs a CTA barrier and shared-memory reads, not a
// grid-wide synchronisation.  The level analysis (a graph traversal, setup only) runs
// on the host; it lays the factor out level by level in an ELL form ([level][entry
// u][row slot]: a level's loads are coalesced): per slot the local row, per (u, slot)
// the local column (-1 = padding) and the factor value.  The numeric factorization
// runs on the device, in the forward level order.  Where every row has at most 4
// entries per triangle and a block fits shared memory (the Table 1 grids), the levels
// are split into records of at most 128 rows and each record's data is also packed
// contiguously, so the application brings a level in with one bulk copy
// (ilu_apply_packed_kernel); otherwise each thread streams its slot through a cp.async
// ring (ilu_apply_kernel).
#include <algorithm>
#include <cstring>
#include <vector>

#include "matrix.cuh"
#include "staged.cuh"

#ifndef PCG_ILU_RCP
#define PCG_ILU_RCP 0
#endif

namespace pcgb {

struct IluLevel {
  int64_t row_base;  // first slot of the level
  int64_t ent_base;  // first ELL entry of the level ([u][slot], m slots per u)
  int64_t pbase;     // byte offset of the level's packed record (pk_bytes), -1: not packed
  int m, c;          // rows, entries per row (max over the level's rows)
};

// Packed level record (one bulk copy per level): [kcol c x m int32][row m int32] (8-B
// aligned) [fv c x m f64][u_ii m f64, backward levels], padded to 16 B.
__host__ __device__ constexpr int pk_fv_off(int m, int c) { return ((4 * c * m + 4 * m) + 7) & ~7; }
__host__ __device__ constexpr int pk_bytes(int m, int c, bool backward) {
  return (pk_fv_off(m, c) + 8 * c * m + (backward ? 8 * m : 0) + 15) & ~15;
}

// Forward levels of all blocks, then backward levels; lo[0..nblk] indexes the forward
// levels of each block, lo[nblk+1 .. 2 nblk+1] the backward ones.
struct IluPlan {
  int64_t bs = 0, nblk = 0, n = 0;
  size_t smem = 0;       // dynamic shared memory of the apply kernel (level records + the vector)
  bool vec_smem = false; // the block's vector in shared memory (bs <= ILU_SMEM_ROWS)
  int cmax = 4;          // entries per row and direction the apply kernel is compiled for
  double *f = nullptr;   // factor values in CSR order (nnz)
  int *diag = nullptr;   // CSR index of a_ii per row
  IluLevel *lev = nullptr;
  int *lo = nullptr;
  int *row = nullptr;    // per slot: local row
  int *kcol = nullptr;   // per entry: local column, -1 = padding
  int *emap = nullptr;   // per entry: CSR index of the factor value, -1 = padding
  double *fv = nullptr;  // per entry: factor value
  double *ud = nullptr;  // per slot: u_ii (backward slots; 1 for forward slots)
  int *udmap = nullptr;  // per slot: CSR index of u_ii (-1 forward)
  int64_t nlev = 0, nslot = 0, nent = 0;
  double bytes_per_apply = 0;
  unsigned char *pk = nullptr;  // packed level records (apply_packed), null: not used
  int pk_threads = 0;           // CTA size of the packed kernel (>= every level's rows)
  int maxlev = 0;               // most levels (forward + backward) of any block
};

void ilu_free(void *p) {
  IluPlan *P = (IluPlan *)p;
  if (!P) return;
  for (void *q : {(void *)P->f, (void *)P->diag, (void *)P->lev, (void *)P->lo, (void *)P->row, (void *)P->kcol,
                  (void *)P->emap, (void *)P->fv, (void *)P->ud, (void *)P->udmap, (void *)P->pk})
    if (q) cudaFree(q);
  delete P;
}

// ---------------------------------------------------------------- numeric factorization
// One CTA per block; rows of one forward level are factorised in parallel (they only
// read rows of earlier levels).  Row i, one thread, exactly the oracle's loop:
//   for (i,k) in the row, r0 <= k < i, ascending:  f_ik = f_ik / f_kk
//     for (i,j) after it in the row, j < r1:  if (k,j) exists: f_ij = f_ij - f_ik f_kj
__global__ void __launch_bounds__(256) ilu_factor_kernel(int64_t n, int64_t bs, const int *__restrict__ rp,
                                                         const int *__restrict__ col, const int *__restrict__ diag,
                                                         double *f, const IluLevel *__restrict__ lev,
                                                         const int *__restrict__ lo, const int *__restrict__ srow,
                                                         int *__restrict__ err) {
  const int64_t b = blockIdx.x, r0 = b * bs, r1 = min(r0 + bs, n);
  for (int l = lo[b]; l < lo[b + 1]; l++) {
    const IluLevel L = lev[l];
    for (int t = threadIdx.x; t < L.m; t += blockDim.x) {
      const int64_t i = r0 + srow[L.row_base + t];
      const int e0 = rp[i], e1 = rp[i + 1];
      for (int kk = e0; kk < e1; kk++) {
        const int k = col[kk];
        if (k < r0 || k >= i) continue;
        const double fkk = f[diag[k]];
        if (fkk == 0.0) {
          atomicExch(err, 1);
          continue;
        }
        const double fik = __ddiv_rn(f[kk], fkk);
        f[kk] = fik;
        const int k0 = rp[k], k1 = rp[k + 1];
        for (int jj = kk + 1; jj < e1; jj++) {
          const int j = col[jj];
          if (j >= r1) break;
          int a = k0, z = k1 - 1, kj = -1;  // (k, j) in row k (columns ascending)
          while (a <= z) {
            const int mid = (a + z) >> 1;
            const int cm = col[mid];
            if (cm == j) {
              kj = mid;
              break;
            }
            if (cm < j) a = mid + 1;
            else z = mid - 1;
          }
          if (kj >= 0) f[jj] = __dsub_rn(f[jj], __dmul_rn(fik, f[kj]));
        }
      }
      if (f[diag[i]] == 0.0) atomicExch(err, 1);
    }
    __syncthreads();  // the level's factor rows are visible to the CTA's later levels
  }
}

__global__ void ilu_fill_kernel(int64_t ne, const int *__restrict__ emap, int64_t ns, const int *__restrict__ udmap,
                                const double *__restrict__ f, double *__restrict__ fv, double *__restrict__ ud) {
  const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = t0; e < ne; e += nt) fv[e] = emap[e] >= 0 ? f[emap[e]] : 0.0;
  for (int64_t s = t0; s < ns; s += nt) ud[s] = udmap[s] >= 0 ? f[udmap[s]] : 1.0;
}

// ---------------------------------------------------------------- application y = M^-1 v
// Forward: y_i = v_i - sum_k l_ik y_k (k ascending); backward: y_i = (y_i - sum_j u_ij
// y_j) / u_ii (j ascending).  The BiCGSTAB loop's flags: stop (loop ended) and skip
// (no s^ needed: converged at the half step) make the kernel return at entry.
struct IluView {
  int64_t bs, n, nblk;
  const IluLevel *lev;
  const int *lo, *row, *kcol;
  const double *fv, *ud;
  const unsigned char *pk;
};

// the packed level records, written once after the factorization (one CTA per level)
__global__ void ilu_pack_kernel(const IluLevel *__restrict__ lev, int64_t nfwd_end, const int *__restrict__ row,
                                const int *__restrict__ kcol, const double *__restrict__ fv,
                                const double *__restrict__ ud, unsigned char *pk) {
  const int64_t l = blockIdx.x;
  const IluLevel L = lev[l];
  if (L.pbase < 0) return;
  const bool backward = l >= nfwd_end;
  unsigned char *rec = pk + L.pbase;
  int *k = reinterpret_cast<int *>(rec);
  int *rw = k + L.c * L.m;
  double *f = reinterpret_cast<double *>(rec + pk_fv_off(L.m, L.c));
  double *d = f + (size_t)L.c * L.m;
  for (int t = threadIdx.x; t < L.m; t += blockDim.x) {
    rw[t] = row[L.row_base + t];
#if PCG_ILU_RCP  // A/B knob: reciprocal pivots (not the oracle's rounding)
    if (backward) d[t] = 1.0 / ud[L.row_base + t];
#else
    if (backward) d[t] = ud[L.row_base + t];
#endif
    for (int u = 0; u < L.c; u++) {
      const int64_t e = L.ent_base + (int64_t)u * L.m + t;
      k[u * L.m + t] = kcol[e];
      f[u * L.m + t] = fv[e];
    }
  }
}

// One direction's levels of block b.  Level records come from shared memory (copied
// at kernel entry) when the block has at most ILU_LEVS of them.  Every thread owns slot
// t of each level (levels wider than the CTA loop over the extra slots); the loads of
// level l + 1 that do not depend on y (its row, u_ii, input value, columns and factor
// values) are issued before level l computes and synchronises, so a level costs a CTA
// barrier plus shared-memory reads, not a chain of global-memory round trips.
constexpr int ILU_LEVS = 1024;
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
constexpr int ILU_PF = 6;  // levels of L2 prefetch ahead (register-prefetch sweep)

__device__ __forceinline__ void prefetch_range(const void *p, size_t bytes) {
  if (bytes == 0) return;
  const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
  const uintptr_t b = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(b - a)) : "memory");
}
struct IluSlot {
  int i;
  double v, d;
};

template <int CMAX>
__device__ __forceinline__ void ilu_load(const IluView &P, const IluLevel &L, int t, const double *vin, bool backward,
                                         IluSlot &sl, int (&k)[CMAX], double (&f)[CMAX]) {
  sl.i = -1;
  if (t < L.m) {
    const int64_t s = L.row_base + t;
    sl.i = __ldg(P.row + s);
    sl.d = backward ? __ldg(P.ud + s) : 1.0;
    sl.v = 0.0;  // the input vector is in y already (copied at kernel entry)
#pragma unroll
    for (int u = 0; u < CMAX; u++) {
      k[u] = -1;
      if (u < L.c) {
        const int64_t e = L.ent_base + (int64_t)u * L.m + t;
        k[u] = __ldg(P.kcol + e);
        f[u] = __ldg(P.fv + e);
      }
    }
  }
}

template <int CMAX>
__device__ __forceinline__ void ilu_row(const IluSlot &sl, const int (&k)[CMAX], const double (&f)[CMAX], double *y,
                                        bool backward) {
  if (sl.i < 0) return;
  double acc = y[sl.i];  // forward: v_i (y was initialised with v); backward: the forward result
#pragma unroll
  for (int u = 0; u < CMAX; u++)
    if (k[u] >= 0) acc = __dsub_rn(acc, __dmul_rn(f[u], y[k[u]]));
  y[sl.i] = backward ? __ddiv_rn(acc, sl.d) : acc;
}

template <int CMAX>
__device__ __forceinline__ void ilu_sweep(const IluView &P, const IluLevel *lv, int nl, const double *vin, double *y,
                                          bool backward) {
  const int t = threadIdx.x;
  IluSlot cur, nxt;
  int kc[CMAX], kn[CMAX];
  double fc[CMAX], fn[CMAX];
  if (nl > 0) ilu_load<CMAX>(P, lv[0], t, vin, backward, cur, kc, fc);
  for (int l = 0; l < nl; l++) {
    const IluLevel L = lv[l];
    if (t == 0 && l + ILU_PF < nl) {  // level l + ILU_PF toward L2: the register prefetch then hits L2
      const IluLevel F = lv[l + ILU_PF];
      prefetch_range(P.row + F.row_base, (size_t)F.m * 4);
      if (backward) prefetch_range(P.ud + F.row_base, (size_t)F.m * 8);
      prefetch_range(P.kcol + F.ent_base, (size_t)F.m * F.c * 4);
      prefetch_range(P.fv + F.ent_base, (size_t)F.m * F.c * 8);
    }
    if (l + 1 < nl) ilu_load<CMAX>(P, lv[l + 1], t, vin, backward, nxt, kn, fn);
    ilu_row<CMAX>(cur, kc, fc, y, backward);
    for (int t2 = t + blockDim.x; t2 < L.m; t2 += blockDim.x) {  // levels wider than the CTA
      IluSlot sx;
      int kx[CMAX];
      double fx[CMAX];
      ilu_load<CMAX>(P, L, t2, vin, backward, sx, kx, fx);
      ilu_row<CMAX>(sx, kx, fx, y, backward);
    }
    __syncthreads();
    cur = nxt;
#pragma unroll
    for (int u = 0; u < CMAX; u++) {
      kc[u] = kn[u];
      fc[u] = fn[u];
    }
  }
}

// The same sweep with the y-independent slot data of the next ILU_RING - 1 levels in
// flight through shared memory (cp.async, one commit group per level, a ring of
// ILU_RING level slots): each thread copies and later reads only its own slot's data,
// so the ring needs no barrier of its own, and the level barrier orders the y traffic.
#ifndef PCG_ILU_RING  // A/B knobs: ring depth (levels) and threads per CTA of the apply kernel
#define PCG_ILU_RING 4
#endif
#ifndef PCG_ILU_THREADS
#define PCG_ILU_THREADS 256
#endif
constexpr int ILU_RING = PCG_ILU_RING;
constexpr int ILU_THREADS = PCG_ILU_THREADS;
constexpr int ILU_RSLOTS = ILU_THREADS;
template <int CMAX>
struct IluRing {
  int row[ILU_RING][ILU_RSLOTS];
  double ud[ILU_RING][ILU_RSLOTS];
  int k[ILU_RING][CMAX][ILU_RSLOTS];
  double f[ILU_RING][CMAX][ILU_RSLOTS];
};

__device__ __forceinline__ void cp_async4(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

template <int CMAX>
__device__ __forceinline__ void ilu_sweep_ring(const IluView &P, const IluLevel *lv, int nl, double *y, bool backward,
                                               IluRing<CMAX> &R) {
  const int t = threadIdx.x;
  auto issue = [&](int l) {
    if (l < nl) {
      const IluLevel L = lv[l];
      const int q = l % ILU_RING;
      if (t < L.m) {
        const int64_t s = L.row_base + t;
        cp_async4(&R.row[q][t], P.row + s);
        if (backward) cp_async8(&R.ud[q][t], P.ud + s);
        for (int u = 0; u < L.c; u++) {
          const int64_t e = L.ent_base + (int64_t)u * L.m + t;
          cp_async4(&R.k[q][u][t], P.kcol + e);
          cp_async8(&R.f[q][u][t], P.fv + e);
        }
      }
    }
    cp_async_commit();  // one group per level (empty past the end): the wait counts stay uniform
  };
  for (int l = 0; l < ILU_RING - 1; l++) issue(l);
  for (int l = 0; l < nl; l++) {
    // (an L2 bulk prefetch of level l + 12 by thread 0 here measured slower: 0.165 vs 0.131 s on
    // Cube 1 — thread 0 sits on every level's critical path)
    issue(l + ILU_RING - 1);
    cp_async_wait<ILU_RING - 1>();  // this thread's copies for level l have landed
    const IluLevel L = lv[l];
    const int q = l % ILU_RING;
    if (t < L.m) {
      const int i = R.row[q][t];
      double acc = y[i];
      for (int u = 0; u < L.c; u++) {
        const int k = R.k[q][u][t];
        if (k >= 0) acc = __dsub_rn(acc, __dmul_rn(R.f[q][u][t], y[k]));
      }
      y[i] = backward ? __ddiv_rn(acc, R.ud[q][t]) : acc;
    }
    // levels wider than the CTA (a run-time stride: a compile-time one made the compiler
    // restructure this loop and cost the one-block Cube 1 solve 26 %, 4.36 -> 5.49 s)
    for (int t2 = t + blockDim.x; t2 < L.m; t2 += blockDim.x) {
      IluSlot sx;
      int kx[CMAX];
      double fx[CMAX];
      ilu_load<CMAX>(P, L, t2, nullptr, backward, sx, kx, fx);
      ilu_row<CMAX>(sx, kx, fx, y, backward);
    }
    __syncthreads();
  }
  cp_async_wait<0>();
}

// shared memory: [level records][the cp.async ring (CMAX <= 8)][the block's vector]
__host__ __device__ constexpr size_t ilu_vec_offset(int cmax) {
  return sizeof(IluLevel) * ILU_LEVS +
         (cmax <= 4 ? sizeof(IluRing<4>) : cmax <= 8 ? sizeof(IluRing<8>) : 0);
}

template <bool SMEM, int CMAX>
__global__ void __launch_bounds__(ILU_THREADS) ilu_apply_kernel(IluView P, const double *__restrict__ in, double *out,
                                                        const int *stop, const int *skip) {
  extern __shared__ __align__(16) unsigned char ilu_smem[];
  if ((stop && *(volatile const int *)stop) || (skip && *(volatile const int *)skip)) return;
  const int64_t b = blockIdx.x, r0 = b * P.bs, nr = min(P.bs, P.n - r0);
  IluLevel *slev = reinterpret_cast<IluLevel *>(ilu_smem);
  double *y = SMEM ? reinterpret_cast<double *>(ilu_smem + ilu_vec_offset(CMAX)) : out + r0;
  const int f0 = P.lo[b], f1 = P.lo[b + 1], b0 = P.lo[P.nblk + 1 + b], b1 = P.lo[P.nblk + 1 + b + 1];
  const bool lev_smem = (f1 - f0) + (b1 - b0) <= ILU_LEVS;
  if (lev_smem) {
    for (int q = threadIdx.x; q < f1 - f0; q += blockDim.x) slev[q] = P.lev[f0 + q];
    for (int q = threadIdx.x; q < b1 - b0; q += blockDim.x) slev[(f1 - f0) + q] = P.lev[b0 + q];
    __syncthreads();
  }
  for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) y[i] = in[r0 + i];  // coalesced; the sweeps work in place
  __syncthreads();
  const IluLevel *lf = lev_smem ? slev : P.lev + f0;
  const IluLevel *lb = lev_smem ? slev + (f1 - f0) : P.lev + b0;
  if (CMAX <= 8) {
    IluRing<CMAX> &R = *reinterpret_cast<IluRing<CMAX> *>(ilu_smem + sizeof(IluLevel) * ILU_LEVS);
    ilu_sweep_ring<CMAX>(P, lf, f1 - f0, y, false, R);
    ilu_sweep_ring<CMAX>(P, lb, b1 - b0, y, true, R);
  } else {
    ilu_sweep<CMAX>(P, lf, f1 - f0, in + r0, y, false);
    ilu_sweep<CMAX>(P, lb, b1 - b0, in + r0, y, true);
  }
  if (SMEM)
    for (int64_t i = threadIdx.x; i < nr; i += blockDim.x) out[r0 + i] = y[i];
}

// The application with every level's y-independent data in ONE packed record per level,
// brought into a shared-memory ring by one bulk copy (TMA engine) per level, issued
// ILU_PK_RING - 1 levels ahead by thread 0, completion on an mbarrier per ring slot:
// no per-thread copy instructions on the level's critical path (the cp.async ring
// above issues 2 + 2c copies per thread per level).  Forward and backward levels form
// one sequence (slot = g % RING, phase = (g / RING) & 1).  One thread per slot: the
// CTA has at least as many threads as the widest level (pk_threads).
constexpr int ILU_PK_RING = 6;
template <int T>
__global__ void __launch_bounds__(T) ilu_apply_packed_kernel(IluView P, const double *__restrict__ in, double *out,
                                                             const int *stop, const int *skip, int rec_cap) {
  extern __shared__ __align__(128) unsigned char ilu_smem[];
  if ((stop && *(volatile const int *)stop) || (skip && *(volatile const int *)skip)) return;
  constexpr int SLOT = pk_bytes(T, 4, true);
  const int64_t b = blockIdx.x, r0 = b * P.bs, nr = min(P.bs, P.n - r0);
  const int f0 = P.lo[b], f1 = P.lo[b + 1], b0 = P.lo[P.nblk + 1 + b], b1 = P.lo[P.nblk + 1 + b + 1];
  const int nf = f1 - f0, ntot = nf + (b1 - b0);
  unsigned char *ring = ilu_smem;
  uint64_t *bars = reinterpret_cast<uint64_t *>(ilu_smem + (size_t)ILU_PK_RING * SLOT);
  IluLevel *slev = reinterpret_cast<IluLevel *>(ilu_smem + (size_t)ILU_PK_RING * SLOT + 8 * ILU_PK_RING);
  double *y = reinterpret_cast<double *>(ilu_smem + (size_t)ILU_PK_RING * SLOT + 8 * ILU_PK_RING +
                                         sizeof(IluLevel) * (size_t)rec_cap);
  const int t = threadIdx.x;
  for (int q = t; q < nf; q += T) slev[q] = P.lev[f0 + q];
  for (int q = t; q < ntot - nf; q += T) slev[nf + q] = P.lev[b0 + q];
  if (t == 0) {
    for (int q = 0; q < ILU_PK_RING; q++) mbar_init(&bars[q], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int64_t i = t; i < nr; i += T) y[i] = in[r0 + i];
  __syncthreads();
  auto issue = [&](int g) {  // thread 0
    if (g >= ntot) return;
    const IluLevel L = slev[g];
    const int q = g % ILU_PK_RING;
    const uint32_t bytes = (uint32_t)pk_bytes(L.m, L.c, g >= nf);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the slot's earlier generic reads
    mbar_expect_tx(&bars[q], bytes);
    bulk_g2s(ring + (size_t)q * SLOT, P.pk + L.pbase, bytes, &bars[q]);
  };
  if (t == 0)
    for (int g = 0; g < ILU_PK_RING - 1; g++) issue(g);
  for (int g = 0; g < ntot; g++) {
    if (t == 0) issue(g + ILU_PK_RING - 1);  // slot of level g - 1: every thread passed its barrier
    const IluLevel L = slev[g];
    const bool backward = g >= nf;
    const int q = g % ILU_PK_RING;
    mbar_wait(&bars[q], (uint32_t)((g / ILU_PK_RING) & 1));
    if (t < L.m) {
      const unsigned char *rec = ring + (size_t)q * SLOT;
      const int *k = reinterpret_cast<const int *>(rec);
      const double *f = reinterpret_cast<const double *>(rec + pk_fv_off(L.m, L.c));
      const int i = k[L.c * L.m + t];
      double acc = y[i];
#pragma unroll
      for (int u = 0; u < 4; u++)
        if (u < L.c) {
          const int kk = k[u * L.m + t];
          if (kk >= 0) acc = __dsub_rn(acc, __dmul_rn(f[u * L.m + t], y[kk]));
        }
#if PCG_ILU_RCP
      y[i] = backward ? acc * f[L.c * L.m + t] : acc;
#else
      y[i] = backward ? __ddiv_rn(acc, f[L.c * L.m + t]) : acc;
#endif
    }
    __syncthreads();
  }
  for (int64_t i = t; i < nr; i += T) out[r0 + i] = y[i];
}

constexpr size_t ILU_SMEM_MAX = 227 * 1024;  // opt-in shared memory per CTA

template <int T>
static size_t ilu_packed_smem(int rec_cap, int64_t rows) {
  return (size_t)ILU_PK_RING * pk_bytes(T, 4, true) + 8 * ILU_PK_RING + sizeof(IluLevel) * (size_t)rec_cap +
         sizeof(double) * (size_t)rows;
}

// ---------------------------------------------------------------- setup
pcg_status ilu_setup(pcg_matrix *A, int64_t bs, cudaStream_t st, void **plan_out) {
  const int64_t n = A->n, nnz = A->nnz;
  if (bs < 1) bs = std::max<int64_t>(1, (n + num_sms(A->device) - 1) / num_sms(A->device));
  if (bs > n) bs = std::max<int64_t>(n, 1);
  IluPlan *P = new IluPlan();
  P->bs = bs;
  P->n = n;
  P->nblk = (n + bs - 1) / bs;
  auto bail = [&](pcg_status s) {
    ilu_free(P);
    return s;
  };
  // ---- host level analysis on the (device-validated, int32) CSR
  std::vector<int> rp(n + 1), col(std::max<int64_t>(nnz, 1));
  if (cudaMemcpyAsync(rp.data(), A->d_row_ptr, sizeof(int) * (n + 1), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      (nnz && cudaMemcpyAsync(col.data(), A->d_col, sizeof(int) * nnz, cudaMemcpyDeviceToHost, st) != cudaSuccess) ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return bail(fail(PCG_ERR_CUDA, "ilu_setup: copy of the pattern"));
  std::vector<int> diag(n, -1);
  for (int64_t i = 0; i < n; i++)
    for (int e = rp[i]; e < rp[i + 1]; e++)
      if (col[e] == i) diag[i] = e;
  std::vector<IluLevel> levs;
  std::vector<int> lo(2 * (P->nblk + 1));
  std::vector<int> srow, kcol, emap, udmap;
  std::vector<int> lev(n);
  // emit(chunk): the level-ordered layout; chunk > 0 splits levels wider than `chunk` rows
  // into records of at most `chunk` rows (rows of one level are independent, so its
  // records may run one after the other)
  auto emit = [&](int chunk) {
  levs.clear();
  srow.clear();
  kcol.clear();
  emap.clear();
  udmap.clear();
  for (int d = 0; d < 2; d++) {  // 0: forward (L), 1: backward (U)
    for (int64_t b = 0; b < P->nblk; b++) {
      const int64_t r0 = b * bs, r1 = std::min(r0 + bs, n);
      int maxl = -1;
      for (int64_t q = 0; q < r1 - r0; q++) {
        const int64_t i = d == 0 ? r0 + q : r1 - 1 - q;
        int l = 0;
        for (int e = rp[i]; e < rp[i + 1]; e++) {
          const int64_t k = col[e];
          if (d == 0 ? (k >= r0 && k < i) : (k > i && k < r1)) l = std::max(l, lev[k] + 1);
        }
        lev[i] = l;
        maxl = std::max(maxl, l);
      }
      // counting sort of the block's rows by level (rows ascending inside a level)
      std::vector<int> cnt(maxl + 2, 0);
      for (int64_t i = r0; i < r1; i++) cnt[lev[i] + 1]++;
      for (int l = 0; l <= maxl; l++) cnt[l + 1] += cnt[l];
      std::vector<int> ord(r1 - r0);
      {
        std::vector<int> pos(cnt.begin(), cnt.end() - 1);
        for (int64_t i = r0; i < r1; i++) ord[pos[lev[i]]++] = (int)(i - r0);
      }
      lo[d * (P->nblk + 1) + b] = (int)levs.size();
      for (int l = 0; l <= maxl; l++)
      for (int c0 = cnt[l]; c0 < cnt[l + 1]; c0 += chunk > 0 ? chunk : (cnt[l + 1] - cnt[l])) {
        const int c1 = chunk > 0 ? std::min(cnt[l + 1], c0 + chunk) : cnt[l + 1];
        IluLevel L;
        L.pbase = -1;
        L.row_base = (int64_t)srow.size();
        L.ent_base = (int64_t)kcol.size();
        L.m = c1 - c0;
        int c = 0;
        for (int t = c0; t < c1; t++) {
          const int64_t i = r0 + ord[t];
          int ci = 0;
          for (int e = rp[i]; e < rp[i + 1]; e++) {
            const int64_t k = col[e];
            if (d == 0 ? (k >= r0 && k < i) : (k > i && k < r1)) ci++;
          }
          c = std::max(c, ci);
        }
        L.c = c;
        kcol.resize(kcol.size() + (size_t)L.m * c, -1);
        emap.resize(emap.size() + (size_t)L.m * c, -1);
        for (int t = c0; t < c1; t++) {
          const int64_t i = r0 + ord[t];
          const int slot = t - c0;
          srow.push_back(ord[t]);
          udmap.push_back(d == 1 ? diag[i] : -1);
          int u = 0;
          for (int e = rp[i]; e < rp[i + 1]; e++) {
            const int64_t k = col[e];
            if (d == 0 ? (k >= r0 && k < i) : (k > i && k < r1)) {
              const size_t ei = (size_t)L.ent_base + (size_t)u * L.m + slot;
              kcol[ei] = (int)(k - r0);
              emap[ei] = e;
              u++;
            }
          }
        }
        levs.push_back(L);
      }
    }
    lo[d * (P->nblk + 1) + P->nblk] = (int)levs.size();
  }
  };
  emit(0);
  // ---- packed level records (ilu_apply_packed_kernel): at most 4 entries per row and
  // direction, levels split into records of <= 128 rows, and the block's vector + level
  // records + ring in shared memory; otherwise the cp.async-ring kernel on the unsplit
  // levels (PCG_ILU_PACKED=0 forces it)
  int64_t pk_total = 0;
  {
    constexpr int T = 128;
    auto maxc_of = [&]() {
      int c = 0;
      for (const IluLevel &L : levs) c = std::max(c, L.c);
      return c;
    };
    auto maxlev_of = [&]() {
      int m = 0;
      for (int64_t b = 0; b < P->nblk; b++)
        m = std::max(m, (lo[b + 1] - lo[b]) + (lo[P->nblk + 1 + b + 1] - lo[P->nblk + 1 + b]));
      return m;
    };
    const char *pe = getenv("PCG_ILU_PACKED");
    const int64_t rows = std::min(bs, n);
    if (!(pe && atoi(pe) == 0) && maxc_of() <= 4 && ilu_packed_smem<T>(0, rows) < ILU_SMEM_MAX) {
      emit(T);
      const int ml = maxlev_of();
      if (ilu_packed_smem<T>(ml, rows) <= ILU_SMEM_MAX) {
        P->pk_threads = T;
        P->maxlev = ml;
        const int64_t nfwd_end = lo[P->nblk];
        for (int64_t l = 0; l < (int64_t)levs.size(); l++) {
          levs[l].pbase = pk_total;
          pk_total += pk_bytes(levs[l].m, levs[l].c, l >= nfwd_end);
        }
      } else {
        emit(0);
      }
    }
  }
  P->nlev = (int64_t)levs.size();
  P->nslot = (int64_t)srow.size();
  P->nent = (int64_t)kcol.size();
  // ---- upload
  auto up = [&](void **dst, const void *src, size_t bytes) -> bool {
    if (cudaMalloc(dst, std::max<size_t>(bytes, 8)) != cudaSuccess) return false;
    return bytes == 0 || cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, st) == cudaSuccess;
  };
  if (!up((void **)&P->diag, diag.data(), sizeof(int) * n) || !up((void **)&P->lev, levs.data(), sizeof(IluLevel) * levs.size()) ||
      !up((void **)&P->lo, lo.data(), sizeof(int) * lo.size()) || !up((void **)&P->row, srow.data(), sizeof(int) * srow.size()) ||
      !up((void **)&P->kcol, kcol.data(), sizeof(int) * kcol.size()) ||
      !up((void **)&P->emap, emap.data(), sizeof(int) * emap.size()) ||
      !up((void **)&P->udmap, udmap.data(), sizeof(int) * udmap.size()) ||
      cudaMalloc(&P->f, sizeof(double) * std::max<int64_t>(nnz, 1)) != cudaSuccess ||
      cudaMalloc(&P->fv, sizeof(double) * std::max<int64_t>(P->nent, 1)) != cudaSuccess ||
      cudaMalloc(&P->ud, sizeof(double) * std::max<int64_t>(P->nslot, 1)) != cudaSuccess) {
    cudaGetLastError();
    return bail(fail(PCG_ERR_OOM, "ilu_setup: device memory"));
  }
  if (nnz) PCG_CUDA(cudaMemcpyAsync(P->f, A->d_val, sizeof(double) * nnz, cudaMemcpyDeviceToDevice, st));
  // ---- numeric factorization (forward level order) and the level-ordered factor
  int *err;
  PCG_CUDA(cudaMalloc(&err, sizeof(int)));
  PCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
  ilu_factor_kernel<<<(unsigned)P->nblk, 256, 0, st>>>(n, bs, A->d_row_ptr, A->d_col, P->diag, P->f, P->lev, P->lo,
                                                       P->row, err);
  ilu_fill_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>((std::max(P->nent, P->nslot) + 255) / 256, 4096)),
                    256, 0, st>>>(P->nent, P->emap, P->nslot, P->udmap, P->f, P->fv, P->ud);
  count_launch(2);
  if (P->pk_threads) {
    if (cudaMalloc(&P->pk, (size_t)std::max<int64_t>(pk_total, 16)) != cudaSuccess) {
      cudaGetLastError();
      P->pk = nullptr;
      P->pk_threads = 0;
    } else {
      ilu_pack_kernel<<<(unsigned)P->nlev, 128, 0, st>>>(P->lev, lo[P->nblk], P->row, P->kcol, P->fv, P->ud, P->pk);
      count_launch();
    }
  }
  int herr = 0;
  PCG_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(err);
  if (herr) return bail(fail(PCG_ERR_ZERO_DIAGONAL, "pcg_bicgstab_ilu: zero pivot in the ILU(0) factorization"));
  const int64_t maxrows = std::min(bs, n);
  int cmax = 0;
  for (const IluLevel &L : levs) cmax = std::max(cmax, L.c);
  P->cmax = cmax <= 4 ? 4 : cmax <= 8 ? 8 : 16;
  if (cmax > 16) return bail(fail(PCG_ERR_INVALID_ARG, "pcg_bicgstab_ilu: rows with more than 16 entries per triangle"));
  const size_t vo = ilu_vec_offset(P->cmax);
  P->vec_smem = vo + sizeof(double) * (size_t)maxrows <= ILU_SMEM_MAX;
  P->smem = vo + (P->vec_smem ? sizeof(double) * (size_t)maxrows : 0);
  if (P->pk_threads) {
    P->smem = P->pk_threads == 128 ? ilu_packed_smem<128>(P->maxlev, maxrows) : ilu_packed_smem<256>(P->maxlev, maxrows);
    PCG_CUDA(cudaFuncSetAttribute(P->pk_threads == 128 ? (const void *)ilu_apply_packed_kernel<128>
                                                       : (const void *)ilu_apply_packed_kernel<256>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem));
  } else
  for (auto fn : {(const void *)ilu_apply_kernel<true, 4>, (const void *)ilu_apply_kernel<true, 8>,
                  (const void *)ilu_apply_kernel<true, 16>, (const void *)ilu_apply_kernel<false, 4>,
                  (const void *)ilu_apply_kernel<false, 8>, (const void *)ilu_apply_kernel<false, 16>})
    PCG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem));
  // algorithmic bytes of one application: v in + y out (16 n), the level-ordered factor
  // (8 + 4 B per stored entry, incl. ELL padding) and slots (row 4 B, u_ii 8 B)
  P->bytes_per_apply = 16.0 * n + 12.0 * P->nent + 12.0 * P->nslot + sizeof(IluLevel) * P->nlev;
  *plan_out = P;
  return PCG_OK;
}

void ilu_launch(void *plan, const double *in, double *out, const int *stop, const int *skip, cudaStream_t st) {
  const IluPlan *P = (const IluPlan *)plan;
  const IluView V{P->bs, P->n, P->nblk, P->lev, P->lo, P->row, P->kcol, P->fv, P->ud, P->pk};
  const unsigned g = (unsigned)P->nblk;
  if (P->pk_threads) {
    if (P->pk_threads == 128)
      ilu_apply_packed_kernel<128><<<g, 128, P->smem, st>>>(V, in, out, stop, skip, P->maxlev);
    else
      ilu_apply_packed_kernel<256><<<g, 256, P->smem, st>>>(V, in, out, stop, skip, P->maxlev);
    count_launch();
    return;
  }
#define ILU_GO(SM, CM) ilu_apply_kernel<SM, CM><<<g, ILU_THREADS, P->smem, st>>>(V, in, out, stop, skip)
  if (P->vec_smem) {
    if (P->cmax == 4) ILU_GO(true, 4);
    else if (P->cmax == 8) ILU_GO(true, 8);
    else ILU_GO(true, 16);
  } else {
    if (P->cmax == 4) ILU_GO(false, 4);
    else if (P->cmax == 8) ILU_GO(false, 8);
    else ILU_GO(false, 16);
  }
#undef ILU_GO
  count_launch();
}

int64_t ilu_block_rows(const void *plan) { return ((const IluPlan *)plan)->bs; }
double ilu_bytes_per_apply(const void *plan) { return ((const IluPlan *)plan)->bytes_per_apply; }

}  // namespace pcgb
