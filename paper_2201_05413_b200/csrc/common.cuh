// common.cuh — internals shared by the product's CUDA translation units.
// (Product code only: nothing here is shared with oracle/.)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <mutex>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "pcg.h"

namespace pcgb {

// NVTX phase ranges (SURVEY §5 tracing): visible in Nsight Systems / ncu --nvtx; the
// header-only NVTX3 calls are no-ops unless a tool is attached.
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange &) = delete;
  NvtxRange &operator=(const NvtxRange &) = delete;
};


// ------------------------------------------------------------------ errors
void set_error(const std::string &msg);
pcg_status fail(pcg_status s, const std::string &msg);
extern std::atomic<int64_t> g_host_launches;  // kernels launched directly from host
inline void count_launch(int64_t k = 1) { g_host_launches += k; }

#define PCG_CUDA(call)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return ::pcgb::fail(e_ == cudaErrorMemoryAllocation ? PCG_ERR_OOM : PCG_ERR_CUDA, \
                          std::string(#call) + ": " + cudaGetErrorString(e_));         \
  } while (0)

#define PCG_TRY(expr)                \
  do {                               \
    pcg_status s_ = (expr);          \
    if (s_ != PCG_OK) return s_;     \
  } while (0)

// ------------------------------------------------------------------ device scalars
// One per solve context.  Written only by "last block" finishers of the fused
// kernels (deterministic fixed-order grid reductions), read by every block at
// kernel entry.  done codes:
enum : int {
  DONE_RUNNING = 0,
  DONE_CONVERGED = 1,  // recurrence residual fired (exit check follows)
  DONE_BREAKDOWN = 2,  // sigma = p^T A p <= 0
  DONE_MAXIT = 3,
  DONE_ZERO_RHS = 4,
  DONE_NONFINITE = 5,
};

struct Scalars {
  double rho, alpha, beta, sigma, gamma;
  double nb, tol, relres_rec, relres_true;
  double rho_part[2];  // (r.z, r.r) partial sums awaiting a cross-GPU allreduce
  double res_part[3];  // (w.w, w.z, b.b) of the residual pass
  double sigma_acc;    // distributed overlap: p.q of the row ranges already done this iteration
  double ahold[3];     // deferred x update: alphas of the held directions p[0..xhold-1]
  long long k, max_iter, replacements;
  int done, parity, stage;  // parity: p[parity] holds the latest direction p_k
  int xhold;                // deferred x update: held directions still owed to x (p[0..xhold-1])
  unsigned int cnt_a, cnt_b, cnt_c, cnt_d;  // last-block arrival counters (self-resetting)
  unsigned long long graph_launches;        // kernels executed from graphs (finishers count)
};

// multi-RHS scalars, one set per column (k <= 32)
constexpr int KMAX = 32;
struct MultiScalars {
  double rho[KMAX], alpha[KMAX], beta[KMAX], sigma[KMAX], gamma[KMAX];
  double nb[KMAX], relres_rec[KMAX], relres_true[KMAX];
  double xpend[KMAX];        // alpha still owed to x (applied by the next K1 / tail)
  double ahold[3][KMAX];     // deferred x update: alphas of the held directions P[0..nheld-1]
  int nheld[KMAX];           // deferred x update: held directions still owed to X
  int lbuf[KMAX];            // deferred x update: the latest direction is in block P[lbuf] (0..3)
  double part[3][KMAX];      // allreduce staging (sigma | rho',gamma | ww,wz,bb)
  long long k[KMAX];
  long long nrep[KMAX];      // residual replacements per column (exit check failed, restarted)
  int done[KMAX];            // per column, same codes as Scalars::done
  int active[KMAX];          // 1 while the column iterates (frozen columns: 0)
  int replace[KMAX];         // residual replacement requested by the exit check
  int parity, n_active, kcols, pad;
  double tol;
  long long max_iter;
  unsigned int cnt_a, cnt_b, cnt_c, cnt_d;
  unsigned long long graph_launches;
};

// ------------------------------------------------------------------ matrix views
struct CsrView {
  int64_t n;            // rows (local)
  int64_t n_cols;       // columns addressable (n + ghosts)
  const int *row_ptr;   // n+1 (int32: nnz < 2^31 per GPU)
  const int *col;       // local column ids
  const double *val;
  int zero;             // run-time 0, opaque to the compiler (rows.cuh cols_ready)
};

struct DiaPat;  // value-free slice pattern (below)
struct SellView {
  int64_t n;
  int64_t n_slices;        // ceil(n/32)
  const int64_t *slice_ptr; // n_slices+1, entry offsets (multiple of 32)
  const int *col;          // [slice][t][lane]
  const double *val;
  int stages;              // TMA-staged variant: shared-memory ring depth
  int64_t stage_entries;   // ... and the largest tile (8 slices) in entries
  const int *lead;         // per tile: max column referenced by tiles 0..t (prefix max)
  int zero;                // always 0 at run time; opaque to the compiler (see cols_ready)
  // 16-bit delta column ids (null: not built).  Entry e of slice s at position t:
  // col = row + cbase[e >> 5] + dcol[e]; cbase has one value per (slice, t) row of 32
  // entries; a slice whose columns do not fit holds CB_INT32 at cbase[slice_ptr[s] >> 5]
  // and is read through `col`.  10.125 instead of 12 bytes per stored entry.
  const int16_t *dcol;
  const int *cbase;
  int64_t row0;  // absolute row of the view's slice 0 (views over a row range; decoding)
  // uniform-offset ("diagonal") positions of the one-chunk engine (null: not built): bit t
  // of dmask[s] set when every real entry of slice s at position t has col = row +
  // doff[8 s + t] (and the padding lanes' row + doff stay in range) — such positions
  // need no column ids, and a slice with only such positions needs one round trip
  const int *doff;
  const uint8_t *dmask;
};
// The uniform-offset engine's further metadata, a separate view so the kernels that do
// not run that engine (the persistent and pipelined kernels, the SpMM) keep the smaller
// parameter block (a larger one measured 7-9 % slower persistent solves: C2, C3, C6).
struct SellViewDia : SellView {
  // value-uniform positions of those slices (CSR-VI-style value sharing; built with doff):
  // bit t of dvmeta[s] set when the 32 stored values of slice s at position t (padding
  // zeros included) are bitwise equal (none with PCG_DIA_VAL=0); that value is
  // dval[8 s + t]; bits 8-11 hold the slice's length.  A slice whose positions are all
  // uniform in offset and value reads neither ids nor values — its 8 offsets and 8 values
  // come with its metadata, and its gathers are its only loads.  The same values in the
  // same order: bitwise the same sums.
  const double *dval;
  const uint16_t *dvmeta;
  // aligned slices (dvmeta bit 12): the positions are the union of the rows' column
  // offsets; bit l of dzmask[8 s + t] set when row l has no entry at position t (it adds
  // 0 * p[row + d]: exact).  Null: not built.
  const unsigned *dzmask;
  // value-free slices grouped by pattern (null dpat: none): dpat[s] indexes ptab, the
  // distinct (offsets, values) of such slices (a lattice stencil has a handful: interior,
  // faces), staged in shared memory once per block; DIA_NOPAT: the slice reads its own.
  // The pattern's offsets and values are the slice's own (checked when built).
  const uint8_t *dpat;
  const DiaPat *ptab;
  const int *plen;  // per pattern: the slice length
  int npat;
};
constexpr int DIA_MAXPAT = 32;
constexpr uint8_t DIA_NOPAT = 0xFF;
struct __align__(16) DiaPat {
  int off[8];
  double val[8];
};
constexpr int CB_INT32 = (int)0x80000000;
// the 16-bit id engine needs ~98 registers unconstrained (2 blocks of 256 per SM); its
// kernels are compiled for 3 resident blocks (<= 80 registers), as the int32 engine runs
#ifndef PCG_D16_MINB
#define PCG_D16_MINB 3
#endif
#ifndef PCG_SELL_MINB  // A/B knob: 0 = unconstrained (80 registers, 3 blocks/SM)
#define PCG_SELL_MINB 0
#endif
#ifndef PCG_DIA_MINB  // the uniform-offset engine: 3 blocks/SM (80 registers, no spills; 4 spill: C5 K1b 1,533 vs 1,810-1,865 us)
#define PCG_DIA_MINB 3
#endif
#ifndef PCG_SHORT_MINB  // the short-row engine (rows.cuh sell_rows_short): resident blocks per SM
#define PCG_SHORT_MINB 4
#endif
#define D16_MINB(FMT)                                                     \
  ((FMT) == FMT_SELL_D16 ? PCG_D16_MINB : (FMT) == FMT_SELL_SHORT ? PCG_SHORT_MINB \
   : (FMT) == FMT_SELL_DIA ? PCG_DIA_MINB \
   : (FMT) == PCG_FORMAT_SELL ? PCG_SELL_MINB : 0)

// internal format code of the TMA-staged SELL kernels (reported as PCG_FORMAT_SELL_TMA)
constexpr int FMT_SELL_TMA = 3;
// internal code of the SELL-32 kernels that read the 16-bit delta column ids (rows.cuh
// sell_rows_d16): the SpMV, K1b and residual passes of the 3-pass schedule
constexpr int FMT_SELL_D16 = 5;
constexpr int FMT_SELL_SHORT = 6;  // SELL-32, every row <= 8 entries: one-chunk engine
constexpr int FMT_SELL_DIA = 7;    // the one-chunk engine with uniform-offset positions (no ids)

// ------------------------------------------------------------------ reductions
constexpr int BLOCK = 256;
constexpr int WARPS = BLOCK / 32;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Fixed-order block sum of NV values; result valid in thread 0.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double (*sm)[WARPS]) {
#pragma unroll
  for (int i = 0; i < NV; i++) v[i] = warp_sum(v[i]);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; i++) sm[i][w] = v[i];
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; i++) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < WARPS; j++) s += sm[i][j];
      v[i] = s;
    }
  }
}

// Writes this block's NV partials, then returns true in exactly one block:
// the last to arrive, after all partials are visible.
template <int NV>
__device__ __forceinline__ bool publish_and_arrive(const double (&v)[NV], double *partials,
                                                   unsigned int *counter) {
  __shared__ bool s_last;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < NV; i++) partials[(size_t)i * gridDim.x + blockIdx.x] = v[i];
    __threadfence();
    unsigned int prev = atomicAdd(counter, 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) __threadfence();
  return s_last;
}

// In the last block: fixed-order sum over all blocks' partials (bypassing L1).
template <int NV>
__device__ __forceinline__ void reduce_partials(const double *partials, double (&out)[NV],
                                                double (*sm)[WARPS]) {
  double v[NV];
#pragma unroll
  for (int i = 0; i < NV; i++) {
    double s = 0.0;
    for (unsigned int b = threadIdx.x; b < gridDim.x; b += BLOCK)
      s += __ldcg(partials + (size_t)i * gridDim.x + b);
    v[i] = s;
  }
  __syncthreads();
  block_sum<NV>(v, sm);
  if (threadIdx.x == 0)
#pragma unroll
    for (int i = 0; i < NV; i++) out[i] = v[i];
}

// streaming loads for matrix data (read once per pass, keep out of L1).  volatile:
// a non-volatile asm with no memory operand counts as side-effect free, and the
// compiler may then hoist it out of the branch that guards its address.
__device__ __forceinline__ double ld_stream(const double *p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int *p) {
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int ld_stream(const int16_t *p) {  // sign-extended to 32 bits
  int v;
  asm volatile("ld.global.nc.L1::no_allocate.s16 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Coherent (weak, L1-cacheable) load for vectors that the SAME kernel also writes —
// the gathers of the persistent cooperative kernels, where a grid barrier separates
// the pass that writes a vector from the pass that reads it.  The PTX memory model
// orders such a plain load after the barrier's acquire (bar.sync carries thread 0's
// ld.acquire.gpu to the CTA), whereas ld.global.nc (__ldg) is defined only for data
// that is read-only for the whole kernel.  volatile for the reason given above; the
// barrier's own asm carries the memory clobber.
__device__ __forceinline__ double ld_weak(const double *p) {
  double v;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

int num_sms(int device);

}  // namespace pcgb
