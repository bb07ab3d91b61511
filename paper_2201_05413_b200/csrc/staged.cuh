// staged.cuh — SELL-32 row engine with the matrix stream staged through shared
// memory by the Tensor Memory Accelerator's bulk-copy path.
//
// A tile is WARPS consecutive SELL slices (256 rows).  SELL stores the slices of
// a tile contiguously, so a tile's values and column ids are two contiguous
// byte ranges: warp 0 issues `cp.async.bulk` global->shared copies per tile
// (values, column ids, and up to NOWN own-row vectors such as x) into a ring of
// S stages, completion tracked by one mbarrier per stage (expect_tx bytes).
//
// Gathers: for stencil-like matrices the only DRAM misses among the gathered
// vector entries are the first touches, i.e. columns beyond every column
// referenced by earlier tiles.  lead[t] = max column referenced by tiles 0..t
// (prefix max, computed at setup), so tile t first touches columns
// (lead[t-1], lead[t]]; when tile t is issued (S rounds ahead) warp 0 also
// issues `cp.async.bulk.prefetch.L2` for that window of each of the NPF gathered
// vectors.  By the time the warps gather, those lines sit in L2.
//
// Warps read their slice's entries from shared memory ([t][lane] layout:
// conflict-free).  The persistent grid walks tiles round-robin (tile =
// block + k*grid); tile k+S is issued as soon as every warp is done with tile k.
#pragma once
#include "common.cuh"

namespace pcgb {

constexpr int TILE_ROWS = WARPS * 32;

struct SellStage {
  int stages;             // ring depth S (>= 1)
  int64_t stage_entries;  // max entries of any tile (multiple of 32)
  __host__ __device__ SellStage(int s, int64_t e) : stages(s), stage_entries(e) {}
  __host__ __device__ SellStage(const SellView &v) : stages(v.stages), stage_entries(v.stage_entries) {}
};

__host__ __device__ inline size_t staged_stage_bytes(const SellStage &c, int nown) {
  // entries doubles + entries ints + own-row vectors + (WARPS+1) slice offsets, 128-B aligned
  const size_t per = (size_t)c.stage_entries * 12 + (size_t)nown * TILE_ROWS * 8 + 8 * (WARPS + 1);
  return (per + 127) & ~(size_t)127;
}
__host__ __device__ inline size_t staged_smem_bytes(const SellStage &c, int nown = 1) {
  return (size_t)c.stages * staged_stage_bytes(c, nown) + 8 * (size_t)c.stages;
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok);
}

template <int NOWN, int NPF>
struct StageIO {
  const double *own[NOWN > 0 ? NOWN : 1];  // own-row vectors staged per tile (padded allocations)
  const double *pf[NPF > 0 ? NPF : 1];     // gathered vectors, L2-prefetched by leading edge
  int64_t pf_len;                          // entries addressable in the gathered vectors
};

// pre(row) -> P (own-row loads issued before the stage wait)
// gather(j) -> value multiplying a_ij
// epi(row, sum, P&, const double* own /* own[k * TILE_ROWS] = k-th staged vector at row */)
template <int CH, int NOWN, int NPF, class Pre, class Gather, class Epi>
__device__ __forceinline__ void sell_staged_rows(const SellView &A, const StageIO<NOWN, NPF> io, Pre pre,
                                                 Gather gather, Epi epi) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int S = A.stages;
  const size_t per = staged_stage_bytes(SellStage(A), NOWN);
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + (size_t)S * per);
  const int64_t E = A.stage_entries;
  auto stage_val = [&](int s) { return reinterpret_cast<double *>(smem + (size_t)s * per); };
  auto stage_col = [&](int s) { return reinterpret_cast<int *>(smem + (size_t)s * per + (size_t)E * 8); };
  auto stage_own = [&](int s) { return reinterpret_cast<double *>(smem + (size_t)s * per + (size_t)E * 12); };
  auto stage_meta = [&](int s) {
    return reinterpret_cast<int64_t *>(smem + (size_t)s * per + (size_t)E * 12 + (size_t)NOWN * TILE_ROWS * 8);
  };
  const int64_t n_tiles = (A.n_slices + WARPS - 1) / WARPS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  auto issue = [&](int64_t t, int s) {  // warp 0
    int64_t *meta = stage_meta(s);
    int64_t v = 0;
    if (lane <= WARPS) {
      int64_t si = t * WARPS + lane;
      if (si > A.n_slices) si = A.n_slices;
      v = __ldg(A.slice_ptr + si);
      meta[lane] = v;
    }
    const int64_t lo = __shfl_sync(0xffffffffu, v, 0), hi = __shfl_sync(0xffffffffu, v, WARPS);
    __syncwarp();
    const int64_t r0 = t * TILE_ROWS;
    int64_t rows = A.n - r0;
    if (rows > TILE_ROWS) rows = TILE_ROWS;
    const int64_t rows2 = (rows + 1) & ~(int64_t)1;  // 16-B multiple (vectors carry >= 1 pad entry)
    if (lane == 0) {
      const int64_t cnt = hi - lo;
      mbar_expect_tx(&bars[s], (uint32_t)(cnt * 12 + (int64_t)NOWN * rows2 * 8));
      if (cnt > 0) {
        bulk_g2s(stage_val(s), A.val + lo, (uint32_t)(cnt * 8), &bars[s]);
        bulk_g2s(stage_col(s), A.col + lo, (uint32_t)(cnt * 4), &bars[s]);
      }
#pragma unroll
      for (int k = 0; k < NOWN; k++)
        bulk_g2s(stage_own(s) + k * TILE_ROWS, io.own[k] + r0, (uint32_t)(rows2 * 8), &bars[s]);
    }
    if (NPF > 0 && lane >= 1 && lane <= NPF && A.lead) {
      // first-touch window of this tile in the gathered vectors
      const int64_t a = t > 0 ? (int64_t)__ldg(A.lead + t - 1) + 1 : 0;
      int64_t b = (int64_t)__ldg(A.lead + t) + 1;
      if (b > io.pf_len) b = io.pf_len;
      const int64_t a16 = a & ~(int64_t)1, b16 = b & ~(int64_t)1;  // 16-B aligned, inside the allocation
      if (b16 > a16 && (b16 - a16) * 8 <= (1 << 20))
        bulk_prefetch_l2(io.pf[lane - 1] + a16, (uint32_t)((b16 - a16) * 8));
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0)
    for (int s = 0; s < S; s++) {
      const int64_t t = (int64_t)blockIdx.x + (int64_t)s * gridDim.x;
      if (t < n_tiles) issue(t, s);
    }
  for (int64_t k = 0;; k++) {
    const int64_t t = (int64_t)blockIdx.x + k * gridDim.x;
    if (t >= n_tiles) break;
    const int s = (int)(k % S);
    const uint32_t parity = (uint32_t)((k / S) & 1);
    const int64_t slice = t * WARPS + warp;
    const int64_t row = slice * 32 + lane;
    const bool ok = row < A.n;
    auto pf = pre(ok ? row : 0);
    mbar_wait(&bars[s], parity);
    if (slice < A.n_slices) {
      const int64_t *meta = stage_meta(s);
      const int off = (int)(meta[warp] - meta[0]);
      const int len = (int)((meta[warp + 1] - meta[warp]) >> 5);
      const double *vs = stage_val(s) + off + lane;
      const int *cs = stage_col(s) + off + lane;
      double sum = 0.0;
      for (int u0 = 0; u0 < len; u0 += CH) {
        double a[CH], g[CH];
#pragma unroll
        for (int u = 0; u < CH; u++)
          if (u0 + u < len) {
            a[u] = vs[(u0 + u) * 32];
            g[u] = gather(cs[(u0 + u) * 32]);
          }
#pragma unroll
        for (int u = 0; u < CH; u++)
          if (u0 + u < len) sum = __fma_rn(a[u], g[u], sum);
      }
      if (ok) epi(row, sum, pf, stage_own(s) + warp * 32 + lane);
    }
    __syncthreads();  // every warp is done with stage s
    if (warp == 0) {
      const int64_t tn = t + (int64_t)S * gridDim.x;
      if (tn < n_tiles) issue(tn, s);
    }
  }
}

}  // namespace pcgb
