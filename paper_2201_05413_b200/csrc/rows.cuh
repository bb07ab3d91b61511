// rows.cuh — row iterators for the two device formats.
//
// Every row sum is formed left to right over the row's stored entries
// (ascending column), i.e. in the order of the paper's MatMult y_i = Σ_j a_ij x_j
// (S:65), with one fused multiply-add per entry.  SELL-32 and CSR with
// L = 1 lane per row therefore produce bitwise-identical sums; CSR with L > 1
// lanes sums L interleaved sub-sums in a fixed shuffle tree.
#pragma once
#include "common.cuh"

namespace pcgb {

// Ordering fence for the SELL loops.  Left alone, the SASS scheduler may emit
// col[u] -> gather[u] -> col[u+1] -> ..., serialising one DRAM round trip per
// entry.  Making every gather index depend on ALL column ids of the chunk
// (j |= xor(j) & zero, with `zero` a run-time 0 the compiler cannot fold) forces
// all column loads to be issued before the first gather address exists.
template <int N>
__device__ __forceinline__ void cols_ready(int (&j)[N], int zero) {
  int x = j[0];
#pragma unroll
  for (int u = 1; u < N; u++) x ^= j[u];
  x &= zero;
#pragma unroll
  for (int u = 0; u < N; u++) j[u] |= x;
}

#ifndef PCG_DIA_SKIPMETA  // pattern slices skip their per-lane offsets/values (waits on the index)
#define PCG_DIA_SKIPMETA 1
#endif
#ifndef PCG_DIA_RUN  // consecutive slices per warp and grid-stride step of the uniform-offset engine
#define PCG_DIA_RUN 8
#endif
#ifndef PCG_SELL_CH  // entries per chunk of the general SELL engine (A/B knob)
#define PCG_SELL_CH 8
#endif

// SELL-32: one warp per slice of 32 consecutive rows, lane = row.  Entries of a
// slice are stored [t][lane] so every load of the t-th entry is one 256-B (val)
// or 128-B (col) coalesced transaction.  Loads are issued 8 entries at a time
// before any gather so each thread keeps 16 independent loads in flight.
// gather(j) -> value multiplied by a_ij;  epi(row, sum) for rows < n.
template <int CH = PCG_SELL_CH, class Gather, class Epi>
__device__ __forceinline__ void sell_rows(const SellView &A, Gather gather, Epi epi) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  // the next slice's offsets are fetched while this slice's entries are in flight (issued
  // after them: an SM's loads complete in issue order), so a slice costs two dependent
  // round trips (entries, gathers) instead of three
  int64_t s = w0, base = 0, next = 0;
  if (s < A.n_slices) {
    base = A.slice_ptr[s];
    next = A.slice_ptr[s + 1];
  }
  for (; s < A.n_slices; s += nw) {
    const int len = (int)((next - base) >> 5);
    const double *vp = A.val + base + lane;
    const int *cp = A.col + base + lane;
    const int64_t s2 = s + nw;
    int64_t base2 = 0, next2 = 0;
    double sum = 0.0;
    for (int t = 0; t < len; t += CH) {
      double a[CH];
      int j[CH];
#pragma unroll
      for (int u = 0; u < CH; u++) j[u] = 0;
#pragma unroll
      for (int u = 0; u < CH; u++) {
        if (t + u < len) {
          a[u] = ld_stream(vp + (size_t)(t + u) * 32);
          j[u] = ld_stream(cp + (size_t)(t + u) * 32);
        }
      }
      if (t == 0 && s2 < A.n_slices) {
        base2 = A.slice_ptr[s2];
        next2 = A.slice_ptr[s2 + 1];
      }
      cols_ready(j, A.zero);
      double g[CH];
#pragma unroll
      for (int u = 0; u < CH; u++)
        if (t + u < len) g[u] = gather(j[u]);
#pragma unroll
      for (int u = 0; u < CH; u++)
        if (t + u < len) sum = __fma_rn(a[u], g[u], sum);
    }
    if (len == 0 && s2 < A.n_slices) {
      base2 = A.slice_ptr[s2];
      next2 = A.slice_ptr[s2 + 1];
    }
    const int64_t row = s * 32 + lane;
    if (row < A.n) epi(row, sum);
    base = base2;
    next = next2;
  }
}

// SELL-32 for systems whose rows hold at most 8 entries (the lattice P1 systems: 7):
// every slice is one chunk, so the chunk loop, its predicates' live ranges and the
// per-chunk state disappear and the kernel fits in fewer registers (more resident warps,
// more slices in flight); the ids are issued before the values (an SM completes loads
// in issue order).  Same entries, same left-to-right sums as sell_rows (bitwise).
template <class Gather, class Epi>
__device__ __forceinline__ void sell_rows_short(const SellView &A, Gather gather, Epi epi) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  int64_t s = w0, base = 0, next = 0;
  if (s < A.n_slices) {
    base = A.slice_ptr[s];
    next = A.slice_ptr[s + 1];
  }
  for (; s < A.n_slices; s += nw) {
    const int len = (int)((next - base) >> 5);  // <= 8 (host-checked)
    const double *vp = A.val + base + lane;
    const int *cp = A.col + base + lane;
    double a[8];
    int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (u < len) j[u] = ld_stream(cp + (size_t)u * 32);
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (u < len) a[u] = ld_stream(vp + (size_t)u * 32);
    const int64_t s2 = s + nw;
    int64_t base2 = 0, next2 = 0;
    if (s2 < A.n_slices) {
      base2 = A.slice_ptr[s2];
      next2 = A.slice_ptr[s2 + 1];
    }
    cols_ready(j, A.zero);
    double g[8];
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (u < len) g[u] = gather(j[u]);
    double sum = 0.0;
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (u < len) sum = __fma_rn(a[u], g[u], sum);
    const int64_t row = s * 32 + lane;
    if (row < A.n) epi(row, sum);
    base = base2;
    next = next2;
  }
}

// The one-chunk engine with uniform-offset positions (SellView::doff / dmask): the next
// slice's mask and offsets are fetched with its slice offsets (indexed by slice: no
// dependent load).  A slice whose positions are all uniform knows its gather addresses
// before any of its loads return and issues values and gathers together: ONE dependent
// round trip instead of two; other slices read their stored ids as sell_rows_short (a
// per-position choice there cost 10 registers for a few bytes).  The same columns as
// sell_rows_short (bitwise the same sums).  A one-trip slice whose values are uniform per
// position as well (SellView::dval) takes them from lanes 0-7 and reads no value stream;
// if its offsets and values are one of the matrix's shared patterns (SellView::dpat) it
// reads them from shared memory instead (six vector loads instead of 24 shuffles).
template <class Gather, class Epi>
__device__ __forceinline__ void sell_rows_dia(const SellViewDia &A, Gather gather, Epi epi) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  // views over a row range (the distributed overlap) start at slice row0 / 32 of the
  // per-slice arrays, and the offsets are relative to the absolute row
  const uint8_t *dmask = A.dmask + (A.row0 >> 5);
  const int *doff = A.doff + (A.row0 >> 5) * 8;
  const uint16_t *dvmeta = A.dvmeta + (A.row0 >> 5);
  const double *dval = A.dval + (A.row0 >> 5) * 8;
  const uint8_t *dpat = A.dpat ? A.dpat + (A.row0 >> 5) : nullptr;
  // the matrix's value-free patterns, staged once per block (every thread of the block
  // runs this engine: the barrier is block-uniform)
  __shared__ DiaPat s_pat[DIA_MAXPAT];
  __shared__ int s_plen[DIA_MAXPAT];
  if (A.npat > 0) {
    for (int t = threadIdx.x; t < A.npat * 12; t += blockDim.x)
      reinterpret_cast<double *>(s_pat)[t] = reinterpret_cast<const double *>(A.ptab)[t];
    for (int t = threadIdx.x; t < A.npat; t += blockDim.x) s_plen[t] = A.plen[t];
    __syncthreads();
  }
  // Each warp takes DIA_RUN consecutive slices per grid-stride step: slices that need two
  // round trips recur with the row-line period of a lattice (Cube 3: 2 of every 16) and a
  // plain grid stride (a multiple of 16 warps) would hand them all to the same warps
  constexpr int RUN = PCG_DIA_RUN;
  auto next_of = [&](int64_t x) { return (x + 1) % RUN != 0 ? x + 1 : x + 1 + (nw - 1) * RUN; };
  // per slice: its first entry; offset mask in bits 0-7, value mask in bits 8-15, length
  // in bits 16-19, pattern index in bits 24-31; lanes 0-7 hold the position offsets and
  // the uniform values
  struct Meta {
    int64_t base;
    unsigned mask;
    int off;
    double val;
    unsigned zm;  // aligned slices: lanes without an entry at position `lane` (lanes 0-7)
  };
  auto meta = [&](int64_t x) {
    Meta m{0, 0u, 0, 0.0, 0u};
    if (x < A.n_slices) {
      const unsigned pid = dpat ? dpat[x] : DIA_NOPAT;
      if (PCG_DIA_SKIPMETA && pid != DIA_NOPAT) {  // a pattern slice: its index is all it needs
        m.mask = pid << 24 | (unsigned)s_plen[pid] << 16;
      } else {
        m.base = A.slice_ptr[x];
        m.mask = (unsigned)dmask[x] | (unsigned)dvmeta[x] << 8 | pid << 24;
        if (lane < 8) {
          m.off = doff[x * 8 + lane];
          m.val = dval[x * 8 + lane];
          if (A.dzmask) m.zm = A.dzmask[(x + (A.row0 >> 5)) * 8 + lane];
        }
      }
    }
    return m;
  };
  auto len_of = [](const Meta &m) { return (int)(m.mask >> 16 & 15u); };
  int64_t s = w0 * RUN;
  // the next slice's metadata is fetched while the current slice is in flight (indexed
  // by slice: no dependent load)
  Meta m0 = meta(s);
  while (s < A.n_slices) {
    const int64_t s2 = next_of(s);
    const int len = len_of(m0);  // <= 8 (host-checked)
    const double *vp = A.val + m0.base + lane;
    const int64_t rowv = s * 32 + lane;         // row within the view (epilogue)
    const int row = (int)(A.row0 + rowv);       // local row (columns)
    const unsigned full = (1u << len) - 1u;
    Meta n1;
    double a[8], g[8];
    double sum = 0.0;
    if ((m0.mask >> 24) != DIA_NOPAT) {  // value-free slice with a shared pattern: no shuffles
      const DiaPat &P = s_pat[m0.mask >> 24];
      const int4 o0 = *reinterpret_cast<const int4 *>(P.off), o1 = *reinterpret_cast<const int4 *>(P.off + 4);
      const int j[8] = {row + o0.x, row + o0.y, row + o0.z, row + o0.w, row + o1.x, row + o1.y, row + o1.z, row + o1.w};
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u < len) g[u] = gather(j[u]);
      n1 = meta(s2);
#pragma unroll
      for (int u = 0; u < 8; u += 2) {
        const double2 v = *reinterpret_cast<const double2 *>(P.val + u);
        a[u] = v.x;
        a[u + 1] = v.y;
      }
    } else if ((m0.mask & full) == full) {  // every position uniform: values and gathers in one round trip
      int j[8];
#pragma unroll
      for (int u = 0; u < 8; u++) j[u] = row + __shfl_sync(0xffffffffu, m0.off, u);
      if ((m0.mask >> 8 & full) == full) {  // ... and every value too: no value stream at all
#pragma unroll
        for (int u = 0; u < 8; u++) a[u] = __shfl_sync(0xffffffffu, m0.val, u);
        if (m0.mask >> 20 & 1u) {  // aligned form: rows without an entry there add 0 * p
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (__shfl_sync(0xffffffffu, m0.zm, u) >> lane & 1u) a[u] = 0.0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (u < len) a[u] = ld_stream(vp + (size_t)u * 32);
      }
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u < len) g[u] = gather(j[u]);
      n1 = meta(s2);
    } else {  // the stored ids (issued first), then the values
      const int *cp = A.col + m0.base + lane;
      int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u < len) j[u] = ld_stream(cp + (size_t)u * 32);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u < len) a[u] = ld_stream(vp + (size_t)u * 32);
      n1 = meta(s2);
      cols_ready(j, A.zero);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (u < len) g[u] = gather(j[u]);
    }
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (u < len) sum = __fma_rn(a[u], g[u], sum);
    if (rowv < A.n) epi(rowv, sum);
    m0 = n1;
    s = s2;
  }
}

// SELL-32 with the 16-bit delta column ids (common.cuh SellView::dcol): the same row
// engine, the same ids (so the same sums, bitwise), 10.125 instead of 12 bytes per entry.
// Per slice the deltas and the per-(slice, t) bases are loaded (indices first: an SM's
// loads complete in issue order), col = row + base + delta; a slice marked CB_INT32 at
// its first base (columns that do not fit 16 bits, rare) reads the int32 ids instead.
// A separate kernel instantiation (FMT_SELL_D16), so the int32 engine above keeps its
// own code.
template <class Gather, class Epi>
__device__ __forceinline__ void sell_rows_d16(const SellView &A, Gather gather, Epi epi) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  // next-slice offsets fetched one slice ahead, as in sell_rows
  int64_t s = w0, base = 0, next = 0;
  if (s < A.n_slices) {
    base = A.slice_ptr[s];
    next = A.slice_ptr[s + 1];
  }
  for (; s < A.n_slices; s += nw) {
    const int len = (int)((next - base) >> 5);
    const int row = (int)(A.row0 + s * 32 + lane);
    const double *vp = A.val + base + lane;
    const int16_t *dp = A.dcol + base + lane;
    const int *cbp = A.cbase + (base >> 5);
    const int64_t s2 = s + nw;
    int64_t base2 = 0, next2 = 0;
    bool fb = false;
    double sum = 0.0;
    for (int t = 0; t < len; t += 8) {
      double a[8];
      int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      // issue order: bases, deltas, values, next offsets (the ids return first)
      const int cbl = (lane < 8 && t + lane < len) ? ld_stream(cbp + t + lane) : 0;
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (t + u < len) j[u] = ld_stream(dp + (size_t)(t + u) * 32);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (t + u < len) a[u] = ld_stream(vp + (size_t)(t + u) * 32);
      if (t == 0 && s2 < A.n_slices) {
        base2 = A.slice_ptr[s2];
        next2 = A.slice_ptr[s2 + 1];
      }
      if (t == 0) fb = __shfl_sync(0xffffffffu, cbl, 0) == CB_INT32;
      if (fb) {
        const int *cp = A.col + base + lane;
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (t + u < len) j[u] = ld_stream(cp + (size_t)(t + u) * 32);
      } else {
#pragma unroll
        for (int u = 0; u < 8; u++) j[u] += row + __shfl_sync(0xffffffffu, cbl, u);
      }
      cols_ready(j, A.zero);
      double g[8];
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (t + u < len) g[u] = gather(j[u]);
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (t + u < len) sum = __fma_rn(a[u], g[u], sum);
    }
    if (len == 0 && s2 < A.n_slices) {
      base2 = A.slice_ptr[s2];
      next2 = A.slice_ptr[s2 + 1];
    }
    if (row - A.row0 < A.n) epi(row - A.row0, sum);
    base = base2;
    next = next2;
  }
}

// CSR: L lanes per row (L in {1,2,4,8,16,32}), lane l takes entries l, l+L, ...
// then the L partial sums meet in a fixed xor-shuffle tree.
template <int L, class Gather, class Epi>
__device__ __forceinline__ void csr_rows(const CsrView &A, Gather gather, Epi epi) {
  const int zero = A.zero;
  const int sub = threadIdx.x & (L - 1);
  const int64_t g0 = ((int64_t)blockIdx.x * BLOCK + threadIdx.x) / L;
  const int64_t ng = (int64_t)gridDim.x * BLOCK / L;
  // all lanes of a warp iterate the same number of times (shuffles need full warps)
  const int64_t iters = (A.n + ng - 1) / ng;
  for (int64_t it = 0; it < iters; it++) {
    const int64_t row = g0 + it * ng;
    double sum = 0.0;
    if (row < A.n) {
      const int rs = A.row_ptr[row], re = A.row_ptr[row + 1];
      for (int k0 = rs + sub; k0 < re; k0 += 8 * L) {  // 8 entries per lane per chunk
        double a[8];
        int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (k0 + u * L < re) {
            a[u] = ld_stream(A.val + k0 + u * L);
            j[u] = ld_stream(A.col + k0 + u * L);
          }
        cols_ready(j, zero);
        double g[8];
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (k0 + u * L < re) g[u] = gather(j[u]);
#pragma unroll
        for (int u = 0; u < 8; u++)
          if (k0 + u * L < re) sum = __fma_rn(a[u], g[u], sum);
      }
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o, L);
    if (row < A.n && sub == 0) epi(row, sum);
  }
}

// Schedule-2 K1 row engine (solver.cu k1_kernel, persist.cu): SpMV + p update + x update + sigma.
// SELL-32 specialisation: one warp per slice, lane = row.  The dependent-load
// chain per slice is kept to two round trips: the own-row vectors (z_i, p_i, x_i)
// are requested together with the slice's matrix entries, and the next slice's
// offsets are fetched one slice ahead (software pipelining).
template <int CH>
__device__ __forceinline__ void k1_sell_rows(const SellView &A, double beta, double alpha_prev,
                                             const double *__restrict__ pold, double *__restrict__ pnew,
                                             const double *__restrict__ z, double *__restrict__ x,
                                             double *__restrict__ q, double &acc) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (int64_t)blockIdx.x * WARPS + (threadIdx.x >> 5);
  const int64_t nw = (int64_t)gridDim.x * WARPS;
  int64_t s = w0;
  int64_t base = 0, next = 0;
  if (s < A.n_slices) {
    base = __ldg(A.slice_ptr + s);
    next = __ldg(A.slice_ptr + s + 1);
  }
  for (; s < A.n_slices; s += nw) {
    const int len = (int)((next - base) >> 5);
    const int64_t row = s * 32 + lane;
    const bool ok = row < A.n;
    // prefetch the following slice's offsets
    const int64_t s2 = s + nw;
    int64_t base2 = 0, next2 = 0;
    if (s2 < A.n_slices) {
      base2 = __ldg(A.slice_ptr + s2);
      next2 = __ldg(A.slice_ptr + s2 + 1);
    }
    // own-row vectors, issued with the matrix stream
    double po = 0.0, zi = 0.0, xi = 0.0;
    if (ok) {
      po = ld_weak(pold + row);  // written by this kernel in the persistent schedule
      zi = ld_weak(z + row);
      xi = __ldcs(x + row);
    }
    const double *vp = A.val + base + lane;
    const int *cp = A.col + base + lane;
    double sum = 0.0;
    for (int t = 0; t < len; t += CH) {
      double a[CH];
      int j[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < CH; u++) {
        if (t + u < len) {
          a[u] = ld_stream(vp + (size_t)(t + u) * 32);
          j[u] = ld_stream(cp + (size_t)(t + u) * 32);
        }
      }
      cols_ready(j, A.zero);
      double g[CH];
#pragma unroll
      for (int u = 0; u < CH; u++)
        if (t + u < len) g[u] = __fma_rn(beta, ld_weak(pold + j[u]), ld_weak(z + j[u]));
#pragma unroll
      for (int u = 0; u < CH; u++)
        if (t + u < len) sum = __fma_rn(a[u], g[u], sum);
    }
    if (ok) {
      const double pi = __fma_rn(beta, po, zi);
      __stcs(pnew + row, pi);
      __stcs(q + row, sum);
      __stcs(x + row, __fma_rn(alpha_prev, po, xi));
      acc = __fma_rn(pi, sum, acc);
    }
    base = base2;
    next = next2;
  }
}

}  // namespace pcgb
