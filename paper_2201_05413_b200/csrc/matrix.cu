// matrix.cu — csr_create: validation, int32 narrowing,
// dinv = 1/a_ii, SELL-32 build and measured format choice; workspace alloc.
//
// Validation follows the CSR invariants of SPEC.md S:28-34 (row_ptr[0] = 0,
// row_ptr[n] = nnz, non-decreasing; columns in range and strictly increasing
// within a row) plus finiteness and the Jacobi preconditioner's need
// for a positive diagonal.  All checks run on the device, one
// thread per row; the first offending row is reported.
#include <climits>
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cstring>

#include "matrix.cuh"
#include "staged.cuh"

namespace pcgb {

enum : int {
  E_DIM = 1,
  E_INDEX = 2,
  E_UNSORTED = 4,
  E_NONFINITE = 8,
  E_ZERO_DIAG = 16,
  E_NEG_DIAG = 32,
};

struct ErrInfo {
  int flags;
  int max_len;
  unsigned long long first_row[6];
};

__device__ __forceinline__ void report(ErrInfo *e, int bit, int64_t row) {
  atomicOr(&e->flags, bit);
  atomicMin(&e->first_row[__ffs(bit) - 1], (unsigned long long)row);
}

// col_map: optional (distributed) global -> local column translation is done by a
// later pass; here columns are checked against [0, n_cols).
__global__ void validate_kernel(int64_t n, int64_t nnz, int64_t n_cols, int64_t diag_offset,
                                const int64_t *__restrict__ rp, const int64_t *__restrict__ col,
                                const double *__restrict__ val, int *__restrict__ rp32,
                                double *__restrict__ dinv, ErrInfo *err) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  const int64_t s = rp[i];
  if (i == n) {
    rp32[n] = (int)s;
    return;
  }
  const int64_t e = rp[i + 1];
  rp32[i] = (int)s;
  if (s < 0 || e < s || e > nnz) {
    report(err, E_DIM, i);
    dinv[i] = 0.0;
    return;
  }
  atomicMax(&err->max_len, (int)(e - s));
  double d = 0.0;
  bool has_d = false;
  int64_t prev = -1;
  for (int64_t k = s; k < e; k++) {
    const int64_t j = col[k];
    const double a = val[k];
    if (j < 0 || j >= n_cols) {
      report(err, E_INDEX, i);
      continue;
    }
    if (j <= prev) report(err, E_UNSORTED, i);
    prev = j;
    if (!isfinite(a)) report(err, E_NONFINITE, i);
    if (j == i + diag_offset) {
      d = a;
      has_d = true;
    }
  }
  if (!has_d || d == 0.0) {
    report(err, E_ZERO_DIAG, i);
    dinv[i] = 0.0;
  } else {
    if (d < 0.0) report(err, E_NEG_DIAG, i);
    dinv[i] = 1.0 / d;
  }
}

__global__ void narrow_kernel(int64_t nnz, const int64_t *__restrict__ col, const double *__restrict__ val,
                              int *__restrict__ col32, double *__restrict__ valo, int64_t col_shift) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    col32[k] = (int)(col[k] - col_shift);
    valo[k] = val[k];
  }
}

// SELL-32: per slice the max row length, times 32 entries
__global__ void slice_len_kernel(int64_t n, int64_t n_slices, const int *__restrict__ rp, int64_t *__restrict__ out) {
  int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > n_slices) return;
  if (s == n_slices) {
    out[s] = 0;
    return;
  }
  int m = 0;
  for (int l = 0; l < 32; l++) {
    int64_t r = s * 32 + l;
    if (r < n) m = max(m, rp[r + 1] - rp[r]);
  }
  out[s] = (int64_t)m * 32;
}

__global__ void sell_fill_kernel(int64_t n, int64_t n_slices, const int *__restrict__ rp,
                                 const int *__restrict__ col, const double *__restrict__ val,
                                 const int64_t *__restrict__ slice_ptr, int *__restrict__ scol,
                                 double *__restrict__ sval) {
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t s = tid >> 5;
  int lane = tid & 31;
  if (s >= n_slices) return;
  int64_t row = s * 32 + lane;
  int64_t base = slice_ptr[s];
  int len = (int)((slice_ptr[s + 1] - base) >> 5);
  int rs = 0, rl = 0;
  if (row < n) {
    rs = rp[row];
    rl = rp[row + 1] - rs;
  }
  for (int t = 0; t < len; t++) {
    int64_t e = base + (int64_t)t * 32 + lane;
    if (t < rl) {
      scol[e] = col[rs + t];
      sval[e] = val[rs + t];
    } else {  // padding: a_ii-position dummy, contributes 0 * finite
      scol[e] = row < n ? (int)row : 0;
      sval[e] = 0.0;
    }
  }
}

// per tile (WARPS slices): the largest column any entry references
__global__ void tile_lead_kernel(int64_t n_slices, const int64_t *__restrict__ slice_ptr, const int *__restrict__ scol,
                                 int *__restrict__ lead) {
  const int64_t t = blockIdx.x;
  int64_t s1 = (t + 1) * WARPS;
  if (s1 > n_slices) s1 = n_slices;
  const int64_t lo = slice_ptr[t * WARPS], hi = slice_ptr[s1];
  int m = 0;
  for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) m = max(m, scol[e]);
  __shared__ int sm[256];
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) sm[threadIdx.x] = max(sm[threadIdx.x], sm[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) lead[t] = sm[0];
}

int num_sms(int device) {
  int v = 0;
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  return v > 0 ? v : 148;
}

// declared in solver.cu
pcg_status launch_spmv_fmt(pcg_matrix *A, int fmt, const double *x, double *y, cudaStream_t st);
int k1_blocks_per_sm(int fmt, int lanes, size_t smem);
pcg_status prepare_staged(size_t smem);

static pcg_status error_from_flags(const ErrInfo &e, int64_t row_offset) {
  static const struct {
    int bit;
    pcg_status st;
    const char *what;
  } order[] = {
      {E_DIM, PCG_ERR_DIMENSION_MISMATCH, "row_ptr not monotone / out of [0, nnz]"},
      {E_INDEX, PCG_ERR_INDEX_OUT_OF_RANGE, "column index out of range"},
      {E_UNSORTED, PCG_ERR_UNSORTED_OR_DUPLICATE, "columns not strictly increasing"},
      {E_NONFINITE, PCG_ERR_NONFINITE, "non-finite value"},
      {E_ZERO_DIAG, PCG_ERR_ZERO_DIAGONAL, "zero or missing diagonal"},
      {E_NEG_DIAG, PCG_ERR_NOT_SPD, "negative diagonal (not SPD)"},
  };
  for (auto &o : order)
    if (e.flags & o.bit)
      return fail(o.st, std::string("csr_create: ") + o.what + " in row " +
                            std::to_string((long long)e.first_row[__builtin_ctz(o.bit)] + row_offset));
  return PCG_OK;
}

// SELL-32 arrays from the device CSR (slice_ptr by a scan of per-slice max row
// lengths; entries [slice][t][lane], padding col = row, val = 0).
pcg_status build_sell(pcg_matrix *A, cudaStream_t st) {
  if (A->d_slice_ptr) return PCG_OK;
  const int64_t n = A->n;
  A->n_slices = (n + 31) / 32;
  PCG_CUDA(cudaMalloc(&A->d_slice_ptr, sizeof(int64_t) * (A->n_slices + 1)));
  int64_t *tmp;
  PCG_CUDA(cudaMalloc(&tmp, sizeof(int64_t) * (A->n_slices + 1)));
  slice_len_kernel<<<(unsigned)((A->n_slices + 1 + 255) / 256), 256, 0, st>>>(n, A->n_slices, A->d_row_ptr, tmp);
  count_launch();
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, tmp, A->d_slice_ptr, A->n_slices + 1, st);
  void *tbuf;
  PCG_CUDA(cudaMalloc(&tbuf, tb));
  cub::DeviceScan::ExclusiveSum(tbuf, tb, tmp, A->d_slice_ptr, A->n_slices + 1, st);
  PCG_CUDA(cudaMemcpyAsync(&A->sell_entries, A->d_slice_ptr + A->n_slices, sizeof(int64_t), cudaMemcpyDeviceToHost,
                           st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(tbuf);
  cudaFree(tmp);
  if (A->sell_entries >= (int64_t(1) << 31)) {
    free_sell(A);
    return fail(PCG_ERR_INVALID_ARG, "csr_create: padded SELL entries exceed 2^31 on one GPU");
  }
  PCG_CUDA(cudaMalloc(&A->d_scol, sizeof(int) * (A->sell_entries > 0 ? A->sell_entries : 1)));
  PCG_CUDA(cudaMalloc(&A->d_sval, sizeof(double) * (A->sell_entries > 0 ? A->sell_entries : 1)));
  if (A->n_slices > 0) {
    sell_fill_kernel<<<(unsigned)((A->n_slices * 32 + 255) / 256), 256, 0, st>>>(
        n, A->n_slices, A->d_row_ptr, A->d_col, A->d_val, A->d_slice_ptr, A->d_scol, A->d_sval);
    count_launch();
    PCG_CUDA(cudaGetLastError());
  }
  A->device_bytes += (double)(A->n_slices + 1) * 8 + (double)A->sell_entries * 12;
  return PCG_OK;
}

// 16-bit delta column ids (common.cuh SellView::dcol), one warp per slice.  Per
// entry row t of the slice, the offsets col - row of the real entries (t < row
// length) must span <= 65535: cbase = min offset + 32768, delta = offset - cbase.
// Padding entries (a = 0) keep a valid column: delta = -cbase (col = row) when it
// fits, else the nearest representable one if it lies in [0, n_cols).  A slice where
// any of this fails is marked CB_INT32 and read through the int32 ids.
__global__ void d16_build_kernel(int64_t n, int64_t n_cols, int64_t n_slices, const int *__restrict__ rp,
                                 const int64_t *__restrict__ slice_ptr, const int *__restrict__ scol,
                                 int16_t *__restrict__ dcol, int *__restrict__ cbase,
                                 unsigned long long *__restrict__ n_ok) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= n_slices) return;
  const int64_t row = s * 32 + lane;
  const int64_t base = slice_ptr[s];
  const int len = (int)((slice_ptr[s + 1] - base) >> 5);
  if (len == 0) return;
  const int rl = row < n ? rp[row + 1] - rp[row] : 0;
  bool ok = true;
  for (int t = 0; t < len; t++) {
    const int64_t e = base + (int64_t)t * 32 + lane;
    const bool real = t < rl;
    const long long off = (long long)scol[e] - row;
    long long lo = real ? off : LLONG_MAX, hi = real ? off : LLONG_MIN;
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, (long long)__shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, (long long)__shfl_xor_sync(0xffffffffu, hi, o));
    }
    long long b = 0;
    if (lo != LLONG_MAX) {
      if (hi - lo > 65535) ok = false;
      b = lo + 32768;
    }
    long long d;
    if (real) {
      d = off - b;
    } else {
      d = -b;  // aim at col = row
      if (d < -32768) d = -32768;
      if (d > 32767) d = 32767;
      const long long c = row + b + d;
      if (c < 0 || c >= n_cols) ok = false;
    }
    if (d < -32768 || d > 32767) ok = false;
    dcol[e] = (int16_t)(ok ? d : 0);
    if (lane == 0) cbase[e >> 5] = (int)b;
  }
  ok = __all_sync(0xffffffffu, ok);
  if (lane == 0) {
    if (ok) atomicAdd(n_ok, 1ull);
    else cbase[base >> 5] = CB_INT32;
  }
}

pcg_status build_d16(pcg_matrix *A, cudaStream_t st) {
  // opt-in (PCG_D16=1): measured on B200 it moves 13 % fewer K1b bytes on C5 but takes
  // the same time (K1b 2,350 us either way; C3 148 us either way), DESIGN.md §7
  const char *e = getenv("PCG_D16");
  if (A->d_sdcol || !A->d_slice_ptr || A->n_slices == 0 || !(e && atoi(e) == 1) || getenv("PCG_NO_D16")) return PCG_OK;
  PCG_CUDA(cudaMalloc(&A->d_sdcol, sizeof(int16_t) * std::max<int64_t>(A->sell_entries, 1)));
  PCG_CUDA(cudaMalloc(&A->d_scbase, sizeof(int) * std::max<int64_t>(A->sell_entries / 32, 1)));
  unsigned long long *d_ok;
  PCG_CUDA(cudaMalloc(&d_ok, sizeof(unsigned long long)));
  PCG_CUDA(cudaMemsetAsync(d_ok, 0, sizeof(unsigned long long), st));
  d16_build_kernel<<<(unsigned)((A->n_slices * 32 + 255) / 256), 256, 0, st>>>(
      A->n, A->n + A->n_ghost, A->n_slices, A->d_row_ptr, A->d_slice_ptr, A->d_scol, A->d_sdcol, A->d_scbase, d_ok);
  count_launch();
  unsigned long long ok = 0;
  PCG_CUDA(cudaMemcpyAsync(&ok, d_ok, sizeof(ok), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_ok);
  A->d16_slices = (int64_t)ok;
  if (ok == 0) {  // nothing compresses: keep the int32 form only
    cudaFree(A->d_sdcol);
    cudaFree(A->d_scbase);
    A->d_sdcol = nullptr;
    A->d_scbase = nullptr;
  } else {
    A->device_bytes += (double)A->sell_entries * 2 + (double)(A->sell_entries / 32) * 4;
  }
  return PCG_OK;
}

// Uniform-offset positions (SellView::doff / dmask), one warp per slice of at most 8
// entries per row: position t of slice s is uniform when every real entry there has
// the same col - row = d, and every padding lane's row + d lies in [0, n_cols) (its
// value is 0: fma(0, p[row + d], s) == s, as with the stored padding column).
// Also the value-uniform positions and the slice length (SellView::dval / dvmeta): the 32
// stored values at position t (padding zeros included) bitwise equal (vals = 0: none).
__global__ void dia_build_kernel(int64_t n, int64_t n_cols, int64_t n_slices, const int *__restrict__ rp,
                                 const int64_t *__restrict__ slice_ptr, const int *__restrict__ scol,
                                 const double *__restrict__ sval, int vals, int *__restrict__ doff,
                                 uint8_t *__restrict__ dmask, double *__restrict__ dval,
                                 uint16_t *__restrict__ dvmeta, unsigned *__restrict__ dzmask,
                                 unsigned long long *__restrict__ n_pos) {
  const int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (s >= n_slices) return;
  const int64_t row = s * 32 + lane;
  const int64_t base = slice_ptr[s];
  const int len = (int)((slice_ptr[s + 1] - base) >> 5);
  const int rl = row < n ? rp[row + 1] - rp[row] : 0;
  unsigned mask = 0, vmask = 0;
  for (int t = 0; t < len && t < 8; t++) {
    const int64_t e = base + (int64_t)t * 32 + lane;
    if (vals) {
      const unsigned long long vb = (unsigned long long)__double_as_longlong(sval[e]);
      const unsigned long long v0 = __shfl_sync(0xffffffffu, vb, 0);
      if (__all_sync(0xffffffffu, vb == v0)) vmask |= 1u << t;
      if (lane == 0) dval[s * 8 + t] = __longlong_as_double((long long)v0);
    }
    const bool real = t < rl;
    const long long off = (long long)scol[e] - row;
    long long lo = real ? off : LLONG_MAX, hi = real ? off : LLONG_MIN;
    for (int o = 16; o > 0; o >>= 1) {
      lo = min(lo, (long long)__shfl_xor_sync(0xffffffffu, lo, o));
      hi = max(hi, (long long)__shfl_xor_sync(0xffffffffu, hi, o));
    }
    bool ok = lo != LLONG_MAX && lo == hi && lo >= INT_MIN && lo <= INT_MAX;
    if (ok && !real) {
      const long long c = row + lo;
      ok = c >= 0 && c < n_cols;
    }
    ok = __all_sync(0xffffffffu, ok);
    if (ok) mask |= 1u << t;
    if (lane == 0) doff[s * 8 + t] = ok ? (int)lo : 0;
  }
  const unsigned fl = (1u << len) - 1u;
  if (vals && dzmask && len <= 8 && (mask & vmask) != fl) {
    // Aligned form: the union of the rows' column offsets as the positions (ascending, so
    // each row keeps its column order), a row without an entry at a position adds
    // 0 * p[row + d] there (exact: the sum never is -0 and p[row + d] is in range).  Kept
    // when every position's present values are bitwise equal (a value-free slice with
    // a zero mask: a lattice's rows at the ends of grid lines).
    int cur = 0, np = 0;
    bool ok = true;
    int aoff[8];
    double aval[8];
    unsigned azm[8];
    for (int t = 0; t < 8 && ok; t++) {
      const long long my = cur < rl ? (long long)scol[base + (int64_t)cur * 32 + lane] - row : LLONG_MAX;
      long long d = my;
      for (int o = 16; o > 0; o >>= 1) d = min(d, (long long)__shfl_xor_sync(0xffffffffu, d, o));
      if (d == LLONG_MAX) break;  // every row consumed
      const bool present = my == d;
      const unsigned pres = __ballot_sync(0xffffffffu, present);
      const unsigned long long vb =
          present ? (unsigned long long)__double_as_longlong(sval[base + (int64_t)cur * 32 + lane]) : 0ull;
      const unsigned long long v0 = __shfl_sync(0xffffffffu, vb, __ffs(pres) - 1);
      const long long c = row + d;
      ok = __all_sync(0xffffffffu, (present ? vb == v0 : (c >= 0 && c < n_cols))) && d >= INT_MIN && d <= INT_MAX;
      aoff[t] = (int)d;
      aval[t] = __longlong_as_double((long long)v0);
      azm[t] = ~pres;
      cur += present;
      np = t + 1;
    }
    ok = ok && __all_sync(0xffffffffu, cur == rl) && np > 0;
    if (ok) {
      if (lane < 8) {
        doff[s * 8 + lane] = lane < np ? aoff[lane] : 0;
        dval[s * 8 + lane] = lane < np ? aval[lane] : 0.0;
        dzmask[s * 8 + lane] = lane < np ? azm[lane] : 0u;
      }
      if (lane == 0) {
        const unsigned f = (1u << np) - 1u;
        dmask[s] = (uint8_t)f;
        dvmeta[s] = (uint16_t)(f | (unsigned)np << 8 | 1u << 12);
        atomicAdd(n_pos, (unsigned long long)np);
        atomicAdd(n_pos + 1, 1ull);
        atomicAdd(n_pos + 3, 1ull);
      }
      return;
    }
  }
  if (lane == 0) {
    dmask[s] = (uint8_t)mask;
    atomicAdd(n_pos, (unsigned long long)__popc(mask));
    const unsigned full = (1u << len) - 1u;
    if (len <= 8 && mask == full) atomicAdd(n_pos + 1, 1ull);  // one-round-trip slice
    dvmeta[s] = (uint16_t)(vmask | (unsigned)min(len, 15) << 8);
    if (len <= 8 && (mask & vmask) == full) atomicAdd(n_pos + 2, 1ull);  // ... without a value stream
  }
}

// Value-free slice patterns: a 64-bit key per value-free one-trip slice (its length, 8
// offsets and 8 value bit patterns; ~0 for the other slices), the host picks the first
// DIA_MAXPAT distinct keys, dia_pat_fill_kernel copies each one's representative and
// dia_pat_assign_kernel gives every slice whose metadata EQUALS a table entry its index
// (a key collision only costs the pattern, never a wrong sum).
__device__ __forceinline__ unsigned long long pat_mix(unsigned long long h, unsigned long long v) {
  h ^= v + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  h ^= h >> 31;
  h *= 0xBF58476D1CE4E5B9ull;
  return h ^ (h >> 29);
}
__device__ __forceinline__ bool value_free(uint8_t dm, uint16_t vm) {
  if (vm >> 12 & 1) return false;  // aligned slices keep their zero masks: no shared pattern
  const int len = vm >> 8 & 15;
  const unsigned full = (1u << len) - 1u;
  return len <= 8 && (dm & full) == full && ((unsigned)vm & full) == full;
}
__global__ void dia_key_kernel(int64_t n_slices, const int *__restrict__ doff, const double *__restrict__ dval,
                               const uint8_t *__restrict__ dmask, const uint16_t *__restrict__ dvmeta,
                               unsigned long long *__restrict__ key) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_slices; s += (int64_t)gridDim.x * blockDim.x) {
    if (!value_free(dmask[s], dvmeta[s])) {
      key[s] = ~0ull;
      continue;
    }
    unsigned long long h = pat_mix(0, dvmeta[s] >> 8);
    for (int t = 0; t < 8; t++) {
      h = pat_mix(h, (unsigned long long)(unsigned)doff[s * 8 + t]);
      h = pat_mix(h, (unsigned long long)__double_as_longlong(dval[s * 8 + t]));
    }
    key[s] = h == ~0ull ? 0 : h;
  }
}
__global__ void dia_pat_fill_kernel(int npat, const int64_t *__restrict__ rep, const int *__restrict__ doff,
                                    const double *__restrict__ dval, const uint16_t *__restrict__ dvmeta,
                                    DiaPat *__restrict__ tab, int *__restrict__ plen) {
  const int p = blockIdx.x, t = threadIdx.x;
  if (p >= npat || t >= 8) return;
  if (t == 0) plen[p] = dvmeta[rep[p]] >> 8 & 15;
  tab[p].off[t] = doff[rep[p] * 8 + t];
  tab[p].val[t] = dval[rep[p] * 8 + t];
}
__global__ void dia_pat_assign_kernel(int64_t n_slices, int npat, const unsigned long long *__restrict__ key,
                                      const unsigned long long *__restrict__ pkey, const int64_t *__restrict__ rep,
                                      const int *__restrict__ doff, const double *__restrict__ dval,
                                      const uint16_t *__restrict__ dvmeta, uint8_t *__restrict__ dpat,
                                      unsigned long long *__restrict__ n_assigned) {
  unsigned long long cnt = 0;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n_slices; s += (int64_t)gridDim.x * blockDim.x) {
    uint8_t id = DIA_NOPAT;
    const unsigned long long k = key[s];
    if (k != ~0ull)
      for (int p = 0; p < npat; p++)
        if (pkey[p] == k) {
          const int64_t r = rep[p];
          bool eq = (dvmeta[s] >> 8) == (dvmeta[r] >> 8);
          for (int t = 0; t < 8 && eq; t++)
            eq = doff[s * 8 + t] == doff[r * 8 + t] &&
                 __double_as_longlong(dval[s * 8 + t]) == __double_as_longlong(dval[r * 8 + t]);
          if (eq) id = (uint8_t)p;
          break;
        }
    dpat[s] = id;
    cnt += id != DIA_NOPAT;
  }
  if (cnt) atomicAdd(n_assigned, cnt);
}

static pcg_status build_dia_patterns(pcg_matrix *A, cudaStream_t st) {
  const char *e = getenv("PCG_DIA_PAT");  // PCG_DIA_PAT=0: every value-free slice reads its own metadata
  if ((e && atoi(e) == 0) || A->dval_slices == 0) return PCG_OK;
  const int64_t ns = A->n_slices;
  unsigned long long *d_key = nullptr;
  PCG_CUDA(cudaMalloc(&d_key, sizeof(unsigned long long) * (size_t)ns));
  const unsigned g = (unsigned)std::min<int64_t>((ns + 255) / 256, 148 * 16);
  dia_key_kernel<<<g, 256, 0, st>>>(ns, A->d_sdoff, A->d_sdval, A->d_sdmask, A->d_sdvmeta, d_key);
  count_launch();
  std::vector<unsigned long long> key((size_t)ns);
  PCG_CUDA(cudaMemcpyAsync(key.data(), d_key, sizeof(unsigned long long) * (size_t)ns, cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  std::vector<unsigned long long> pkey;
  std::vector<int64_t> rep;
  unsigned long long last = ~0ull;
  for (int64_t s = 0; s < ns; s++) {  // first DIA_MAXPAT distinct keys, in slice order
    const unsigned long long k = key[(size_t)s];
    if (k == ~0ull || k == last) continue;
    last = k;
    if (std::find(pkey.begin(), pkey.end(), k) != pkey.end()) continue;
    if ((int)pkey.size() == DIA_MAXPAT) continue;
    pkey.push_back(k);
    rep.push_back(s);
  }
  const int np = (int)pkey.size();
  if (np == 0) {
    cudaFree(d_key);
    return PCG_OK;
  }
  unsigned long long *d_pkey = nullptr, *d_cnt = nullptr;
  int64_t *d_rep = nullptr;
  PCG_CUDA(cudaMalloc(&d_pkey, sizeof(unsigned long long) * np));
  PCG_CUDA(cudaMalloc(&d_rep, sizeof(int64_t) * np));
  PCG_CUDA(cudaMalloc(&d_cnt, sizeof(unsigned long long)));
  PCG_CUDA(cudaMalloc(&A->d_ptab, sizeof(DiaPat) * np));
  PCG_CUDA(cudaMalloc(&A->d_plen, sizeof(int) * np));
  PCG_CUDA(cudaMalloc(&A->d_sdpat, (size_t)ns));
  PCG_CUDA(cudaMemcpyAsync(d_pkey, pkey.data(), sizeof(unsigned long long) * np, cudaMemcpyHostToDevice, st));
  PCG_CUDA(cudaMemcpyAsync(d_rep, rep.data(), sizeof(int64_t) * np, cudaMemcpyHostToDevice, st));
  PCG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), st));
  dia_pat_fill_kernel<<<np, 32, 0, st>>>(np, d_rep, A->d_sdoff, A->d_sdval, A->d_sdvmeta,
                                      A->d_ptab, A->d_plen);
  count_launch();
  dia_pat_assign_kernel<<<g, 256, 0, st>>>(ns, np, d_key, d_pkey, d_rep, A->d_sdoff, A->d_sdval, A->d_sdvmeta,
                                           A->d_sdpat, d_cnt);
  count_launch();
  unsigned long long cnt = 0;
  PCG_CUDA(cudaMemcpyAsync(&cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_key);
  cudaFree(d_pkey);
  cudaFree(d_rep);
  cudaFree(d_cnt);
  A->npat = np;
  A->pat_slices = (int64_t)cnt;
  A->device_bytes += (double)ns + sizeof(DiaPat) * (double)np;
  return PCG_OK;
}

pcg_status build_dia(pcg_matrix *A, cudaStream_t st) {
  const char *e = getenv("PCG_DIA");  // PCG_DIA=0: ids at every position
  if (A->d_sdoff || !A->d_slice_ptr || A->n_slices == 0 || !A->short_rows || (e && atoi(e) == 0)) return PCG_OK;
  PCG_CUDA(cudaMalloc(&A->d_sdoff, sizeof(int) * 8 * (size_t)A->n_slices));
  PCG_CUDA(cudaMalloc(&A->d_sdmask, (size_t)A->n_slices));
  PCG_CUDA(cudaMemsetAsync(A->d_sdoff, 0, sizeof(int) * 8 * (size_t)A->n_slices, st));
  const char *ev = getenv("PCG_DIA_VAL");  // PCG_DIA_VAL=0: values read from the stream at every position
  const int vals = !(ev && atoi(ev) == 0);
  PCG_CUDA(cudaMalloc(&A->d_sdval, sizeof(double) * 8 * (size_t)A->n_slices));
  PCG_CUDA(cudaMalloc(&A->d_sdvmeta, sizeof(uint16_t) * (size_t)A->n_slices));
  PCG_CUDA(cudaMemsetAsync(A->d_sdval, 0, sizeof(double) * 8 * (size_t)A->n_slices, st));
  const char *ea = getenv("PCG_DIA_ALIGN");  // PCG_DIA_ALIGN=0: no aligned (zero-mask) slices
  if (vals && !(ea && atoi(ea) == 0)) {
    PCG_CUDA(cudaMalloc(&A->d_sdzmask, sizeof(unsigned) * 8 * (size_t)A->n_slices));
    PCG_CUDA(cudaMemsetAsync(A->d_sdzmask, 0, sizeof(unsigned) * 8 * (size_t)A->n_slices, st));
  }
  unsigned long long *d_n;
  PCG_CUDA(cudaMalloc(&d_n, 4 * sizeof(unsigned long long)));
  PCG_CUDA(cudaMemsetAsync(d_n, 0, 4 * sizeof(unsigned long long), st));
  dia_build_kernel<<<(unsigned)((A->n_slices * 32 + 255) / 256), 256, 0, st>>>(
      A->n, A->n + A->n_ghost, A->n_slices, A->d_row_ptr, A->d_slice_ptr, A->d_scol, A->d_sval, vals,
      A->d_sdoff, A->d_sdmask, A->d_sdval, A->d_sdvmeta, A->d_sdzmask, d_n);
  count_launch();
  unsigned long long np[4] = {0, 0, 0, 0};
  PCG_CUDA(cudaMemcpyAsync(np, d_n, sizeof(np), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_n);
  A->dia_positions = (int64_t)np[0];
  A->dia_slices = (int64_t)np[1];
  A->dval_slices = (int64_t)np[2] + (int64_t)np[3];
  A->aligned_slices = (int64_t)np[3];
  if (A->d_sdzmask) A->device_bytes += 32.0 * (double)A->n_slices;
  A->device_bytes += 33.0 * (double)A->n_slices;
  A->device_bytes += 66.0 * (double)A->n_slices;
  PCG_TRY(build_dia_patterns(A, st));
  return PCG_OK;
}

void free_sell(pcg_matrix *A) {
  if (A->d_sdoff) {
    cudaFree(A->d_sdoff);
    cudaFree(A->d_sdmask);
    A->device_bytes -= 33.0 * (double)A->n_slices;
    A->d_sdoff = nullptr;
    A->d_sdmask = nullptr;
    A->dia_positions = 0;
    A->dia_slices = 0;
  }
  if (A->d_sdval) {
    cudaFree(A->d_sdval);
    cudaFree(A->d_sdvmeta);
    A->device_bytes -= 66.0 * (double)A->n_slices;
    A->d_sdval = nullptr;
    A->d_sdvmeta = nullptr;
  }
  if (A->d_sdzmask) {
    cudaFree(A->d_sdzmask);
    A->device_bytes -= 32.0 * (double)A->n_slices;
    A->d_sdzmask = nullptr;
    A->aligned_slices = 0;
  }
  if (A->d_sdpat) {
    cudaFree(A->d_sdpat);
    cudaFree(A->d_ptab);
    cudaFree(A->d_plen);
    A->d_plen = nullptr;
    A->device_bytes -= (double)A->n_slices + sizeof(DiaPat) * (double)A->npat;
    A->d_sdpat = nullptr;
    A->d_ptab = nullptr;
    A->npat = 0;
    A->pat_slices = 0;
    A->dval_slices = 0;
  }
  if (A->d_wdesc) cudaFree(A->d_wdesc);
  if (A->d_wlidx) cudaFree(A->d_wlidx);
  A->d_wdesc = nullptr;
  A->d_wlidx = nullptr;
  A->wplan = 0;
  if (A->d_sdcol) {
    cudaFree(A->d_sdcol);
    cudaFree(A->d_scbase);
    A->device_bytes -= (double)A->sell_entries * 2 + (double)(A->sell_entries / 32) * 4;
    A->d_sdcol = nullptr;
    A->d_scbase = nullptr;
    A->d16_slices = 0;
  }
  for (void *p : {(void *)A->d_slice_ptr, (void *)A->d_scol, (void *)A->d_sval})
    if (p) cudaFree(p);
  if (A->d_slice_ptr) A->device_bytes -= (double)(A->n_slices + 1) * 8 + (double)A->sell_entries * 12;
  A->d_slice_ptr = nullptr;
  A->d_scol = nullptr;
  A->d_sval = nullptr;
  A->sell_entries = 0;
}

// PCG_DROP_ZEROS: off-diagonal entries whose value is exactly 0.0 are not stored.
// Row by row, order kept; the diagonal (local column i) always stays.
__global__ void dz_count_kernel(int64_t n, const int *__restrict__ rp, const int *__restrict__ col,
                                const double *__restrict__ val, int *__restrict__ cnt) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int k = rp[i]; k < rp[i + 1]; k++) c += (val[k] != 0.0 || col[k] == (int)i);
    cnt[i] = c;
  }
}
__global__ void dz_copy_kernel(int64_t n, const int *__restrict__ rp, const int *__restrict__ col,
                               const double *__restrict__ val, const int *__restrict__ rp2, int *__restrict__ col2,
                               double *__restrict__ val2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int o = rp2[i];
    for (int k = rp[i]; k < rp[i + 1]; k++)
      if (val[k] != 0.0 || col[k] == (int)i) {
        col2[o] = col[k];
        val2[o] = val[k];
        o++;
      }
  }
}

static pcg_status drop_zeros(pcg_matrix *A, cudaStream_t st) {
  const int64_t n = A->n;
  if (n == 0 || A->nnz == 0) return PCG_OK;
  int *cnt = nullptr, *rp2 = nullptr, *col2 = nullptr, *mx = nullptr;
  double *val2 = nullptr;
  PCG_CUDA(cudaMalloc(&cnt, sizeof(int) * (n + 1)));
  PCG_CUDA(cudaMalloc(&rp2, sizeof(int) * (n + 1)));
  PCG_CUDA(cudaMalloc(&mx, sizeof(int)));
  const unsigned g = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16);
  dz_count_kernel<<<g, 256, 0, st>>>(n, A->d_row_ptr, A->d_col, A->d_val, cnt);
  PCG_CUDA(cudaMemsetAsync(cnt + n, 0, sizeof(int), st));
  size_t tb = 0, tm = 0;
  PCG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, rp2, (int)(n + 1), st));
  PCG_CUDA(cub::DeviceReduce::Max(nullptr, tm, cnt, mx, (int)n, st));
  void *tmp = nullptr;
  PCG_CUDA(cudaMalloc(&tmp, std::max(tb, tm)));
  PCG_CUDA(cub::DeviceReduce::Max(tmp, tm, cnt, mx, (int)n, st));
  PCG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, rp2, (int)(n + 1), st));
  int nnz2 = 0, maxlen = 0;
  PCG_CUDA(cudaMemcpyAsync(&nnz2, rp2 + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaMemcpyAsync(&maxlen, mx, sizeof(int), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  PCG_CUDA(cudaMalloc(&col2, sizeof(int) * std::max(nnz2, 1)));
  PCG_CUDA(cudaMalloc(&val2, sizeof(double) * std::max(nnz2, 1)));
  dz_copy_kernel<<<g, 256, 0, st>>>(n, A->d_row_ptr, A->d_col, A->d_val, rp2, col2, val2);
  count_launch(2);
  PCG_CUDA(cudaGetLastError());
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(A->d_row_ptr);
  cudaFree(A->d_col);
  cudaFree(A->d_val);
  cudaFree(cnt);
  cudaFree(mx);
  cudaFree(tmp);
  A->d_row_ptr = rp2;
  A->d_col = col2;
  A->d_val = val2;
  A->nnz = nnz2;
  A->max_row_len = maxlen;
  return PCG_OK;
}

// Core of csr_create / csr_create_dist: columns already translated so that the
// local matrix is n x n_cols (n_cols = n + n_ghost) with diagonal at i + 0.
// d_col_check: columns as given by the caller (global ids on a distributed handle),
// validated against [0, n_cols_check) with the diagonal at i + diag_offset;
// d_col_store: the local ids the kernels gather with (same array on one GPU).
pcg_status create_local(pcg_matrix *A, int64_t n, int64_t nnz, const int64_t *d_rp, const int64_t *d_col_check,
                        const int64_t *d_col_store, const double *d_val, int64_t n_cols_check,
                        int64_t diag_offset, int flags, cudaStream_t st) {
  A->n = n;
  A->nnz = nnz;
  ErrInfo *d_err;
  PCG_CUDA(cudaMalloc(&d_err, sizeof(ErrInfo)));
  ErrInfo h_err;
  memset(&h_err, 0, sizeof(h_err));
  for (auto &r : h_err.first_row) r = ~0ull;
  PCG_CUDA(cudaMemcpyAsync(d_err, &h_err, sizeof(ErrInfo), cudaMemcpyHostToDevice, st));
  PCG_CUDA(cudaMalloc(&A->d_row_ptr, sizeof(int) * (n + 1)));
  PCG_CUDA(cudaMalloc(&A->d_col, sizeof(int) * (nnz > 0 ? nnz : 1)));
  PCG_CUDA(cudaMalloc(&A->d_val, sizeof(double) * (nnz > 0 ? nnz : 1)));
  PCG_CUDA(cudaMalloc(&A->d_dinv, sizeof(double) * (n > 0 ? n : 1)));
  validate_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(n, nnz, n_cols_check, diag_offset, d_rp, d_col_check,
                                                                     d_val, A->d_row_ptr, A->d_dinv, d_err);
  count_launch();
  PCG_CUDA(cudaGetLastError());
  PCG_CUDA(cudaMemcpyAsync(&h_err, d_err, sizeof(ErrInfo), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_err);
  PCG_TRY(error_from_flags(h_err, A->row_begin));
  A->max_row_len = h_err.max_len;
  if (nnz > 0) {
    narrow_kernel<<<1184, 256, 0, st>>>(nnz, d_col_store, d_val, A->d_col, A->d_val, 0);
    count_launch();
    PCG_CUDA(cudaGetLastError());
  }
  if (flags & PCG_DROP_ZEROS) PCG_TRY(drop_zeros(A, st));
  nnz = A->nnz;
  if ((flags & PCG_REORDER_RCM) && n > 0) {
    if (A->comm)
      return fail(PCG_ERR_INVALID_ARG,
                  "csr_create_dist: PCG_REORDER_RCM is one-GPU only; order the global matrix with csr_rcm_order "
                  "before partitioning");
    int *perm = nullptr;
    PCG_CUDA(cudaMalloc(&perm, sizeof(int) * n));
    pcg_status s = rcm_order(n, A->d_row_ptr, A->d_col, perm, st);
    if (s != PCG_OK) {
      cudaFree(perm);
      return s;
    }
    PCG_TRY(apply_perm(A, perm, st));
    A->reorder = 1;
  }
  // ---- SELL-32
  const int fmt_req = flags & 0xF0;
  A->n_slices = (n + 31) / 32;
  bool want_sell = fmt_req != PCG_FMT_CSR && n > 0;
  double pad_nat = 1.0;
  if (want_sell) {
    PCG_TRY(build_sell(A, st));
    pad_nat = nnz > 0 ? (double)A->sell_entries / (double)nnz : 1.0;
    if (fmt_req == PCG_FMT_AUTO && pad_nat > 1.25) {
      want_sell = false;  // padding too large: natural-order SELL would move >25% extra bytes
      free_sell(A);
    }
    if (fmt_req == PCG_FMT_SELL_SIGMA) want_sell = false;  // only the permuted SELL is a candidate
  }
  // SELL-C-sigma candidate (sigma.cu): one GPU, and only where natural slices pad
  const bool try_sigma = !A->comm && n > 0 &&
                         (fmt_req == PCG_FMT_SELL_SIGMA || (fmt_req == PCG_FMT_AUTO && pad_nat > 1.02));
  // ---- CSR lanes per row from the mean row length (power of two, <= 32)
  const double mean = n > 0 ? (double)nnz / (double)n : 1.0;
  int L = 1;
  while (L < 32 && L * 4 < mean) L <<= 1;
  A->csr_lanes = L;
  // ---- TMA-staged SELL: largest tile (WARPS slices) sets the shared-memory stage size
  A->stage_entries = 0;
  if (fmt_req == PCG_FMT_SELL_TMA && want_sell && A->n_slices > 0) {
    std::vector<int64_t> sp(A->n_slices + 1);
    PCG_CUDA(cudaMemcpy(sp.data(), A->d_slice_ptr, sizeof(int64_t) * sp.size(), cudaMemcpyDeviceToHost));
    int64_t mx = 0;
    for (int64_t t = 0; t * WARPS < A->n_slices; t++)
      mx = std::max(mx, sp[std::min<int64_t>((t + 1) * WARPS, A->n_slices)] - sp[t * WARPS]);
    const char *e = getenv("PCG_STAGES");
    A->stages = e ? std::max(1, std::min(4, atoi(e))) : 2;
    A->stage_entries = mx;
    const size_t smem = staged_smem_bytes(SellStage(A->stages, mx));
    if (smem > 200 * 1024 || mx == 0) {
      A->stage_entries = 0;
    } else {
      PCG_TRY(prepare_staged(smem));
      // prefix-max lead column per tile -> L2 prefetch windows
      const int64_t nt = (A->n_slices + WARPS - 1) / WARPS;
      PCG_CUDA(cudaMalloc(&A->d_lead, sizeof(int) * nt));
      tile_lead_kernel<<<(unsigned)nt, 256, 0, st>>>(A->n_slices, A->d_slice_ptr, A->d_scol, A->d_lead);
      count_launch();
      std::vector<int> ld(nt);
      PCG_CUDA(cudaMemcpyAsync(ld.data(), A->d_lead, sizeof(int) * nt, cudaMemcpyDeviceToHost, st));
      PCG_CUDA(cudaStreamSynchronize(st));
      for (int64_t t = 1; t < nt; t++) ld[t] = std::max(ld[t], ld[t - 1]);
      PCG_CUDA(cudaMemcpy(A->d_lead, ld.data(), sizeof(int) * nt, cudaMemcpyHostToDevice));
      if (getenv("PCG_NO_L2PF")) {  // tuning knob: disable the L2 prefetch windows
        cudaFree(A->d_lead);
        A->d_lead = nullptr;
      }
    }
  }
  // ---- launch geometry: persistent grids, a multiple of the SM count
  const int sms = num_sms(A->device);
  auto configure = [&](int fmt) {
    A->format = fmt;
    A->dyn_smem = fmt == FMT_SELL_TMA ? staged_smem_bytes(SellStage(A->stages, A->stage_entries)) : 0;
    int bps = k1_blocks_per_sm(fmt, A->csr_lanes, A->dyn_smem);
    int64_t g = (int64_t)sms * (bps > 0 ? bps : 1);
    int64_t need = fmt == FMT_SELL_TMA   ? (A->n_slices + WARPS - 1) / WARPS
                   : fmt == PCG_FORMAT_SELL ? (A->n_slices + WARPS - 1) / WARPS
                                            : (n * A->csr_lanes + BLOCK - 1) / BLOCK;
    if (need < 1) need = 1;
    A->grid_spmv = (int)(g < need ? g : need);
  };
  const int64_t need_vec = (n / 2 + BLOCK - 1) / BLOCK;
  A->grid_vec = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * 8, need_vec));
  std::vector<int> cands;
  if (fmt_req == PCG_FMT_CSR || (!want_sell && fmt_req != PCG_FMT_SELL_SIGMA)) cands = {PCG_FORMAT_CSR};
  else if (fmt_req == PCG_FMT_SELL) cands = {PCG_FORMAT_SELL};
  else if (fmt_req == PCG_FMT_SELL_SIGMA) cands = {};
  else if (fmt_req == PCG_FMT_SELL_TMA) {
    if (!A->stage_entries) return fail(PCG_ERR_INVALID_ARG, "csr_create: TMA-staged SELL unavailable for this matrix");
    cands = {FMT_SELL_TMA};
  } else if (pad_nat <= 1.02) {
    // near-uniform slices: natural SELL-32 moves the fewest bytes and was the fastest
    // format on every such matrix measured (C1, C4, C5); no timing (it is also what a
    // profiler's serialised replays would corrupt)
    cands = {PCG_FORMAT_SELL};
  } else {
    // the TMA-staged SELL (PCG_FMT_SELL_TMA) never won a measurement and is only
    // built/used on request
    cands = {PCG_FORMAT_CSR, PCG_FORMAT_SELL};
  }
  // ---- format choice.  Default: a deterministic rule on the padding of the slices
  // (pcg.h promises bitwise-identical results for identical inputs, and the formats
  // sum in different orders): natural SELL-32 if its slices pad <= 2 %; otherwise
  // SELL-C-sigma if sorting the sigma-windows cuts the padding by >= 1 % and leaves
  // <= 25 %, else natural SELL-32 if it pads <= 25 %, else CSR.  The measured choice
  // (time 5 SpMVs per candidate, round 1's rule) is kept behind PCG_FMT_TIMED=1.
  const bool fmt_timed = getenv("PCG_FMT_TIMED") != nullptr;
  if (!fmt_timed && fmt_req == PCG_FMT_AUTO && cands.size() > 1)
    cands = {want_sell ? PCG_FORMAT_SELL : PCG_FORMAT_CSR};
  const bool timed = n > 0 && (cands.size() > 1 || (try_sigma && fmt_req == PCG_FMT_AUTO && fmt_timed));
  float best = 1e30f;
  int best_fmt = cands.empty() ? PCG_FORMAT_SELL : cands[0];
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  auto time_fmt = [&](int fmt, float *ms) -> pcg_status {
    double *x = A->work.stage_x, *y = A->work.w;
    configure(fmt);
    PCG_TRY(launch_spmv_fmt(A, fmt, x, y, st));  // warm-up
    cudaEventRecord(e0, st);
    for (int r = 0; r < 5; r++) PCG_TRY(launch_spmv_fmt(A, fmt, x, y, st));
    cudaEventRecord(e1, st);
    PCG_CUDA(cudaEventSynchronize(e1));
    cudaEventElapsedTime(ms, e0, e1);
    return PCG_OK;
  };
  if (timed || try_sigma) {
    PCG_TRY(ensure_work(A));
    PCG_CUDA(cudaMemsetAsync(A->work.stage_x, 0, sizeof(double) * (n + A->n_ghost), st));
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
  }
  if (timed) {
    for (int fmt : cands) {
      float ms = 0;
      PCG_TRY(time_fmt(fmt, &ms));
      if (fmt == PCG_FORMAT_CSR) A->spmv_us_csr = ms * 1e3 / 5;
      else if (fmt == PCG_FORMAT_SELL) A->spmv_us_sell = ms * 1e3 / 5;
      else A->spmv_us_tma = ms * 1e3 / 5;
      if (ms < best) {
        best = ms;
        best_fmt = fmt;
      }
    }
  }
  if (try_sigma) {
    // build P A P^T, swap it in (the natural CSR/SELL move to S), build its SELL, time it
    SigmaSys S;
    PCG_TRY(sigma_build(A, st, &S));
    sigma_swap(A, &S);
    pcg_status bs = build_sell(A, st);
    if (bs != PCG_OK) {
      free_sell(A);
      sigma_swap(A, &S);
      sigma_free(&S);
      if (fmt_req == PCG_FMT_SELL_SIGMA) return bs;
    } else {
      float ms = 0;
      const double pad_sig = nnz > 0 ? (double)A->sell_entries / (double)nnz : 1.0;
      bool keep;
      if (fmt_timed) {
        PCG_TRY(time_fmt(PCG_FORMAT_SELL, &ms));
        A->spmv_us_sigma = ms * 1e3 / 5;
        keep = ms < best;
      } else {
        keep = pad_sig <= 1.25 && pad_sig <= pad_nat - 0.01;
      }
      if (fmt_req == PCG_FMT_SELL_SIGMA || keep) {  // keep the permuted system
        sigma_free(&S);
        if (A->d_lead) cudaFree(A->d_lead);
        A->d_lead = nullptr;
        A->stage_entries = 0;
        best_fmt = PCG_FORMAT_SELL;
      } else {  // back to the natural system
        free_sell(A);
        sigma_swap(A, &S);
        sigma_free(&S);
      }
    }
  }
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  configure(best_fmt);
  if (A->format == PCG_FORMAT_SELL) PCG_TRY(build_d16(A, st));
  {  // rows of at most 8 entries: the one-chunk SELL engine and its grid (PCG_SHORT=0: off)
    const char *se = getenv("PCG_SHORT");
    A->short_rows = A->format == PCG_FORMAT_SELL && !A->d_sdcol && A->max_row_len <= 8 && !(se && atoi(se) == 0);
    if (A->short_rows) {
      PCG_TRY(build_dia(A, st));
      const int64_t need = (A->n_slices + WARPS - 1) / WARPS;
      const int64_t g = (int64_t)sms * k1_blocks_per_sm(A->d_sdoff ? FMT_SELL_DIA : FMT_SELL_SHORT, 1, 0);
      A->grid_spmv = (int)std::max<int64_t>(1, std::min(g, need));
    }
  }
  {
    const char *sch = getenv("PCG_SCHEDULE");
    A->schedule = (sch && atoi(sch) == 2) ? 2 : 3;
  }
  if (A->work.graph_ready) free_work(A);  // geometry changed after a provisional workspace
  if (A->work.dslice) {  // dinv may have been permuted since (SELL-C-sigma, RCM)
    cudaFree(A->work.dslice);
    A->work.dslice = nullptr;
  }
  A->device_bytes += (double)(n + 1) * 4 + (double)nnz * 12 + (double)n * 8;
  return PCG_OK;
}

static pcg_status stage_in(const void *src, size_t bytes, bool dev, void **dst, bool *owned, cudaStream_t st) {
  if (dev) {
    *dst = const_cast<void *>(src);
    *owned = false;
    return PCG_OK;
  }
  PCG_CUDA(cudaMalloc(dst, bytes > 0 ? bytes : 8));
  *owned = true;
  if (bytes) PCG_CUDA(cudaMemcpyAsync(*dst, src, bytes, cudaMemcpyHostToDevice, st));
  return PCG_OK;
}

pcg_status csr_create_impl(int64_t n, int64_t nnz, const int64_t *row_ptr, const int64_t *col_idx,
                           const double *val, int flags, cudaStream_t st, pcg_matrix *A) {
  const bool dev = (flags & PCG_PTR_DEVICE) != 0;
  int64_t ends[2] = {0, 0};
  if (dev) {
    PCG_CUDA(cudaMemcpyAsync(&ends[0], row_ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaMemcpyAsync(&ends[1], row_ptr + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaStreamSynchronize(st));
  } else {
    ends[0] = row_ptr[0];
    ends[1] = row_ptr[n];
  }
  if (ends[0] != 0 || ends[1] != nnz)
    return fail(PCG_ERR_DIMENSION_MISMATCH, "csr_create: row_ptr[0] must be 0 and row_ptr[n] must equal nnz");
  void *drp, *dcol, *dval;
  bool o1, o2, o3;
  PCG_TRY(stage_in(row_ptr, sizeof(int64_t) * (n + 1), dev, &drp, &o1, st));
  PCG_TRY(stage_in(col_idx, sizeof(int64_t) * nnz, dev, &dcol, &o2, st));
  PCG_TRY(stage_in(val, sizeof(double) * nnz, dev, &dval, &o3, st));
  pcg_status s = create_local(A, n, nnz, (const int64_t *)drp, (const int64_t *)dcol, (const int64_t *)dcol,
                              (const double *)dval, n, 0, flags, st);
  cudaStreamSynchronize(st);
  if (o1) cudaFree(drp);
  if (o2) cudaFree(dcol);
  if (o3) cudaFree(dval);
  return s;
}

// ---------------------------------------------------------------- workspace
// SolveWork::dslice: per 32-row slice the common dinv, NaN when the slice's entries differ
// (the last slice: its existing rows)
__global__ void dinv_slice_kernel(int64_t n, const double *__restrict__ dinv, double *__restrict__ dslice,
                                  unsigned long long *__restrict__ n_shared) {
  const int64_t ns = (n + 31) / 32;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ns * 32; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = t >> 5;
    const int lane = (int)(t & 31);
    const unsigned long long b = t < n ? (unsigned long long)__double_as_longlong(dinv[t]) : ~0ull;
    const unsigned long long b0 = __shfl_sync(0xffffffffu, b, 0);
    const bool same = __all_sync(0xffffffffu, b == b0 || t >= n);  // (the last slice's missing rows)
    if (lane == 0) {
      dslice[s] = same ? __longlong_as_double((long long)b0) : __longlong_as_double(0x7ff8000000000000ll);
      if (same) atomicAdd(n_shared, 1ull);
    }
  }
}

pcg_status ensure_work(pcg_matrix *A) {
  SolveWork &w = A->work;
  if (!w.dslice) {  // (dropped when the format choice swaps dinv: rebuilt from the final one)
    const char *ed = getenv("PCG_DINV_SLICE");  // PCG_DINV_SLICE=0: K2 reads dinv per row
    if (A->n > 0 && !(ed && atoi(ed) == 0)) {
      const int64_t ns = (A->n + 31) / 32;
      unsigned long long *d_cnt = nullptr, cnt = 0;
      PCG_CUDA(cudaMalloc(&w.dslice, sizeof(double) * (size_t)ns));
      PCG_CUDA(cudaMalloc(&d_cnt, sizeof(unsigned long long)));
      PCG_CUDA(cudaMemset(d_cnt, 0, sizeof(unsigned long long)));
      dinv_slice_kernel<<<(unsigned)std::min<int64_t>((ns * 32 + 255) / 256, 148 * 64), 256>>>(A->n, A->d_dinv,
                                                                                          w.dslice, d_cnt);
      count_launch();
      PCG_CUDA(cudaGetLastError());
      PCG_CUDA(cudaMemcpy(&cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost));  // (synchronises)
      cudaFree(d_cnt);
      w.dslice_all = (int64_t)cnt == ns;
      if (2 * (int64_t)cnt < ns) {  // mostly per-row diagonals (a jittered mesh): not worth a branch
        cudaFree(w.dslice);
        w.dslice = nullptr;
      }
    }
  }
  if (w.sc) return PCG_OK;
  // +64 entries of padding: TMA tile copies round row counts up to 16-B multiples
  const size_t n = (size_t)A->n, ng = (size_t)(A->n + A->n_ghost);
  const size_t nb = sizeof(double) * (n + 64), ngb = sizeof(double) * (ng + 64);
  PCG_CUDA(cudaMalloc(&w.r, nb));
  PCG_CUDA(cudaMalloc(&w.z, ngb));
  PCG_CUDA(cudaMalloc(&w.q, nb));
  PCG_CUDA(cudaMalloc(&w.p[0], ngb));
  PCG_CUDA(cudaMalloc(&w.p[1], ngb));
  PCG_CUDA(cudaMalloc(&w.x, ngb));
  PCG_CUDA(cudaMalloc(&w.w, nb));
  PCG_CUDA(cudaMalloc(&w.stage_b, nb));
  PCG_CUDA(cudaMalloc(&w.stage_x, ngb));
  const int sms = num_sms(A->device);
  const size_t maxg = (size_t)sms * 32;
  PCG_CUDA(cudaMalloc(&w.partials, sizeof(double) * 6 * maxg));
  PCG_CUDA(cudaMalloc(&w.sc, sizeof(Scalars)));
  PCG_CUDA(cudaMemset(w.sc, 0, sizeof(Scalars)));
  PCG_CUDA(cudaMallocHost(&w.h_sc, sizeof(Scalars)));
  // zero-init vectors so ghosts / pads never hold NaN garbage
  PCG_CUDA(cudaMemset(w.z, 0, ngb));
  PCG_CUDA(cudaMemset(w.p[0], 0, ngb));
  PCG_CUDA(cudaMemset(w.p[1], 0, ngb));
  PCG_CUDA(cudaMemset(w.x, 0, ngb));
  PCG_CUDA(cudaMemset(w.stage_x, 0, ngb));
  A->device_bytes += 9.0 * ngb;
  return PCG_OK;
}

void free_work(pcg_matrix *A) {
  SolveWork &w = A->work;
  if (w.loop_exec) cudaGraphExecDestroy(w.loop_exec);
  if (w.loop_graph) cudaGraphDestroy(w.loop_graph);
  if (w.mloop_exec) cudaGraphExecDestroy(w.mloop_exec);
  if (w.mloop_graph) cudaGraphDestroy(w.mloop_graph);
  if (w.bg_exec) cudaGraphExecDestroy(w.bg_exec);
  if (w.bg_graph) cudaGraphDestroy(w.bg_graph);
  if (w.ilu) ilu_free(w.ilu);
  for (double *p : {w.r, w.z, w.q, w.p[0], w.p[1], w.p23[0], w.p23[1], w.x, w.w, w.stage_b, w.stage_x, w.partials,
                    w.dslice, w.mr, w.mz, w.mq, w.mp[0], w.mp[1], w.mp23[0], w.mp23[1], w.mx, w.mb, w.mw, w.mpart})
    if (p) cudaFree(p);
  if (w.sc) cudaFree(w.sc);
  if (w.h_sc) cudaFreeHost(w.h_sc);
  if (w.msc) cudaFree(w.msc);
  if (w.pbar) cudaFree(w.pbar);
  for (void *q : {(void *)w.bv, w.bstate, w.bbar, (void *)w.bminv, w.bgsc, (void *)w.pv, w.pstate, w.ppbar, w.pdsc})
    if (q) cudaFree(q);
  if (w.h_msc) cudaFreeHost(w.h_msc);
  for (void *q : {(void *)w.bcg, (void *)w.bcg_part, w.bcg_st, w.bspmm_sc, (void *)w.bspmm_part})
    if (q) cudaFree(q);
  if (w.bcg_hst) cudaFreeHost(w.bcg_hst);
  w = SolveWork();
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status csr_create(int64_t n, int64_t nnz, const int64_t *row_ptr, const int64_t *col_idx,
                                 const double *val, int flags, void *stream, pcg_matrix_t *out) {
  pcgb::NvtxRange nvtx_("pcg:csr_create");
  if (!out) return fail(PCG_ERR_INVALID_ARG, "csr_create: out is null");
  *out = nullptr;
  if (n < 0 || nnz < 0) return fail(PCG_ERR_INVALID_ARG, "csr_create: n and nnz must be >= 0");
  if (!row_ptr || (nnz > 0 && (!col_idx || !val)))
    return fail(PCG_ERR_INVALID_ARG, "csr_create: null array");
  if (nnz >= (int64_t(1) << 31)) return fail(PCG_ERR_INVALID_ARG, "csr_create: nnz per GPU must be < 2^31");
  auto t0 = std::chrono::steady_clock::now();
  pcg_matrix *A = new pcg_matrix();
  cudaGetDevice(&A->device);
  A->row_end = n;
  A->n_global = n;
  pcg_status s = csr_create_impl(n, nnz, row_ptr, col_idx, val, flags, (cudaStream_t)stream, A);
  if (s != PCG_OK) {
    csr_destroy(A);
    return s;
  }
  A->t_setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = A;
  return PCG_OK;
}

extern "C" pcg_status csr_destroy(pcg_matrix_t A) {
  if (!A) return PCG_OK;
  cudaSetDevice(A->device);
  cudaDeviceSynchronize();
  free_work(A);
  if (A->ov_side) cudaStreamDestroy(A->ov_side);
  if (A->ov_fork) cudaEventDestroy(A->ov_fork);
  if (A->ov_join) cudaEventDestroy(A->ov_join);
  for (void *p : {(void *)A->d_row_ptr, (void *)A->d_col, (void *)A->d_val, (void *)A->d_dinv,
                  (void *)A->d_slice_ptr, (void *)A->d_scol, (void *)A->d_sval, (void *)A->d_lead, (void *)A->halo.d_send_idx,
                  (void *)A->d_perm, (void *)A->d_iperm, (void *)A->d_sdcol, (void *)A->d_scbase, A->d_wdesc,
                  (void *)A->d_wlidx, (void *)A->halo.d_send_buf})
    if (p) cudaFree(p);
  delete A;
  return PCG_OK;
}

extern "C" pcg_status pcg_matrix_get_stats(pcg_matrix_t A, pcg_matrix_stats *o) {
  if (!A || !o) return fail(PCG_ERR_INVALID_ARG, "pcg_matrix_get_stats: null argument");
  memset(o, 0, sizeof(*o));
  o->n = A->n;
  o->nnz = A->nnz;
  o->format = A->sigma ? PCG_FORMAT_SELL_SIGMA : A->format;
  o->max_row_len = A->max_row_len;
  o->sell_entries = A->sell_entries;
  o->t_setup_s = A->t_setup_s;
  o->device_bytes = A->device_bytes;
  o->spmv_us_csr = A->spmv_us_csr;
  o->spmv_us_sell = A->spmv_us_sell;
  o->spmv_us_tma = A->spmv_us_tma;
  o->stage_entries = A->stage_entries;
  o->stages = A->stages;
  o->schedule = A->schedule;
  o->n_ghost = A->n_ghost;
  o->row_begin = A->row_begin;
  o->row_end = A->row_end;
  o->n_global = A->n_global;
  o->spmv_us_sigma = A->spmv_us_sigma;
  o->sigma = A->sigma;
  o->reorder = A->reorder;
  o->overlap_rows = A->ov ? A->ov_ib - A->ov_ia : 0;
  o->d16_slices = A->d16_slices;
  o->spmm_windowed = A->wplan;
  o->short_rows = A->short_rows ? 1 : 0;
  o->dia_positions = A->dia_positions;
  o->dia_slices = (int32_t)std::min<int64_t>(A->dia_slices, INT32_MAX);
  o->dval_slices = A->dval_slices;
  o->npat = A->npat;
  o->aligned_slices = A->aligned_slices;
  o->pat_slices = A->pat_slices;
  return PCG_OK;
}
