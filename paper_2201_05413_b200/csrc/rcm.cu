// rcm.cu — reverse Cuthill-McKee ordering on the device ("RCM or
// graph-partitioned multi-GPU" for irregular meshes whose numbering is arbitrary).
//
// Definition (oracle.h orc_rcm, the sequential algorithm): component start = the
// unnumbered node of least (degree, id); George-Liu pseudo-peripheral search; from
// the start r a FIFO queue in which every dequeued node appends its unnumbered
// neighbours in increasing (degree, id); components in that order; reversed.
//
// Level-synchronous form used here (same order, exactly): the Cuthill-McKee queue
// visits the BFS levels of r one after another, and a node v of level L+1 is
// appended by its neighbour of least queue position in level L (any earlier
// neighbour would have put v in level <= L).  So level L+1, in queue order, is its
// node set sorted by (least parent position, degree, id).  Per level: one expansion
// kernel (atomicMin of the parent position; the first toucher appends v), a sort
// of the new nodes by id (their append order is not deterministic), then a stable
// radix sort by (parent position << 32 | degree), then placement.  Degree-0 nodes
// are the first components in id order (each is least (degree, id) while any
// remain) and are placed in one pass.
//
// One host synchronisation per BFS level (the size of the next level); setup only.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>

#include "matrix.cuh"

namespace pcgb {

static unsigned rgrid(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

__global__ void rcm_deg_kernel(int64_t n, const int *__restrict__ rp, const int *__restrict__ col, int *__restrict__ deg,
                               int *__restrict__ iso) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int d = 0;
    for (int k = rp[i]; k < rp[i + 1]; k++) d += col[k] != (int)i;
    deg[i] = d;
    iso[i] = d == 0;
  }
}

// least (degree, id) over the nodes not yet placed
__global__ void rcm_min_unplaced_kernel(int64_t n, const int *__restrict__ deg, const int *__restrict__ mark,
                                        unsigned long long *__restrict__ best) {
  unsigned long long m = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!mark[i]) m = min(m, ((unsigned long long)(unsigned)deg[i] << 32) | (unsigned)i);
  for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(best, m);
}

// BFS level expansion (peripheral search): lvl[v] = L+1 for every unreached neighbour
__global__ void bfs_expand_kernel(const int *__restrict__ front, int fsize, const int *__restrict__ rp,
                                  const int *__restrict__ col, int *__restrict__ lvl, int L, int *__restrict__ next,
                                  int *__restrict__ cnt) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < fsize; t += gridDim.x * blockDim.x) {
    const int u = front[t];
    for (int k = rp[u]; k < rp[u + 1]; k++) {
      const int v = col[k];
      if (v != u && lvl[v] < 0 && atomicCAS(&lvl[v], -1, L + 1) == -1) next[atomicAdd(cnt, 1)] = v;
    }
  }
}

__global__ void level_min_kernel(const int *__restrict__ front, int fsize, const int *__restrict__ deg,
                                 unsigned long long *__restrict__ best) {
  unsigned long long m = ~0ull;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < fsize; t += gridDim.x * blockDim.x) {
    const int v = front[t];
    m = min(m, ((unsigned long long)(unsigned)deg[v] << 32) | (unsigned)v);
  }
  for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m != ~0ull) atomicMin(best, m);
}

// Cuthill-McKee level expansion: queue positions [ls, le) are the current level
__global__ void cm_expand_kernel(const int *__restrict__ order, int ls, int le, const int *__restrict__ rp,
                                 const int *__restrict__ col, const int *__restrict__ mark, int *__restrict__ parent,
                                 int *__restrict__ next, int *__restrict__ cnt) {
  for (int k = ls + blockIdx.x * blockDim.x + threadIdx.x; k < le; k += gridDim.x * blockDim.x) {
    const int u = order[k];
    for (int e = rp[u]; e < rp[u + 1]; e++) {
      const int v = col[e];
      if (v != u && !mark[v] && atomicMin(&parent[v], k) == INT_MAX) next[atomicAdd(cnt, 1)] = v;
    }
  }
}

__global__ void cm_keys_kernel(const int *__restrict__ ids, int m, const int *__restrict__ parent,
                               const int *__restrict__ deg, unsigned long long *__restrict__ key) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
    const int v = ids[t];
    key[t] = ((unsigned long long)(unsigned)parent[v] << 32) | (unsigned)deg[v];
  }
}

__global__ void cm_place_kernel(const int *__restrict__ ids, int m, int base, int *__restrict__ order,
                                int *__restrict__ mark) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < m; t += gridDim.x * blockDim.x) {
    order[base + t] = ids[t];
    mark[ids[t]] = 1;
  }
}

__global__ void rcm_reverse_kernel(int64_t n, const int *__restrict__ order, int *__restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    perm[i] = order[n - 1 - i];
}

namespace {
struct Rcm {
  int64_t n = 0;
  const int *rp = nullptr, *col = nullptr;
  cudaStream_t st = nullptr;
  int *deg = nullptr, *iso = nullptr, *lvl = nullptr, *mark = nullptr, *parent = nullptr, *order = nullptr;
  int *fa = nullptr, *fb = nullptr, *ids2 = nullptr, *cnt = nullptr, *nsel = nullptr;
  unsigned long long *key = nullptr, *key2 = nullptr, *best = nullptr;
  int *h = nullptr;  // pinned: [0] count, [1..2] best
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  int bits = 1;

  ~Rcm() {
    for (void *p : {(void *)deg, (void *)iso, (void *)lvl, (void *)mark, (void *)parent, (void *)order, (void *)fa,
                    (void *)fb, (void *)ids2, (void *)cnt, (void *)nsel, (void *)key, (void *)key2, (void *)best, tmp})
      if (p) cudaFree(p);
    if (h) cudaFreeHost(h);
  }

  pcg_status read_cnt(int *out) {
    PCG_CUDA(cudaMemcpyAsync(h, cnt, sizeof(int), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaStreamSynchronize(st));
    *out = h[0];
    return PCG_OK;
  }
  pcg_status read_best(unsigned long long *out) {
    PCG_CUDA(cudaMemcpyAsync(h + 1, best, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaStreamSynchronize(st));
    memcpy(out, h + 1, sizeof(*out));
    return PCG_OK;
  }

  // BFS from s; *ecc = last level; *last = least (degree, id) node of the last level
  pcg_status bfs(int s, int *ecc, int *last) {
    PCG_CUDA(cudaMemsetAsync(lvl, 0xff, sizeof(int) * n, st));
    PCG_CUDA(cudaMemcpyAsync(fa, &s, sizeof(int), cudaMemcpyHostToDevice, st));
    const int zero = 0;
    PCG_CUDA(cudaMemcpyAsync(lvl + s, &zero, sizeof(int), cudaMemcpyHostToDevice, st));
    int fsize = 1, L = 0;
    int *front = fa, *next = fb;
    for (;;) {
      PCG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), st));
      bfs_expand_kernel<<<rgrid(fsize), 256, 0, st>>>(front, fsize, rp, col, lvl, L, next, cnt);
      count_launch();
      int m = 0;
      PCG_TRY(read_cnt(&m));
      if (m == 0) break;
      std::swap(front, next);
      fsize = m;
      L++;
    }
    PCG_CUDA(cudaMemsetAsync(best, 0xff, sizeof(unsigned long long), st));
    level_min_kernel<<<rgrid(fsize), 256, 0, st>>>(front, fsize, deg, best);
    count_launch();
    unsigned long long b = 0;
    PCG_TRY(read_best(&b));
    *ecc = L;
    *last = (int)(b & 0xffffffffu);
    return PCG_OK;
  }

  pcg_status run(int *perm) {
    if (n == 0) return PCG_OK;
    while ((1ll << bits) < n) bits++;
    const size_t ni = sizeof(int) * (size_t)n;
    PCG_CUDA(cudaMalloc(&deg, ni));
    PCG_CUDA(cudaMalloc(&iso, ni));
    PCG_CUDA(cudaMalloc(&lvl, ni));
    PCG_CUDA(cudaMalloc(&mark, ni));
    PCG_CUDA(cudaMalloc(&parent, ni));
    PCG_CUDA(cudaMalloc(&order, ni));
    PCG_CUDA(cudaMalloc(&fa, ni));
    PCG_CUDA(cudaMalloc(&fb, ni));
    PCG_CUDA(cudaMalloc(&ids2, ni));
    PCG_CUDA(cudaMalloc(&key, sizeof(unsigned long long) * n));
    PCG_CUDA(cudaMalloc(&key2, sizeof(unsigned long long) * n));
    PCG_CUDA(cudaMalloc(&cnt, sizeof(int)));
    PCG_CUDA(cudaMalloc(&nsel, sizeof(int)));
    PCG_CUDA(cudaMalloc(&best, sizeof(unsigned long long)));
    PCG_CUDA(cudaMallocHost(&h, 4 * sizeof(int)));
    size_t t1 = 0, t2 = 0, t3 = 0;
    PCG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t1, fa, fb, (int)n, 0, bits, st));
    PCG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t2, key, key2, fa, fb, (int)n, 0, 64, st));
    PCG_CUDA(cub::DeviceSelect::Flagged(nullptr, t3, cub::CountingInputIterator<int>(0), iso, order, nsel, (int)n, st));
    tmp_bytes = std::max(t1, std::max(t2, t3));
    PCG_CUDA(cudaMalloc(&tmp, tmp_bytes));

    rcm_deg_kernel<<<rgrid(n), 256, 0, st>>>(n, rp, col, deg, iso);
    count_launch();
    PCG_CUDA(cudaMemsetAsync(mark, 0, ni, st));
    fill_int(parent, INT_MAX);
    // degree-0 nodes: the first components, in id order
    PCG_CUDA(cub::DeviceSelect::Flagged(tmp, tmp_bytes, cub::CountingInputIterator<int>(0), iso, order, nsel, (int)n, st));
    PCG_CUDA(cudaMemcpyAsync(h, nsel, sizeof(int), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaStreamSynchronize(st));
    int pos = h[0];
    if (pos > 0) {
      cm_place_kernel<<<rgrid(pos), 256, 0, st>>>(order, pos, 0, order, mark);
      count_launch();
    }
    while (pos < n) {
      PCG_CUDA(cudaMemsetAsync(best, 0xff, sizeof(unsigned long long), st));
      rcm_min_unplaced_kernel<<<rgrid(n), 256, 0, st>>>(n, deg, mark, best);
      count_launch();
      unsigned long long b = 0;
      PCG_TRY(read_best(&b));
      int r = (int)(b & 0xffffffffu), ecc_r = 0, x = 0;
      PCG_TRY(bfs(r, &ecc_r, &x));
      for (;;) {  // George-Liu
        int ecc_x = 0, x2 = 0;
        PCG_TRY(bfs(x, &ecc_x, &x2));
        if (ecc_x > ecc_r) {
          r = x;
          ecc_r = ecc_x;
          x = x2;
        } else {
          break;
        }
      }
      // Cuthill-McKee from r, level by level
      PCG_CUDA(cudaMemcpyAsync(order + pos, &r, sizeof(int), cudaMemcpyHostToDevice, st));
      const int one = 1;
      PCG_CUDA(cudaMemcpyAsync(mark + r, &one, sizeof(int), cudaMemcpyHostToDevice, st));
      int ls = pos, le = pos + 1;
      for (;;) {
        PCG_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), st));
        cm_expand_kernel<<<rgrid(le - ls), 256, 0, st>>>(order, ls, le, rp, col, mark, parent, fa, cnt);
        count_launch();
        int m = 0;
        PCG_TRY(read_cnt(&m));
        if (m == 0) break;
        PCG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, fa, fb, m, 0, bits, st));
        cm_keys_kernel<<<rgrid(m), 256, 0, st>>>(fb, m, parent, deg, key);
        PCG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key2, fb, ids2, m, 0, 64, st));
        cm_place_kernel<<<rgrid(m), 256, 0, st>>>(ids2, m, le, order, mark);
        count_launch(4);
        ls = le;
        le += m;
      }
      pos = le;
    }
    rcm_reverse_kernel<<<rgrid(n), 256, 0, st>>>(n, order, perm);
    count_launch();
    PCG_CUDA(cudaGetLastError());
    PCG_CUDA(cudaStreamSynchronize(st));
    return PCG_OK;
  }

  void fill_int(int *p, int v);
};

__global__ void fill_int_kernel(int64_t n, int *__restrict__ p, int v) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
void Rcm::fill_int(int *p, int v) {
  fill_int_kernel<<<rgrid(n), 256, 0, st>>>(n, p, v);
  count_launch();
}
}  // namespace

// perm[k] = original index of the node placed k-th (device, n ints); rp/col: the
// device int32 CSR of a symmetric pattern (diagonal entries ignored)
pcg_status rcm_order(int64_t n, const int *rp, const int *col, int *perm, cudaStream_t st) {
  if (n >= INT_MAX) return fail(PCG_ERR_INVALID_ARG, "rcm: n must be < 2^31");
  Rcm R;
  R.n = n;
  R.rp = rp;
  R.col = col;
  R.st = st;
  return R.run(perm);
}

}  // namespace pcgb

namespace pcgb {
// int64 CSR pattern -> int32 device copy, with the structural checks of csr_rcm_order
__global__ void rcm_narrow_kernel(int64_t n, int64_t nnz, const int64_t *__restrict__ rp, const int64_t *__restrict__ col,
                                  int *__restrict__ rp32, int *__restrict__ col32, int *__restrict__ err) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    rp32[i] = (int)rp[i];
    if (i < n && rp[i + 1] < rp[i]) atomicOr(err, 1);
  }
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = col[k];
    if (c < 0 || c >= n) atomicOr(err, 2);
    col32[k] = (int)c;
  }
}
__global__ void widen_kernel(int64_t n, const int *__restrict__ a, int64_t *__restrict__ b) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status csr_rcm_order(int64_t n, int64_t nnz, const int64_t *row_ptr, const int64_t *col_idx, int flags,
                                    void *stream, int64_t *perm) {
  if (n < 0 || nnz < 0) return fail(PCG_ERR_INVALID_ARG, "csr_rcm_order: n and nnz must be >= 0");
  if (!row_ptr || (n > 0 && !perm) || (nnz > 0 && !col_idx)) return fail(PCG_ERR_INVALID_ARG, "csr_rcm_order: null array");
  if (n >= INT_MAX || nnz >= INT_MAX) return fail(PCG_ERR_INVALID_ARG, "csr_rcm_order: n and nnz must be < 2^31");
  if (n == 0) return PCG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool dev = (flags & PCG_PTR_DEVICE) != 0;
  int64_t ends[2];
  PCG_CUDA(cudaMemcpyAsync(&ends[0], row_ptr, sizeof(int64_t), cudaMemcpyDefault, st));
  PCG_CUDA(cudaMemcpyAsync(&ends[1], row_ptr + n, sizeof(int64_t), cudaMemcpyDefault, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  if (ends[0] != 0 || ends[1] != nnz)
    return fail(PCG_ERR_DIMENSION_MISMATCH, "csr_rcm_order: row_ptr[0] must be 0 and row_ptr[n] must equal nnz");
  int64_t *d64 = nullptr;  // staged host inputs / the int64 result
  int *rp32 = nullptr, *col32 = nullptr, *p32 = nullptr, *err = nullptr;
  pcg_status s = PCG_OK;
  auto run = [&]() -> pcg_status {
    const int64_t *drp = row_ptr, *dcol = col_idx;
    PCG_CUDA(cudaMalloc(&d64, sizeof(int64_t) * (dev ? n : (n + 1 + nnz + n))));
    if (!dev) {
      PCG_CUDA(cudaMemcpyAsync(d64, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
      if (nnz) PCG_CUDA(cudaMemcpyAsync(d64 + n + 1, col_idx, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
      drp = d64;
      dcol = d64 + n + 1;
    }
    PCG_CUDA(cudaMalloc(&rp32, sizeof(int) * (n + 1)));
    PCG_CUDA(cudaMalloc(&col32, sizeof(int) * std::max<int64_t>(nnz, 1)));
    PCG_CUDA(cudaMalloc(&p32, sizeof(int) * n));
    PCG_CUDA(cudaMalloc(&err, sizeof(int)));
    PCG_CUDA(cudaMemsetAsync(err, 0, sizeof(int), st));
    rcm_narrow_kernel<<<rgrid(std::max(n + 1, nnz)), 256, 0, st>>>(n, nnz, drp, dcol, rp32, col32, err);
    count_launch();
    int herr = 0;
    PCG_CUDA(cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaStreamSynchronize(st));
    if (herr & 1) return fail(PCG_ERR_DIMENSION_MISMATCH, "csr_rcm_order: row_ptr must be nondecreasing");
    if (herr & 2) return fail(PCG_ERR_INDEX_OUT_OF_RANGE, "csr_rcm_order: column index out of range");
    PCG_TRY(rcm_order(n, rp32, col32, p32, st));
    int64_t *out64 = dev ? perm : d64 + (n + 1 + nnz);
    widen_kernel<<<rgrid(n), 256, 0, st>>>(n, p32, out64);
    count_launch();
    if (!dev) PCG_CUDA(cudaMemcpyAsync(perm, out64, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
    PCG_CUDA(cudaGetLastError());
    PCG_CUDA(cudaStreamSynchronize(st));
    return PCG_OK;
  };
  s = run();
  for (void *p : {(void *)d64, (void *)rp32, (void *)col32, (void *)p32, (void *)err})
    if (p) cudaFree(p);
  return s;
}
