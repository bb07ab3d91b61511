// dist.cu — multi-GPU row partition, halo plan and NCCL exchange.
//
// One process per GPU.  Rank g owns the contiguous rows [r_g, r_{g+1}) given by
// the nnz-balanced rule of SURVEY §8(c).10.  Per PCG iteration the only data
// exchange is the halo of z (the ghost copies of p advance locally by the same
// recurrence, see solver.cu) plus two scalar allreduces (sigma; rho', gamma) —
// the analogue of the paper's MatMult halo scatter and VecDot reductions
// (P:194).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "matrix.cuh"

#define PCG_NCCL(call)                                                                         \
  do {                                                                                         \
    ncclResult_t r_ = (call);                                                                  \
    if (r_ != ncclSuccess)                                                                     \
      return ::pcgb::fail(PCG_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_)); \
  } while (0)

namespace pcgb {

pcg_status create_local(pcg_matrix *A, int64_t n, int64_t nnz, const int64_t *d_rp, const int64_t *d_col_check,
                        const int64_t *d_col_store, const double *d_val, int64_t n_cols_check,
                        int64_t diag_offset, int flags, cudaStream_t st);

__global__ void mark_remote_kernel(int64_t nnz, const int64_t *__restrict__ col, int64_t r0, int64_t r1,
                                   int64_t n_global, uint8_t *__restrict__ flag) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = col[k];
    if (j < 0 || j >= n_global) continue;  // reported by validation
    if (j < r0 || j >= r1) flag[j] = 1;
  }
}

// global column -> local id: owned j -> j - r0 ; ghost j -> n + index in sorted ghost list
__global__ void map_cols_kernel(int64_t nnz, const int64_t *__restrict__ col, int64_t r0, int64_t r1, int64_t n,
                                const int64_t *__restrict__ ghost, int64_t n_ghost, int64_t *__restrict__ out) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = col[k];
    if (j >= r0 && j < r1) {
      out[k] = j - r0;
    } else {
      int64_t lo = 0, hi = n_ghost;
      while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (ghost[mid] < j) lo = mid + 1;
        else hi = mid;
      }
      out[k] = n + lo;
    }
  }
}

__global__ void pack_kernel(int64_t m, const int *__restrict__ idx, const double *__restrict__ v,
                            double *__restrict__ buf) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x)
    buf[s] = v[idx[s]];
}

__global__ void to_local_rows_kernel(int64_t m, const int64_t *__restrict__ g, int64_t r0, int *__restrict__ out) {
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < m; s += (int64_t)gridDim.x * blockDim.x)
    out[s] = (int)(g[s] - r0);
}

// ---------------------------------------------------------------- failure detection
// A collective whose peer died, hung or failed never completes, and a plain
// cudaStreamSynchronize would block every surviving rank forever.  Every host wait of
// the distributed paths therefore polls an event on the stream and, between polls,
// ncclCommGetAsyncError; an asynchronous NCCL error or `timeout_s` without completion
// aborts the communicator (ncclCommAbort unblocks the NCCL kernels queued on this
// rank) and returns PCG_ERR_NCCL.  Every rank runs the same rule, so when one rank
// fails the others fail too, within their timeout, instead of hanging.  The handle's
// communicator is unusable afterwards (aborted: every later call returns PCG_ERR_NCCL).
static pcg_status abort_comm(pcg_comm *C, const std::string &why) {
  if (C->nccl) ncclCommAbort(C->nccl);
  C->nccl = nullptr;
  C->aborted = true;
  return fail(PCG_ERR_NCCL, "NCCL communicator aborted: " + why);
}

pcg_status comm_wait(pcg_comm *C, cudaStream_t st) {
  if (C && C->aborted) return fail(PCG_ERR_NCCL, "NCCL communicator was aborted");
  if (!C || C->use_ops || !C->nccl) {
    PCG_CUDA(cudaStreamSynchronize(st));
    return PCG_OK;
  }
  NvtxRange r_("pcg:comm_wait");
  if (!C->wait_ev) PCG_CUDA(cudaEventCreateWithFlags(&C->wait_ev, cudaEventDisableTiming));
  PCG_CUDA(cudaEventRecord(C->wait_ev, st));
  const auto t0 = std::chrono::steady_clock::now();
  for (int poll = 0;; poll++) {
    const cudaError_t q = cudaEventQuery(C->wait_ev);
    if (C->dar && dar_failed(C->dar))  // a device allreduce saw no peer progress for ~8 s
      return abort_comm(C, "device allreduce: a peer stopped making progress");
    if (q == cudaSuccess) return PCG_OK;
    if (q != cudaErrorNotReady) {
      cudaGetLastError();
      return fail(PCG_ERR_CUDA, std::string("comm_wait: ") + cudaGetErrorString(q));
    }
    ncclResult_t ae = ncclSuccess;
    if (ncclCommGetAsyncError(C->nccl, &ae) != ncclSuccess || (ae != ncclSuccess && ae != ncclInProgress))
      return abort_comm(C, std::string("asynchronous error: ") + ncclGetErrorString(ae));
    const double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (dt > C->timeout_s)
      return abort_comm(C, "no progress for " + std::to_string(dt) + " s (PCG_COMM_TIMEOUT_S)");
    if (poll > 64) std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
}

// ---------------------------------------------------------------- communicator backends
// NCCL (the product path, stream-ordered and graph-capturable) or caller-supplied
// host callbacks (pcg_comm_init_ops: device data staged through host memory).
bool comm_uses_graphs(const pcg_comm *c) { return c && !c->use_ops; }

#define PCG_OPS(call, what)                                                             \
  do {                                                                                  \
    if ((call) != 0) return ::pcgb::fail(PCG_ERR_NCCL, std::string(what) + ": host communicator callback failed"); \
  } while (0)

static pcg_status comm_alive(pcg_comm *C) {
  return C->aborted ? fail(PCG_ERR_NCCL, "NCCL communicator was aborted") : PCG_OK;
}

static pcg_status comm_allreduce_f64(pcg_comm *C, double *dbuf, int count, cudaStream_t st) {
  PCG_TRY(comm_alive(C));
  // a 1-rank NCCL communicator still issues the (trivial) collective: it keeps the
  // captured-graph + NCCL path testable on one GPU
  if (count == 0 || (C->use_ops && C->size == 1)) return PCG_OK;
  if (!C->use_ops && C->dar) return dar_allreduce(C->dar, dbuf, count, st);  // opt-in, dar.cu
  if (!C->use_ops) {
    PCG_NCCL(ncclAllReduce(dbuf, dbuf, (size_t)count, ncclDouble, ncclSum, C->nccl, st));
    return PCG_OK;
  }
  std::vector<double> h(count);
  PCG_CUDA(cudaMemcpyAsync(h.data(), dbuf, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  PCG_OPS(C->ops.allreduce_sum_f64(C->ops.ctx, h.data(), count), "allreduce_sum_f64");
  PCG_CUDA(cudaMemcpyAsync(dbuf, h.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}

static pcg_status comm_allreduce_max_i32(pcg_comm *C, int *dbuf, int count, cudaStream_t st) {
  PCG_TRY(comm_alive(C));
  if (C->size == 1 || count == 0) return PCG_OK;
  if (!C->use_ops) {
    PCG_NCCL(ncclAllReduce(dbuf, dbuf, (size_t)count, ncclInt32, ncclMax, C->nccl, st));
    return PCG_OK;
  }
  std::vector<int32_t> h(count);
  PCG_CUDA(cudaMemcpyAsync(h.data(), dbuf, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  PCG_OPS(C->ops.allreduce_max_i32(C->ops.ctx, h.data(), count), "allreduce_max_i32");
  PCG_CUDA(cudaMemcpyAsync(dbuf, h.data(), sizeof(int32_t) * count, cudaMemcpyHostToDevice, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}

// all[r*count + i] = rank r's mine[i]; mine is C->rank's slot of all (device)
static pcg_status comm_allgather_i64(pcg_comm *C, int64_t *dall, int count, cudaStream_t st) {
  PCG_TRY(comm_alive(C));
  if (C->size == 1) return PCG_OK;
  if (!C->use_ops) {
    PCG_NCCL(ncclAllGather(dall + (size_t)count * C->rank, dall, (size_t)count, ncclInt64, C->nccl, st));
    return PCG_OK;
  }
  std::vector<int64_t> mine(count), all((size_t)count * C->size);
  PCG_CUDA(cudaMemcpyAsync(mine.data(), dall + (size_t)count * C->rank, sizeof(int64_t) * count,
                           cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  PCG_OPS(C->ops.allgather_i64(C->ops.ctx, mine.data(), count, all.data()), "allgather_i64");
  PCG_CUDA(cudaMemcpyAsync(dall, all.data(), sizeof(int64_t) * all.size(), cudaMemcpyHostToDevice, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}

struct Xfer {
  int peer;
  const void *send;  // device
  int64_t scount;    // elements
  void *recv;        // device
  int64_t rcount;
};

// grouped point-to-point exchange of `esize`-byte elements (NCCL type `ty`)
static pcg_status comm_exchange(pcg_comm *C, const std::vector<Xfer> &xs, ncclDataType_t ty, size_t esize,
                                cudaStream_t st) {
  if (xs.empty()) return PCG_OK;
  PCG_TRY(comm_alive(C));
  if (!C->use_ops) {
    PCG_NCCL(ncclGroupStart());
    for (const Xfer &x : xs) {
      if (x.scount > 0) PCG_NCCL(ncclSend(x.send, (size_t)x.scount, ty, x.peer, C->nccl, st));
      if (x.rcount > 0) PCG_NCCL(ncclRecv(x.recv, (size_t)x.rcount, ty, x.peer, C->nccl, st));
    }
    PCG_NCCL(ncclGroupEnd());
    return PCG_OK;
  }
  const size_t np = xs.size();
  std::vector<std::vector<char>> hs(np), hr(np);
  std::vector<const void *> sp(np);
  std::vector<void *> rp(np);
  std::vector<int64_t> sb(np), rb(np);
  std::vector<int32_t> peers(np);
  for (size_t t = 0; t < np; t++) {
    peers[t] = xs[t].peer;
    sb[t] = xs[t].scount * (int64_t)esize;
    rb[t] = xs[t].rcount * (int64_t)esize;
    hs[t].resize(sb[t] > 0 ? sb[t] : 1);
    hr[t].resize(rb[t] > 0 ? rb[t] : 1);
    sp[t] = hs[t].data();
    rp[t] = hr[t].data();
    if (sb[t] > 0) PCG_CUDA(cudaMemcpyAsync(hs[t].data(), xs[t].send, sb[t], cudaMemcpyDeviceToHost, st));
  }
  PCG_CUDA(cudaStreamSynchronize(st));
  PCG_OPS(C->ops.exchange(C->ops.ctx, (int32_t)np, peers.data(), sp.data(), sb.data(), rp.data(), rb.data()),
          "exchange");
  for (size_t t = 0; t < np; t++)
    if (rb[t] > 0) PCG_CUDA(cudaMemcpyAsync(xs[t].recv, hr[t].data(), rb[t], cudaMemcpyHostToDevice, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  return PCG_OK;
}

pcg_status halo_exchange(pcg_matrix *A, double *vec, int width, cudaStream_t st) {
  (void)width;
  NvtxRange r_("pcg:halo_exchange");
  if (!A->comm || A->halo.nbr.empty()) return PCG_OK;
  HaloPlan &hp = A->halo;
  if (hp.n_send > 0) {
    pack_kernel<<<(unsigned)std::min<int64_t>((hp.n_send + 255) / 256, 1184), 256, 0, st>>>(hp.n_send, hp.d_send_idx,
                                                                                          vec, hp.d_send_buf);
    count_launch();
  }
  std::vector<Xfer> xs;
  for (size_t t = 0; t < hp.nbr.size(); t++)
    xs.push_back({hp.nbr[t], hp.d_send_buf + hp.send_off[t], hp.send_cnt[t], vec + A->n + hp.recv_off[t],
                  hp.recv_cnt[t]});
  return comm_exchange(A->comm, xs, ncclDouble, sizeof(double), st);
}

pcg_status allreduce_sum(pcg_matrix *A, double *buf, int count, cudaStream_t st) {
  if (!A->comm) return PCG_OK;
  return comm_allreduce_f64(A->comm, buf, count, st);
}

// rows that reference a ghost column (need the halo before their SpMV)
__global__ void ghost_rows_kernel(int64_t n, const int *__restrict__ rp, const int *__restrict__ col,
                                  uint8_t *__restrict__ flag) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint8_t f = 0;
    for (int k = rp[i]; k < rp[i + 1]; k++) f |= col[k] >= (int)n;
    flag[i] = f;
  }
}

// The longest run of rows without ghost columns, aligned to SELL slices, becomes the
// interior range whose SpMV runs while the z halo is in flight (north_star
// (c): "halos ... overlapped with the interior SpMV").  Contiguous blocks of a banded
// order (lattice, RCM) have their boundary rows at both ends.  Off if the range is
// under a quarter of the rows, for the TMA-staged format, or with PCG_NO_OVERLAP=1.
static pcg_status overlap_plan(pcg_matrix *A, cudaStream_t st) {
  A->ov = false;
  const int64_t n = A->n;
  // PCG_FORCE_OVERLAP=1 (tests): the split schedule even without a halo (1-rank NCCL handle),
  // interior = the middle half, so the captured fork/join graph runs on one GPU
  const bool force = getenv("PCG_FORCE_OVERLAP") && n >= 256;
  if (getenv("PCG_NO_OVERLAP") || ((A->halo.nbr.empty() || n < 64) && !force)) return PCG_OK;
  if (A->format != PCG_FORMAT_SELL && A->format != PCG_FORMAT_CSR) return PCG_OK;
  if (force) {
    if (!A->ov_side) {
      PCG_CUDA(cudaStreamCreateWithFlags(&A->ov_side, cudaStreamNonBlocking));
      PCG_CUDA(cudaEventCreateWithFlags(&A->ov_fork, cudaEventDisableTiming));
      PCG_CUDA(cudaEventCreateWithFlags(&A->ov_join, cudaEventDisableTiming));
    }
    A->ov_ia = (n / 4) & ~int64_t(31);
    A->ov_ib = (3 * n / 4) & ~int64_t(31);
    A->ov = true;
    return PCG_OK;
  }
  uint8_t *d_flag;
  PCG_CUDA(cudaMalloc(&d_flag, n));
  ghost_rows_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(n, A->d_row_ptr, A->d_col,
                                                                                           d_flag);
  count_launch();
  std::vector<uint8_t> f(n);
  PCG_CUDA(cudaMemcpyAsync(f.data(), d_flag, n, cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d_flag);
  int64_t best_a = 0, best_b = 0;
  for (int64_t i = 0; i < n;) {
    if (f[i]) {
      i++;
      continue;
    }
    int64_t j = i;
    while (j < n && !f[j]) j++;
    if (j - i > best_b - best_a) {
      best_a = i;
      best_b = j;
    }
    i = j;
  }
  const int64_t ia = best_a == 0 ? 0 : (best_a + 31) & ~int64_t(31);
  const int64_t ib = best_b == n ? n : best_b & ~int64_t(31);
  if (ib - ia < n / 4 || (ia == 0 && ib == n)) return PCG_OK;
  if (!A->ov_side) {
    PCG_CUDA(cudaStreamCreateWithFlags(&A->ov_side, cudaStreamNonBlocking));
    PCG_CUDA(cudaEventCreateWithFlags(&A->ov_fork, cudaEventDisableTiming));
    PCG_CUDA(cudaEventCreateWithFlags(&A->ov_join, cudaEventDisableTiming));
  }
  A->ov_ia = ia;
  A->ov_ib = ib;
  A->ov = true;
  return PCG_OK;
}

static pcg_status create_dist_impl(pcg_comm *C, int64_t n_global, int64_t r0, int64_t r1, int64_t nnz,
                                   const int64_t *row_ptr, const int64_t *col, const double *val, int flags,
                                   cudaStream_t st, pcg_matrix *A) {
  const int64_t n = r1 - r0;
  const bool dev = (flags & PCG_PTR_DEVICE) != 0;
  // stage inputs on the device
  int64_t *drp = (int64_t *)row_ptr, *dcol = (int64_t *)col;
  double *dval = (double *)val;
  std::vector<void *> owned;
  if (!dev) {
    PCG_CUDA(cudaMalloc(&drp, sizeof(int64_t) * (n + 1)));
    PCG_CUDA(cudaMalloc(&dcol, sizeof(int64_t) * (nnz > 0 ? nnz : 1)));
    PCG_CUDA(cudaMalloc(&dval, sizeof(double) * (nnz > 0 ? nnz : 1)));
    owned = {drp, dcol, dval};
    PCG_CUDA(cudaMemcpyAsync(drp, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, st));
    if (nnz) PCG_CUDA(cudaMemcpyAsync(dcol, col, sizeof(int64_t) * nnz, cudaMemcpyHostToDevice, st));
    if (nnz) PCG_CUDA(cudaMemcpyAsync(dval, val, sizeof(double) * nnz, cudaMemcpyHostToDevice, st));
  }
  int64_t ends[2];
  PCG_CUDA(cudaMemcpyAsync(&ends[0], drp, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  PCG_CUDA(cudaMemcpyAsync(&ends[1], drp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  PCG_TRY(comm_wait(C, st));
  if (ends[0] != 0 || ends[1] != nnz)
    return fail(PCG_ERR_DIMENSION_MISMATCH, "csr_create_dist: row_ptr_local[0] must be 0 and [n] = nnz_local");
  // ---- ghost list: sorted unique remote columns (device mark + compaction)
  uint8_t *flag;
  PCG_CUDA(cudaMalloc(&flag, n_global > 0 ? n_global : 1));
  PCG_CUDA(cudaMemsetAsync(flag, 0, n_global, st));
  // out-of-range columns are caught by validation below; clamp marking to valid ones
  mark_remote_kernel<<<1184, 256, 0, st>>>(nnz, dcol, r0, r1, n_global, flag);
  count_launch();
  int64_t *ghost, *d_cnt;
  PCG_CUDA(cudaMalloc(&ghost, sizeof(int64_t) * (n_global > 0 ? n_global : 1)));
  PCG_CUDA(cudaMalloc(&d_cnt, sizeof(int64_t)));
  {
    thrust::counting_iterator<int64_t> it(0);
    size_t tb = 0;
    cub::DeviceSelect::Flagged(nullptr, tb, it, flag, ghost, d_cnt, n_global, st);
    void *tbuf;
    PCG_CUDA(cudaMalloc(&tbuf, tb));
    cub::DeviceSelect::Flagged(tbuf, tb, it, flag, ghost, d_cnt, n_global, st);
    PCG_CUDA(cudaMemcpyAsync(&A->n_ghost, d_cnt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PCG_TRY(comm_wait(C, st));
    cudaFree(tbuf);
  }
  cudaFree(flag);
  const int64_t ng = A->n_ghost;
  std::vector<int64_t> h_ghost(ng);
  if (ng) PCG_CUDA(cudaMemcpy(h_ghost.data(), ghost, sizeof(int64_t) * ng, cudaMemcpyDeviceToHost));
  // ---- validate on global columns (diag at global row), then map to local ids
  int64_t *dloc;
  PCG_CUDA(cudaMalloc(&dloc, sizeof(int64_t) * (nnz > 0 ? nnz : 1)));
  {
    // validation of structure happens in create_local against n_cols on the mapped
    // ids; out-of-range globals must be caught first
    map_cols_kernel<<<1184, 256, 0, st>>>(nnz, dcol, r0, r1, n, ghost, ng, dloc);
    count_launch();
  }
  cudaFree(ghost);
  cudaFree(d_cnt);
  // ---- all ranks' bounds
  const int G = C->size, me = C->rank;
  int64_t *d_bounds;
  PCG_CUDA(cudaMalloc(&d_bounds, sizeof(int64_t) * 2 * G));
  int64_t mine[2] = {r0, r1};
  PCG_CUDA(cudaMemcpyAsync(d_bounds + 2 * me, mine, sizeof(mine), cudaMemcpyHostToDevice, st));
  PCG_TRY(comm_allgather_i64(C, d_bounds, 2, st));
  std::vector<int64_t> hb(2 * G);
  PCG_CUDA(cudaMemcpyAsync(hb.data(), d_bounds, sizeof(int64_t) * 2 * G, cudaMemcpyDeviceToHost, st));
  PCG_TRY(comm_wait(C, st));
  cudaFree(d_bounds);
  for (int g = 0; g < G; g++)
    if (g > 0 && hb[2 * g] != hb[2 * g - 1])
      return fail(PCG_ERR_INVALID_ARG, "csr_create_dist: rank row ranges are not contiguous in rank order");
  // ---- receive lists: ghosts owned by each rank (contiguous runs of the sorted list)
  std::vector<int64_t> bnd(G + 1), need(G, 0), need_off(G, 0);
  for (int g = 0; g < G; g++) bnd[g] = hb[2 * g];
  bnd[G] = hb[2 * G - 1];
  PCG_TRY(pcg_halo_recv_plan(ng, h_ghost.data(), G, bnd.data(), need.data(), need_off.data()));
  // counts matrix M[h][g] = #rows rank h needs from rank g
  int64_t *d_M;
  PCG_CUDA(cudaMalloc(&d_M, sizeof(int64_t) * G * G));
  PCG_CUDA(cudaMemcpyAsync(d_M + (size_t)G * me, need.data(), sizeof(int64_t) * G, cudaMemcpyHostToDevice, st));
  PCG_TRY(comm_allgather_i64(C, d_M, G, st));
  std::vector<int64_t> M((size_t)G * G);
  PCG_CUDA(cudaMemcpyAsync(M.data(), d_M, sizeof(int64_t) * G * G, cudaMemcpyDeviceToHost, st));
  PCG_TRY(comm_wait(C, st));
  cudaFree(d_M);
  HaloPlan &hp = A->halo;
  int64_t send_total = 0;
  for (int g = 0; g < G; g++) {
    if (g == me) continue;
    const int64_t sc = M[(size_t)G * g + me], rc = need[g];
    if (sc == 0 && rc == 0) continue;
    hp.nbr.push_back(g);
    hp.recv_off.push_back(need_off[g]);
    hp.recv_cnt.push_back(rc);
    hp.send_off.push_back(send_total);
    hp.send_cnt.push_back(sc);
    send_total += sc;
  }
  hp.n_send = send_total;
  // ---- exchange index lists (global row ids) -> local send rows
  int64_t *d_recv_idx = nullptr, *d_send_g = nullptr;
  PCG_CUDA(cudaMalloc(&d_recv_idx, sizeof(int64_t) * (ng > 0 ? ng : 1)));
  PCG_CUDA(cudaMalloc(&d_send_g, sizeof(int64_t) * (send_total > 0 ? send_total : 1)));
  if (ng) PCG_CUDA(cudaMemcpyAsync(d_recv_idx, h_ghost.data(), sizeof(int64_t) * ng, cudaMemcpyHostToDevice, st));
  {  // every rank sends the global ids it needs from a peer; what arrives is the peer's send list
    std::vector<Xfer> xs;
    for (size_t t = 0; t < hp.nbr.size(); t++)
      xs.push_back({hp.nbr[t], d_recv_idx + hp.recv_off[t], hp.recv_cnt[t], d_send_g + hp.send_off[t], hp.send_cnt[t]});
    PCG_TRY(comm_exchange(C, xs, ncclInt64, sizeof(int64_t), st));
  }
  PCG_CUDA(cudaMalloc(&hp.d_send_idx, sizeof(int) * (send_total > 0 ? send_total : 1)));
  PCG_CUDA(cudaMalloc(&hp.d_send_buf, sizeof(double) * KMAX * (send_total > 0 ? send_total : 1)));
  if (send_total) {
    to_local_rows_kernel<<<(unsigned)std::min<int64_t>((send_total + 255) / 256, 1184), 256, 0, st>>>(
        send_total, d_send_g, r0, hp.d_send_idx);
    count_launch();
  }
  PCG_TRY(comm_wait(C, st));
  cudaFree(d_recv_idx);
  cudaFree(d_send_g);
  // ---- local matrix: n rows, n + n_ghost columns, diagonal at local i
  A->comm = C;
  A->row_begin = r0;
  A->row_end = r1;
  A->n_global = n_global;
  pcg_status s = create_local(A, n, nnz, drp, dcol, dloc, dval, n_global, r0, flags, st);
  if (s == PCG_OK) s = overlap_plan(A, st);
  cudaStreamSynchronize(st);
  // all ranks fail together (a local validation error must not leave peers waiting)
  {
    int *d_s;
    int hs = (int)s;
    if (cudaMalloc(&d_s, sizeof(int)) == cudaSuccess) {
      cudaMemcpyAsync(d_s, &hs, sizeof(int), cudaMemcpyHostToDevice, st);
      (void)comm_allreduce_max_i32(C, d_s, 1, st);
      int all = 0;
      cudaMemcpyAsync(&all, d_s, sizeof(int), cudaMemcpyDeviceToHost, st);
      const pcg_status ws = comm_wait(C, st);
      cudaFree(d_s);
      if (ws != PCG_OK) all = (int)ws;
      if (s == PCG_OK && all != PCG_OK) s = fail((pcg_status)all, "csr_create_dist: another rank failed validation");
    }
  }
  cudaFree(dloc);
  for (void *p : owned) cudaFree(p);
  return s;
}

}  // namespace pcgb

using namespace pcgb;

extern "C" pcg_status pcg_partition_rows(int64_t n, const int64_t *row_ptr, int32_t G, int64_t *bounds) {
  if (n < 0 || G < 1 || !row_ptr || !bounds) return fail(PCG_ERR_INVALID_ARG, "pcg_partition_rows: bad argument");
  const int64_t nnz = row_ptr[n];
  bounds[0] = 0;
  bounds[G] = n;
  for (int g = 1; g < G; g++) {
    const int64_t target = ((int64_t)g * nnz) / G;
    bounds[g] = std::lower_bound(row_ptr, row_ptr + n + 1, target) - row_ptr;
    if (bounds[g] > n) bounds[g] = n;
  }
  return PCG_OK;
}

extern "C" pcg_status pcg_halo_ghosts(int64_t r0, int64_t r1, int64_t nnz, const int64_t *col, int64_t *ghosts,
                                      int64_t cap, int64_t *n_ghost) {
  if (!n_ghost || (nnz > 0 && !col) || r1 < r0 || nnz < 0) return fail(PCG_ERR_INVALID_ARG, "pcg_halo_ghosts: bad argument");
  std::vector<int64_t> g;
  for (int64_t k = 0; k < nnz; k++)
    if (col[k] < r0 || col[k] >= r1) g.push_back(col[k]);
  std::sort(g.begin(), g.end());
  g.erase(std::unique(g.begin(), g.end()), g.end());
  *n_ghost = (int64_t)g.size();
  if (ghosts)
    for (int64_t i = 0; i < (int64_t)g.size() && i < cap; i++) ghosts[i] = g[i];
  return PCG_OK;
}

extern "C" pcg_status pcg_halo_recv_plan(int64_t ng, const int64_t *ghosts, int32_t G, const int64_t *bounds,
                                         int64_t *need, int64_t *need_off) {
  if (G < 1 || !bounds || !need || !need_off || (ng > 0 && !ghosts))
    return fail(PCG_ERR_INVALID_ARG, "pcg_halo_recv_plan: bad argument");
  for (int g = 0; g < G; g++) need[g] = 0;
  for (int64_t t = 0, g = 0; t < ng; t++) {
    while (g < G && ghosts[t] >= bounds[g + 1]) g++;
    if (g >= G || ghosts[t] < bounds[g])
      return fail(PCG_ERR_INDEX_OUT_OF_RANGE, "pcg_halo_recv_plan: ghost column outside every rank's rows");
    need[g]++;
  }
  need_off[0] = 0;
  for (int g = 1; g < G; g++) need_off[g] = need_off[g - 1] + need[g - 1];
  return PCG_OK;
}

extern "C" pcg_status pcg_comm_unique_id(void *id128) {
  if (!id128) return fail(PCG_ERR_INVALID_ARG, "pcg_comm_unique_id: null");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  PCG_NCCL(ncclGetUniqueId(&id));
  memcpy(id128, &id, sizeof(id));
  return PCG_OK;
}

extern "C" pcg_status pcg_comm_init(int32_t rank, int32_t size, const void *id128, pcg_comm_t *out) {
  if (!id128 || !out || size < 1 || rank < 0 || rank >= size)
    return fail(PCG_ERR_INVALID_ARG, "pcg_comm_init: bad argument");
  pcg_comm *c = new pcg_comm();
  c->rank = rank;
  c->size = size;
  ncclUniqueId id;
  memcpy(&id, id128, sizeof(id));
  if (const char *e = getenv("PCG_COMM_TIMEOUT_S")) c->timeout_s = atof(e) > 0 ? atof(e) : c->timeout_s;
  ncclResult_t r = ncclCommInitRank(&c->nccl, size, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return fail(PCG_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  }
  if (const char *e = getenv("PCG_DEVICE_ALLREDUCE")) {  // collective: every rank must set it alike
    if (atoi(e) == 1) {
      pcg_status s = dar_setup(c->nccl, rank, size, &c->dar);
      if (s != PCG_OK) {
        ncclCommDestroy(c->nccl);
        delete c;
        return s;
      }
    }
  }
  *out = c;
  return PCG_OK;
}

extern "C" pcg_status pcg_comm_init_ops(int32_t rank, int32_t size, const pcg_comm_ops *ops, pcg_comm_t *out) {
  if (!ops || !out || size < 1 || rank < 0 || rank >= size || !ops->allreduce_sum_f64 || !ops->allreduce_max_i32 ||
      !ops->allgather_i64 || !ops->exchange)
    return fail(PCG_ERR_INVALID_ARG, "pcg_comm_init_ops: bad argument");
  pcg_comm *c = new pcg_comm();
  c->rank = rank;
  c->size = size;
  c->use_ops = true;
  c->ops = *ops;
  *out = c;
  return PCG_OK;
}

extern "C" pcg_status pcg_comm_destroy(pcg_comm_t c) {
  if (!c) return PCG_OK;
  if (c->nccl) ncclCommDestroy(c->nccl);
  if (c->wait_ev) cudaEventDestroy(c->wait_ev);
  if (c->dar) dar_free(c->dar);
  delete c;
  return PCG_OK;
}

extern "C" pcg_status pcg_comm_abort(pcg_comm_t c) {
  if (!c) return fail(PCG_ERR_INVALID_ARG, "pcg_comm_abort: null communicator");
  if (c->use_ops) {
    c->aborted = true;
    return PCG_OK;
  }
  if (!c->aborted) (void)abort_comm(c, "pcg_comm_abort");
  return PCG_OK;
}

extern "C" pcg_status pcg_comm_get_info(pcg_comm_t c, int32_t *rank, int32_t *size, int32_t *device_allreduce) {
  if (!c) return fail(PCG_ERR_INVALID_ARG, "pcg_comm_get_info: null communicator");
  if (rank) *rank = c->rank;
  if (size) *size = c->size;
  if (device_allreduce) *device_allreduce = c->dar != nullptr;
  return PCG_OK;
}

extern "C" pcg_status pcg_comm_set_timeout(pcg_comm_t c, double seconds) {
  if (!c || !(seconds > 0.0)) return fail(PCG_ERR_INVALID_ARG, "pcg_comm_set_timeout: bad argument");
  c->timeout_s = seconds;
  return PCG_OK;
}

extern "C" pcg_status csr_create_dist(pcg_comm_t comm, int64_t n_global, int64_t row_begin, int64_t row_end,
                                      int64_t nnz_local, const int64_t *row_ptr_local,
                                      const int64_t *col_idx_global, const double *val, int flags, void *stream,
                                      pcg_matrix_t *out) {
  pcgb::NvtxRange nvtx_("pcg:csr_create_dist");
  if (!comm || !out || !row_ptr_local || (nnz_local > 0 && (!col_idx_global || !val)))
    return fail(PCG_ERR_INVALID_ARG, "csr_create_dist: null argument");
  *out = nullptr;
  if (n_global < 0 || row_begin < 0 || row_end < row_begin || row_end > n_global || nnz_local < 0)
    return fail(PCG_ERR_INVALID_ARG, "csr_create_dist: bad row range");
  if (nnz_local >= (int64_t(1) << 31)) return fail(PCG_ERR_INVALID_ARG, "csr_create_dist: nnz per GPU must be < 2^31");
  auto t0 = std::chrono::steady_clock::now();
  pcg_matrix *A = new pcg_matrix();
  cudaGetDevice(&A->device);
  pcg_status s = create_dist_impl(comm, n_global, row_begin, row_end, nnz_local, row_ptr_local, col_idx_global, val,
                                  flags, (cudaStream_t)stream, A);
  if (s != PCG_OK) {
    A->comm = nullptr;
    csr_destroy(A);
    return s;
  }
  A->t_setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  *out = A;
  return PCG_OK;
}
