// matrix.cuh — the opaque pcg_matrix handle (device formats + solver workspace).
#pragma once
#include <nccl.h>

#include <vector>

#include "common.cuh"

struct pcg_comm {
  ncclComm_t nccl = nullptr;   // NCCL backend (null when ops are used)
  int rank = 0, size = 1;
  cudaStream_t comm_stream = nullptr;
  bool use_ops = false;        // host-callback backend (pcg_comm_init_ops)
  pcg_comm_ops ops{};
  // failure detection: waits poll ncclCommGetAsyncError and give up after
  // timeout_s (PCG_COMM_TIMEOUT_S, default 300) with ncclCommAbort -> PCG_ERR_NCCL
  double timeout_s = 300.0;
  bool aborted = false;
  cudaEvent_t wait_ev = nullptr;
  void *dar = nullptr;  // device-initiated allreduce over NVLink peer memory (dar.cu), opt-in
};

namespace pcgb {

pcg_status dar_setup(ncclComm_t nccl, int rank, int size, void **out);
pcg_status dar_allreduce(void *dar, double *buf, int count, cudaStream_t st);
bool dar_failed(const void *dar);
void dar_free(void *dar);
pcg_status ilu_setup(pcg_matrix *A, int64_t bs, cudaStream_t st, void **plan_out);
void ilu_launch(void *plan, const double *in, double *out, const int *stop, const int *skip, cudaStream_t st);
void ilu_free(void *plan);
int64_t ilu_block_rows(const void *plan);
double ilu_bytes_per_apply(const void *plan);
// Wait for the work queued on `st` (distributed handles: with NCCL failure detection
// and the communicator's timeout; see dist.cu comm_wait).
pcg_status comm_wait(pcg_comm *C, cudaStream_t st);

// Halo plan for a distributed handle: this rank's rows are
// [row_begin,row_end); local column ids: owned j -> j-row_begin, ghosts -> n+g.
struct HaloPlan {
  std::vector<int> nbr;                 // neighbour ranks (ascending)
  std::vector<int64_t> recv_off, recv_cnt;  // ghost slots per neighbour (into [n, n+n_ghost))
  std::vector<int64_t> send_off, send_cnt;  // slots into d_send_idx per neighbour
  int *d_send_idx = nullptr;            // local row ids to pack, concatenated per neighbour
  double *d_send_buf = nullptr;         // packed values (k doubles per row in multi mode)
  int64_t n_send = 0;
};

struct SolveWork {
  // single-RHS vectors (n + n_ghost entries where gathered)
  double *r = nullptr, *z = nullptr, *q = nullptr, *p[2] = {nullptr, nullptr}, *x = nullptr;
  double *w = nullptr;  // spmv scratch (exit check / standalone spmv)
  double *stage_b = nullptr, *stage_x = nullptr;  // device staging for host pointers
  double *partials = nullptr;  // 4 * max_grid
  // per 32-row slice the slice's dinv when its 32 entries are bitwise equal, NaN otherwise
  // (K2 then reads 8 bytes per 32 rows instead of 8 per row: a lattice's Jacobi diagonal)
  double *dslice = nullptr;
  bool dslice_all = false;  // every slice shares one: K2 stores no z, K1a forms it from r
  Scalars *sc = nullptr;       // device scalars
  Scalars *h_sc = nullptr;     // pinned host mirror
  cudaGraphExec_t loop_exec = nullptr;
  cudaGraph_t loop_graph = nullptr;
  bool graph_ready = false;
  int graph_kind = 0;  // 1 = conditional while node, 2 = unrolled chunk
  int unroll = 0;
  int xdefer = 0;  // 3-pass graph loop: x updated every xdefer-th iteration (2 or 4; 0 = every one)
  double *p23[2] = {nullptr, nullptr};  // direction buffers p[2], p[3] of the 4-cycle
  // multi-RHS workspace (row-major n x kcap)
  int kcap = 0;
  double *mr = nullptr, *mz = nullptr, *mq = nullptr, *mp[2] = {nullptr, nullptr}, *mp23[2] = {nullptr, nullptr}, *mx = nullptr,
         *mb = nullptr, *mw = nullptr;
  MultiScalars *msc = nullptr, *h_msc = nullptr;
  double *mpart = nullptr;
  cudaGraphExec_t mloop_exec = nullptr;
  cudaGraph_t mloop_graph = nullptr;
  int mgraph_k = 0;
  // persistent cooperative solve (persist.cu)
  void *pbar = nullptr;  // grid barrier state
  int pgrid = 0;
  // BiCGSTAB (bicgstab.cu): x r r^ p p^ v s^ t, state, barrier, Block-Jacobi inverses
  double *bv = nullptr;
  void *bstate = nullptr, *bbar = nullptr;
  double *bminv = nullptr;
  void *ilu = nullptr;  // ILU(0) Block-Jacobi plan (ilu.cu), cached per block size
  int bminv_bs = 0, bgrid = 0, bgrid_bs = 0;
  // pipelined PCG (pipelined.cu): x r u w m0 m1 z q s p, state, barrier, grid
  double *pv = nullptr;
  void *pstate = nullptr, *ppbar = nullptr, *pdsc = nullptr;
  int ppgrid = 0;
  // block CG (blockcg.cu): X R Z P Q B blocks, state (+ pinned mirror), Gram partials
  double *bcg = nullptr, *bcg_part = nullptr;
  int64_t bcg_cap = 0, bcg_part_cap = 0;
  void *bcg_st = nullptr, *bcg_hst = nullptr;
  void *bspmm_sc = nullptr;  // scratch MultiScalars of the block-CG SpMM (multi.cu block_spmm)
  double *bspmm_part = nullptr;
  // BiCGSTAB graph schedule: device scalars, loop graph (per block size)
  void *bgsc = nullptr;
  cudaGraphExec_t bg_exec = nullptr;
  cudaGraph_t bg_graph = nullptr;
  int bg_bs = 0;
};

// single-RHS solver vectors (p0/p1: direction double buffer of the 2-pass schedule)
struct Vecs {
  double *r, *z, *q, *p0, *p1, *x;
  const double *dinv;
  double *p2, *p3;  // deferred x update with a 4-cycle (null otherwise)
};

// a symmetrically permuted copy of the system (SELL-C-sigma, sigma.cu)
struct SigmaSys {
  int *perm = nullptr, *iperm = nullptr;  // perm[i'] = original row of permuted row i'
  int *row_ptr = nullptr, *col = nullptr;
  double *val = nullptr, *dinv = nullptr;
  int64_t *slice_ptr = nullptr;
  int *scol = nullptr;
  double *sval = nullptr;
  int64_t sell_entries = 0;
  int sigma = 0;
};

}  // namespace pcgb

struct pcg_matrix {
  int device = 0;
  int64_t n = 0, nnz = 0;  // local rows / nnz
  int32_t max_row_len = 0;
  bool short_rows = false;  // SELL with rows <= 8 entries: the one-chunk engine (rows.cuh)
  int format = PCG_FORMAT_CSR;
  // CSR (int32)
  int *d_row_ptr = nullptr, *d_col = nullptr;
  double *d_val = nullptr, *d_dinv = nullptr;
  // SELL-32
  int64_t n_slices = 0, sell_entries = 0;
  int64_t *d_slice_ptr = nullptr;
  int *d_scol = nullptr;
  double *d_sval = nullptr;
  // CSR kernel lanes per row
  int csr_lanes = 4;
  int schedule = 3;  // 3: K1a + K1b + K2 (96n B), 2: fused K1 + K2 (88n B)
  // launch geometry
  int grid_vec = 0, grid_spmv = 0;  // persistent grid sizes (multiples of the SM count)
  double t_setup_s = 0, spmv_us_csr = 0, spmv_us_sell = 0, spmv_us_tma = 0, spmv_us_sigma = 0;
  double device_bytes = 0;
  // distributed
  pcg_comm *comm = nullptr;
  int64_t n_ghost = 0, row_begin = 0, row_end = 0, n_global = 0;
  int64_t n_interior = 0;  // rows [0,n_interior) reference no ghost (not used by the 1-GPU path)
  pcgb::HaloPlan halo;
  pcgb::SolveWork work;
  std::mutex mu;
  pcgb::CsrView csr() const { return {n, n + n_ghost, d_row_ptr, d_col, d_val, 0}; }
  int stages = 2;
  int64_t stage_entries = 0;  // 0: TMA-staged SELL unavailable
  size_t dyn_smem = 0;        // dynamic shared memory of the chosen format's kernels
  int *d_lead = nullptr;      // per-tile prefix-max column (TMA L2 prefetch windows)
  // SELL-C-sigma: the device system is P A P^T (vectors in permuted order) when d_perm != null
  // (also PCG_REORDER_RCM: perm = the RCM order, composed with the sigma sort if both)
  int *d_perm = nullptr, *d_iperm = nullptr;
  int sigma = 0;
  int reorder = 0;  // 1: PCG_REORDER_RCM applied
  // distributed: halo exchange overlapped with the interior SpMV (dist.cu overlap_plan).
  // Rows [ov_ia, ov_ib) reference no ghost; the z halo runs on ov_side meanwhile.
  bool ov = false;
  int64_t ov_ia = 0, ov_ib = 0;
  cudaStream_t ov_side = nullptr;
  cudaEvent_t ov_fork = nullptr, ov_join = nullptr;
  // windowed SpMM plan (multi.cu): per 512-row tile up to 4 column windows staged in shared
  // memory by TMA, per SELL entry its 16-bit offset in the concatenated windows
  void *d_wdesc = nullptr;
  uint16_t *d_wlidx = nullptr;
  int wplan = 0;  // 0: not built, 1: usable, -1: the matrix does not fit the windows
  // 16-bit delta column ids of the SELL entries (common.cuh SellView::dcol)
  int16_t *d_sdcol = nullptr;
  int *d_scbase = nullptr;
  int64_t d16_slices = 0;
  // uniform-offset positions of the one-chunk engine (common.cuh SellView::doff / dmask)
  int *d_sdoff = nullptr;
  uint8_t *d_sdmask = nullptr;
  int64_t dia_positions = 0;  // positions without ids, over all slices
  int64_t dia_slices = 0;     // slices made only of such positions (one dependent round trip)
  // value-uniform positions of those slices (common.cuh SellView::dval / dvmeta)
  double *d_sdval = nullptr;
  uint16_t *d_sdvmeta = nullptr;
  unsigned *d_sdzmask = nullptr;
  int64_t aligned_slices = 0;  // value-free slices in the aligned (zero-mask) form
  int64_t dval_slices = 0;    // one-trip slices whose values are all per-position uniform (no value stream)
  // their patterns (common.cuh SellView::dpat / ptab)
  uint8_t *d_sdpat = nullptr;
  pcgb::DiaPat *d_ptab = nullptr;
  int *d_plen = nullptr;
  int npat = 0;
  int64_t pat_slices = 0;     // value-free slices that read a shared pattern
  pcgb::SellView sell() const {
    return {n, n_slices, d_slice_ptr, d_scol, d_sval, stages, stage_entries, d_lead, 0, d_sdcol, d_scbase, 0,
            d_sdoff, d_sdmask};
  }
  pcgb::SellViewDia sell_dia() const {
    pcgb::SellViewDia v;
    static_cast<pcgb::SellView &>(v) = sell();
    v.dval = d_sdval;
    v.dvmeta = d_sdvmeta;
    v.dzmask = d_sdzmask;
    v.dpat = d_sdpat;
    v.ptab = d_ptab;
    v.plen = d_plen;
    v.npat = npat;
    return v;
  }
};

namespace pcgb {
pcg_status ensure_work(pcg_matrix *A);
pcg_status ensure_multi_work(pcg_matrix *A, int k);
pcg_status build_sell(pcg_matrix *A, cudaStream_t st);
int persist_schedule(const pcg_matrix *A);
bool persist_wanted(const pcg_matrix *A);
pcg_status persist_launch(pcg_matrix *A, Vecs v, cudaStream_t st);
int sigma_window();
pcg_status sigma_build(pcg_matrix *A, cudaStream_t st, SigmaSys *S);
void sigma_swap(pcg_matrix *A, SigmaSys *S);
void sigma_free(SigmaSys *S);
pcg_status apply_perm(pcg_matrix *A, int *perm, cudaStream_t st);
pcg_status rcm_order(int64_t n, const int *rp, const int *col, int *perm, cudaStream_t st);
pcg_status block_spmm(pcg_matrix *A, const double *P, double *Q, int k, int64_t ld, const int *d_done,
                      cudaStream_t st);
pcg_status perm_in(pcg_matrix *A, const double *src_dev, double *dst, cudaStream_t st);
pcg_status perm_out(pcg_matrix *A, const double *src, double *dst_dev, cudaStream_t st);
pcg_status perm_in_cols(pcg_matrix *A, int k, const double *src, int64_t lds, double *dst, int64_t ldd, cudaStream_t st);
pcg_status perm_out_cols(pcg_matrix *A, int k, const double *src, int64_t lds, double *dst, int64_t ldd, cudaStream_t st);
void free_sell(pcg_matrix *A);
void free_work(pcg_matrix *A);
pcg_status launch_spmv(pcg_matrix *A, const double *x, double *y, cudaStream_t st);
pcg_status halo_exchange(pcg_matrix *A, double *vec, int width, cudaStream_t st);
pcg_status allreduce_sum(pcg_matrix *A, double *buf, int count, cudaStream_t st);
bool comm_uses_graphs(const pcg_comm *c);
bool is_device_ptr(const void *p);
}  // namespace pcgb
