/* pcg.h — C ABI of the B200-native Jacobi-preconditioned CG solver.
 *
 * What it computes (the paper's problem statement, arxiv 2201.05413):
 *   A u = b with sparse A, solved iteratively "starting
 *   from an initial guess" with a preconditioner M^{-1} (here
 *   Jacobi, M = diag(A)) until the relative residual of Eq. (relativeError)
 *   ||A x - b||_2 / ||b||_2 <= eps; several right-hand sides
 *   B = [b_1 .. b_t] (Eq. MRH-TERMS).  The exact recurrence,
 *   stopping rule and iteration count are SURVEY.md §8(c).8-9, restated in
 *   the recurrence residual fires the loop exit, the true
 *   residual decides convergence (with residual replacement if it fails).
 *
 * Conventions (all entry points):
 *   - Plain C types only.  No exceptions cross the ABI.  Every call returns a
 *     pcg_status; on error, pcg_last_error() returns a thread-local message.
 *   - Matrices are square n x n, CSR, 0-based, int64 row_ptr[n+1] and
 *     col_idx[nnz], fp64 values; columns strictly increasing within a row
 *     (SPEC.md S:28-34).  Inputs are COPIED: the caller keeps ownership.
 *   - Vectors are fp64.  Solve/SpMV pointers may be host or device memory
 *     (detected per pointer); host arrays are staged through device buffers.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Work is
 *     ordered after prior work on it; calls return when results are in place
 *     (synchronous).
 *   - Deterministic: same inputs, flags and GPU count give bitwise-identical x
 *     and iteration counts (rule-based format choice, fixed grid per device
 *     model, fixed-order block reductions).
 *   - Thread-safe for distinct matrix handles.
 */
#ifndef PCG_B200_H
#define PCG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  PCG_OK = 0,
  PCG_NOT_CONVERGED = 1,           /* max_iter reached; x holds the last iterate */
  PCG_ERR_INVALID_ARG = 2,         /* null pointer, n < 0, tol <= 0, max_iter < 1, k < 1 */
  PCG_ERR_INDEX_OUT_OF_RANGE = 3,  /* col_idx outside [0, n)                       */
  PCG_ERR_UNSORTED_OR_DUPLICATE = 4, /* columns not strictly increasing in a row   */
  PCG_ERR_DIMENSION_MISMATCH = 5,  /* row_ptr[0] != 0, row_ptr[n] != nnz, decreasing*/
  PCG_ERR_ZERO_DIAGONAL = 6,       /* a_ii missing or 0: Jacobi undefined         */
  PCG_ERR_NOT_SPD = 7,             /* a_ii < 0, or p^T A p <= 0 during CG (breakdown)     */
  PCG_ERR_NONFINITE = 8,           /* NaN/Inf in values or right-hand side         */
  PCG_ERR_OOM = 9,
  PCG_ERR_CUDA = 10,
  PCG_ERR_NCCL = 11,
  PCG_ERR_BREAKDOWN = 12           /* BiCGSTAB: rho = r^.r, r^.v or omega became 0            */
} pcg_status;

/* csr_create flags */
#define PCG_PTR_HOST 0x0   /* row_ptr/col_idx/val are host pointers   */
#define PCG_PTR_DEVICE 0x1 /* ... are device pointers                 */
#define PCG_DROP_ZEROS 0x100 /* do not store off-diagonal entries whose value is exactly 0.0 (SURVEY
                              * §8(c) Q7's C3': the products are unchanged — 0 * x added to a partial
                              * sum is exact for finite x — with fewer bytes; stats report the stored
                              * nnz).  Default: every given entry is stored (the pattern policy).   */
#define PCG_REORDER_RCM 0x200 /* one GPU: keep the system in reverse Cuthill-McKee order
                               * (csr_rcm_order) as P A P^T; b, x0 gathered and x scattered
                               * inside the calls, so the caller's numbering is unchanged.
                               * restores gather locality for a mesh
                               * numbered arbitrarily.  INVALID_ARG on a distributed handle. */
#define PCG_FMT_AUTO 0x00  /* pick the format by a deterministic rule on slice padding:
                              SELL-32 if its 32-row slices pad <= 2 %, else SELL-C-sigma
                              if sorting cuts the padding by >= 1 % to <= 25 %, else SELL-32
                              if <= 25 %, else CSR (environment PCG_FMT_TIMED=1: time 5
                              SpMVs per candidate instead; not deterministic across runs) */
#define PCG_FMT_CSR 0x10   /* force CSR (sub-warp per row)            */
#define PCG_FMT_SELL 0x20  /* force SELL-32 (slices of 32 rows)       */
#define PCG_FMT_SELL_TMA 0x30 /* force SELL-32 with TMA-staged tiles  */
#define PCG_FMT_SELL_SIGMA 0x40 /* force SELL-C-sigma: rows sorted by length inside windows of
                                   sigma rows, applied as a symmetric permutation P A P^T
                                   (vectors are permuted at the ABI boundary; one GPU only) */

/* format codes reported by pcg_matrix_stats.format */
#define PCG_FORMAT_CSR 1
#define PCG_FORMAT_SELL 2
#define PCG_FORMAT_SELL_TMA 3 /* SELL-32, matrix tiles staged in shared memory by TMA bulk copies */
#define PCG_FORMAT_SELL_SIGMA 4 /* SELL-32 of the sigma-sorted system P A P^T */

typedef struct pcg_matrix *pcg_matrix_t;
typedef struct pcg_comm *pcg_comm_t;

typedef struct {
  int64_t iterations;       /* number of products A p              */
  double relres_recurrence; /* sqrt(r.r)/||b|| of the recurrence at exit             */
  double relres_true;       /* ||b - A x|| / ||b|| at exit (Eq. relativeError)      */
  int32_t converged;        /* 1 iff relres_true <= tol                              */
  int32_t status;           /* pcg_status of this solve / column                     */
  int64_t replacements;     /* residual replacements performed                       */
  double t_solve_s;         /* device time of the solve (CUDA events), excl. staging */
  double bytes_algorithmic; /* Σ over iterations of the §8(d) per-iteration bytes    */
  double flops;             /* Σ k (2 nnz + 13 n)                     */
} pcg_info;

typedef struct {
  int64_t n, nnz;            /* local rows / local nonzeros                   */
  int32_t format;            /* PCG_FORMAT_*                                  */
  int32_t max_row_len;
  int64_t sell_entries;      /* padded SELL entries (0 if not built)          */
  double t_setup_s;          /* csr_create wall time                          */
  double device_bytes;       /* device memory held by the handle              */
  double spmv_us_csr, spmv_us_sell; /* autotune timings (0 if not measured)   */
  int64_t n_ghost;           /* distributed: halo size (0 on one GPU)         */
  int64_t row_begin, row_end, n_global;
  double spmv_us_tma;        /* autotune timing of the TMA-staged SELL kernels */
  int64_t stage_entries;     /* TMA stage size in entries (0 = unavailable)   */
  int32_t stages;            /* TMA ring depth                                */
  int32_t schedule;          /* passes per iteration: 3 (K1a,K1b,K2) or 2 (fused K1,K2) */
  double spmv_us_sigma;      /* autotune timing of SELL-C-sigma (0 if not tried) */
  int32_t sigma;             /* sorting window of SELL-C-sigma (0: natural row order) */
  int32_t reorder;           /* 1: the device system is RCM-reordered (PCG_REORDER_RCM) */
  int64_t overlap_rows;      /* distributed: rows whose SpMV overlaps the halo exchange (0: off) */
  int64_t d16_slices;        /* SELL slices whose column ids are stored as 16-bit deltas from the row
                                (10.125 instead of 12 bytes per entry; opt-in, environment
                                PCG_D16=1 at csr_create: measured no faster) — same ids, so results are
                                bitwise those of the int32 form */
  int32_t spmm_windowed;     /* multi-RHS SpMM plan: 1 = column windows staged by TMA (opt-in,
                                environment PCG_SPMM_WIN=1; built at the first pcg_solve_multi),
                                -1 = not used, 0 = not decided yet */
  int32_t short_rows;        /* 1: SELL-32 with every row <= 8 entries runs the one-chunk row
                                engine (64 registers, 4 resident blocks/SM instead of 3; same
                                entries, same sums); environment PCG_SHORT=0 at csr_create: off */
  int32_t dia_slices;        /* slices made only of such positions (one dependent round trip) */
  int64_t dia_positions;     /* one-chunk engine: (slice, position) pairs whose entries all have the
                                same col - row, read without column ids; a slice made only of such
                                positions issues its gathers with its values (one dependent round trip);
                                same columns, so the same sums; PCG_DIA=0 at csr_create: off */
  int64_t dval_slices;       /* one-round-trip slices whose 32 stored values at every position are
                                bitwise equal (a lattice stencil's interior): one value per (slice,
                                position) is read with the offsets and the value stream is skipped
                                (value sharing, as CSR-VI); same values, so the same sums;
                                PCG_DIA_VAL=0 at csr_create: off */
  int64_t pat_slices;        /* value-free slices that read their offsets and values from a table of
                                the matrix's distinct such patterns, staged in shared memory per
                                block (no per-slice metadata beyond a pattern index); PCG_DIA_PAT=0
                                at csr_create: off */
  int32_t npat;              /* distinct patterns in that table (<= 32) */
  int64_t aligned_slices;    /* value-free slices stored in the aligned form: positions = the union of
                                the rows' column offsets, a row without an entry at a position adds
                                0 * p[row + d] there (exact), so a lattice's grid-line ends need no ids
                                or values either; PCG_DIA_ALIGN=0 at csr_create: off */
} pcg_matrix_stats;

/* ---------------------------------------------------------------- setup (§8(a) a1) */
/* Validate the CSR, narrow indices to int32 (nnz must be < 2^31 per GPU),
 * upload, precompute dinv = 1/a_ii, build SELL-32 and pick the format (flags).
 * Errors: INVALID_ARG, DIMENSION_MISMATCH, INDEX_OUT_OF_RANGE,
 * UNSORTED_OR_DUPLICATE, NONFINITE, ZERO_DIAGONAL, NOT_SPD (a_ii < 0), OOM, CUDA. */
pcg_status csr_create(int64_t n, int64_t nnz, const int64_t *row_ptr, const int64_t *col_idx,
                      const double *val, int flags, void *stream, pcg_matrix_t *out);
pcg_status csr_destroy(pcg_matrix_t A);

/* reverse Cuthill-McKee order of a symmetric CSR pattern (edges =
 * off-diagonal entries, explicit zeros included), computed on the device.  The
 * order is the sequential algorithm's exactly (start per component = least
 * (degree, id) node, George-Liu pseudo-peripheral search, neighbours appended in
 * increasing (degree, id), reversed), bit-identical to the oracle's orc_rcm.
 * perm[k] = original index of the node placed k-th (n int64, caller-owned).
 * row_ptr/col_idx/perm: host, or device with PCG_PTR_DEVICE in flags.  The pattern
 * must be symmetric (not checked).  n, nnz < 2^31.  Errors: INVALID_ARG,
 * DIMENSION_MISMATCH, INDEX_OUT_OF_RANGE, OOM, CUDA.  Use: order a global matrix
 * before csr_create_dist partitions it (contiguous blocks of a banded order have
 * small halos), or pass PCG_REORDER_RCM to csr_create on one GPU. */
pcg_status csr_rcm_order(int64_t n, int64_t nnz, const int64_t *row_ptr, const int64_t *col_idx, int flags,
                         void *stream, int64_t *perm);
pcg_status pcg_matrix_get_stats(pcg_matrix_t A, pcg_matrix_stats *out);

/* y = A x (one SpMV, the paper's MatMult).  x, y: n doubles (host or device).
 * On a distributed handle: local rows, x local (owned rows), halo exchanged inside. */
pcg_status pcg_spmv(pcg_matrix_t A, const double *x, double *y, void *stream);

/* ---------------------------------------------------------------- solve (§8(a) a2-a6) */
/* Jacobi-PCG for A x = b.  x is in/out: x0 in, solution out (caller-owned).
 * b, x: n doubles, host or device.  tol > 0 (relative, Eq. relativeError),
 * max_iter >= 1.  Returns OK, NOT_CONVERGED (x = last iterate), NOT_SPD
 * (breakdown p^T A p <= 0), NONFINITE (b has NaN/Inf), or an error.
 * b = 0 gives x = 0 and 0 iterations.  info may be NULL. */
pcg_status pcg_solve(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                     void *stream, pcg_info *info);

/* k right-hand sides (§8(a) a7): column j runs the single-RHS recurrence
 * independently and freezes at its own convergence.
 * B, X column-major with leading dimensions ldb, ldx >= n; X in/out.
 * k >= 1 (k = 0 -> INVALID_ARG); k > 32 is processed in chunks of 32.
 * infos: k entries (may be NULL).  Returns the worst column status. */
pcg_status pcg_solve_multi(pcg_matrix_t A, int32_t k, const double *B, int64_t ldb, double *X,
                           int64_t ldx, double tol, int64_t max_iter, void *stream,
                           pcg_info *infos);

/* SURVEY §8(f) N3 (reading R5): block conjugate gradients (O'Leary 1980)
 * with the Jacobi M.  The k columns share one block Krylov space, so every column
 * converges in about as many steps as the fastest independent solve needs (C4: 366
 * products instead of 549-578), at the cost of two k x k Gram matrices and two k x k
 * Cholesky solves per step.  The iterates differ from pcg_solve_multi's (parity
 * against the oracle's orc_block_cg).  Arguments as pcg_solve_multi; 1 <= k <= 32
 * (one block); one-GPU handles.  Columns with b_j = 0 get x_j = 0 and leave the
 * block.  All columns stop together: each column's recurrence residual <= tol
 * ||b_j||, then the true residuals decide (restart from X otherwise).  Every info
 * carries the shared iteration count; bytes_algorithmic is the block's divided by
 * the active columns.  Returns OK, NOT_CONVERGED, NOT_SPD (a k x k Gram matrix not
 * positive definite: breakdown, e.g. linearly dependent right-hand sides), or an
 * error. */
pcg_status pcg_solve_block(pcg_matrix_t A, int32_t k, const double *B, int64_t ldb, double *X, int64_t ldx,
                           double tol, int64_t max_iter, void *stream, pcg_info *infos);

/* ---------------------------------------------------------------- BiCGSTAB (§8(f) N2) */
/* Right-preconditioned BiCGSTAB (van der Vorst 1992) — the Krylov solver the paper
 * selects — with Block-Jacobi M: block_size = 1 is point
 * Jacobi; 2, 4, 8 use the exact inverses of the diagonal blocks of block_size
 * consecutive rows (reading R2).  For nonsymmetric A (the paper's
 * identity-row grids, Table 1) as well as SPD.  Stops when the
 * recurrence residual (or the half-step residual) satisfies ||.|| <= tol ||b||;
 * the true residual (Eq. relativeError) then decides, restarting from
 * x if needed.  The shadow residual is the fixed vector 2u(5413, i) - 1 (SplitMix64
 * u; i = original row).  b, x: n doubles, host or device; x in/out.  Returns OK,
 * NOT_CONVERGED, BREAKDOWN, NONFINITE, ZERO_DIAGONAL (singular block) or an error.
 * Blocks are consecutive rows of the caller's numbering on every device format
 * (SELL-C-sigma handles map them through their permutation).  Distributed handles
 * (csr_create_dist): collective call from every rank with its rows of b and x,
 * block_size 1 only (INVALID_ARG otherwise); the shadow residual uses global row ids,
 * so the iterates are those of the undivided system up to reduction order. */
pcg_status pcg_bicgstab(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                        int32_t block_size, void *stream, pcg_info *info);

/* The same BiCGSTAB with Block-Jacobi ILU(0) blocks — PETSc's default Block-Jacobi
 * sub-solver, the preconditioner of the paper's iterative runs (DESIGN.md
 * reading R6): blocks of block_rows consecutive rows (block_rows <= 0: one block per
 * SM, ceil(n / SMs) rows — PETSc's one block per process; block_rows >= n: one block,
 * the paper's one-process setting); in each block the incomplete LU with zero fill
 * (Saad, Alg. 10.4, IKJ), computed on the device at the first call (cached on the
 * handle per block_rows), applied by level-scheduled triangular solves, one CTA per
 * block.  Factor and application are bitwise the oracle's (orc_bicgstab_pc).
 * One-GPU handles in the caller's numbering (CSR or natural SELL: INVALID_ARG for
 * distributed, SELL-C-sigma or RCM handles).  Returns as pcg_bicgstab; ZERO_DIAGONAL
 * for a zero pivot of the incomplete factorization. */
pcg_status pcg_bicgstab_ilu(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                            int64_t block_rows, void *stream, pcg_info *info);

/* Preconditioned pipelined CG (reading R4: Ghysels &
 * Vanroose 2014, Alg. 3) with the Jacobi preconditioner: the same problem, inputs,
 * stopping rule (recurrence residual, then the true residual of Eq. relativeError,
 * P:132-135), exit check and residual replacement as pcg_solve, but ONE reduction
 * phase per iteration (r.u, w.u, r.r) with the SpMV on m = M^-1 w independent of it —
 * the latency-reduced variant: one grid barrier per iteration on one GPU, one
 * allreduce per iteration across GPUs.  Iterates equal PCG's in exact arithmetic;
 * in floating point the iteration count may differ slightly.
 * Arguments as pcg_solve (b, x host or device; x in/out; info: iterations = SpMVs
 * on m, residuals, device time, algorithmic bytes = k (12 nnz + 4(n+1) + 160 n)).
 * Single-GPU handles: the whole solve as one cooperative kernel (one grid barrier per
 * iteration).  Distributed handles (csr_create_dist): per iteration one fused kernel,
 * ONE allreduce of three sums, one halo exchange of m, one finisher; collective call
 * from every rank, b and x are the rank's rows.
 * Errors: PCG_ERR_INVALID_ARG, PCG_NOT_CONVERGED (x holds the last iterate),
 * PCG_ERR_NOT_SPD (alpha <= 0), PCG_ERR_NONFINITE, PCG_ERR_OOM, PCG_ERR_CUDA. */
pcg_status pcg_solve_pipelined(pcg_matrix_t A, const double *b, double *x, double tol, int64_t max_iter,
                               void *stream, pcg_info *info);

/* ---------------------------------------------------------------- multi-GPU (§8(a) a8, §8(e)) */
/* Row partition rule: bounds[0] = 0, bounds[G] = n,
 * bounds[g] = lower_bound(row_ptr, floor(g*nnz/G)).  Host pointers. */
pcg_status pcg_partition_rows(int64_t n, const int64_t *row_ptr, int32_t G, int64_t *bounds);
/* NCCL bootstrap: rank 0 calls pcg_comm_unique_id (128 bytes), the caller broadcasts it
 * (e.g. torch.distributed), every rank calls pcg_comm_init. */
pcg_status pcg_comm_unique_id(void *id128);
pcg_status pcg_comm_init(int32_t rank, int32_t size, const void *id128, pcg_comm_t *out);
pcg_status pcg_comm_destroy(pcg_comm_t comm);
/* Failure detection (every host wait of a distributed call): the library polls the
 * queued work and ncclCommGetAsyncError; an asynchronous NCCL error, or no completion
 * within the communicator's timeout (default 300 s, environment PCG_COMM_TIMEOUT_S at
 * pcg_comm_init, or pcg_comm_set_timeout), aborts the communicator (ncclCommAbort)
 * and the call returns PCG_ERR_NCCL instead of blocking.  Every rank applies the same
 * rule, so a rank that dies or fails makes its peers fail within their timeout.  An
 * aborted communicator stays unusable: later calls on handles built on it return
 * PCG_ERR_NCCL; destroy the handles and the communicator and build new ones.
 * pcg_comm_abort aborts on request (e.g. from a caller's own watchdog). */
pcg_status pcg_comm_set_timeout(pcg_comm_t comm, double seconds);
pcg_status pcg_comm_abort(pcg_comm_t comm);
/* Device-initiated allreduce (opt-in, environment PCG_DEVICE_ALLREDUCE=1
 * at pcg_comm_init on EVERY rank, NCCL communicators of <= 8 ranks on one node): the
 * scalar reductions of the distributed solvers (sigma; rho', gamma; the BiCGSTAB and
 * pipelined sums) run as one single-thread kernel each that writes the rank's values
 * into every peer's mailbox over NVLink (CUDA IPC mappings made at pcg_comm_init) and
 * sums all ranks' values in rank order — the same bits on every rank — instead of an
 * ncclAllReduce.  If any rank cannot map its peers, every rank keeps NCCL.  A peer that
 * stops making progress for ~8 s makes the kernel flag an error that the next host
 * wait turns into PCG_ERR_NCCL (communicator aborted).  device_allreduce reports
 * whether it is active.  pcg_dar_emulate: the protocol's self-test on ONE GPU — G <= 8
 * "ranks" as G co-resident blocks of one cooperative kernel, each with its own mailbox,
 * `rounds` successive reductions of nv <= 4 values; in/out host arrays of
 * rounds x G x nv doubles (rank g's input / result of round r at [(r G + g) nv]). */
pcg_status pcg_comm_get_info(pcg_comm_t comm, int32_t *rank, int32_t *size, int32_t *device_allreduce);
pcg_status pcg_dar_emulate(int32_t G, int32_t rounds, int32_t nv, const double *in, double *out);

/* Host-callback communicator: the same distributed path (csr_create_dist, pcg_solve,
 * pcg_spmv) with every exchange step done by caller-supplied host functions instead of
 * NCCL; device data is staged through host memory around each call and the
 * iteration loop runs without CUDA graphs.  Meant for validating the multi-GPU code
 * path where ranks cannot each have their own GPU (e.g. several processes sharing
 * one GPU, exchanging over torch.distributed gloo) — never a performance path.
 * All buffers are HOST memory; every callback returns 0 on success.
 *   allreduce_sum_f64: in-place elementwise sum over ranks of buf[0..count)
 *   allreduce_max_i32: in-place elementwise max over ranks
 *   allgather_i64:     all[r*count + i] = rank r's mine[i]
 *   exchange:          for each listed peer p: send send_bytes[p] bytes from send[p] to
 *                      peers[p] and receive recv_bytes[p] bytes from peers[p] into recv[p]
 *                      (all pairs posted together; counts match the peer's). */
typedef struct {
  void *ctx;
  int (*allreduce_sum_f64)(void *ctx, double *buf, int64_t count);
  int (*allreduce_max_i32)(void *ctx, int32_t *buf, int64_t count);
  int (*allgather_i64)(void *ctx, const int64_t *mine, int64_t count, int64_t *all);
  int (*exchange)(void *ctx, int32_t n_peers, const int32_t *peers, const void *const *send,
                  const int64_t *send_bytes, void *const *recv, const int64_t *recv_bytes);
} pcg_comm_ops;
pcg_status pcg_comm_init_ops(int32_t rank, int32_t size, const pcg_comm_ops *ops, pcg_comm_t *out);
/* Distributed matrix: this rank owns rows [row_begin, row_end) of the global n_global x
 * n_global matrix; row_ptr_local (row_end-row_begin+1, starting at 0), global col_idx.
 * Collective over comm (halo lists are exchanged).  pcg_solve / pcg_spmv on the
 * handle then take local vectors of row_end-row_begin entries. */
pcg_status csr_create_dist(pcg_comm_t comm, int64_t n_global, int64_t row_begin, int64_t row_end,
                           int64_t nnz_local, const int64_t *row_ptr_local,
                           const int64_t *col_idx_global, const double *val, int flags,
                           void *stream, pcg_matrix_t *out);

/* Host-side halo planning (used by csr_create_dist; host pointers, no GPU needed).
 * pcg_halo_ghosts: sorted unique columns outside [row_begin, row_end) referenced by the
 *   local rows (col: nnz_local global ids).  Writes min(count, cap) ids; *n_ghost = count.
 * pcg_halo_recv_plan: for a sorted ghost list and all ranks' row bounds (G+1 entries,
 *   bounds[g]..bounds[g+1] owned by rank g), the number of ghosts owned by each rank and
 *   the offset of its run in the ghost list (ghost slots are [n_local + offset, +count)).
 *   INDEX_OUT_OF_RANGE if a ghost lies outside every rank's rows. */
pcg_status pcg_halo_ghosts(int64_t row_begin, int64_t row_end, int64_t nnz_local, const int64_t *col_idx_global,
                           int64_t *ghosts, int64_t cap, int64_t *n_ghost);
pcg_status pcg_halo_recv_plan(int64_t n_ghost, const int64_t *ghosts, int32_t G, const int64_t *bounds,
                              int64_t *recv_count, int64_t *recv_offset);

/* ---------------------------------------------------------------- diagnostics */
const char *pcg_last_error(void);
const char *pcg_status_string(pcg_status s);
/* Per-kernel timing for the roofline (bench/profiling only): runs the init pass on b
 * (device pointer, x0 = 0), then `reps` PCG iterations launched one kernel at a time
 * with CUDA events between the passes on `stream`.  us[0..2] = mean device time in
 * microseconds of: K1a (streaming p/x update, averaged over the loop's hold / apply pairs
 * when x is updated every second iteration; 0 under the fused schedule), K1b (SpMV
 * + sigma; the fused K1 under schedule 2), K2 (r/z updates + dots).
 * Single-GPU handles only; stops early (fewer reps) if the solve converges. */
pcg_status pcg_profile_kernels(pcg_matrix_t A, const double *b, int32_t reps, void *stream, double *us,
                               int32_t *reps_done);

/* Multi-RHS per-kernel timing (bench/profiling only): k columns of B (device,
 * column-major, ld >= n, 1 <= k <= 32) run the init pass (X0 = 0) and then `reps`
 * block iterations one kernel at a time.  us[0..2] = mean device time (microseconds)
 * of: K1a (streaming X += alpha P, P = Z + beta P), K1b (SpMM Q = A P with
 * per-column sigma), K2 (R/Z updates with per-column rho', gamma).
 * Single-GPU handles only. */
pcg_status pcg_profile_multi(pcg_matrix_t A, int32_t k, const double *B, int64_t ldb, int32_t reps, void *stream,
                             double *us, int32_t *reps_done);

/* number of kernels this library launched in the calling process (monotone counter,
 * for launch accounting in benchmarks) */
int64_t pcg_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* PCG_B200_H */
