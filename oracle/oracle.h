/* oracle.h — plain, slow, obviously-correct fp64 CPU oracle for the
 * Jacobi-PCG hot path (arxiv 2201.05413, north_star in BASELINE.json).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA product under
 * paper_2201_05413_b200/ and include/; neither side includes the other.
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n; "S:n" = SPEC.md line n;
 * "§8(c).k" = SURVEY.md §8(c) step k (the readings listed in DESIGN.md §3).
 */
#ifndef ORACLE_H
#define ORACLE_H
#include <stdint.h>

#define ORC_OK 0
#define ORC_NOT_CONVERGED 1
#define ORC_ERR_INVALID_ARG 2
#define ORC_ERR_ZERO_DIAGONAL 3
#define ORC_ERR_NOT_SPD 4
#define ORC_ERR_POLICY 5 /* a policy-dropped entry was not exactly 0.0 */
#define ORC_ERR_OOM 6
#define ORC_ERR_INDEX 7  /* an index outside its dimension (coo_to_csr)     */

/* element families (§8(c).1) */
#define ORC_P1_TRI 1  /* 2D lattice, "/" split, 3 nodes per element      */
#define ORC_P1_TET 2  /* 3D lattice, Kuhn split, 4 nodes per element     */
#define ORC_P2_TRI 3  /* 2D P2 on the "/" split, 6 DOFs per element      */

/* load functions f of -Δu = f (§8(c).4, BASELINE.json configs) */
#define ORC_F_ZERO 0
#define ORC_F_CONST 1   /* f = fparam[0]                                  */
#define ORC_F_SIN2D 2   /* f = 2π² sin πx sin πy                          */
#define ORC_F_SIN3D 3   /* f = 3π² sin πx sin πy sin πz                   */
#define ORC_F_BUMP3D 4  /* f = exp(-|x-c|²/(2σ²)), fparam = {cx,cy,cz,σ}  */
#define ORC_F_LINEAR 5  /* f = p0 + p1 x + p2 y + p3 z, fparam = {p0..p3} */

/* pattern policies (§8(c).6) */
#define ORC_PAT_ELEMENT 0 /* element graph, explicit zeros stored          */
#define ORC_PAT_AXIS 1    /* lattice axis neighbours only; dropped == 0.0  */

typedef struct {
  int dim;           /* 2 or 3 */
  int family;        /* ORC_P1_TRI / ORC_P1_TET / ORC_P2_TRI */
  int c;             /* cells per axis */
  int64_t n_nodes;   /* DOF count (all, incl. boundary) */
  int64_t n_elem;
  int npe;           /* DOFs per element */
  double *coord;     /* n_nodes*dim */
  int32_t *elem;     /* n_elem*npe */
  uint8_t *boundary; /* n_nodes: 1 if on ∂Ω */
  int64_t n_reset;   /* jitter repair: nodes reset to the lattice */
} orc_mesh;

typedef struct {
  int64_t n, nnz;
  int64_t *row_ptr; /* n+1 */
  int64_t *col;     /* nnz */
  double *val;      /* nnz */
} orc_csr;

/* SplitMix64 output number idx of stream `seed` (§8(c).2):
 * mix(seed + (idx+1)*0x9E3779B97F4A7C15). */
uint64_t orc_splitmix64(uint64_t seed, uint64_t idx);
/* top 53 bits × 2^-53, in [0,1) */
double orc_uniform(uint64_t seed, uint64_t idx);

int orc_mesh_build(int family, int c, int jitter, uint64_t seed, orc_mesh *m);
void orc_mesh_free(orc_mesh *m);

/* element matrices: coords of the element's nodes (npe*dim), Ke npe*npe */
int orc_elem_stiffness(int family, const double *xe, double *Ke);
/* element load: fe[a] += Σ_q w_q f(x_q) φ_a(x_q) */
int orc_elem_load(int family, const double *xe, int fkind, const double *fparam, double *fe);

/* Neumann stiffness (element-graph pattern, before BCs) and load F */
int orc_assemble(const orc_mesh *m, int fkind, const double *fparam, orc_csr *K, double *F);
/* load vector F only */
int orc_assemble_load(const orc_mesh *m, int fkind, const double *fparam, double *F);
/* Dirichlet elimination + pattern policy:  K_FF, b_F = F_F - K_FB g_B.
 * g: n_nodes values (only boundary entries are read). */
int orc_dirichlet(const orc_mesh *m, const orc_csr *K, const double *F, const double *g,
                  int policy, orc_csr *Kff, double *bF /* n_free */, int64_t *free_of_node);
void orc_csr_free(orc_csr *A);

/* y = A x  (left-to-right within a row) */
void orc_spmv(const orc_csr *A, const double *x, double *y);
/* a.b to (almost) exact rounding (Dot2, Ogita-Rump-Oishi 2005); reading R1 */
double orc_dot(int64_t n, const double *a, const double *b);

/* Jacobi-PCG, §8(c).8.  x in/out.  alpha_hist/beta_hist may be NULL. */
int orc_pcg(const orc_csr *A, const double *b, double *x, double tol, int64_t max_iter,
            int64_t *iters, double *relres_rec, double *relres_true,
            double *alpha_hist, double *beta_hist, int64_t hist_len);

/* orc_pcg plus the residual-replacement record: *replacements = number of failed
 * exit checks (each restarts the loop from the current x, §8(c).8); x_first (n
 * values) and *k_first = the iterate and iteration count at the first one (k_first
 * = -1 if none).  Any of the three may be NULL. */
int orc_pcg_ex(const orc_csr *A, const double *b, double *x, double tol, int64_t max_iter,
               int64_t *iters, double *relres_rec, double *relres_true,
               double *alpha_hist, double *beta_hist, int64_t hist_len,
               int64_t *replacements, double *x_first, int64_t *k_first);

/* §8(c).3-6 for the lattice P1 configs only (C1, C4, C5: family P1_TRI / P1_TET
 * without jitter, homogeneous Dirichlet data g = 0, AXIS pattern policy), without
 * the Neumann K: K_FF and b_F = F_F are accumulated element by element in the
 * order of orc_assemble (elements ascending, local (a,b) ascending), so every
 * entry receives the same additions in the same order as orc_assemble followed by
 * orc_dirichlet(ORC_PAT_AXIS) and is bitwise equal to it (pinned in tests).  Row i
 * of K_FF holds the free axis neighbours of node i and i itself, ascending.  An
 * element coupling between two free non-axis nodes must be exactly 0.0
 * (ORC_ERR_POLICY otherwise: per element, which implies orc_dirichlet's check on
 * the sum).  Memory: the mesh + K_FF + one n_nodes load vector (the C5 system at
 * c = 512 in ~35 GB instead of the Neumann K's ~75 GB). */
int orc_assemble_free_lattice(const orc_mesh *m, int fkind, const double *fparam, orc_csr *Kff, double *bF);

/* row partition, §8(c).10: bounds[0..G] */
void orc_partition(int64_t n, const int64_t *row_ptr, int G, int64_t *bounds);
/* halo list of rows [r0,r1): sorted unique remote columns; returns count,
 * writes at most cap entries to out (out may be NULL to count) */
int64_t orc_halo(const orc_csr *A, int64_t r0, int64_t r1, int64_t *out, int64_t cap);

/* Table 1 FD identity-boundary-row convention: nnz for N^3 nodes */
int64_t orc_fd_identity_rows_nnz(int64_t N);

/* the Table 1 system as a problem (Laplace, Dirichlet u = f on the
 * boundary, identity boundary rows; nonsymmetric) and preconditioned BiCGSTAB */
#define ORC_FD_X2MY2 1  /* f = x^2 - y^2 (discrete solution == f exactly) */
#define ORC_FD_EXPSIN 2 /* f = exp(pi x) sin(pi y)                        */
/* BiCGSTAB shadow residual r^_i = 2 u(seed, i) - 1, u = orc_uniform (reading R2) */
#define ORC_BICG_SEED 5413ULL
int orc_fd_cube(int64_t N, int fkind, orc_csr *A, double *b /* N^3 */);
int orc_bicgstab(const orc_csr *A, const double *b, double *x, double tol, int64_t max_iter, int64_t bs,
                 int64_t *iters, double *relres_rec, double *relres_true);
/* the same BiCGSTAB with the preconditioner chosen by pc: ORC_PC_BJ_LU (Block-Jacobi,
 * dense LU blocks of bs rows; bs = 1 point Jacobi — orc_bicgstab) or ORC_PC_BJ_ILU0
 * (Block-Jacobi with ILU(0) blocks of bs consecutive rows, PETSc's default sub-solver,
 * DESIGN.md reading R6; bs = n: one block, the paper's one-process run) */
#define ORC_PC_BJ_LU 0
#define ORC_PC_BJ_ILU0 1
int orc_bicgstab_pc(const orc_csr *A, const double *b, double *x, double tol, int64_t max_iter, int pc, int64_t bs,
                    int64_t *iters, double *relres_rec, double *relres_true);
/* ILU(0) of the Block-Jacobi blocks (bs rows each), Saad Alg. 10.4: the factor values in
 * A's pattern (f: nnz; L strictly lower with unit diagonal, U upper; entries whose column
 * lies outside the row's block are copied unchanged); and y = M^{-1} v. */
int orc_ilu0_factor(const orc_csr *A, int64_t bs, double *f);
int orc_ilu0_apply(const orc_csr *A, int64_t bs, const double *v, double *y);

/* SURVEY §8(f) N3 (reading R4): preconditioned pipelined CG (Ghysels &
 * Vanroose 2014, "Hiding global synchronization latency in the preconditioned
 * Conjugate Gradient algorithm", Alg. 3) with the Jacobi preconditioner: one
 * reduction phase (r.u, w.u, r.r) per iteration, the SpMV on m = M^-1 w overlapping
 * it.  Same stopping rule, exit check and replacement as orc_pcg (§8(c).8). */
int orc_pcg_pipelined(const orc_csr *A, const double *b, double *x, double tol, int64_t max_iter, int64_t *iters,
                      double *relres_rec, double *relres_true);

/* SURVEY §8(f) N1 / SPEC coo_to_csr: COO triplets -> CSR.  Entries ordered
 * by (row, col); the values of equal (row, col) entries are summed left to right in
 * INPUT order starting from 0.0, i.e. A[r][c] = sum over the entries (r, c, v) in order
 * (SPEC: "duplicates summed").  Caller-owned outputs: row_ptr[n_rows+1], col_out[nnz],
 * val_out[nnz]; *nnz_out = unique entries.  ORC_ERR_INDEX if an index is out of range. */
int orc_coo_to_csr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t *row, const int64_t *col,
                   const double *val, int64_t *row_ptr, int64_t *col_out, double *val_out, int64_t *nnz_out);

/* SURVEY §8(f) N3 (reading R5): block conjugate gradients (O'Leary 1980, "The block
 * conjugate gradient algorithm and related methods", Lin. Alg. Appl. 29) with the
 * Jacobi M: the k right-hand sides share one Krylov space.  B, X column-major n x k
 * (ld = n), X in/out.  Columns with b_j = 0 get x_j = 0 and are left out.  With
 * the m remaining columns as n x m blocks:
 *   R = B - A X; Z = M^-1 R; P = Z; Gam = R^T Z
 *   loop: Q = A P; G = P^T Q; alpha = G^-1 Gam; X += P alpha; R -= Q alpha;
 *         stop test (every column: ||r_j|| <= tol ||b_j||, then the true residuals
 *         decide; replacement = restart from X otherwise);
 *         Z = M^-1 R; Gam' = R^T Z; beta = Gam^-1 Gam'; P = Z + P beta; Gam = Gam'.
 * k x k systems by Cholesky; a non-positive pivot is ORC_ERR_NOT_SPD (breakdown).
 * *iters = number of block products A P.  relres_true[k] per column. */
int orc_block_cg(const orc_csr *A, int k, const double *B, double *X, double tol, int64_t max_iter, int64_t *iters,
                 double *relres_true);

/* reverse Cuthill-McKee ordering of the graph of a symmetric
 * pattern (edges = off-diagonal entries; explicit zeros are edges).  Plain
 * sequential algorithm (Cuthill & McKee 1969, reversed per George 1971), start
 * nodes by the George-Liu pseudo-peripheral search (1979), ties by node id:
 *   component start s = the unnumbered node of least (degree, id);
 *   r = s; repeat { x = least (degree, id) node of the last BFS level of r;
 *                   if ecc(x) > ecc(r) then r = x else stop };
 *   from r, a FIFO queue: each dequeued node appends its unnumbered neighbours
 *   in increasing (degree, id);
 *   components in that order; finally the whole order is reversed.
 * perm[k] = the original index of the node placed k-th (new -> old).  The
 * pattern must be symmetric (not checked). */
int orc_rcm(int64_t n, const int64_t *row_ptr, const int64_t *col, int64_t *perm);

#endif
