/* fem_gen.h — on-device assembly of the benchmark systems K u = f (the step
 * before the solver).
 *
 * Builds, row by row on the GPU, the SPD stiffness matrix K_FF and load
 * vector(s) b_F of -Δu = f on the unit square/cube with Dirichlet data g
 * ("Laplace equation ... Dirichlet condition u=f on the
 * boundary"; FEM discretisation P:78), following the readings of
 * SURVEY.md §8(c) steps 1-7 restated in DESIGN.md §3:
 *   meshes: c cells per axis, node id lexicographic (x fastest); 2D "/" split;
 *           3D Kuhn split (6 tets per cube sharing the main diagonal); P2 on
 *           the half-lattice;  jitter (P1_TRI only): d = (2u-1)(0.3h),
 *           u = SplitMix64(seed, 2*node+axis), one-pass lattice reset of the
 *           interior vertices of non-positive-area triangles;
 *   K_e = |T| G G^T (P1), 3-point edge-midpoint rule (P2); degree-2 load rules;
 *   Dirichlet elimination, b_F = F_F - K_FB g_B; pattern policy AXIS (lattice
 *   P1: axis neighbours only; dropped entries must be exactly 0) or ELEMENT
 *   (element graph, explicit zeros stored); columns ascending.
 * Rows are numbered by free DOF (lexicographic, boundary skipped), so a row
 * range [row_begin, row_end) is exactly one rank's slab under csr_create_dist.
 *
 * All array arguments are DEVICE pointers owned by the caller.  Errors:
 * PCG_ERR_INVALID_ARG (bad spec / range / a policy-dropped entry that is not
 * exactly 0), PCG_ERR_CUDA.
 */
#ifndef FEM_GEN_B200_H
#define FEM_GEN_B200_H
#include <stdint.h>

#include "pcg.h"

#ifdef __cplusplus
extern "C" {
#endif

#define FEM_P1_TRI 1
#define FEM_P1_TET 2
#define FEM_P2_TRI 3

#define FEM_F_ZERO 0
#define FEM_F_ONE 1
#define FEM_F_SIN2D 2  /* 2π² sin πx sin πy        (u = sin πx sin πy)       */
#define FEM_F_SIN3D 3  /* 3π² sin πx sin πy sin πz (u = sin πx sin πy sin πz) */
#define FEM_F_BUMP3D 4 /* column s: exp(-|x-c_s|²/(2σ²)), c_s,axis = U(seed, 3s+axis) */

#define FEM_G_ZERO 0
#define FEM_G_X2MY2 1    /* g = x² - y² on the boundary                                   */
#define FEM_G_LINEAR3D 2 /* g = 1 + 2x - 3y + z/2 (3D; P1 reproduces it exactly: reading R3) */

#define FEM_PAT_ELEMENT 0
#define FEM_PAT_AXIS 1

typedef struct {
  int32_t family; /* FEM_P1_TRI / FEM_P1_TET / FEM_P2_TRI */
  int32_t c;      /* cells per axis, >= 2 */
  int32_t jitter; /* 0/1, FEM_P1_TRI only */
  int32_t fkind;  /* FEM_F_* */
  int32_t gkind;  /* FEM_G_* */
  int32_t policy; /* FEM_PAT_* */
  int32_t k;      /* right-hand sides: 1, or the bump count for FEM_F_BUMP3D (<= 32) */
  int32_t pad;
  uint64_t seed;  /* jitter / bump-centre stream */
  double sigma;   /* bump width */
} fem_spec;

/* n_free: rows of K_FF; nnz_total: its nonzeros (closed form); n_nodes: all DOFs */
pcg_status fem_problem_size(const fem_spec *spec, int64_t *n_free, int64_t *nnz_total, int64_t *n_nodes);

/* Two phases over rows [row_begin, row_end):
 *   phase 1 (d_col == NULL): writes d_row_ptr (row_end-row_begin+1 entries, starting at 0)
 *            and *nnz_out (host) — the caller then allocates col/val;
 *   phase 2: fills d_col (GLOBAL free-DOF column ids, int64), d_val, and d_B
 *            (k column-major columns, leading dimension ldb >= rows; may be NULL). */
pcg_status fem_assemble(const fem_spec *spec, int64_t row_begin, int64_t row_end, int64_t *d_row_ptr,
                        int64_t *d_col, double *d_val, double *d_B, int64_t ldb, void *stream);
pcg_status fem_count(const fem_spec *spec, int64_t row_begin, int64_t row_end, int64_t *d_row_ptr,
                     int64_t *nnz_out, void *stream);

/* ---------------------------------------------------------------- the paper's Table 1 systems
 * (reading R2): FD Laplace on N^3 nodes of
 * the unit cube (h = 1/(N-1)), node id i + N(j + N l); interior rows 6 / -1 x 6 (columns
 * ascending), b = 0; boundary rows identity, b = f(node).  Nonsymmetric.  nnz(N^3) =
 * 7(N-2)^3 + N^3 - (N-2)^3 (Cube 1, N = 128: 14,099,408).  Two phases over rows
 * [row_begin, row_end) like fem_count / fem_assemble; d_b (rows entries) may be NULL. */
#define FD_F_X2MY2 1  /* f = x^2 - y^2 (the discrete solution equals f) */
#define FD_F_EXPSIN 2 /* f = exp(pi x) sin(pi y)                        */
pcg_status fd_cube_count(int64_t N, int64_t row_begin, int64_t row_end, int64_t *d_row_ptr, int64_t *nnz_out,
                         void *stream);
pcg_status fd_cube_assemble(int64_t N, int32_t fkind, int64_t row_begin, int64_t row_end, const int64_t *d_row_ptr,
                            int64_t *d_col, double *d_val, double *d_b, void *stream);

/* Element-by-element assembly, step 1 (generic path): the
 * elements' stiffness matrices K_e as COO triplets over ALL lattice nodes (Neumann,
 * before Dirichlet elimination; node id lexicographic, x fastest, boundary included).
 * Elements are enumerated as the row-wise generator visits them (cells
 * lexicographic, then the split's element order); element e's triplets sit at
 * [(e - e0) * npe^2, (e - e0 + 1) * npe^2), local (a, b) row-major.  coo_to_csr of all
 * elements' triplets is the assembled Neumann stiffness (explicit zeros kept).
 *   P1: K_e = |T| G G^T (barycentric gradients G; §8(c).3);
 *   P2: K_e[a][b] = sum over the 3 edge midpoints of |T|/3 grad phi_a . grad phi_b.
 * fem_element_count: n_elem (2c^2 triangles, 6c^3 tets), npe (3 / 6 / 4), n_nodes.
 * d_row, d_col (int64) and d_val (f64): DEVICE buffers of (e1 - e0) * npe^2 entries,
 * caller-owned.  Synchronous on `stream`.  Errors: PCG_ERR_INVALID_ARG (bad spec or
 * range, null buffer), PCG_ERR_CUDA. */
pcg_status fem_element_count(const fem_spec *spec, int64_t *n_elem, int32_t *npe, int64_t *n_nodes);
pcg_status fem_element_coo(const fem_spec *spec, int64_t e0, int64_t e1, int64_t *d_row, int64_t *d_col,
                           double *d_val, void *stream);

/* Generic COO -> CSR on the device (SURVEY §8(f) N1 "generic COO -> CSR (sort +
 * segmented reduce)"; SPEC coo_to_csr: "duplicates summed; CSR invariants
 * hold", IndexOutOfRange), the staging step of element-by-element assembly.
 * Output entries are ordered by (row, col), columns strictly increasing within a
 * row.  The values of the entries that share a (row, col) are summed left to right
 * in INPUT order starting from 0.0 (a stable radix sort keeps that order), so the
 * result is bitwise the dense accumulation A[row][col] += val over the entries in
 * order; a group that sums to 0.0 stays an explicit entry.
 *   row[nnz], col[nnz] (int64), val[nnz] (f64): DEVICE pointers, read only, caller-owned.
 *   row_ptr[n_rows + 1] (int64), col_out[nnz] (int64), val_out[nnz] (f64): DEVICE buffers,
 *   caller-owned (nnz entries always suffice); *nnz_out (HOST) = number of unique entries.
 * Sizes: 0 <= n_rows, n_cols < 2^31, 0 <= nnz < 2^31.  Scratch (~44 B per entry) is
 * allocated and freed inside; returns when the result is complete (synchronous on
 * `stream`).  Errors: PCG_ERR_INVALID_ARG (null pointer, sizes out of range; outputs
 * untouched), PCG_ERR_INDEX_OUT_OF_RANGE (an index outside [0, n_rows) x [0, n_cols);
 * outputs unspecified), PCG_ERR_OOM, PCG_ERR_CUDA.
 * Example: (0,0,1), (0,0,3), (1,1,2) in 2 x 2 -> row_ptr {0,1,2}, col {0,1}, val {4,2}. */
pcg_status coo_to_csr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t *row, const int64_t *col,
                      const double *val, int64_t *row_ptr, int64_t *col_out, double *val_out, int64_t *nnz_out,
                      void *stream);

#ifdef __cplusplus
}
#endif
#endif
