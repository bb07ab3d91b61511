"""Pins of the oracle's ILU(0) Block-Jacobi preconditioner (DESIGN.md
reading R6): PETSc's default Block-Jacobi sub-solver, Saad Alg. 10.4.

What fixes it independently of oracle.c:
  * the defining property of ILU(0): (L U)_ij = a_ij for every (i, j) in the pattern of
    the block (L unit lower, U upper, both in A's pattern), checked with dense products;
  * no fill is needed for a tridiagonal (1D) block or a dense block, so there ILU(0) is
    the exact LU and M = A: BiCGSTAB converges in one step;
  * the application y = (L U)^{-1} v solves M y = v (dense solve of the factors);
  * block structure: blocks are independent (a block-diagonal matrix is solved exactly
    block by block, and entries coupling blocks are ignored by M);
  * the paper's reference point: BiCGSTAB + Block-Jacobi/ILU(0) on Cube 1 (128^3
    nodes) in one process takes 128 iterations; the oracle's count on the same
    Table 1 grids grows linearly with N (the h^-1 conditioning of ILU(0)-preconditioned
    Laplacians) and extrapolates to within 15 % of it.
"""
import numpy as np
import pytest

import oracle as O


def _csr(D):
    n = D.shape[0]
    rp, cols, vals = [0], [], []
    for i in range(n):
        nz = np.nonzero(D[i])[0]
        cols += list(nz)
        vals += list(D[i, nz])
        rp.append(len(cols))
    return O.Csr(n, rp, cols, vals)


def _factors(A, f, bs):
    """dense L (unit lower) and U of the block-diagonal part, from the factor values"""
    n = A.n
    L, U = np.eye(n), np.zeros((n, n))
    for i in range(n):
        r0 = (i // bs) * bs
        r1 = min(r0 + bs, n)
        for e in range(A.row_ptr[i], A.row_ptr[i + 1]):
            j = A.col[e]
            if j < r0 or j >= r1:
                continue
            if j < i:
                L[i, j] = f[e]
            else:
                U[i, j] = f[e]
    return L, U


def _blockdiag(A, bs):
    D = A.to_dense()
    n = A.n
    B = np.zeros_like(D)
    for r0 in range(0, n, bs):
        r1 = min(r0 + bs, n)
        B[r0:r1, r0:r1] = D[r0:r1, r0:r1]
    return B


def _random_sparse(n, density, seed, sym=False):
    rng = np.random.default_rng(seed)
    D = rng.standard_normal((n, n)) * (rng.random((n, n)) < density)
    if sym:
        D = D + D.T
    D += np.diag(np.abs(D).sum(1) + 1.0)
    return D


@pytest.mark.parametrize("case,bs", [("fd6", 216), ("fd6", 36), ("fd6", 50), ("c1", 225), ("c1", 40),
                                     ("rand", 80), ("rand", 17), ("randsym", 33)])
def test_ilu0_lu_equals_a_on_the_pattern(case, bs):
    if case == "fd6":
        A, _ = O.fd_cube(6, O.FD_EXPSIN)
    elif case == "c1":
        A = O.build_problem("C1", c=16)["A"]
    else:
        A = _csr(_random_sparse(80, 0.08, 3, sym=case == "randsym"))
    f = O.ilu0_factor(A, bs)
    L, U = _factors(A, f, bs)
    LU = L @ U
    B = _blockdiag(A, bs)
    scale = np.abs(B).max()
    for i in range(A.n):
        r0 = (i // bs) * bs
        r1 = min(r0 + bs, A.n)
        for e in range(A.row_ptr[i], A.row_ptr[i + 1]):
            j = A.col[e]
            if r0 <= j < r1:
                assert abs(LU[i, j] - B[i, j]) <= 1e-12 * scale, (i, j)
    # and the product has fill only outside the pattern (else ILU(0) would be exact LU)
    assert np.all(np.tril(L, -1)[B == 0] == 0) and np.all(np.triu(U)[B == 0] == 0)


def test_ilu0_is_exact_lu_without_fill():
    """Tridiagonal block (1D Laplacian) and a dense block: no fill, ILU(0) = LU, M = A,
    BiCGSTAB in one step; the factors reproduce A exactly (to rounding) everywhere."""
    n = 40
    T = np.diag(np.full(n, 2.0)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1)
    D = _random_sparse(30, 1.0, 9)  # dense, diagonally dominant
    for M in (T, D):
        A = _csr(M)
        L, U = _factors(A, O.ilu0_factor(A, A.n), A.n)
        assert np.allclose(L @ U, M, rtol=0, atol=1e-12 * np.abs(M).max())
        b = np.random.default_rng(1).standard_normal(A.n)
        r = O.bicgstab_ilu(A, b, tol=1e-12)
        assert r.status == O.OK and r.iterations == 1
        assert np.allclose(r.x, np.linalg.solve(M, b), rtol=0, atol=1e-10)


@pytest.mark.parametrize("bs", [216, 36, 50, 1])
def test_ilu0_apply_solves_the_factors(bs):
    A, _ = O.fd_cube(6, O.FD_EXPSIN)
    v = np.random.default_rng(5).standard_normal(A.n)
    y = O.ilu0_apply(A, bs, v)
    L, U = _factors(A, O.ilu0_factor(A, bs), bs)
    assert np.allclose(L @ (U @ y), v, rtol=0, atol=1e-12 * np.abs(v).max())
    if bs == 1:  # 1 x 1 blocks: point Jacobi
        d = np.array([A.to_dense()[i, i] for i in range(A.n)])
        assert np.array_equal(y, v / d)


def test_ilu0_block_diagonal_matrix_is_solved_exactly():
    """A matrix that IS block diagonal with tridiagonal blocks: M = A exactly."""
    nb, m = 4, 25
    T = np.diag(np.full(m, 3.0)) - np.diag(np.ones(m - 1), 1) - np.diag(np.full(m - 1, 0.5), -1)
    M = np.kron(np.eye(nb), T)
    A = _csr(M)
    b = np.arange(1.0, nb * m + 1)
    r = O.bicgstab_ilu(A, b, tol=1e-13, block=m)
    assert r.status == O.OK and r.iterations == 1
    assert np.allclose(r.x, np.linalg.solve(M, b), rtol=0, atol=1e-11)


def test_bicgstab_ilu_reproduces_the_harmonic_quadratic():
    """The Table 1 system with boundary data x^2 - y^2 (reading R2): exact discrete solution."""
    N = 14
    A, b = O.fd_cube(N)
    h = 1.0 / (N - 1)
    i = np.arange(N)
    X, Y = np.tile(i, N * N) * h, np.tile(np.repeat(i, N), N) * h
    for bs in (A.n, N * N, 100):
        r = O.bicgstab_ilu(A, b, tol=1e-13, block=bs)
        assert r.status == O.OK and r.relres_true <= 1e-13
        assert np.max(np.abs(r.x - (X * X - Y * Y))) <= 1e-11


def test_bicgstab_ilu_iterations_against_the_paper():
    """BiCGSTAB + Block-Jacobi (one block per process, ILU(0)) on Cube 1, one
    process, eps = 1e-12: 128 iterations.  The oracle's one-block counts on the Table 1
    grids grow linearly in N; their fit extrapolates to Cube 1 (N = 128) within 15 %.
    ILU(0) must also beat point Jacobi by > 2.5x (the paper: Block-Jacobi roughly halves
    the iterations of the unpreconditioned solver)."""
    Ns = [16, 24, 32, 40]
    its = []
    for N in Ns:
        A, b = O.fd_cube(N)
        r = O.bicgstab_ilu(A, b, tol=1e-12)
        assert r.status == O.OK
        its.append(r.iterations)
        if N == 32:
            assert O.bicgstab(A, b, tol=1e-12).iterations > 2.5 * r.iterations
    slope, icpt = np.polyfit(Ns, its, 1)
    est = slope * 128 + icpt
    assert abs(est - 128) <= 0.15 * 128, (its, est)


def test_bicgstab_ilu_status_and_zero_pivot():
    A, b = O.fd_cube(8, O.FD_EXPSIN)
    r = O.bicgstab_ilu(A, b, tol=1e-14, max_iter=2)
    assert r.status == O.NOT_CONVERGED and r.iterations == 2
    r = O.bicgstab_ilu(A, np.zeros(A.n))
    assert r.status == O.OK and r.iterations == 0
    Z = O.Csr(2, [0, 2, 4], [0, 1, 0, 1], [0.0, 1.0, 1.0, 2.0])
    r = O.bicgstab_ilu(Z, np.ones(2))
    assert r.status == O.ERR_ZERO_DIAGONAL
