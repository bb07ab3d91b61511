"""Pins of the oracle against what the paper and mathematics fix (CPU only).

Each test names the fact it pins.  None re-types an oracle formula: the
references are printed values (tests/golden/, cited), closed forms, textbook
matrices, exact library solves (DST-I, dense Cholesky), invariants and brute
force on tiny inputs.  P:n = /root/reference/PAPER.md line n; S:n = SPEC.md.
"""
import math
import os

import numpy as np
import pytest

import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------- PRNG
def test_splitmix64_reference_sequence():
    want = [int(r[0], 16) for r in _golden_rows("splitmix64_seed0.txt")]
    got = [O.splitmix64(0, i) for i in range(len(want))]
    assert got == want


def test_uniform_range_and_mean():
    u = np.array([O.uniform(7, i) for i in range(20000)])
    assert u.min() >= 0.0 and u.max() < 1.0
    assert abs(u.mean() - 0.5) < 0.01


# ---------------------------------------------------------------- structure
def test_table1_nonzeros_paper():
    """PAPER Table 1 nnz under the identity-boundary-row FD convention."""
    for N, rows, nnz in _golden_rows("table1_nnz.txt"):
        assert int(N) ** 3 == int(rows)
        assert O.fd_identity_rows_nnz(int(N)) == int(nnz)


def test_kuhn_p1_is_h_times_fd_stencil():
    """Kuhn P1 stiffness on the lattice == h * 7-point FD Laplacian (P:78 'w(i,j)=1')."""
    c = 8
    h = 1.0 / c
    P = O.build_problem("C5", c=c)
    A = P["A"].to_dense() / h
    m = c - 1
    n = m ** 3
    L = np.zeros((n, n))
    for l in range(m):
        for j in range(m):
            for i in range(m):
                r = i + m * (j + m * l)
                L[r, r] = 6.0
                for di, dj, dl in [(1, 0, 0), (-1, 0, 0), (0, 1, 0), (0, -1, 0), (0, 0, 1), (0, 0, -1)]:
                    a, b, cc = i + di, j + dj, l + dl
                    if 0 <= a < m and 0 <= b < m and 0 <= cc < m:
                        L[r, a + m * (b + m * cc)] = -1.0
    assert np.max(np.abs(A - L)) < 1e-13


def test_p1_lattice_2d_is_5point_stencil():
    c = 8
    A = O.build_problem("C1", c=c)["A"].to_dense()
    m = c - 1
    L = 4 * np.eye(m * m)
    for j in range(m):
        for i in range(m):
            r = i + m * j
            if i + 1 < m:
                L[r, r + 1] = L[r + 1, r] = -1
            if j + 1 < m:
                L[r, r + m] = L[r + m, r] = -1
    assert np.max(np.abs(A - L)) < 1e-14


@pytest.mark.parametrize("name,c", [("C1", 16), ("C1", 64), ("C2", 16), ("C2", 33), ("C3", 8),
                                    ("C3", 32), ("C4", 8), ("C4", 13), ("C5", 16)])
def test_config_sizes_closed_forms(name, c):
    """n and nnz closed forms of §8(c).7 (C1: 5m²-4m, C2: 7m²-8m+2, C3: 46c²-96c+53,
    C4/C5: 7m³-6m²)."""
    P = O.build_problem(name, c=c, k=1)
    A = P["A"]
    m = c - 1
    want = {"C1": (m * m, 5 * m * m - 4 * m), "C2": (m * m, 7 * m * m - 8 * m + 2),
            "C3": ((2 * c - 1) ** 2, 46 * c * c - 96 * c + 53),
            "C4": (m ** 3, 7 * m ** 3 - 6 * m * m), "C5": (m ** 3, 7 * m ** 3 - 6 * m * m)}[name]
    assert (A.n, A.nnz) == want
    # CSR invariants: monotone row_ptr, strictly increasing columns, diag present
    assert A.row_ptr[0] == 0 and np.all(np.diff(A.row_ptr) >= 1)
    for i in range(A.n):
        cols = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
        assert np.all(np.diff(cols) > 0) and i in cols


# ---------------------------------------------------------------- element matrices
def test_p1_right_triangle_textbook():
    """Right angle at vertex 0: K_e = [[1,-1/2,-1/2],[-1/2,1/2,0],[-1/2,0,1/2]] (h-free)."""
    h = 0.125
    K = O.elem_stiffness(O.P1_TRI, [0, 0, h, 0, 0, h])
    want = np.array([[1, -.5, -.5], [-.5, .5, 0], [-.5, 0, .5]])
    assert np.max(np.abs(K - want)) < 1e-15


def test_p1_cot_formula_2d():
    """K_ij = -1/2 cot(θ_k), θ_k the angle opposite edge ij (the 2D form of P:78's w)."""
    rng = np.random.default_rng(1)
    for _ in range(50):
        x = rng.random((3, 2))
        K = O.elem_stiffness(O.P1_TRI, x.ravel())
        for i, j, k in [(0, 1, 2), (1, 2, 0), (0, 2, 1)]:
            u, v = x[i] - x[k], x[j] - x[k]
            cosang = u @ v / (np.linalg.norm(u) * np.linalg.norm(v))
            ang = math.acos(np.clip(cosang, -1, 1))
            assert abs(K[i, j] - (-0.5 / math.tan(ang))) < 1e-10 * max(1, abs(K[i, j]))


def test_p1_cot_formula_3d_paper():
    """w(i,j) = 1/6 Σ_k l_k cot α_k: per tet, K_ij = -(1/6) l_kl cot α_kl with l_kl the
    length of the edge opposite ij and α_kl the dihedral angle at that edge."""
    rng = np.random.default_rng(2)
    for _ in range(50):
        x = rng.random((4, 3))
        K = O.elem_stiffness(O.P1_TET, x.ravel())
        for i in range(4):
            for j in range(i + 1, 4):
                k, l = [t for t in range(4) if t not in (i, j)]
                e = x[l] - x[k]
                # dihedral angle at edge kl between faces (k,l,i) and (k,l,j)
                def perp(p):
                    d = x[p] - x[k]
                    return d - (d @ e) / (e @ e) * e
                a, b = perp(i), perp(j)
                cosang = a @ b / (np.linalg.norm(a) * np.linalg.norm(b))
                ang = math.acos(np.clip(cosang, -1, 1))
                w = np.linalg.norm(e) / 6.0 / math.tan(ang)
                assert abs(K[i, j] + w) < 1e-9 * max(1, abs(w))


def test_p2_reference_triangle_textbook():
    want = np.array(_golden_rows("p2_reference_stiffness.txt"), dtype=float) / 6.0
    K = O.elem_stiffness(O.P2_TRI, [0, 0, 1, 0, 0, 1, .5, 0, .5, .5, 0, .5])
    assert np.max(np.abs(K - want)) < 1e-14


@pytest.mark.parametrize("fam", [O.P1_TRI, O.P2_TRI, O.P1_TET])
def test_element_rowsum_symmetry(fam):
    rng = np.random.default_rng(3)
    for _ in range(20):
        if fam == O.P1_TET:
            x = rng.random((4, 3))
        else:
            v = rng.random((3, 2))
            x = v if fam == O.P1_TRI else np.vstack([v, (v[0] + v[1]) / 2, (v[1] + v[2]) / 2,
                                                     (v[0] + v[2]) / 2])
        K = O.elem_stiffness(fam, x.ravel())
        assert np.array_equal(K, K.T)
        assert np.max(np.abs(K.sum(1))) < 1e-12 * np.max(np.abs(K))


@pytest.mark.parametrize("name,c", [("C1", 16), ("C2", 32), ("C3", 16), ("C5", 8)])
def test_neumann_stiffness_symmetric_zero_rowsum(name, c):
    """north_star: 'the stiffness matrix is symmetric with zero row sums before BCs'."""
    cfg = O.configs()[name]
    mesh = O.Mesh(O.FAMILY[cfg["family"]], c, cfg["jitter"], cfg["seed"])
    K, _ = O.assemble(mesh, O.F_ZERO)
    S = K.to_scipy()
    assert (S - S.T).nnz == 0 or np.max(np.abs((S - S.T).data)) == 0.0
    rs = np.asarray(S.sum(axis=1)).ravel()
    assert np.max(np.abs(rs)) <= 1e-15 * 8 * np.max(np.abs(S.diagonal()))


# ---------------------------------------------------------------- load vectors
@pytest.mark.parametrize("name,c,vol", [("C1", 16, 2), ("C5", 8, 3)])
def test_load_constant_and_linear_exact(name, c, vol):
    """Degree-2 rules integrate f·φ_i exactly for linear f; the lattice patch of an interior
    node is point-symmetric, so F_i = f(x_i)·h^d (∫φ_i = h^d)."""
    cfg = O.configs()[name]
    mesh = O.Mesh(O.FAMILY[cfg["family"]], c)
    h = 1.0 / c
    coef = (0.7, 1.3, -2.1, 0.4)
    F = O.assemble_load(mesh, O.F_LINEAR, coef)
    X = mesh.coord
    f = coef[0] + coef[1] * X[:, 0] + coef[2] * X[:, 1] + (coef[3] * X[:, 2] if vol == 3 else 0)
    inner = ~mesh.boundary
    assert np.max(np.abs(F[inner] - f[inner] * h ** vol)) < 1e-14
    F1 = O.assemble_load(mesh, O.F_CONST, (1.0,))
    assert np.max(np.abs(F1[inner] - h ** vol)) < 1e-16


def test_load_p2_constant_exact():
    """P2, f = 1: ∫φ_vertex = 0, ∫φ_midpoint = |T|/3 per triangle (exact integrals)."""
    c = 8
    h = 1.0 / c
    mesh = O.Mesh(O.P2_TRI, c)
    F = O.assemble_load(mesh, O.F_CONST, (1.0,))
    np_ = 2 * c + 1
    for idx in np.nonzero(~mesh.boundary)[0]:
        a, b = idx % np_, idx // np_
        if a % 2 == 0 and b % 2 == 0:
            assert abs(F[idx]) < 1e-17
        else:
            assert abs(F[idx] - 2 * (h * h / 2) / 3) < 1e-16


# ---------------------------------------------------------------- exact discrete solves
def _dst_solve(b, m, dim, h):
    from scipy.fft import dstn, idstn
    j = np.arange(1, m + 1)
    lam1 = 2 - 2 * np.cos(j * np.pi / (m + 1))
    if dim == 2:
        lam = lam1[None, :] + lam1[:, None]
        B = b.reshape(m, m)
    else:
        lam = h * (lam1[None, None, :] + lam1[None, :, None] + lam1[:, None, None])
        B = b.reshape(m, m, m)
    return idstn(dstn(B, type=1) / lam, type=1).ravel()


@pytest.mark.parametrize("name,c", [("C1", 64), ("C5", 32), ("C4", 16)])
def test_pcg_matches_dst_exact_solution(name, c):
    """Lattice K_FF is diagonalised by DST-I (closed-form spectrum); PCG to 1e-13 must
    match the exact discrete solution."""
    P = O.build_problem(name, c=c, k=2)
    dim = 2 if name == "C1" else 3
    for col in range(P["B"].shape[1]):
        b = P["B"][:, col]
        r = O.pcg(P["A"], b, tol=1e-13)
        assert r.status == O.OK
        xe = _dst_solve(b, c - 1, dim, 1.0 / c)
        assert np.linalg.norm(r.x - xe) / np.linalg.norm(xe) < 1e-11


@pytest.mark.parametrize("name,c", [("C1", 32), ("C5", 16)])
def test_sin_mode_is_eigenvector(name, c):
    """K s = λ s, s = sampled sin mode: λ = 8 sin²(πh/2) (2D), 12 h sin²(πh/2) (3D)."""
    P = O.build_problem(name, c=c)
    X = P["mesh"].coord[P["free_nodes"]]
    h = 1.0 / c
    s = np.prod(np.sin(np.pi * X), axis=1)
    lam = (8 if name == "C1" else 12 * h) * math.sin(math.pi * h / 2) ** 2
    y = O.spmv(P["A"], s)
    assert np.max(np.abs(y - lam * s)) < 1e-14 * max(1, lam)


@pytest.mark.parametrize("name,c", [("C1", 6), ("C2", 8), ("C3", 4), ("C4", 4), ("C5", 5)])
def test_pcg_vs_dense_cholesky(name, c):
    P = O.build_problem(name, c=c, k=1)
    A = P["A"].to_dense()
    b = P["B"][:, 0]
    Lc = np.linalg.cholesky(A)
    xe = np.linalg.solve(Lc.T, np.linalg.solve(Lc, b))
    r = O.pcg(P["A"], b, tol=1e-14)
    assert r.status == O.OK
    assert np.linalg.norm(r.x - xe) / np.linalg.norm(xe) < 1e-12


# ---------------------------------------------------------------- patch tests
def test_p1_jittered_patch_linear_exact():
    """P1 reproduces linear harmonic fields exactly on any (jittered) mesh."""
    c = 32
    mesh = O.Mesh(O.P1_TRI, c, True, 99)
    K, F = O.assemble(mesh, O.F_ZERO)
    X = mesh.coord
    g = 1 + 2 * X[:, 0] - 3 * X[:, 1]
    A, b, fmap = O.dirichlet(mesh, K, F, g, O.PAT_ELEMENT)
    r = O.pcg(A, b, tol=1e-14)
    u = g[fmap >= 0]
    assert np.linalg.norm(r.x - u) / np.linalg.norm(u) < 1e-11


@pytest.mark.parametrize("kind", ["harmonic", "poisson"])
def test_p2_patch_quadratic_exact(kind):
    """P2 reproduces quadratics exactly: x²-y² (f=0) and x²+y² (f=-4)."""
    c = 8
    mesh = O.Mesh(O.P2_TRI, c)
    X = mesh.coord
    if kind == "harmonic":
        K, F = O.assemble(mesh, O.F_ZERO)
        g = X[:, 0] ** 2 - X[:, 1] ** 2
    else:
        K, F = O.assemble(mesh, O.F_CONST, (-4.0,))
        g = X[:, 0] ** 2 + X[:, 1] ** 2
    A, b, fmap = O.dirichlet(mesh, K, F, g, O.PAT_ELEMENT)
    r = O.pcg(A, b, tol=1e-14)
    u = g[fmap >= 0]
    assert np.linalg.norm(r.x - u) / np.linalg.norm(u) < 1e-12


def test_p2_unit_square_centre_value():
    """C3 reading: -Δu = 1, u = 0 on ∂[0,1]²: u(½,½) from the exact series
    u = x(1-x)/2 - (4/π³) Σ_{m odd} sin(mπx) cosh(mπ(y-½)) / (m³ cosh(mπ/2)); P2 error O(h⁴)."""
    exact = 0.125 - 4 / math.pi ** 3 * sum(
        math.sin(m * math.pi / 2) / (m ** 3 * math.cosh(m * math.pi / 2)) for m in range(1, 200, 2))
    assert abs(exact - 0.0736713532815138) < 1e-15
    errs = []
    for c in (16, 32):
        P = O.build_problem("C3", c=c)
        r = O.pcg(P["A"], P["B"][:, 0], tol=1e-14)
        X = P["mesh"].coord[P["free_nodes"]]
        i = np.nonzero((np.abs(X[:, 0] - .5) < 1e-12) & (np.abs(X[:, 1] - .5) < 1e-12))[0][0]
        errs.append(abs(r.x[i] - exact))
    assert errs[1] < 2e-8
    assert 10 < errs[0] / errs[1] < 25  # ~16 for O(h^4)


def test_c1_discretisation_error_second_order():
    """x_err (Eq. ERROR-METRIC) vs sampled sin(πx)sin(πy) shrinks as O(h²)."""
    errs = []
    for c in (32, 64):
        P = O.build_problem("C1", c=c)
        r = O.pcg(P["A"], P["B"][:, 0], tol=1e-12)
        X = P["mesh"].coord[P["free_nodes"]]
        u = np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1])
        errs.append(np.linalg.norm(u - r.x) / np.linalg.norm(u))
    assert 1e-4 < errs[1] < 4e-4
    assert 3.5 < errs[0] / errs[1] < 4.5


# ---------------------------------------------------------------- PCG recurrence
def _csr_from_dense(A):
    n = A.shape[0]
    rp, cols, vals = [0], [], []
    for i in range(n):
        nz = np.nonzero(A[i])[0]
        cols += list(nz)
        vals += list(A[i, nz])
        rp.append(len(cols))
    return O.Csr(n, rp, cols, vals)


def test_spec_spmv_vector():
    """[2,-1;-1,2,-1;-1,2]·[1,1,1] = [1,0,1]."""
    A = _csr_from_dense(np.array([[2., -1, 0], [-1, 2, -1], [0, -1, 2]]))
    assert np.array_equal(O.spmv(A, np.ones(3)), [1., 0., 1.])


def test_identity_and_diagonal_converge_in_one_iteration():
    """Jacobi-PCG on a diagonal (or identity) matrix needs one iteration."""
    rng = np.random.default_rng(4)
    for D in (np.eye(7), np.diag(rng.random(7) + 0.5)):
        r = O.pcg(_csr_from_dense(D), rng.random(7), tol=1e-12)
        assert r.status == O.OK and r.iterations == 1
        assert np.allclose(D @ r.x, D @ np.linalg.solve(D, D @ r.x))


def test_1d_laplacian_vs_dense():
    """1D n=10 Dirichlet Laplacian, PCG vs dense solve within 1e-9."""
    n = 10
    A = 2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)
    b = np.arange(1, n + 1, dtype=float)
    r = O.pcg(_csr_from_dense(A), b, tol=1e-12)
    assert np.linalg.norm(r.x - np.linalg.solve(A, b)) / np.linalg.norm(np.linalg.solve(A, b)) < 1e-9


def test_finite_termination_three_distinct_eigenvalues():
    """CG terminates in m iterations when the preconditioned operator has m distinct
    eigenvalues.  S = Q Λ Qᵀ with Q a normalised Hadamard matrix has constant diagonal
    mean(Λ); A = D^{1/2} S D^{1/2} then has diag(A)⁻¹A ~ S/mean(Λ): 3 distinct eigenvalues."""
    from scipy.linalg import hadamard
    rng = np.random.default_rng(5)
    n = 16
    Q = hadamard(n) / 4.0
    lam = np.array([1.0] * 6 + [2.0] * 5 + [5.0] * 5)
    S = Q @ np.diag(lam) @ Q.T
    d = rng.random(n) + 0.5
    A = np.sqrt(d)[:, None] * S * np.sqrt(d)[None, :]
    A = (A + A.T) / 2
    r = O.pcg(_csr_from_dense(A), rng.standard_normal(n), tol=1e-10)
    assert r.status == O.OK and r.iterations == 3


def test_lanczos_ritz_values_hit_jacobi_spectrum():
    """α, β of PCG define the Lanczos tridiagonal of D⁻¹K; its extreme eigenvalues converge to
    the closed-form extremes 1 ∓ cos(π/c) of the 2D lattice's D⁻¹K."""
    c = 32
    P = O.build_problem("C1", c=c)
    b = np.random.default_rng(6).standard_normal(P["A"].n)  # excites every mode
    r = O.pcg(P["A"], b, tol=1e-12, hist=1000)
    k = r.iterations - 1
    a, bt = r.alpha[:k], r.beta[:k]
    T = np.zeros((k, k))
    for j in range(k):
        T[j, j] = 1 / a[j] + (bt[j - 1] / a[j - 1] if j else 0)
        if j + 1 < k:
            T[j, j + 1] = T[j + 1, j] = math.sqrt(bt[j]) / a[j]
    ev = np.linalg.eigvalsh(T)
    lo, hi = 1 - math.cos(math.pi / c), 1 + math.cos(math.pi / c)
    assert abs(ev[0] - lo) < 1e-8 * hi and abs(ev[-1] - hi) < 1e-8 * hi


def test_status_codes_and_edge_cases():
    A = _csr_from_dense(np.array([[2., -1, 0], [-1, 2, -1], [0, -1, 2]]))
    # b = 0 -> x = 0, 0 iterations
    r = O.pcg(A, np.zeros(3), x0=np.ones(3))
    assert r.status == O.OK and r.iterations == 0 and np.all(r.x == 0)
    # exact initial guess -> 0 iterations
    r = O.pcg(A, np.array([1., 0, 1]), x0=np.ones(3))
    assert r.status == O.OK and r.iterations == 0
    # zero / negative diagonal, indefinite, bad args
    assert O.pcg(_csr_from_dense(np.array([[0., 1], [1, 2]])), np.ones(2)).status == O.ERR_ZERO_DIAGONAL
    assert O.pcg(_csr_from_dense(np.diag([1., -1])), np.ones(2)).status == O.ERR_NOT_SPD
    indef = np.array([[1., 3], [3, 1]])
    assert O.pcg(_csr_from_dense(indef), np.array([1., 0])).status == O.ERR_NOT_SPD
    assert O.pcg(A, np.ones(3), tol=0.0).status == O.ERR_INVALID_ARG
    assert O.pcg(A, np.ones(3), max_iter=0).status == O.ERR_INVALID_ARG
    # max_iter reached: NOT_CONVERGED, x holds the last iterate
    P = O.build_problem("C1", c=16)
    r = O.pcg(P["A"], P["B"][:, 0], tol=1e-12, max_iter=5)
    assert r.status == O.NOT_CONVERGED and r.iterations == 5 and r.relres_true > 1e-12


@pytest.mark.parametrize("name,c", [("C1", 32), ("C2", 32), ("C3", 16), ("C4", 12)])
def test_exit_contract_true_residual(name, c):
    """S:397 / Eq. relativeError: converged ⇔ ||b-Ax||/||b|| ≤ ε."""
    P = O.build_problem(name, c=c, k=2)
    for j in range(P["B"].shape[1]):
        b = P["B"][:, j]
        r = O.pcg(P["A"], b, tol=1e-10)
        t = np.linalg.norm(b - P["A"].to_scipy() @ r.x) / np.linalg.norm(b)
        assert r.status == O.OK and t <= 1e-10 and abs(t - r.relres_true) < 1e-13


def test_multi_rhs_linearity():
    """Eq. MRH-TERMS: independent columns; solutions are linear in B."""
    P = O.build_problem("C4", c=10, k=3)
    B = P["B"]
    X, res = O.pcg_multi(P["A"], np.column_stack([B[:, 0], B[:, 1], B[:, 0] + B[:, 1]]), tol=1e-13)
    assert all(r.status == O.OK for r in res)
    assert np.linalg.norm(X[:, 2] - X[:, 0] - X[:, 1]) / np.linalg.norm(X[:, 2]) < 1e-11


# ---------------------------------------------------------------- jitter + partition
def test_jitter_repair_invariants():
    c = 256
    h = 1.0 / c
    mesh = O.Mesh(O.P1_TRI, c, True, O.configs()["C2"]["seed"])
    X = mesh.coord
    T = mesh.elem
    a2 = ((X[T[:, 1], 0] - X[T[:, 0], 0]) * (X[T[:, 2], 1] - X[T[:, 0], 1])
          - (X[T[:, 2], 0] - X[T[:, 0], 0]) * (X[T[:, 1], 1] - X[T[:, 0], 1]))
    assert a2.min() > 0
    np_ = c + 1
    lat = np.stack([np.arange(mesh.n_nodes) % np_, np.arange(mesh.n_nodes) // np_], 1) * h
    d = X - lat
    assert np.all(d[mesh.boundary] == 0)
    assert np.max(np.abs(d)) <= 0.3 * h
    on_lattice = np.all(d == 0, axis=1) & ~mesh.boundary
    assert on_lattice.sum() == mesh.n_reset  # reset nodes are exactly the interior lattice ones
    assert mesh.n_reset > 0


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_partition_rule_and_halo_brute_force(G):
    P = O.build_problem("C2", c=24)
    A = P["A"]
    b = O.partition(A, G)
    assert b[0] == 0 and b[G] == A.n and np.all(np.diff(b) >= 0)
    for g in range(1, G):
        assert b[g] == np.searchsorted(A.row_ptr, (g * A.nnz) // G, side="left")
    for g in range(G):
        r0, r1 = b[g], b[g + 1]
        cols = set(A.col[A.row_ptr[r0]:A.row_ptr[r1]].tolist())
        want = sorted(j for j in cols if j < r0 or j >= r1)
        assert O.halo(A, r0, r1).tolist() == want


# ---------------------------------------------------------------- inner products (reading R1)
def _exact_dot(a, b):
    """Σ a_i b_i in exact rational arithmetic, then rounded once to fp64."""
    from fractions import Fraction
    return float(sum(Fraction(float(x)) * Fraction(float(y)) for x, y in zip(a, b)))


def test_dot_is_exactly_rounded_on_random_vectors():
    rng = np.random.default_rng(11)
    for n in (1, 7, 100, 2000):
        a = rng.standard_normal(n) * np.exp(rng.uniform(-20, 20, n))
        b = rng.standard_normal(n)
        e = _exact_dot(a, b)
        got = O.dot(a, b)
        # Dot2 error bound: |got - e| <= u|e| + gamma_n^2 Σ|a_i b_i|  (Ogita-Rump-Oishi, Prop. 5.5)
        u = 2.0 ** -53
        g = n * u / (1 - n * u)
        assert abs(got - e) <= u * abs(e) + g * g * float(np.sum(np.abs(a * b))) + 1e-300


def test_dot_survives_cancellation_that_breaks_a_plain_sum():
    # Σ = 1 exactly; a left-to-right fp64 sum returns 0
    a = np.array([1e16, 1.0, -1e16])
    b = np.ones(3)
    assert float(a[0] * b[0] + a[1] * b[1] + a[2] * b[2]) == 0.0
    assert O.dot(a, b) == 1.0
    # ill-conditioned (cond ~ 1e20): still the exactly rounded value
    rng = np.random.default_rng(3)
    x = rng.standard_normal(50) * 1e10
    a = np.concatenate([x[:25], x[:25], [3.0]])
    b = np.concatenate([np.ones(25), -np.ones(25), [0.5]])
    assert O.dot(a, b) == _exact_dot(a, b) == 1.5


# ---------------------------------------------------------------- N2: Table 1 systems + BiCGSTAB (reading R2)
@pytest.mark.parametrize("N,want", [(16, 20560), (128, 14099408)])
def test_fd_cube_is_table1(N, want):
    """The identity-boundary-row FD system has exactly the non-zero count the paper
    prints for Cube 1 (128^3 nodes: 14,099,408) and SPEC's 16^3 = 20,560."""
    A, b = O.fd_cube(N)
    assert A.n == N ** 3 and A.nnz == want
    rl = np.diff(A.row_ptr)
    assert set(np.unique(rl)) == {1, 7}
    assert np.all(np.diff(A.col[A.row_ptr[N * N + N + 1]:A.row_ptr[N * N + N + 2]]) > 0)


def _grid(N):
    h = 1.0 / (N - 1)
    i = np.arange(N)
    return np.tile(i, N * N) * h, np.tile(np.repeat(i, N), N) * h


@pytest.mark.parametrize("bs", [1, 2, 5])
def test_bicgstab_reproduces_the_harmonic_quadratic(bs):
    """Second differences are exact for quadratics: the discrete solution of the
    Table 1 system with boundary data x^2 - y^2 is x^2 - y^2 at every node."""
    N = 14
    A, b = O.fd_cube(N)
    X, Y = _grid(N)
    r = O.bicgstab(A, b, tol=1e-13, block=bs)
    assert r.status == O.OK and r.relres_true <= 1e-13
    assert np.max(np.abs(r.x - (X * X - Y * Y))) <= 1e-11


def test_bicgstab_block_equal_to_matrix_is_one_step():
    """M = A (one Block-Jacobi block covering the matrix): the first step is exact."""
    A, b = O.fd_cube(6, O.FD_EXPSIN)
    r = O.bicgstab(A, b, tol=1e-12, block=A.n)
    assert r.status == O.OK and r.iterations == 1
    assert np.allclose(r.x, np.linalg.solve(A.to_dense(), b), rtol=0, atol=1e-12)


@pytest.mark.parametrize("bs", [1, 3, 7])
def test_bicgstab_matches_dense_solve_on_nonsymmetric(bs):
    rng = np.random.default_rng(21)
    n = 60
    D = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.15)
    D += np.diag(np.abs(D).sum(1) + 1.0)  # strictly diagonally dominant, nonsymmetric
    rp, cols, vals = [0], [], []
    for i in range(n):
        nz = np.nonzero(D[i])[0]
        cols += list(nz)
        vals += list(D[i, nz])
        rp.append(len(cols))
    A = O.Csr(n, rp, cols, vals)
    bb = rng.standard_normal(n)
    r = O.bicgstab(A, bb, tol=1e-13, block=bs)
    assert r.status == O.OK
    xe = np.linalg.solve(D, bb)
    assert np.linalg.norm(r.x - xe) / np.linalg.norm(xe) <= 1e-11


def test_bicgstab_on_spd_lattice_matches_dst():
    """On the SPD C1 lattice system BiCGSTAB reaches the DST-I exact solution too."""
    from scipy.fft import dstn, idstn
    c = 32
    P = O.build_problem("C1", c=c)
    A, b = P["A"], P["B"][:, 0]
    m = c - 1
    jj = np.arange(1, m + 1)
    l1 = 2 - 2 * np.cos(jj * np.pi / c)
    xe = idstn(dstn(b.reshape(m, m), type=1) / (l1[None, :] + l1[:, None]), type=1).ravel()
    r = O.bicgstab(A, b, tol=1e-13)
    assert r.status == O.OK
    assert np.linalg.norm(r.x - xe) / np.linalg.norm(xe) <= 1e-11


def test_bicgstab_status_codes():
    A, b = O.fd_cube(10, O.FD_EXPSIN)
    r = O.bicgstab(A, b, tol=1e-12, max_iter=3)
    assert r.status == O.NOT_CONVERGED and r.iterations == 3
    r = O.bicgstab(A, np.zeros(A.n))
    assert r.status == O.OK and r.iterations == 0 and np.all(r.x == 0)
    I = O.Csr(5, list(range(6)), list(range(5)), [2.0] * 5)
    r = O.bicgstab(I, np.arange(1.0, 6.0), tol=1e-14)
    assert r.status == O.OK and r.iterations == 1 and np.allclose(r.x, np.arange(1.0, 6.0) / 2)


# ---------------------------------------------------------------- N4: C6 jittered Kuhn tets (reading R3)
def test_kuhn_tet_volume_bound_at_015h():
    """Multilinear corner bound: with every vertex of a Kuhn tet moved by at most 0.15h per
    coordinate, the signed volume keeps its sign and stays >= 0.1 of the lattice volume
    (so the C6 mesh needs no repair); at 0.2h a fixed-vertex tet already degenerates."""
    import itertools

    def kuhn(p):
        v = [np.zeros(3)]
        for k in range(3):
            w = v[-1].copy()
            w[p[k]] += 1
            v.append(w)
        return v

    def vol(V):
        return np.linalg.det(np.array([V[1] - V[0], V[2] - V[0], V[3] - V[0]])) / 6

    corners = list(itertools.product([-1, 1], repeat=3))
    for d, lo in ((0.15, 0.1 / 6 - 1e-12), (0.2, None)):
        worst = 1e9
        for p in itertools.permutations(range(3)):
            V = kuhn(p)
            s0 = np.sign(vol(V))
            for cs in itertools.product(corners, repeat=4):
                worst = min(worst, s0 * vol([v + d * np.array(c) for v, c in zip(V, cs)]))
        if lo is not None:
            assert worst >= lo
        else:
            assert worst < 0


def test_c6_mesh_jitter_is_bounded_and_deterministic():
    c = 8
    m1 = O.Mesh(O.P1_TET, c, True, O.configs()["C6"]["seed"])
    m2 = O.Mesh(O.P1_TET, c, True, O.configs()["C6"]["seed"])
    assert np.array_equal(m1.coord, m2.coord)
    h = 1.0 / c
    np_ = c + 1
    idx = np.arange(m1.n_nodes)
    lat = np.stack([idx % np_, (idx // np_) % np_, idx // (np_ * np_)], 1) * h
    d = m1.coord - lat
    assert np.all(d[m1.boundary] == 0)
    assert np.max(np.abs(d)) <= 0.15 * h and np.max(np.abs(d)) > 0.1 * h


def test_c6_patch_test_reproduces_the_linear_field():
    """P1 reproduces linear fields exactly: with g = 1 + 2x - 3y + z/2 and f = 0 the discrete
    solution on the jittered mesh equals g at every free node."""
    P = O.build_problem("C6", c=10)
    r = O.pcg(P["A"], P["B"][:, 0], tol=1e-13)
    X = P["mesh"].coord[P["free_nodes"]]
    ex = ((1.0 + 2.0 * X[:, 0]) - 3.0 * X[:, 1]) + 0.5 * X[:, 2]
    assert r.status == O.OK and np.max(np.abs(r.x - ex)) <= 1e-11


def test_c6_neumann_stiffness_symmetric_zero_rowsums_and_dense_solve():
    m = O.Mesh(O.P1_TET, 5, True, O.configs()["C6"]["seed"])
    K, F = O.assemble(m, O.F_ZERO)
    D = K.to_dense()
    assert np.max(np.abs(D - D.T)) <= 1e-15 * np.abs(D).max()
    assert np.max(np.abs(D.sum(1))) <= 1e-14 * np.abs(D).max()
    P = O.build_problem("C6", c=5)
    A, b = P["A"], P["B"][:, 0]
    xe = np.linalg.solve(A.to_dense(), b)
    r = O.pcg(A, b, tol=1e-14)
    assert np.linalg.norm(r.x - xe) / np.linalg.norm(xe) <= 1e-12


# ---------------------------------------------------------------- COO -> CSR
def test_coo_to_csr_spec_examples():
    rp, c, v = O.coo_to_csr(2, 2, [0, 0, 1], [0, 0, 1], [1.0, 3.0, 2.0])  # S:55 duplicate summation
    assert rp.tolist() == [0, 1, 2] and c.tolist() == [0, 1] and v.tolist() == [4.0, 2.0]
    rp, c, v = O.coo_to_csr(3, 3, [], [], [])  # S:56 empty
    assert rp.tolist() == [0, 0, 0, 0] and c.size == 0
    rp, c, v = O.coo_to_csr(3, 3, [2, 0, 1], [2, 0, 1], [1.0, 1.0, 1.0])  # S:57 identity (any order)
    assert rp.tolist() == [0, 1, 2, 3] and c.tolist() == [0, 1, 2] and v.tolist() == [1.0, 1.0, 1.0]
    with pytest.raises(IndexError):  # S:53 IndexOutOfRange
        O.coo_to_csr(2, 3, [0, 2], [0, 0], [1.0, 1.0])
    with pytest.raises(IndexError):
        O.coo_to_csr(2, 3, [0], [-1], [1.0])


@pytest.mark.parametrize("seed,nr,nc,nnz", [(1, 7, 5, 60), (2, 40, 40, 900), (3, 1, 9, 30), (4, 13, 1, 25)])
def test_coo_to_csr_brute_force_dense(seed, nr, nc, nnz):
    """Dense accumulation in input order (A[r][c] += v) is the definition: bitwise equal
    values, pattern = the set of positions present (explicit zero sums kept)."""
    from coo_inputs import triplets
    r, c, v = triplets(seed, nr, nc, nnz)
    rp, co, vo = O.coo_to_csr(nr, nc, r, c, v)
    D = np.zeros((nr, nc))
    present = np.zeros((nr, nc), dtype=bool)
    for k in range(nnz):
        D[r[k], c[k]] += v[k]
        present[r[k], c[k]] = True
    assert rp[0] == 0 and rp[-1] == co.size == present.sum()
    for i in range(nr):
        cols = co[rp[i]:rp[i + 1]]
        assert np.all(np.diff(cols) > 0)  # strictly increasing within a row
        assert cols.tolist() == np.nonzero(present[i])[0].tolist()
        assert np.array_equal(vo[rp[i]:rp[i + 1]], D[i, cols])  # bitwise
    assert np.any(vo == 0.0) or nr * nc < 40  # the cancelling pair stays an explicit entry


@pytest.mark.parametrize("fam,c,jit", [(O.P1_TRI, 6, False), (O.P1_TRI, 8, True), (O.P2_TRI, 4, False),
                                       (O.P1_TET, 3, False)])
def test_coo_to_csr_of_element_triplets_is_the_assembly(fam, c, jit):
    """Element-by-element assembly through COO (triplets (t_a, t_b, Ke[a][b]) emitted in
    element order, local (a, b) order) is orc_assemble's stiffness, bitwise: the two
    oracle paths (incidence-list pattern + csr_find, versus sort + ordered sum) agree."""
    m = O.Mesh(fam, c, jitter=jit, seed=77)
    K, _ = O.assemble(m, O.F_ZERO)
    rows, cols, vals = [], [], []
    for e in range(m.n_elem):
        t = m.elem[e]
        Ke = O.elem_stiffness(fam, m.coord[t].ravel())
        for a in range(m.npe):
            for b in range(m.npe):
                rows.append(t[a])
                cols.append(t[b])
                vals.append(Ke[a, b])
    rp, co, vo = O.coo_to_csr(m.n_nodes, m.n_nodes, rows, cols, vals)
    assert np.array_equal(rp, K.row_ptr) and np.array_equal(co, K.col)
    assert np.array_equal(vo, K.val)


# ---------------------------------------------------------------- pipelined PCG (reading R4)
def _csr_from_dense(D):
    n = D.shape[0]
    rp, col, val = [0], [], []
    for i in range(n):
        for j in range(n):
            if D[i, j] != 0.0 or i == j:
                col.append(j)
                val.append(D[i, j])
        rp.append(len(col))
    return O.Csr(n, rp, col, val)


def test_pipelined_identity_and_diagonal_one_step():
    b = np.random.default_rng(5).uniform(-1, 1, 40)
    r = O.pcg_pipelined(_csr_from_dense(np.eye(40)), b, tol=1e-14)
    assert r.status == O.OK and r.iterations == 1 and np.array_equal(r.x, b)
    d = np.random.default_rng(6).uniform(0.5, 3.0, 40)
    r = O.pcg_pipelined(_csr_from_dense(np.diag(d)), b, tol=1e-12)
    assert r.status == O.OK and r.iterations == 1 and np.allclose(r.x, b / d, rtol=4e-16, atol=0)


@pytest.mark.parametrize("name,c", [("C1", 8), ("C3", 4), ("C5", 4)])
def test_pipelined_equals_pcg_in_exact_arithmetic(name, c):
    """Ghysels-Vanroose's recurrences are PCG's rewritten: after k steps the iterate is
    PCG's k-th iterate, up to rounding (checked for k = 1..8)."""
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    for k in range(1, 9):
        xc = O.pcg(A, b, tol=1e-15, max_iter=k).x
        xp = O.pcg_pipelined(A, b, tol=1e-15, max_iter=k).x
        assert np.linalg.norm(xp - xc) <= 1e-12 * np.linalg.norm(xc), k


@pytest.mark.parametrize("name,c", [("C1", 32), ("C2", 32), ("C4", 16), ("C6", 8)])
def test_pipelined_converges_like_pcg(name, c):
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()[name]["tol"]
    rc = O.pcg(A, b, tol=tol)
    rp = O.pcg_pipelined(A, b, tol=tol)
    assert rp.status == O.OK and rp.relres_true <= tol
    assert abs(rp.iterations - rc.iterations) <= max(2, 0.03 * rc.iterations), (rp.iterations, rc.iterations)
    assert np.linalg.norm(rp.x - rc.x) <= 1e-8 * np.linalg.norm(rc.x)


def test_pipelined_max_iter():
    P = O.build_problem("C1", c=16, k=1)
    r = O.pcg_pipelined(P["A"], P["B"][:, 0], tol=1e-12, max_iter=5)
    assert r.status == O.NOT_CONVERGED and r.iterations == 5


# ---------------------------------------------------------------- round 2 pins
def test_sin3d_load_discretisation_error_sequence():
    """C5's load f = 3π² sin πx sin πy sin πz (BASELINE.json configs[4]): x_err (Eq.
    ERROR-METRIC) against the sampled u = sin πx sin πy sin πz follows the
    O(h²) sequence SURVEY §8(c) fixes from its independent probe: 1.64e-3 (c = 32),
    4.11e-4 (c = 64).  A 3π² -> 2π² slip (u scaled by 2/3) gives x_err ≈ 0.33."""
    want = {32: 1.64e-3, 64: 4.11e-4}
    errs = {}
    for c in want:
        P = O.build_problem("C5", c=c)
        r = O.pcg(P["A"], P["B"][:, 0], tol=1e-12)
        X = P["mesh"].coord[P["free_nodes"]]
        u = np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])
        errs[c] = np.linalg.norm(u - r.x) / np.linalg.norm(u)
        assert abs(errs[c] - want[c]) <= 0.01 * want[c], (c, errs[c])
    assert 3.9 < errs[32] / errs[64] < 4.1


@pytest.mark.parametrize("centre", [(0.5, 0.5, 0.5), (0.37, 0.52, 0.61)])
def test_bump3d_load_integrates_the_gaussian(centre):
    """C4's load f = exp(-|x - c|²/(2σ²)) (BASELINE.json configs[3], σ = 0.05, reading
    Q10): for an interior bump the Neumann load vector sums to ∫f = (2πσ²)^{3/2} (the
    Gaussian integral; the tail outside the cube is < 1e-20).  σ² in place of 2σ²
    changes the sum by 2^{-3/2}; a dropped quadrature weight by 4/3 or more."""
    sigma = 0.05
    m = O.Mesh(O.P1_TET, 32)
    F = O.assemble_load(m, O.F_BUMP3D, (centre[0], centre[1], centre[2], sigma))
    want = (2 * math.pi * sigma ** 2) ** 1.5
    assert abs(F.sum() - want) <= 1e-9 * want


def _splitmix64_py(seed, idx):
    """SplitMix64 (Steele, Lea, Flood 2014) in Python integers, itself pinned below by
    the published sequence test (tests/golden/splitmix64_seed0.txt)."""
    M = (1 << 64) - 1
    z = (seed + (idx + 1) * 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def test_splitmix64_python_twin_matches_published_sequence():
    rows = _golden_rows("splitmix64_seed0.txt")
    for i, row in enumerate(rows):
        assert _splitmix64_py(0, i) == int(row[0], 16)


def test_bump_centres_index_mapping():
    """§8(c).11: c_s = (u(seed, 3s), u(seed, 3s+1), u(seed, 3s+2)), u = top 53 bits of
    SplitMix64 × 2^-53, computed here from the Python twin (not the oracle's C)."""
    seed = O.configs()["C4"]["seed"]
    cs = O.bump_centres(seed, 16)
    for s in range(16):
        for a in range(3):
            u = (_splitmix64_py(seed, 3 * s + a) >> 11) * 2.0 ** -53
            assert cs[s, a] == u, (s, a)


@pytest.mark.parametrize("name,c", [("C1", 16), ("C1", 64), ("C4", 8), ("C5", 12)])
def test_free_lattice_assembly_is_bitwise_the_pipeline(name, c):
    """orc_assemble_free_lattice (the C5 full-size golden's builder) equals
    orc_assemble + orc_dirichlet(AXIS) bitwise: same pattern, same values, same b."""
    P = O.build_problem(name, c=c, k=1 if name == "C4" else None)
    cfg = P["cfg"]
    if cfg["f"] == "BUMP3D":
        cs = O.bump_centres(cfg["seed"], 1)[0]
        fk, fp = O.F_BUMP3D, (cs[0], cs[1], cs[2], cfg["sigma"])
    else:
        fk, fp = {"SIN2D": O.F_SIN2D, "SIN3D": O.F_SIN3D}[cfg["f"]], (1.0, 0.0, 0.0, 0.0)
    A, b = O.assemble_free_lattice(P["mesh"], fk, fp)
    assert np.array_equal(A.row_ptr, P["A"].row_ptr) and np.array_equal(A.col, P["A"].col)
    assert A.val.tobytes() == P["A"].val.tobytes()
    assert b.tobytes() == P["B"][:, 0].tobytes()


def test_residual_replacement_fires_and_is_a_restart():
    """§8(c).8 exit: when the recurrence residual passes tol but the true residual
    (Eq. relativeError) does not, the loop restarts from the current x with
    r = b - Ax, z = dinv r, p = z, counting on.  At tol = 1e-15 on C1 the recurrence
    drops below the attainable accuracy (true relres floor ~1e-13), so replacements
    fire; the continuation after the first one must be exactly a fresh solve from that
    iterate with the remaining iteration budget (same x bits, same count)."""
    P = O.build_problem("C1")
    A, b = P["A"], P["B"][:, 0]
    r = O.pcg_ex(A, b, tol=1e-15, max_iter=400)
    assert r.status == O.NOT_CONVERGED and r.iterations == 400
    assert r.replacements >= 2 and 100 <= r.k_first < 400
    assert r.relres_true < 1e-12  # replacement keeps the iterate at attainable accuracy
    r2 = O.pcg_ex(A, b, x0=r.x_first, tol=1e-15, max_iter=400 - r.k_first)
    assert r2.iterations == 400 - r.k_first and r2.replacements == r.replacements - 1
    assert r2.x.tobytes() == r.x.tobytes()
    # without replacement firing, pcg_ex is pcg
    r3 = O.pcg_ex(A, b, tol=1e-10)
    r4 = O.pcg(A, b, tol=1e-10)
    assert r3.replacements == 0 and r3.k_first == -1 and r3.x.tobytes() == r4.x.tobytes()


def test_residual_replacement_then_convergence():
    """A replacement followed by convergence (status OK): C4 construction at c = 16,
    bump 0, tol = 1e-15 — the true residual fails the exit check once, the restart
    converges in the next iteration."""
    P = O.build_problem("C4", c=16, k=1)
    r = O.pcg_ex(P["A"], P["B"][:, 0], tol=1e-15, max_iter=300)
    assert r.status == O.OK and r.replacements >= 1 and r.relres_true <= 1e-15
