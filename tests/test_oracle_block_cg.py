"""Pins of the oracle's block CG (oracle.h orc_block_cg, reading R5).

k = 1 is Jacobi-PCG (the pinned orc_pcg), finite termination in about n/k steps on a
small dense SPD system (checked against a dense solve), one step for a diagonal
system, zero right-hand sides, and the shared Krylov space needing fewer products
than the independent solves on C4.
"""
import numpy as np
import pytest

import oracle as O


def _dense_csr(M):
    n = M.shape[0]
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    col = np.tile(np.arange(n, dtype=np.int64), n)
    return O.Csr(n, rp, col, M.reshape(-1).copy())


def _spd(n, seed, cond=50.0):
    rng = np.random.default_rng(seed)
    Qm, _ = np.linalg.qr(rng.standard_normal((n, n)))
    ev = np.geomspace(1.0, cond, n)
    return (Qm * ev) @ Qm.T


@pytest.mark.parametrize("name,c", [("C1", None), ("C2", 32), ("C4", 12)])
def test_block_cg_k1_is_pcg(name, c):
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    r = O.pcg(A, b, tol=1e-10)
    X, it, rt, st = O.block_cg(A, b[:, None], tol=1e-10)
    assert st == O.OK and rt[0] <= 1e-10
    assert abs(it - r.iterations) <= 1
    assert np.linalg.norm(X[:, 0] - r.x) / np.linalg.norm(r.x) <= 1e-10


@pytest.mark.parametrize("n,k,seed", [(24, 4, 1), (40, 8, 2), (33, 3, 3)])
def test_block_cg_finite_termination_dense(n, k, seed):
    M = _spd(n, seed)
    B = np.random.default_rng(seed + 10).standard_normal((n, k))
    X, it, rt, st = O.block_cg(_dense_csr(M), B, tol=1e-12)
    assert st == O.OK
    assert it <= -(-n // k) + 3  # block Krylov space of dimension k*j fills R^n after ceil(n/k) steps
    Xd = np.linalg.solve(M, B)
    assert np.linalg.norm(X - Xd) / np.linalg.norm(Xd) <= 1e-9


def test_block_cg_diagonal_one_step():
    n, k = 50, 5
    d = 1.0 + np.arange(n) % 7
    A = O.Csr(n, np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int64), d)
    B = np.random.default_rng(4).standard_normal((n, k))
    X, it, rt, st = O.block_cg(A, B, tol=1e-12)
    assert st == O.OK and it == 1
    assert np.allclose(X, B / d[:, None], rtol=1e-14, atol=0)


def test_block_cg_zero_columns():
    P = O.build_problem("C1", k=1)
    A, b = P["A"], P["B"][:, 0]
    B = np.stack([np.zeros(A.n), b, np.zeros(A.n), 2 * b + 1], 1)
    X, it, rt, st = O.block_cg(A, B, tol=1e-10)
    assert st == O.OK
    assert np.all(X[:, 0] == 0) and np.all(X[:, 2] == 0)
    import scipy.sparse.linalg as sla
    K = A.to_scipy().tocsc()
    for j in (1, 3):
        xd = sla.spsolve(K, B[:, j])
        assert np.linalg.norm(X[:, j] - xd) / np.linalg.norm(xd) <= 1e-8
        assert rt[j] <= 1e-10


def test_block_cg_shared_krylov_space_fewer_products():
    P = O.build_problem("C4", c=16)
    A, B = P["A"], P["B"]
    X, it, rt, st = O.block_cg(A, B, tol=1e-10)
    assert st == O.OK and np.all(rt <= 1e-10)
    its = [O.pcg(A, B[:, j], tol=1e-10).iterations for j in range(B.shape[1])]
    assert it < min(its)
    import scipy.sparse.linalg as sla
    K = A.to_scipy().tocsc()
    Xd = sla.spsolve(K, B)
    assert np.linalg.norm(X - Xd) / np.linalg.norm(Xd) <= 1e-7
