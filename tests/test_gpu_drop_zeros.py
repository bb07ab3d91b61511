"""PCG_DROP_ZEROS (SURVEY §8(c) Q7, C3'): explicit zero entries not stored.

C3's bilinear Q1 stencil on a cross-diffusion grid carries explicit zeros (40228 of
101429 entries at c=48).  Dropping them leaves every product unchanged (0 * x added
to a partial sum is exact for finite x), so with the one-thread-per-row SELL-32
order the iterates are bitwise those of the full pattern; any format matches the
oracle at the parity bar of test_gpu_parity.py.
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pcg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_05413_b200 as p
    return p


def _dev(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a)).cuda()


def _mk(pcg, A, fmt, drop):
    return pcg.Matrix.from_csr(_dev(A.row_ptr), _dev(A.col), _dev(A.val), fmt=fmt, drop_zeros=drop)


def test_drop_zeros_stats_and_spmv(pcg):
    A = O.build_problem("C3", c=48, k=1)["A"]
    M = _mk(pcg, A, "auto", True)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    keep = (A.val != 0) | (A.col == rows)
    assert M.nnz == int(keep.sum()) == M.stats()["nnz"]
    assert M.nnz < len(A.val)
    x = np.random.default_rng(3).standard_normal(A.n)
    y = M.spmv(_dev(x)).cpu().numpy()
    ref = A.to_scipy() @ x
    mag = np.abs(A.to_scipy()) @ np.abs(x)
    assert np.all(np.abs(y - ref) <= 2 * 9 * 2.0 ** -53 * mag + 1e-300)


def test_drop_zeros_sell_bitwise(pcg):
    P = O.build_problem("C3", c=48, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()["C3"]["tol"]
    x0, i0 = _mk(pcg, A, "sell", False).solve(_dev(b), tol=tol)
    x1, i1 = _mk(pcg, A, "sell", True).solve(_dev(b), tol=tol)
    assert i0["status"] == i1["status"] == 0
    assert i0["iterations"] == i1["iterations"]
    assert bool((x0 == x1).all()), "dropping exact zeros must not change a one-thread-per-row sum"


@pytest.mark.parametrize("fmt", ["auto", "csr", "sigma"])
def test_drop_zeros_oracle_parity(pcg, fmt):
    P = O.build_problem("C3", c=48, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()["C3"]["tol"]
    r = O.pcg(A, b, tol=tol)
    x, info = _mk(pcg, A, fmt, True).solve(_dev(b), tol=tol)
    x = x.cpu().numpy()
    assert info["status"] == 0 and info["relres_true"] <= tol
    assert np.linalg.norm(x - r.x) / np.linalg.norm(r.x) <= 1e-9
    assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)


def test_drop_zeros_diagonal_only(pcg):
    # every off-diagonal entry zero: the stored matrix is the diagonal; PCG converges in 1 step
    n = 1000
    cols = [[j for j in (i - 1, i, i + 1) if 0 <= j < n] for i in range(n)]  # tridiagonal pattern, sorted
    rp = np.concatenate([[0], np.cumsum([len(c) for c in cols])]).astype(np.int64)
    col = np.concatenate(cols).astype(np.int64)
    rows = np.repeat(np.arange(n), np.diff(rp))
    dg = 1.0 + np.arange(n) % 5
    val = np.where(col == rows, dg[rows], 0.0)
    M = pcg.Matrix.from_csr(_dev(rp), _dev(col), _dev(val), drop_zeros=True)
    assert M.nnz == n
    b = np.random.default_rng(1).standard_normal(n)
    x, info = M.solve(_dev(b), tol=1e-12)
    assert info["status"] == 0 and info["iterations"] <= 1
    assert np.allclose(x.cpu().numpy(), b / dg, rtol=1e-14, atol=0)
