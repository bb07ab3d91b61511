"""Irregular sparsity through the whole path (format choice, CSR lanes, SELL padding
limits, SELL-C-sigma, multi-RHS, BiCGSTAB, pipelined): seeded SPD matrices whose
row-length distribution is far from the FEM stencils — an arrowhead (one dense row
and column), a power-law degree distribution, and rows of 1..300 entries — solved
against the oracle with the parity bars of DESIGN.md §5."""
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


def _spd_from_pattern(n, rows, cols, seed):
    """Symmetric pattern (rows, cols) + diagonal; off-diagonal values in [-1, 0), the
    diagonal 1 + row sum of |off-diagonals| (strictly diagonally dominant: SPD)."""
    rng = np.random.default_rng(seed)
    keep = rows != cols
    r, c = rows[keep], cols[keep]
    r, c = np.concatenate([r, c]), np.concatenate([c, r])
    key = np.unique(r.astype(np.int64) * n + c)
    r, c = key // n, key % n
    v = -rng.uniform(0.1, 1.0, r.size)
    # symmetric values: take the value of the (min, max) orientation
    lo, hi = np.minimum(r, c), np.maximum(r, c)
    sym = {}
    for a, b_, x in zip(lo, hi, v):
        sym.setdefault((a, b_), x)
    v = np.array([sym[(a, b_)] for a, b_ in zip(lo, hi)])
    d = 1.0 + np.bincount(r, weights=np.abs(v), minlength=n)
    R = np.concatenate([r, np.arange(n)])
    Cc = np.concatenate([c, np.arange(n)])
    V = np.concatenate([v, d])
    rp, co, va = O.coo_to_csr(n, n, R, Cc, V)
    return O.Csr(n, rp, co, va)


def _arrowhead(n):
    rows = np.concatenate([np.zeros(n - 1, np.int64), np.arange(1, n - 1)])
    cols = np.concatenate([np.arange(1, n), np.arange(2, n)])
    return _spd_from_pattern(n, rows, cols, 1)


def _powerlaw(n, m):
    rng = np.random.default_rng(2)
    deg = np.minimum((rng.pareto(1.5, n) + 1).astype(np.int64), n // 4)
    rows = np.repeat(np.arange(n), deg)
    cols = rng.integers(0, n, rows.size)
    return _spd_from_pattern(n, rows[:m], cols[:m], 3)


def _wide(n):
    rng = np.random.default_rng(4)
    lens = rng.integers(1, 300, n)
    rows = np.repeat(np.arange(n), lens)
    cols = np.clip(rows + rng.integers(-2000, 2000, rows.size), 0, n - 1)
    return _spd_from_pattern(n, rows, cols, 5)


CASES = {"arrowhead": lambda: _arrowhead(20000), "powerlaw": lambda: _powerlaw(30000, 400000),
         "wide": lambda: _wide(6000)}


@pytest.mark.parametrize("case", sorted(CASES))
@pytest.mark.parametrize("fmt", ["auto", "csr", "sigma"])
def test_irregular_pcg(pcg, case, fmt):
    import torch
    A = CASES[case]()
    b = np.random.default_rng(9).uniform(-1, 1, A.n)
    M = pcg.Matrix.from_csr(torch.as_tensor(A.row_ptr).cuda(), torch.as_tensor(A.col).cuda(),
                            torch.as_tensor(A.val).cuda(), fmt=fmt)
    r = O.pcg(A, b, tol=1e-10)
    x, info = M.solve(torch.as_tensor(b).cuda(), tol=1e-10)
    x = x.cpu().numpy()
    assert info["status"] == 0 and info["relres_true"] <= 1e-10
    assert np.linalg.norm(x - r.x) <= 1e-9 * np.linalg.norm(r.x)
    assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
    # SpMV within the forward error bound
    xr = np.random.default_rng(10).standard_normal(A.n)
    y = M.spmv(torch.as_tensor(xr).cuda()).cpu().numpy()
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    mag = np.bincount(rows, weights=np.abs(A.val) * np.abs(xr)[A.col], minlength=A.n)
    assert np.all(np.abs(y - O.spmv(A, xr)) <= 2 * np.diff(A.row_ptr) * 2.0 ** -53 * mag * (1 + 1e-9))


@pytest.mark.parametrize("case", sorted(CASES))
def test_irregular_multi_bicgstab_pipelined(pcg, case):
    import torch
    A = CASES[case]()
    M = pcg.Matrix.from_csr(torch.as_tensor(A.row_ptr).cuda(), torch.as_tensor(A.col).cuda(),
                            torch.as_tensor(A.val).cuda())
    B = np.random.default_rng(11).uniform(-1, 1, (A.n, 5))
    X, infos = M.solve_multi(torch.as_tensor(B).cuda(), tol=1e-10)
    X = X.cpu().numpy()
    for j in range(5):
        r = O.pcg(A, B[:, j], tol=1e-10)
        assert infos[j]["status"] == 0 and np.linalg.norm(X[:, j] - r.x) <= 1e-9 * np.linalg.norm(r.x)
    b = B[:, 0]
    rb = O.bicgstab(A, b, tol=1e-10)
    x, info = M.bicgstab(torch.as_tensor(b).cuda(), tol=1e-10)
    assert info["status"] == 0 and np.linalg.norm(x.cpu().numpy() - rb.x) <= 1e-9 * np.linalg.norm(rb.x)
    rp = O.pcg_pipelined(A, b, tol=1e-10)
    x, info = M.solve_pipelined(torch.as_tensor(b).cuda(), tol=1e-10)
    assert info["status"] == 0 and np.linalg.norm(x.cpu().numpy() - rp.x) <= 1e-8 * np.linalg.norm(rp.x)
