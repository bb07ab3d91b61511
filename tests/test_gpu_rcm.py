"""GPU reverse Cuthill-McKee (include/pcg.h csr_rcm_order, PCG_REORDER_RCM).

The order is index work: bit-exact against the oracle's sequential orc_rcm.  Solves on
the reordered device system (P A P^T, vectors gathered/scattered inside the calls) meet
the PCG parity bar of test_gpu_parity.py against the oracle on the caller's numbering.
"""
import numpy as np
import pytest

import oracle as O
from paper_2201_05413_b200 import inputs as I

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


def _graph(n, edges):
    rows = [[i] for i in range(n)]
    for a, b in edges:
        rows[a].append(b)
        rows[b].append(a)
    rows = [sorted(set(r)) for r in rows]
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int64)
    col = np.concatenate(rows).astype(np.int64) if n else np.zeros(0, dtype=np.int64)
    return O.Csr(n, rp, col, np.ones(len(col)))


def _relabelled(name, c, seed=11):
    P = O.build_problem(name, c=c, k=1)
    A = P["A"]
    q = I.relabel_order(A.n, seed)
    rp, col, val = I.relabel_csr_numpy(A.row_ptr, A.col, A.val, q)
    return O.Csr(A.n, rp, col, val), P["B"][:, 0][q]


def _lattice(c):
    E = [(j * c + i, j * c + i + 1) for j in range(c) for i in range(c - 1)]
    E += [(j * c + i, (j + 1) * c + i) for j in range(c - 1) for i in range(c)]
    return _graph(c * c, E)


GRAPHS = {
    "degree_order": lambda: _graph(8, [(0, 1), (0, 2), (0, 3), (1, 4), (2, 4), (2, 5), (3, 6), (6, 7), (5, 7)]),
    "peripheral": lambda: _graph(6, [(1, 2), (2, 3), (3, 4), (4, 5), (0, 3)]),
    "components_isolated": lambda: _graph(6, [(1, 3), (0, 2), (2, 4)]),
    "all_isolated": lambda: _graph(5, []),
    "single": lambda: _graph(1, []),
    "lattice33": lambda: _lattice(33),
    "C1": lambda: O.build_problem("C1", k=1)["A"],
    "C3_c24": lambda: O.build_problem("C3", c=24, k=1)["A"],
    "C2_relabelled": lambda: _relabelled("C2", 48)[0],
    "C6_relabelled": lambda: _relabelled("C6", 12)[0],
    "blocks_plus_isolated": lambda: _graph(40, [(i, i + 1) for i in range(10)] + [(20 + i, 21 + i) for i in range(9)]
                                           + [(12, 14), (14, 16)]),
}


@pytest.mark.parametrize("name", list(GRAPHS))
@pytest.mark.parametrize("side", ["host", "device"])
def test_rcm_order_bit_exact(pcg, name, side):
    A = GRAPHS[name]()
    ref = O.rcm(A)
    if side == "host":
        p = pcg.csr_rcm_order(A.row_ptr, A.col)
    else:
        p = pcg.csr_rcm_order(_dev(A.row_ptr), _dev(A.col)).cpu().numpy()
    assert p.dtype == np.int64
    assert np.array_equal(p, ref)


def test_rcm_order_empty_and_errors(pcg):
    assert pcg.csr_rcm_order(np.zeros(1, dtype=np.int64), np.zeros(0, dtype=np.int64)).size == 0
    with pytest.raises(pcg.PcgError):
        pcg.csr_rcm_order(np.array([0, 1, 2]), np.array([0, 5]))  # column out of range
    with pytest.raises(pcg.PcgError):
        pcg.csr_rcm_order(np.array([0, 2, 1]), np.array([0]))  # row_ptr[n] != nnz


@pytest.mark.parametrize("name,c,fmt", [("C2", 48, "auto"), ("C6", 12, "auto"), ("C3", 24, "sigma"),
                                        ("C6", 12, "csr"), ("C2", 48, "sell")])
def test_rcm_solve_parity(pcg, name, c, fmt):
    A, b = _relabelled(name, c)
    tol = O.configs()[name]["tol"]
    r = O.pcg(A, b, tol=tol)
    M = pcg.Matrix.from_csr(_dev(A.row_ptr), _dev(A.col), _dev(A.val), fmt=fmt, reorder="rcm")
    st = M.stats()
    assert st["reorder"] == 1
    assert (st["format"] == 4) == (st["sigma"] > 0)  # PCG_FORMAT_SELL_SIGMA iff a sigma window
    x, info = M.solve(_dev(b), tol=tol)
    x = x.cpu().numpy()
    assert info["status"] == 0 and info["relres_true"] <= tol
    assert np.linalg.norm(x - r.x) / np.linalg.norm(r.x) <= 1e-9
    assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
    # SpMV through the permuted system: y = P^T (P A P^T)(P x), caller's numbering
    xr = np.random.default_rng(5).standard_normal(A.n)
    y = M.spmv(_dev(xr)).cpu().numpy()
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    mag = np.bincount(rows, weights=np.abs(A.val) * np.abs(xr)[A.col], minlength=A.n)
    assert np.all(np.abs(y - O.spmv(A, xr)) <= 2 * np.diff(A.row_ptr) * 2.0 ** -53 * mag + 1e-300)


def test_rcm_other_solvers(pcg):
    A, b = _relabelled("C6", 12)
    tol = 1e-10
    M = pcg.Matrix.from_csr(_dev(A.row_ptr), _dev(A.col), _dev(A.val), reorder="rcm")
    r = O.pcg(A, b, tol=tol)
    xp, ip = M.solve_pipelined(_dev(b), tol=tol)
    assert ip["status"] == 0 and np.linalg.norm(xp.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-8
    xb, ib = M.bicgstab(_dev(b), tol=tol)
    assert ib["status"] == 0 and ib["relres_true"] <= tol
    B = np.stack([b, 2 * b + 1], 1)
    X, infos = M.solve_multi(_dev(B), tol=tol)
    X = X.cpu().numpy()
    for j in range(2):
        rj = O.pcg(A, B[:, j], tol=tol)
        assert infos[j]["status"] == 0
        assert np.linalg.norm(X[:, j] - rj.x) / np.linalg.norm(rj.x) <= 1e-9


def test_rcm_with_drop_zeros(pcg):
    # C3' reordered: the RCM order of the dropped pattern, same solution
    A, b = _relabelled("C3", 24)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    keep = (A.val != 0) | (A.col == rows)
    rp = np.concatenate([[0], np.cumsum(np.bincount(rows[keep], minlength=A.n))]).astype(np.int64)
    Ad = O.Csr(A.n, rp, A.col[keep], A.val[keep])
    assert np.array_equal(pcg.csr_rcm_order(Ad.row_ptr, Ad.col), O.rcm(Ad))
    M = pcg.Matrix.from_csr(_dev(A.row_ptr), _dev(A.col), _dev(A.val), drop_zeros=True, reorder="rcm")
    assert M.nnz == Ad.nnz
    r = O.pcg(A, b, tol=1e-10)
    x, info = M.solve(_dev(b), tol=1e-10)
    assert info["status"] == 0
    assert np.linalg.norm(x.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-9


def test_rcm_restores_locality(pcg):
    # the relabelled C6 has a bandwidth ~n; after RCM it is O(n^(2/3))
    A, _ = _relabelled("C6", 16)
    p = pcg.csr_rcm_order(A.row_ptr, A.col)
    ip = np.empty(A.n, dtype=np.int64)
    ip[p] = np.arange(A.n)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    bw0 = np.max(np.abs(rows - A.col))
    bw1 = np.max(np.abs(ip[rows] - ip[A.col]))
    assert bw1 < 0.1 * bw0
