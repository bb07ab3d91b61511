"""The deferred x update of the single-GPU graph loop (solver.cu k1a_deferred): x is
updated every second iteration with the same fused multiply-adds in the same order, so
x must be BITWISE the every-iteration update's (PCG_XDEFER=0) at every kind of stop:
converged after a hold or an apply iteration, max_iter odd and even, residual
replacement (§8(c).8), breakdown (p^T A p <= 0) after either kind, warm start.  The
oracle bars of the graph schedule are in tests/test_gpu_schedules.py.
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


def _pair(pcg, monkeypatch, A, graph=True, mode="2"):
    """(deferred handle, every-iteration handle) of the same matrix on the graph path;
    mode: the deferral cycle (x every 2nd or every 4th iteration)"""
    monkeypatch.setenv("PCG_PERSIST", "0")
    if not graph:
        monkeypatch.setenv("PCG_NO_GRAPH", "1")
    out = []
    for xd in (mode, "0"):
        monkeypatch.setenv("PCG_XDEFER", xd)
        M = pcg.Matrix.from_csr(_dev(A.row_ptr), _dev(A.col), _dev(A.val), fmt="sell")
        _solve(M, np.ones(A.n), max_iter=3)  # builds the loop graph under this env
        out.append(M)
    monkeypatch.delenv("PCG_XDEFER")
    return out


def _solve(M, b, **kw):
    import torch
    from paper_2201_05413_b200 import PcgError
    x = torch.zeros(len(b), dtype=torch.float64, device="cuda")
    if "x0" in kw:
        x.copy_(_dev(kw.pop("x0")))
    try:
        _, info = M.solve(_dev(b), out=x, **kw)
        st = info["status"]
    except PcgError as e:
        info, st = None, e.status
    return x.cpu().numpy(), st, info


@pytest.mark.parametrize("mode", ["2", "4"])
@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("name,c", [("C1", None), ("C2", 48), ("C4", 16)])
def test_deferred_x_bitwise_converged(pcg, monkeypatch, graph, name, c, mode):
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    Md, Me = _pair(pcg, monkeypatch, A, graph, mode)
    tol = O.configs()[name]["tol"]
    xd, sd, infd = _solve(Md, b, tol=tol)
    xe, se, infe = _solve(Me, b, tol=tol)
    assert sd == se == 0 and infd["iterations"] == infe["iterations"]
    assert np.array_equal(xd, xe)
    # the oracle, for the record of what the bitwise pair computes
    r = O.pcg(A, b, tol=tol)
    assert np.linalg.norm(xd - r.x) / np.linalg.norm(r.x) <= 1e-9


@pytest.mark.parametrize("mode", ["2", "4"])
def test_deferred_x_bitwise_stop_parities(pcg, monkeypatch, mode):
    """max_iter 1..9 stops after every pass of the cycle; tolerances that converge at
    every position of the cycle; a warm start."""
    P = O.build_problem("C1", c=32)
    A, b = P["A"], P["B"][:, 0]
    Md, Me = _pair(pcg, monkeypatch, A, True, mode)
    for mi in range(1, 10):
        xd, sd, _ = _solve(Md, b, tol=1e-12, max_iter=mi)
        xe, se, _ = _solve(Me, b, tol=1e-12, max_iter=mi)
        assert sd == se == 1 and np.array_equal(xd, xe), mi
    its = set()
    for tol in (1e-2, 3e-3, 1e-3, 3e-4, 1e-4, 3e-5, 1e-5, 3e-6, 1e-6, 3e-7, 1e-7, 3e-8, 1e-8):
        xd, sd, infd = _solve(Md, b, tol=tol)
        xe, se, infe = _solve(Me, b, tol=tol)
        assert sd == se and infd["iterations"] == infe["iterations"] and np.array_equal(xd, xe), tol
        its.add(infd["iterations"] % int(mode))
    assert len(its) >= 2  # several positions of the cycle exercised
    x0 = np.random.default_rng(3).standard_normal(A.n)
    xd, _, infd = _solve(Md, b, tol=1e-10, x0=x0)
    xe, _, infe = _solve(Me, b, tol=1e-10, x0=x0)
    assert infd["iterations"] == infe["iterations"] and np.array_equal(xd, xe)


@pytest.mark.parametrize("mode", ["2", "4"])
def test_deferred_x_bitwise_replacement(pcg, monkeypatch, mode):
    """below attainable accuracy: replacements restart the deferred loop (p in p[0])"""
    P = O.build_problem("C1")
    A, b = P["A"], P["B"][:, 0]
    Md, Me = _pair(pcg, monkeypatch, A, True, mode)
    for mi in (397, 398, 399, 400):
        xd, sd, infd = _solve(Md, b, tol=1e-15, max_iter=mi)
        xe, se, infe = _solve(Me, b, tol=1e-15, max_iter=mi)
        assert sd == se == 1 and infd["replacements"] == infe["replacements"] >= 2
        assert np.array_equal(xd, xe)


@pytest.mark.parametrize("mode", ["2", "4"])
def test_deferred_x_bitwise_breakdown(pcg, monkeypatch, mode):
    """symmetric indefinite systems (C1 Laplacian - s I, random b): CG breaks down
    (NOT_SPD) at iterations of both parities (the oracle's count); x holds every applied
    update, bitwise the same on both paths"""
    import scipy.sparse as sp
    P = O.build_problem("C1", c=24)
    A0 = P["A"].to_scipy().tocsr()
    b = np.random.default_rng(1).standard_normal(A0.shape[0])
    lam = np.linalg.eigvalsh(A0.toarray())
    parities = set()
    for f in (0.0005, 0.001, 0.002, 0.005, 0.01, 0.02, 0.05, 0.1, 0.2, 0.3):
        s = lam[0] + f * (lam[-1] - lam[0])
        B = (A0 - s * sp.identity(A0.shape[0])).tocsr()
        B.sort_indices()
        C = O.Csr(B.shape[0], B.indptr, B.indices, B.data)
        r = O.pcg(C, b, tol=1e-12, max_iter=2000)
        assert r.status == O.ERR_NOT_SPD
        Md, Me = _pair(pcg, monkeypatch, C, True, mode)
        xd, sd, _ = _solve(Md, b, tol=1e-12, max_iter=2000)
        xe, se, _ = _solve(Me, b, tol=1e-12, max_iter=2000)
        assert sd == se == 7, (f, sd, se)  # PCG_ERR_NOT_SPD
        assert np.array_equal(xd, xe), f
        parities.add(r.iterations % int(mode))
    assert len(parities) >= 2


# ---------------------------------------------------------------- k right-hand sides (mk1a_deferred)
def _mpair(pcg, monkeypatch, A, k, mode="4"):
    out = []
    for xd in (mode, "0"):
        monkeypatch.setenv("PCG_XDEFER", xd)
        M = pcg.Matrix.from_csr(_dev(A.row_ptr), _dev(A.col), _dev(A.val), fmt="sell")
        _msolve(M, np.ones((A.n, k)), max_iter=3)  # builds the k-column loop graph under this env
        out.append(M)
    monkeypatch.delenv("PCG_XDEFER")
    return out


def _msolve(M, B, **kw):
    import torch
    from paper_2201_05413_b200 import PcgError
    X = torch.zeros((B.shape[1], B.shape[0]), dtype=torch.float64, device="cuda").t()  # column-major
    try:
        _, infos = M.solve_multi(_dev(B), out=X, **kw)
        st = [i["status"] for i in infos]
        its = [i["iterations"] for i in infos]
        reps = [i["replacements"] for i in infos]
    except PcgError as e:
        infos, st, its, reps = None, e.status, None, None
    return X.cpu().numpy(), st, its, reps


@pytest.mark.parametrize("mode", ["2", "4"])
def test_deferred_x_multi_bitwise(pcg, monkeypatch, mode):
    """C4's k = 16 Gaussian-bump columns converge at different iterations (549-578), so
    columns freeze after hold and after apply passes; max_iter odd and even; below
    attainable accuracy (per-column replacements).  X bitwise the every-iteration X."""
    P = O.build_problem("C4", c=16, k=16)
    A, B = P["A"], P["B"]
    Md, Me = _mpair(pcg, monkeypatch, A, 16, mode)
    xd, sd, itd, _ = _msolve(Md, B, tol=1e-10)
    xe, se, ite, _ = _msolve(Me, B, tol=1e-10)
    assert sd == se and itd == ite and np.array_equal(xd, xe)
    assert len({i % int(mode) for i in itd}) >= 2, itd  # frozen after several passes of the cycle
    for j in range(16):
        r = O.pcg(A, B[:, j], tol=1e-10)
        assert np.linalg.norm(xd[:, j] - r.x) / np.linalg.norm(r.x) <= 1e-9
    for mi in (5, 6, 7, 8):
        xd, _, _, _ = _msolve(Md, B, tol=1e-10, max_iter=mi)
        xe, _, _, _ = _msolve(Me, B, tol=1e-10, max_iter=mi)
        assert np.array_equal(xd, xe), mi
    xd, sd, itd, rd = _msolve(Md, B[:, :5], tol=1e-16, max_iter=251)
    xe, se, ite, re = _msolve(Me, B[:, :5], tol=1e-16, max_iter=251)
    assert rd == re and min(rd) >= 1 and np.array_equal(xd, xe)


@pytest.mark.parametrize("mode", ["2", "4"])
def test_deferred_x_multi_bitwise_breakdown(pcg, monkeypatch, mode):
    """indefinite C1 Laplacian - s I, k = 4 random columns: per-column breakdown at
    iterations of both parities; X bitwise the every-iteration X"""
    import scipy.sparse as sp
    P = O.build_problem("C1", c=24)
    A0 = P["A"].to_scipy().tocsr()
    lam = np.linalg.eigvalsh(A0.toarray())
    B = np.random.default_rng(2).standard_normal((A0.shape[0], 4))
    for f in (0.001, 0.01, 0.05):
        s = lam[0] + f * (lam[-1] - lam[0])
        Bm = (A0 - s * sp.identity(A0.shape[0])).tocsr()
        Bm.sort_indices()
        C = O.Csr(Bm.shape[0], Bm.indptr, Bm.indices, Bm.data)
        Md, Me = _mpair(pcg, monkeypatch, C, 4, mode)
        xd, sd, _, _ = _msolve(Md, B, tol=1e-12, max_iter=2000)
        xe, se, _, _ = _msolve(Me, B, tol=1e-12, max_iter=2000)
        assert sd == se and np.array_equal(xd, xe), f


@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 65, 97])
def test_deferred_x_tiny_and_ragged_graph_loop(pcg, monkeypatch, n):
    """the graph loop (one-chunk SpMV, x every 4th iteration) on tiny / ragged systems:
    n below one slice, odd n (the streaming passes' pair tail), a ragged last slice;
    bitwise the every-iteration x, and the oracle's solution"""
    rng = np.random.default_rng(n)
    T = np.diag(np.full(n, 2.5)) - np.diag(np.ones(n - 1), 1) - np.diag(np.ones(n - 1), -1) if n > 1 else np.eye(1) * 2.0
    A = O.Csr(n, *[np.asarray(v) for v in _csr_arrays(T)])
    b = rng.standard_normal(n)
    Md, Me = _pair(pcg, monkeypatch, A, True, "4")
    xd, sd, infd = _solve(Md, b, tol=1e-12)
    xe, se, infe = _solve(Me, b, tol=1e-12)
    assert sd == se == 0 and infd["iterations"] == infe["iterations"] and np.array_equal(xd, xe)
    r = O.pcg(A, b, tol=1e-12)
    assert np.linalg.norm(xd - r.x) <= 1e-9 * np.linalg.norm(r.x)
    for mi in (1, 2, 3, 5):
        xd, _, _ = _solve(Md, b, tol=1e-14, max_iter=mi)
        xe, _, _ = _solve(Me, b, tol=1e-14, max_iter=mi)
        assert np.array_equal(xd, xe), mi


def _csr_arrays(D):
    rp, cols, vals = [0], [], []
    for i in range(D.shape[0]):
        nz = np.nonzero(D[i])[0]
        cols += list(nz)
        vals += list(D[i, nz])
        rp.append(len(cols))
    return np.array(rp, dtype=np.int64), np.array(cols, dtype=np.int64), np.array(vals, dtype=np.float64)
