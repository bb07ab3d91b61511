"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same
seeded inputs.  Tolerances:
  * integer structure (row_ptr, col, partitions): bit-exact;
  * SpMV: |y_gpu - y_orc|_i <= 2 nnz_i u Σ_j |a_ij x_j|  (forward error of any
    summation order, u = 2^-53);
  * PCG: rel-L2(x_gpu, x_orc) <= 1e-9, true relres <= tol, iterations within
    max(2%, 1) of the oracle (north_star).
"""
import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


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


def torch_cpu(a):
    import torch
    return torch.as_tensor(np.ascontiguousarray(a))


def _matrix(pcg, A, fmt="auto"):
    return pcg.Matrix.from_csr(_dev(A.row_ptr), _dev(A.col), _dev(A.val), fmt=fmt)


def _spmv_bound(A, x):
    absx = np.abs(x)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    mag = np.bincount(rows, weights=np.abs(A.val) * absx[A.col], minlength=A.n)
    ln = np.diff(A.row_ptr)
    return 2 * ln * U * mag + 1e-300


CASES = [("C1", None), ("C2", 96), ("C3", 48), ("C5", 32), ("C4", 16), ("C6", 20)]


@pytest.mark.parametrize("name,c", CASES)
@pytest.mark.parametrize("fmt", ["auto", "csr", "sell", "tma", "sigma"])
def test_spmv_parity(pcg, name, c, fmt):
    P = O.build_problem(name, c=c, k=1)
    A = P["A"]
    M = _matrix(pcg, A, fmt)
    x = np.random.default_rng(7).standard_normal(A.n)
    y = M.spmv(_dev(x)).cpu().numpy()
    yo = O.spmv(A, x)
    assert np.all(np.abs(y - yo) <= _spmv_bound(A, x))
    if fmt != "auto":
        assert M.stats()["format"] == {"csr": 1, "sell": 2, "tma": 3, "sigma": 4}[fmt]
    if fmt == "sigma":  # rows keep their entry order: bitwise the natural SELL SpMV
        ys = _matrix(pcg, A, "sell").spmv(_dev(x)).cpu().numpy()
        assert np.array_equal(y, ys)
        yh = M.spmv(torch_cpu(x)).numpy()  # host pointers through the permutation
        assert np.array_equal(yh, y)


@pytest.mark.parametrize("name,c", CASES)
def test_pcg_parity(pcg, name, c):
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()[name]["tol"]
    r = O.pcg(A, b, tol=tol)
    assert r.status == O.OK
    M = _matrix(pcg, A)
    x, info = M.solve(_dev(b), tol=tol)
    x = x.cpu().numpy()
    assert info["status"] == 0, info
    assert info["relres_true"] <= tol
    rel = np.linalg.norm(x - r.x) / np.linalg.norm(r.x)
    assert rel <= 1e-9, rel
    assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations), (info["iterations"], r.iterations)
    # the true residual reported by the GPU agrees with the oracle's definition
    t = np.linalg.norm(b - A.to_scipy() @ x) / np.linalg.norm(b)
    assert abs(t - info["relres_true"]) <= 1e-3 * tol


@pytest.mark.parametrize("fmt", ["csr", "sell", "tma"])
def test_pcg_both_formats_and_determinism(pcg, fmt):
    P = O.build_problem("C2", c=64)
    M = _matrix(pcg, P["A"], fmt)
    b = _dev(P["B"][:, 0])
    x1, i1 = M.solve(b)
    x2, i2 = M.solve(b)
    assert i1["iterations"] == i2["iterations"]
    assert bool((x1 == x2).all()), "solve must be bitwise reproducible"


def test_pcg_host_pointers_equal_device(pcg):
    P = O.build_problem("C1", c=32)
    M = _matrix(pcg, P["A"])
    import torch
    b = torch.as_tensor(P["B"][:, 0])
    xh, ih = M.solve(b)  # host tensors (staged by the library)
    xd, idv = M.solve(b.cuda())
    assert xh.device.type == "cpu"
    assert ih["iterations"] == idv["iterations"]
    assert np.array_equal(xh.numpy(), xd.cpu().numpy())


def test_pcg_x0_warm_start_and_zero_rhs(pcg):
    P = O.build_problem("C1", c=32)
    A, b = P["A"], P["B"][:, 0]
    M = _matrix(pcg, A)
    r = O.pcg(A, b, tol=1e-12)
    x, info = M.solve(_dev(b), x0=_dev(r.x), tol=1e-10)  # already converged: 0 iterations
    assert info["iterations"] == 0 and info["status"] == 0
    x, info = M.solve(_dev(np.zeros(A.n)), x0=_dev(np.ones(A.n)))
    assert info["iterations"] == 0 and info["status"] == 0 and float(x.abs().max()) == 0.0
    # warm start from a partial solve matches the oracle from the same x0
    x0 = O.pcg(A, b, tol=1e-3).x
    ro = O.pcg(A, b, x0=x0, tol=1e-10)
    x, info = M.solve(_dev(b), x0=_dev(x0), tol=1e-10)
    assert abs(info["iterations"] - ro.iterations) <= max(1, 0.02 * ro.iterations)
    assert np.linalg.norm(x.cpu().numpy() - ro.x) / np.linalg.norm(ro.x) <= 1e-9


def test_pcg_max_iter_not_converged(pcg):
    P = O.build_problem("C1", c=32)
    A, b = P["A"], P["B"][:, 0]
    M = _matrix(pcg, A)
    ro = O.pcg(A, b, tol=1e-10, max_iter=7)
    x, info = M.solve(_dev(b), tol=1e-10, max_iter=7)
    assert info["status"] == 1 and info["iterations"] == 7 and ro.status == O.NOT_CONVERGED
    assert np.linalg.norm(x.cpu().numpy() - ro.x) / np.linalg.norm(ro.x) <= 1e-12


def _csr(D):
    n = D.shape[0]
    rp, cols, vals = [0], [], []
    for i in range(n):
        nz = np.nonzero(D[i])[0]
        cols += list(nz)
        vals += list(D[i, nz])
        rp.append(len(cols))
    return O.Csr(n, rp, cols, vals)


def test_error_paths(pcg):
    from paper_2201_05413_b200 import PcgError
    bad = {
        "unsorted": (np.array([0, 2, 3]), np.array([1, 0, 1]), np.array([1., 2., 3.]), 4),
        "out_of_range": (np.array([0, 1, 2]), np.array([0, 5]), np.array([1., 1.]), 3),
        "dim": (np.array([0, 2, 1]), np.array([0, 1]), np.array([1., 1.]), 5),
        "zero_diag": (np.array([0, 1, 2]), np.array([1, 1]), np.array([1., 1.]), 6),
        "neg_diag": (np.array([0, 1, 2]), np.array([0, 1]), np.array([-1., 1.]), 7),
        "nan": (np.array([0, 1, 2]), np.array([0, 1]), np.array([np.nan, 1.]), 8),
    }
    for what, (rp, ci, va, code) in bad.items():
        with pytest.raises(PcgError) as e:
            pcg.Matrix.from_csr(_dev(rp), _dev(ci), _dev(va))
        assert e.value.status == code, what
    # indefinite matrix with positive diagonal: CG breakdown -> NOT_SPD
    M = _matrix(pcg, _csr(np.array([[1., 3.], [3., 1.]])))
    with pytest.raises(PcgError) as e:
        M.solve(_dev(np.array([1., 0.])))
    assert e.value.status == 7
    # non-finite right-hand side
    M = _matrix(pcg, _csr(np.diag([2., 3., 4.])))
    with pytest.raises(PcgError) as e:
        M.solve(_dev(np.array([1., np.inf, 0.])))
    assert e.value.status == 8
    # diagonal / identity: one iteration
    x, info = M.solve(_dev(np.array([2., 3., 4.])))
    assert info["iterations"] == 1 and np.allclose(x.cpu().numpy(), 1.0)


def test_empty_and_tiny(pcg):
    M = _matrix(pcg, _csr(np.array([[4.0]])))
    x, info = M.solve(_dev(np.array([2.0])))
    assert info["iterations"] == 1 and float(x[0]) == 0.5
    M = _matrix(pcg, O.Csr(0, [0], [], []))
    x, info = M.solve(_dev(np.zeros(0)))
    assert info["iterations"] == 0


@pytest.mark.parametrize("k", [1, 3, 16])
def test_multi_rhs_parity(pcg, k):
    P = O.build_problem("C4", c=32, k=max(k, 1))
    A, B = P["A"], P["B"][:, :k]
    M = _matrix(pcg, A)
    X, infos = M.solve_multi(_dev(B), tol=1e-10)
    X = X.cpu().numpy()
    for j in range(k):
        r = O.pcg(A, B[:, j], tol=1e-10)
        assert infos[j]["status"] == 0 and infos[j]["relres_true"] <= 1e-10
        assert np.linalg.norm(X[:, j] - r.x) / np.linalg.norm(r.x) <= 1e-9
        assert abs(infos[j]["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)


def test_multi_rhs_frozen_columns_and_zero_column(pcg):
    """Columns converge at different iterations and freeze; a zero column gives x = 0."""
    P = O.build_problem("C1", c=48)
    A = P["A"]
    rng = np.random.default_rng(3)
    B = np.column_stack([P["B"][:, 0], np.zeros(A.n), rng.standard_normal(A.n), 1e-3 * P["B"][:, 0]])
    M = _matrix(pcg, A)
    X, infos = M.solve_multi(_dev(B), tol=1e-10)
    X = X.cpu().numpy()
    assert infos[1]["iterations"] == 0 and np.all(X[:, 1] == 0)
    its = []
    for j in (0, 2, 3):
        r = O.pcg(A, B[:, j], tol=1e-10)
        its.append(r.iterations)
        assert abs(infos[j]["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
        assert np.linalg.norm(X[:, j] - r.x) / np.linalg.norm(r.x) <= 1e-9
    assert len(set(its)) > 1  # the columns really froze at different steps


@pytest.mark.parametrize("name,c", [("C1", 64), ("C2", 64), ("C3", 32), ("C4", 16), ("C5", 32), ("C6", 16)])
def test_generator_structure_parity(pcg, name, c):
    """GPU FEM assembly: CSR structure bit-exact vs the oracle; values and RHS within
    a few ulps of the row magnitude (different but equivalent summation)."""
    spec = pcg.fem_spec(name, c=c)
    G = pcg.fem_build(spec)
    P = O.build_problem(name, c=c)
    A = P["A"]
    assert np.array_equal(G["row_ptr"].cpu().numpy(), A.row_ptr)
    assert np.array_equal(G["col"].cpu().numpy(), A.col)
    val = G["val"].cpu().numpy()
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    rowmax = np.zeros(A.n)
    np.maximum.at(rowmax, rows, np.abs(A.val))
    assert np.all(np.abs(val - A.val) <= 64 * U * rowmax[rows])
    B = G["B"].cpu().numpy()
    assert B.shape == P["B"].shape
    scale = np.max(np.abs(P["B"]), axis=0)
    assert np.all(np.abs(B - P["B"]) <= 1e-12 * scale[None, :])


@pytest.mark.parametrize("name,c", [("C3", 48), ("C2", 64), ("C1", None)])
def test_sigma_pcg_parity(pcg, name, c):
    """SELL-C-sigma (symmetric permutation P A P^T inside the library) against the oracle;
    host and device pointers; multi-RHS through the same permuted handle."""
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()[name]["tol"]
    r = O.pcg(A, b, tol=tol)
    M = _matrix(pcg, A, "sigma")
    st = M.stats()
    assert st["format"] == 4 and st["sigma"] >= 64
    for bb in (_dev(b), torch_cpu(b)):
        x, info = M.solve(bb, tol=tol)
        x = x.cpu().numpy()
        assert info["status"] == 0 and info["relres_true"] <= tol
        assert np.linalg.norm(x - r.x) / np.linalg.norm(r.x) <= 1e-9
        assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
    rng = np.random.default_rng(1)
    B = np.column_stack([b, rng.standard_normal(A.n), np.zeros(A.n)])
    X, infos = M.solve_multi(_dev(B), tol=tol)
    X = X.cpu().numpy()
    assert infos[2]["iterations"] == 0 and np.all(X[:, 2] == 0)
    for j in range(2):
        rj = O.pcg(A, B[:, j], tol=tol)
        assert np.linalg.norm(X[:, j] - rj.x) / np.linalg.norm(rj.x) <= 1e-9
        assert abs(infos[j]["iterations"] - rj.iterations) <= max(1, 0.02 * rj.iterations)


def test_host_out_not_pinned_receives_the_solution(pcg):
    """a non-pinned host `out` is staged through pinned memory and must hold
    x on return (solve, solve_multi)."""
    import torch
    P = O.build_problem("C1", c=32)
    A, b = P["A"], P["B"][:, 0]
    M = _matrix(pcg, A)
    out = torch.zeros(A.n, dtype=torch.float64)
    x, info = M.solve(torch.as_tensor(b), out=out)
    assert x is out and info["status"] == 0
    xd, _ = M.solve(_dev(b))
    assert np.array_equal(out.numpy(), xd.cpu().numpy())
    B = np.column_stack([b, 2 * b])
    outk = torch.zeros(2, A.n, dtype=torch.float64).t()  # (n, 2) column-major
    X, infos = M.solve_multi(torch.as_tensor(B), out=outk)
    assert X.data_ptr() == outk.data_ptr()
    Xd, _ = M.solve_multi(_dev(B))  # the same multi-RHS solve from device buffers
    assert np.array_equal(outk.numpy(), Xd.cpu().numpy())


@pytest.mark.parametrize("name,c", [("C3", 48), ("C2", 96), ("C6", 20)])
def test_format_choice_is_deterministic(pcg, name, c):
    """pcg.h: identical inputs give bitwise-identical results — the AUTO format rule
    depends on the pattern only, so two handles of one matrix agree exactly."""
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    M1, M2 = _matrix(pcg, A), _matrix(pcg, A)
    s1, s2 = M1.stats(), M2.stats()
    assert (s1["format"], s1["sigma"]) == (s2["format"], s2["sigma"])
    x1, i1 = M1.solve(_dev(b))
    x2, i2 = M2.solve(_dev(b))
    assert i1["iterations"] == i2["iterations"] and bool((x1 == x2).all())


@pytest.mark.parametrize("name,c,fmt", [("C5", 32, "auto"), ("C4", 24, "sell"), ("C3", 40, "sigma"), ("C2", 64, "sell"),
                                        ("C6", 16, "sell")])
def test_d16_column_form_is_bitwise_the_int32_form(pcg, monkeypatch, name, c, fmt):
    """The 16-bit delta column ids (pcg.h d16_slices) decode to the same ids as the
    int32 SELL array, so SpMV, single- and multi-RHS solves are bitwise identical with
    and without them, and match the oracle.  The int32 handle runs the same chunked
    engine and grid (PCG_SHORT=0): the one-chunk engines visit slices in another order,
    so their dot products round differently."""
    P = O.build_problem(name, c=c, k=2 if name == "C4" else 1)
    A = P["A"]
    monkeypatch.delenv("PCG_NO_D16", raising=False)
    monkeypatch.setenv("PCG_D16", "1")
    M1 = _matrix(pcg, A, fmt)
    monkeypatch.delenv("PCG_D16")
    monkeypatch.setenv("PCG_SHORT", "0")
    M0 = _matrix(pcg, A, fmt)
    monkeypatch.delenv("PCG_SHORT")
    s1, s0 = M1.stats(), M0.stats()
    assert s0["d16_slices"] == 0
    assert s1["d16_slices"] > 0.5 * ((A.n + 31) // 32), s1
    x = np.random.default_rng(11).standard_normal(A.n)
    y1, y0 = M1.spmv(_dev(x)).cpu().numpy(), M0.spmv(_dev(x)).cpu().numpy()
    assert np.array_equal(y1, y0)
    assert np.all(np.abs(y1 - O.spmv(A, x)) <= _spmv_bound(A, x))
    b = P["B"][:, 0]
    x1, i1 = M1.solve(_dev(b))
    x0, i0 = M0.solve(_dev(b))
    assert i1["iterations"] == i0["iterations"] and bool((x1 == x0).all())
    if P["B"].shape[1] > 1:
        X1, _ = M1.solve_multi(_dev(P["B"]))
        X0, _ = M0.solve_multi(_dev(P["B"]))
        assert bool((X1 == X0).all())


@pytest.mark.parametrize("name,c", [("C1", None), ("C2", 40), ("C4", 12), ("C5", 24)])
def test_short_row_engine_is_bitwise_the_chunked_engine(pcg, monkeypatch, name, c):
    """Rows of at most 8 entries (the lattice P1 systems) run the one-chunk SELL engine
    (pcg.h short_rows): the same entries summed in the same order, so the SpMV is
    bitwise the chunked engine's (PCG_SHORT=0); the graph-loop solve (the C5 bench
    path) meets the oracle bars with it; C3 (P2, up to 19 entries) keeps the chunked one."""
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    monkeypatch.setenv("PCG_PERSIST", "0")
    monkeypatch.setenv("PCG_SHORT", "0")
    M0 = _matrix(pcg, A, "sell")
    monkeypatch.delenv("PCG_SHORT")
    M1 = _matrix(pcg, A, "sell")
    assert M0.stats()["short_rows"] == 0 and M1.stats()["short_rows"] == 1
    x = np.random.default_rng(12).standard_normal(A.n)
    y1, y0 = M1.spmv(_dev(x)).cpu().numpy(), M0.spmv(_dev(x)).cpu().numpy()
    assert np.array_equal(y1, y0)
    tol = O.configs()[name]["tol"]
    r = O.pcg(A, b, tol=tol)
    xs, info = M1.solve(_dev(b), tol=tol)
    assert info["status"] == 0 and info["relres_true"] <= tol
    assert np.linalg.norm(xs.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-9
    assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
    P3 = O.build_problem("C3", c=16, k=1)
    assert _matrix(pcg, P3["A"], "sell").stats()["short_rows"] == 0


def _banded_mix(n, seed):
    """SPD, rows of <= 7 entries: a 5-point-like band (uniform offsets per slice
    position) on the first half, random extra couplings on the second (non-uniform)"""
    rng = np.random.default_rng(seed)
    D = np.zeros((n, n))
    for i in range(n):
        for d in (-40, -1, 1, 40):
            if 0 <= i + d < n:
                D[i, i + d] = -1.0
    for i in range(n // 2, n):
        j = int(rng.integers(0, n))
        if j != i and np.count_nonzero(D[i]) < 5 and np.count_nonzero(D[j]) < 5:
            D[i, j] = D[j, i] = -0.5
    D += np.diag(np.abs(D).sum(1) + 1.0)
    return _csr(D)


def _grid_values(m, seed):
    """5-point Laplacian on an m x m grid (m > 32: slices inside a grid line are one-trip
    and value-uniform) with every 37th x-coupling scaled by 0.75 (symmetric, diagonally
    dominant): one-trip slices whose values are not uniform, and boundary slices that
    are not one-trip"""
    n = m * m
    M = np.zeros((n, n))
    for i in range(n):
        x, y = i % m, i // m
        for dx, dy in ((-1, 0), (1, 0), (0, -1), (0, 1)):
            if 0 <= x + dx < m and 0 <= y + dy < m:
                M[i, i + dx + m * dy] = -1.0
        M[i, i] = 4.0
    for i in range(0, n - 1, 37):
        if (i + 1) % m:
            M[i, i + 1] = M[i + 1, i] = -0.75
    return _csr(M)


@pytest.mark.parametrize("name,c", [("C1", None), ("C1", 512), ("C5", 32), ("C5", 64), ("C4", 16), ("mix", 900),
                                    ("mixv", 70)])
def test_uniform_offset_positions_are_bitwise_the_id_form(pcg, monkeypatch, name, c):
    """The one-chunk engine's id-free uniform-offset positions (pcg.h dia_positions)
    and value-uniform slices (pcg.h dval_slices): the same columns and values, so the
    SpMV is bitwise the id form (PCG_DIA=0), the value-stream form (PCG_DIA_VAL=0) and
    the chunked engine (PCG_SHORT=0); the graph-loop solve meets the oracle bars; a
    pattern mixing uniform and non-uniform slices takes every path of the engine."""
    if name in ("mix", "mixv"):
        A = _banded_mix(c, 5) if name == "mix" else _grid_values(c, 5)
        b = np.random.default_rng(6).standard_normal(A.n)
        tol = 1e-10
    else:
        P = O.build_problem(name, c=c, k=1)
        A, b = P["A"], P["B"][:, 0]
        tol = O.configs()[name]["tol"]
    monkeypatch.setenv("PCG_PERSIST", "0")
    hs = {}
    knobs = ("PCG_DIA", "PCG_SHORT", "PCG_DIA_VAL", "PCG_DIA_PAT", "PCG_DIA_ALIGN")
    for key, env in (("dia", {}), ("ids", {"PCG_DIA": "0"}), ("chunked", {"PCG_SHORT": "0"}),
                     ("novals", {"PCG_DIA_VAL": "0"}), ("nopat", {"PCG_DIA_PAT": "0"}),
                     ("noalign", {"PCG_DIA_ALIGN": "0"})):
        for k in knobs:
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        hs[key] = _matrix(pcg, A, "sell")
    for k in knobs:
        monkeypatch.delenv(k, raising=False)
    st = hs["dia"].stats()
    n_slices = (A.n + 31) // 32
    assert st["short_rows"] == 1 and 0 < st["dia_positions"] <= 8 * n_slices, st
    assert hs["ids"].stats()["dia_positions"] == 0
    # lattice stencils and the constant band: value-uniform one-trip slices exist; the
    # scaled couplings of mixv leave some one-trip slices reading their values
    # (below c = 64 every 32-row slice of a lattice meets a boundary row: only the aligned
    # form, positions = the union of the rows' offsets, makes such slices one-trip)
    assert st["aligned_slices"] <= st["dval_slices"] <= st["dia_slices"], st
    if name in ("mixv", "C5", "C1"):
        assert st["aligned_slices"] > 0, st
    if name == "mixv" or (name == "C5" and c >= 64):
        assert st["dval_slices"] > st["aligned_slices"], st
    assert hs["noalign"].stats()["aligned_slices"] == 0
    if name == "mixv":
        assert st["dval_slices"] < st["dia_slices"], st
    # the value-free slices read a shared pattern (a lattice has a handful: interior, faces)
    assert st["pat_slices"] <= st["dval_slices"] and st["npat"] <= 32, st
    if st["dval_slices"] > st["aligned_slices"]:  # (aligned slices keep their own zero masks)
        assert st["pat_slices"] > 0 and st["npat"] > 0, st
    assert hs["nopat"].stats()["pat_slices"] == 0 and hs["nopat"].stats()["dval_slices"] == st["dval_slices"]
    assert hs["novals"].stats()["dval_slices"] == 0 and hs["novals"].stats()["pat_slices"] == 0
    assert hs["novals"].stats()["dia_slices"] == st["dia_slices"] - st["aligned_slices"]
    x = np.random.default_rng(12).standard_normal(A.n)
    ys = {k: M.spmv(_dev(x)).cpu().numpy() for k, M in hs.items()}
    for k in ("ids", "chunked", "novals", "nopat", "noalign"):
        assert np.array_equal(ys["dia"], ys[k]), k
    # the multi-RHS SpMM reads the shared patterns too: bitwise the stream form
    B3 = np.random.default_rng(13).standard_normal((A.n, 3))
    X3 = {k: hs[k].solve_multi(_dev(B3), tol=1e-8)[0].cpu().numpy() for k in ("dia", "nopat", "ids")}
    assert np.array_equal(X3["dia"], X3["nopat"]) and np.array_equal(X3["dia"], X3["ids"])
    r = O.pcg(A, b, tol=tol)
    xs, info = hs["dia"].solve(_dev(b), tol=tol)
    assert info["status"] == 0 and info["relres_true"] <= tol
    assert np.linalg.norm(xs.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-9
    assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)


@pytest.mark.parametrize("k", [1, 5, 16])
def test_windowed_spmm_multi_rhs_parity(pcg, monkeypatch, k):
    """The multi-RHS SpMM with TMA-staged column windows (pcg.h spmm_windowed): the plan
    is built for the lattice system (opt-in, PCG_SPMM_WIN=1), and every column matches the
    oracle's single-RHS solve within the north_star bars; PCG_SPMM_WIN=0 keeps the
    register-gather SpMM."""
    P = O.build_problem("C4", c=40, k=k)
    A, B = P["A"], P["B"]
    monkeypatch.setenv("PCG_SPMM_WIN", "1")
    M = _matrix(pcg, A)
    X, infos = M.solve_multi(_dev(B), tol=1e-10)
    assert M.stats()["spmm_windowed"] == 1
    X = X.cpu().numpy()
    for j in range(k):
        r = O.pcg(A, B[:, j], tol=1e-10)
        assert infos[j]["status"] == 0 and infos[j]["relres_true"] <= 1e-10
        assert np.linalg.norm(X[:, j] - r.x) / np.linalg.norm(r.x) <= 1e-9
        assert abs(infos[j]["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
    monkeypatch.setenv("PCG_SPMM_WIN", "0")
    M0 = _matrix(pcg, A)
    X0, infos0 = M0.solve_multi(_dev(B), tol=1e-10)
    assert M0.stats()["spmm_windowed"] == -1
    assert np.linalg.norm(X0.cpu().numpy() - X) <= 1e-9 * np.linalg.norm(X)


def test_multi_rhs_chunking_and_leading_dimensions(pcg):
    """pcg.h pcg_solve_multi promises k > 32 (chunked internally by 32 columns) and
    leading dimensions ldb, ldx > n (column-major, SPEC DenseBlock S:39-42): called
    through the raw C ABI with k = 37 columns in padded host and device buffers, every
    column matches its own oracle solve, and the padding rows are left untouched."""
    import ctypes as C
    import torch
    from paper_2201_05413_b200 import _lib
    P = O.build_problem("C1", c=24)
    A = P["A"]
    n, k, ldb, ldx = A.n, 37, A.n + 5, A.n + 11
    rng = np.random.default_rng(4)
    B = rng.standard_normal((n, k))
    Bp = np.full((k, ldb), 7.0)
    Bp[:, :n] = B.T
    M = _matrix(pcg, A)
    for dev in (False, True):
        Xp = np.full((k, ldx), -3.0)
        tb = torch.as_tensor(Bp).contiguous()
        tx = torch.as_tensor(Xp).contiguous()
        if dev:
            tb, tx = tb.cuda(), tx.cuda()
        else:
            tb, tx = tb.pin_memory(), tx.pin_memory()
        tx[:, :n] = 0.0
        infos = (_lib.PcgInfo * k)()
        st = _lib.lib().pcg_solve_multi(M._h, k, C.c_void_p(tb.data_ptr()), ldb, C.c_void_p(tx.data_ptr()), ldx,
                                        1e-10, 50000, C.c_void_p(torch.cuda.current_stream().cuda_stream), infos)
        assert st == 0
        X = tx.cpu().numpy()
        assert np.all(X[:, n:] == -3.0)  # padding untouched
        for j in (0, 1, 31, 32, 36):
            r = O.pcg(A, B[:, j], tol=1e-10)
            assert infos[j].status == 0
            assert np.linalg.norm(X[j, :n] - r.x) / np.linalg.norm(r.x) <= 1e-9
            assert abs(infos[j].iterations - r.iterations) <= max(1, 0.02 * r.iterations)


@pytest.mark.parametrize("name,c", [("C5", 64), ("C1", 512), ("C3", 48), ("C2", 96)])
def test_dinv_slices_are_bitwise_the_per_row_dinv(pcg, monkeypatch, name, c):
    """K2 reads one dinv per 32-row slice where the slice's 32 entries are equal (a
    lattice's Jacobi diagonal; SolveWork::dslice): the same values, so the graph-loop
    solve is bitwise the per-row form (PCG_DINV_SLICE=0) — also on systems without such
    slices (C2 jittered, C3 P2 and SELL-C-sigma permuted) and after the format choice
    permuted dinv."""
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()[name]["tol"]
    monkeypatch.setenv("PCG_PERSIST", "0")
    out = {}
    for key, env in (("slice", None), ("row", "0")):
        if env is None:
            monkeypatch.delenv("PCG_DINV_SLICE", raising=False)
        else:
            monkeypatch.setenv("PCG_DINV_SLICE", env)
        M = _matrix(pcg, A)
        out[key] = M.solve(_dev(b), tol=tol)
        B2 = np.stack([b, np.random.default_rng(7).standard_normal(A.n)], axis=1)
        out[key + "_k"] = M.solve_multi(_dev(B2), tol=1e-8)[0].cpu().numpy()  # the multi-RHS K2 too
    monkeypatch.delenv("PCG_DINV_SLICE", raising=False)
    assert np.array_equal(out["slice_k"], out["row_k"])
    (xs, infs), (xr, infr) = out["slice"], out["row"]
    assert infs["status"] == 0 and infs["iterations"] == infr["iterations"]
    assert np.array_equal(xs.cpu().numpy(), xr.cpu().numpy())
    r = O.pcg(A, b, tol=tol)
    assert np.linalg.norm(xs.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-9
