"""Full-size GPU parity at BASELINE.json's exact configs, in the launch configuration
bench.py times (device-generated system, PCG_FMT_AUTO, 3-pass schedule).

C1-C4: against tests/golden/oracle_full.json, written by oracle/make_golden.py (oracle
only): iterations within max(2 %, 1), x on 257 sampled indices within the 1e-9 bar,
||x||_2 within 1e-9 (a full-vector consequence of rel-L2 <= 1e-9), structure
(row_ptr at the sampled rows, n, nnz) exact.
C5 (133M unknowns, beyond the oracle's budget): properties that hold at any size:
true relres <= tol (recomputed by an independent SpMV), the solution against the
exact discrete solution by DST-I (closed-form spectrum of the lattice operator,
scipy on the host), the iteration count against the oracle's doubling ladder
(c = 32..256), and the CSR structure of sampled rows against the AXIS-policy
definition (free axis neighbours, values h*(6, -1)).
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "oracle_full.json")


def _gold():
    if not os.path.exists(GOLD):
        pytest.skip("oracle_full.json not generated")
    with open(GOLD) as fh:
        return json.load(fh)


@pytest.fixture(scope="module")
def pcg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_05413_b200 as p
    return p


@pytest.fixture(params=["default", "graph"])
def schedule(request, monkeypatch):
    """default: the library's own choice (the persistent kernel below 32M rows);
    graph: PCG_PERSIST=0, the conditional-WHILE graph schedule the C5 bench times."""
    for k in ("PCG_PERSIST", "PCG_SCHEDULE", "PCG_NO_GRAPH"):
        monkeypatch.delenv(k, raising=False)
    if request.param == "graph":
        monkeypatch.setenv("PCG_PERSIST", "0")
    return request.param


@pytest.mark.parametrize("name", ["C1", "C2", "C4", "C3", "C6"])
def test_fullsize_vs_oracle_golden(pcg, name, schedule):
    _golden_case(pcg, name)


def _golden_case(pcg, name, key=None, c=None):
    g = _gold()
    key = key or name
    if key not in g:
        pytest.skip(f"{key} golden not generated")
    g = g[key]
    spec = pcg.fem_spec(name, c=c) if c else pcg.fem_spec(name)
    P = pcg.fem_build(spec)
    n = P["row_ptr"].numel() - 1
    assert n == g["n"] and P["col"].numel() == g["nnz"]
    idx = np.array(g["sample_idx"])
    assert np.array_equal(P["row_ptr"].cpu().numpy()[idx], g["row_ptr_sample"])
    A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
    B = P["B"]
    cfg = pcg.problems.configs()[name]
    if B.shape[1] == 1:
        x, info = A.solve(B[:, 0].contiguous(), tol=cfg["tol"], max_iter=cfg["max_iter"])
        X, infos = x[:, None], [info]
    else:
        X, infos = A.solve_multi(B, tol=cfg["tol"], max_iter=cfg["max_iter"])
    X = X.cpu().numpy()
    for j, ref in enumerate(g["rhs"]):
        info = infos[j]
        assert info["status"] == 0 and info["relres_true"] <= cfg["tol"]
        assert abs(info["iterations"] - ref["iterations"]) <= max(1, 0.02 * ref["iterations"]), \
            (j, info["iterations"], ref["iterations"])
        xs, xo = X[idx, j], np.array(ref["x_sample"])
        assert np.linalg.norm(xs - xo) <= 1e-9 * np.linalg.norm(xo), j
        assert abs(np.linalg.norm(X[:, j]) - ref["x_norm"]) <= 1e-9 * ref["x_norm"]


def test_c5_c256_vs_oracle_golden(pcg, schedule):
    """The C5 construction at c = 256 (16.6M unknowns, 116M nnz) against the oracle's
    solve through the standard pipeline (tests/golden oracle_full.json "C5c256")."""
    _golden_case(pcg, "C5", key="C5c256", c=256)


def test_c5_fullsize_vs_oracle_golden(pcg, monkeypatch):
    """C5 itself (c = 512, 133M unknowns, 932M nnz) in the launch configuration
    bench.py times (device generator, PCG_FMT_AUTO, n > 32M -> the graph schedule)
    against the oracle's full-size solve ("C5full": orc_assemble_free_lattice, bitwise
    the standard pipeline, + orc_pcg): iterations within max(2 %, 1), x on 257
    sampled entries and ||x|| within 1e-9, structure at the sampled rows exact."""
    for k in ("PCG_PERSIST", "PCG_SCHEDULE", "PCG_NO_GRAPH"):
        monkeypatch.delenv(k, raising=False)
    _golden_case(pcg, "C5", key="C5full")


def test_c5_fullsize_properties(pcg):
    import torch
    from scipy.fft import dstn, idstn
    name = "C5"
    cfg = pcg.problems.configs()[name]
    c = cfg["c"]
    m, h = c - 1, 1.0 / c
    spec = pcg.fem_spec(name)
    P = pcg.fem_build(spec)
    n = m ** 3
    assert P["row_ptr"].numel() == n + 1 and P["col"].numel() == 7 * m ** 3 - 6 * m ** 2
    # sampled rows: AXIS pattern and lattice values h*(6, -1)
    rp = P["row_ptr"]
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([[0, n - 1, n // 2, m * m - 1], rng.integers(0, n, 300)]))
    for r in rows:
        s, e = int(rp[r]), int(rp[r + 1])
        cols = P["col"][s:e].cpu().numpy()
        vals = P["val"][s:e].cpu().numpy()
        i, j, k = r % m, (r // m) % m, r // (m * m)
        want = []
        for dk, dj, di in [(-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0), (0, 0, 1), (0, 1, 0), (1, 0, 0)]:
            a, b_, cc = i + di, j + dj, k + dk
            if 0 <= a < m and 0 <= b_ < m and 0 <= cc < m:
                want.append(a + m * (b_ + m * cc))
        assert cols.tolist() == want
        assert np.allclose(vals, np.where(cols == r, 6 * h, -h), rtol=1e-14, atol=0)
    A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
    b = P["B"][:, 0].contiguous()
    del P
    x, info = A.solve(b, tol=cfg["tol"], max_iter=cfg["max_iter"])
    assert info["status"] == 0 and info["relres_true"] <= cfg["tol"]
    # independent true residual: SpMV through the library on the final x
    r = b - A.spmv(x)
    assert float(torch.linalg.norm(r) / torch.linalg.norm(b)) <= cfg["tol"] * (1 + 1e-6)
    # iteration count vs the oracle's ladder (ratio per doubling of c: 2.07, 1.97, 1.95)
    g = _gold().get("C5ladder")
    if g:
        ratio = info["iterations"] / g["256"]["iterations"]
        assert 1.85 <= ratio <= 2.0, ratio
    # exact discrete solution by DST-I (K = h * sum of three 1D second differences)
    bh = b.cpu().numpy().reshape(m, m, m)
    jj = np.arange(1, m + 1)
    l1 = 2 - 2 * np.cos(jj * np.pi / c)
    lam = h * (l1[None, None, :] + l1[None, :, None] + l1[:, None, None])
    xe = idstn(dstn(bh, type=1, workers=-1) / lam, type=1, workers=-1).ravel()
    xg = x.cpu().numpy()
    assert np.linalg.norm(xg - xe) / np.linalg.norm(xe) <= 1e-8
