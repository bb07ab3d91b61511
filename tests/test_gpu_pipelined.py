"""GPU parity for the pipelined Jacobi-PCG (pcg_solve_pipelined; SURVEY §8(f) N3,
DESIGN.md reading R4) against the oracle (oracle.c orc_pcg_pipelined).

Bars: true relres <= tol; solution within 1e-8 (relative) of the oracle's pipelined
solution AND of its standard PCG solution (both solve the same system to 1e-10);
iterations within max(2, 3 %) of the oracle's where no restart occurs (C1, C2, C4,
C6).  The P2 system C3 sits at pipelined CG's stability edge: there the recurrences
drift, alpha turns <= 0 and the solve restarts (reading R4) at rounding-sensitive
points — the oracle needs 154 steps at c = 32 (PCG 153) and 522 at c = 64 (PCG 297),
and a different summation order (SELL-C-sigma) moves the restarts.  For C3 the bar
is convergence to the same solution with a count between 0.9 x PCG's and 2 x the
oracle's.
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


def _solve(pcg, name, c, fmt="auto"):
    import torch
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    M = pcg.Matrix.from_csr(torch.as_tensor(A.row_ptr).cuda(), torch.as_tensor(A.col).cuda(),
                            torch.as_tensor(A.val).cuda(), fmt=fmt)
    return A, b, M


@pytest.mark.parametrize("name,c,fmt", [("C1", None, "auto"), ("C2", 64, "auto"), ("C4", 32, "auto"),
                                        ("C6", 16, "auto"), ("C1", None, "csr")])
def test_pipelined_parity(pcg, name, c, fmt):
    import torch
    A, b, M = _solve(pcg, name, c, fmt)
    tol = O.configs()[name]["tol"]
    ro = O.pcg_pipelined(A, b, tol=tol)
    rc = O.pcg(A, b, tol=tol)
    for bb in (torch.as_tensor(b).cuda(), torch.as_tensor(b)):
        x, info = M.solve_pipelined(bb, tol=tol)
        x = x.cpu().numpy()
        assert info["status"] == 0 and info["relres_true"] <= tol
        assert np.linalg.norm(x - ro.x) <= 1e-8 * np.linalg.norm(ro.x)
        assert np.linalg.norm(x - rc.x) <= 1e-8 * np.linalg.norm(rc.x)
        assert abs(info["iterations"] - ro.iterations) <= max(2, 0.03 * ro.iterations), (info, ro.iterations)


@pytest.mark.parametrize("c,fmt", [(32, "sigma"), (32, "sell"), (64, "auto")])
def test_pipelined_restart_path(pcg, c, fmt):
    import torch
    A, b, M = _solve(pcg, "C3", c, fmt)
    ro = O.pcg_pipelined(A, b, tol=1e-10)
    rc = O.pcg(A, b, tol=1e-10)
    assert ro.status == O.OK
    x, info = M.solve_pipelined(torch.as_tensor(b).cuda(), tol=1e-10)
    assert info["status"] == 0 and info["relres_true"] <= 1e-10
    assert 0.9 * rc.iterations <= info["iterations"] <= 2 * ro.iterations, (info["iterations"], ro.iterations)
    assert np.linalg.norm(x.cpu().numpy() - rc.x) <= 1e-8 * np.linalg.norm(rc.x)
    if c == 64:  # the oracle itself restarts here; so must the GPU
        assert ro.iterations > 1.3 * rc.iterations and info["replacements"] >= 1


def test_pipelined_edges(pcg):
    import torch
    A, b, M = _solve(pcg, "C1", 16)
    bd = torch.as_tensor(b).cuda()
    x, info = M.solve_pipelined(torch.zeros_like(bd), x0=torch.ones_like(bd))
    assert info["iterations"] == 0 and float(x.abs().max()) == 0.0  # b = 0: x = 0
    xs, _ = M.solve_pipelined(bd, tol=1e-14)
    x, info = M.solve_pipelined(bd, x0=xs, tol=1e-10)
    assert info["iterations"] == 0 and info["status"] == 0  # converged on entry
    ro = O.pcg_pipelined(A, b, tol=1e-12, max_iter=7)
    x, info = M.solve_pipelined(bd, tol=1e-12, max_iter=7)
    assert info["status"] == 1 and info["iterations"] == 7 and ro.status == O.NOT_CONVERGED
    assert np.linalg.norm(x.cpu().numpy() - ro.x) <= 1e-12 * np.linalg.norm(ro.x)
