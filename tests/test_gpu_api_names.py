"""The Python binding under the C ABI's names (include/pcg.h): each alias gives the
result of the method it forwards to, bitwise (same kernels, same inputs)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_abi_named_entry_points():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_05413_b200 as pcg
    P = pcg.fem_build(pcg.fem_spec("C1"))
    b = P["B"][:, 0].contiguous()
    A = pcg.csr_create(P["row_ptr"], P["col"], P["val"])
    M = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
    assert torch.equal(pcg.pcg_spmv(A, b), M.spmv(b))
    x1, i1 = pcg.pcg_solve(A, b, tol=1e-10)
    x2, i2 = M.solve(b, tol=1e-10)
    assert torch.equal(x1, x2) and i1["iterations"] == i2["iterations"]
    B = torch.stack([b, 2.0 * b], dim=1)
    X1, I1 = pcg.pcg_solve_multi(A, B, tol=1e-10)
    X2, I2 = M.solve_multi(B, tol=1e-10)
    assert torch.equal(X1, X2) and [i["iterations"] for i in I1] == [i["iterations"] for i in I2]
    y1, j1 = pcg.pcg_bicgstab(A, b, tol=1e-10, block_size=1)
    y2, j2 = M.bicgstab(b, tol=1e-10, block=1)
    assert torch.equal(y1, y2) and j1["iterations"] == j2["iterations"]
    bounds = pcg.pcg_partition_rows(P["row_ptr"].cpu().numpy(), 4)
    assert bounds[0] == 0 and bounds[-1] == A.n and np.all(np.diff(bounds) >= 0)
    pcg.csr_destroy(A)
    M.close()
