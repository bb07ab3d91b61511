"""GPU parity for the generic COO -> CSR (include/fem_gen.h coo_to_csr; SURVEY §8(f) N1,
SPEC coo_to_csr S:50-57) against the oracle (oracle.c orc_coo_to_csr).

Bar: bitwise — integers (row_ptr, col) and values: both sides sum each duplicate group
left to right in input order from 0.0 (the oracle's definition), so no tolerance.
"""
import numpy as np
import pytest

import oracle as O
from coo_inputs import triplets

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pcg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_05413_b200 as p
    return p


def _gpu(pcg, r, c, v, nr, nc):
    import torch
    out = pcg.coo_to_csr(torch.as_tensor(r).cuda(), torch.as_tensor(c).cuda(), torch.as_tensor(v).cuda(), nr, nc)
    return out["row_ptr"].cpu().numpy(), out["col"].cpu().numpy(), out["val"].cpu().numpy()


def _same(a, b):
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert np.array_equal(a[2].view(np.int64), b[2].view(np.int64))  # bitwise, incl. signed zeros


def test_spec_examples(pcg):
    _same(_gpu(pcg, [0, 0, 1], [0, 0, 1], [1.0, 3.0, 2.0], 2, 2), ([0, 1, 2], [0, 1], np.array([4.0, 2.0])))
    rp, c, v = _gpu(pcg, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0), 3, 3)
    assert rp.tolist() == [0, 0, 0, 0] and c.size == 0
    _same(_gpu(pcg, [2, 0, 1], [2, 0, 1], [1.0, 1.0, 1.0], 3, 3), ([0, 1, 2, 3], [0, 1, 2], np.ones(3)))


@pytest.mark.parametrize("seed,nr,nc,nnz,keys", [
    (11, 7, 5, 60, None), (12, 40, 40, 900, None), (13, 1000, 1000, 100_003, 30_001),
    (14, 3000, 17, 50_000, None), (15, 1, 1, 4097, None), (16, 2_000_000, 2_000_000, 8_000_000, 3_000_000),
    (17, 50_000_000, 3, 1000, None), (18, 5, 2**31 - 1, 20_000, 5_000)])
def test_parity_with_oracle(pcg, seed, nr, nc, nnz, keys):
    r, c, v = triplets(seed, nr, nc, nnz, keys)
    _same(_gpu(pcg, r, c, v, nr, nc), O.coo_to_csr(nr, nc, r, c, v))


def test_one_long_run(pcg):
    """Every entry on one position: a single duplicate group of 2^20 + 3 values."""
    rng = np.random.default_rng(19)
    n = (1 << 20) + 3
    r = np.full(n, 4, np.int64)
    c = np.full(n, 2, np.int64)
    v = rng.uniform(-1, 1, n)
    _same(_gpu(pcg, r, c, v, 9, 9), O.coo_to_csr(9, 9, r, c, v))


def test_errors(pcg):
    import torch
    from paper_2201_05413_b200 import PcgError
    for r, c in (([0, 2], [0, 0]), ([0, 1], [0, 3]), ([-1], [0]), ([0], [-5])):
        with pytest.raises(PcgError) as e:
            _gpu(pcg, np.array(r, np.int64), np.array(c, np.int64), np.ones(len(r)), 2, 3)
        assert e.value.status == 3  # PCG_ERR_INDEX_OUT_OF_RANGE
    t = torch.zeros(1, dtype=torch.int64, device="cuda")
    with pytest.raises(PcgError) as e:
        pcg.coo_to_csr(t, t, torch.zeros(1, dtype=torch.float64, device="cuda"), 2, 2**31)
    assert e.value.status == 2  # PCG_ERR_INVALID_ARG
