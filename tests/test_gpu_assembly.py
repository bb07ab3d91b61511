"""GPU element-by-element assembly (generic path): fem_element_coo
emits every element's stiffness K_e as COO triplets, coo_to_csr sums them in element
order.  Compared with the oracle's assembly (oracle.c orc_assemble: incidence-list
pattern + per-element accumulation) on the same meshes: the Neumann stiffness over
all nodes — pattern bit-exact; values within 64 ulps of the row magnitude, the bar
of the row-wise generator (test_gpu_parity.py): both sides add the elements' K_e
entries in element order, but K_e itself is evaluated with different contraction
(nvcc fuses multiply-adds, the oracle is compiled with -ffp-contract=off), so
entries agree to rounding, bitwise only where the lattice arithmetic is exact.
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


def _oracle_K(name, c):
    cfg = O.configs()[name]
    m = O.Mesh(O.FAMILY[cfg["family"]], c, jitter=bool(cfg["jitter"]), seed=cfg["seed"])
    K, _ = O.assemble(m, O.F_ZERO)
    return K


@pytest.mark.parametrize("name,c", [("C1", 8), ("C1", 33), ("C2", 16), ("C2", 64), ("C3", 6), ("C3", 24),
                                    ("C5", 4), ("C5", 12), ("C6", 6), ("C6", 20)])
def test_element_assembly_matches_oracle(pcg, name, c):
    from paper_2201_05413_b200.problems import fem_assemble_elements, fem_element_triplets, fem_spec
    spec = fem_spec(name, c=c)
    T = fem_element_triplets(spec)
    npe = T["npe"]
    assert T["row"].numel() == T["val"].numel() and T["row"].numel() % (npe * npe) == 0
    G = fem_assemble_elements(spec)
    K = _oracle_K(name, c)
    assert np.array_equal(G["row_ptr"].cpu().numpy(), K.row_ptr)
    assert np.array_equal(G["col"].cpu().numpy(), K.col)
    v = G["val"].cpu().numpy()
    rows = np.repeat(np.arange(K.n), np.diff(K.row_ptr))
    rowmax = np.zeros(K.n)
    np.maximum.at(rowmax, rows, np.abs(K.val))
    assert np.all(np.abs(v - K.val) <= 64 * np.finfo(float).eps * rowmax[rows])
    if c & (c - 1) == 0 and not O.configs()[name]["jitter"]:  # power-of-two lattice: exact arithmetic
        assert np.array_equal(v, K.val)


def test_element_count_and_errors(pcg):
    import ctypes as C
    from paper_2201_05413_b200 import PcgError
    from paper_2201_05413_b200._lib import check, lib
    from paper_2201_05413_b200.problems import fem_spec
    for name, c, ne, npe in (("C1", 5, 50, 3), ("C3", 5, 50, 6), ("C5", 3, 162, 4)):
        spec = fem_spec(name, c=c)
        n_e, n_p, n_n = C.c_int64(), C.c_int32(), C.c_int64()
        check(lib().fem_element_count(C.byref(spec), C.byref(n_e), C.byref(n_p), C.byref(n_n)), "count")
        assert (n_e.value, n_p.value) == (ne, npe)
    spec = fem_spec("C1", c=5)
    with pytest.raises(PcgError):
        check(lib().fem_element_coo(C.byref(spec), 0, 51, None, None, None, None), "fem_element_coo")
