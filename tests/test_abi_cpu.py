"""CPU-side checks of the product boundary: the C-ABI library loads, exports every
symbol include/*.h declares, and its host-only entry points behave (no GPU)."""
import os
import re

import numpy as np
import pytest

import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    names = []
    for h in ("pcg.h", "fem_gen.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        names += re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+(?:\s+|\s*\*\s*)([a-z_0-9]+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def pcg():
    from paper_2201_05413_b200 import build
    build.build()
    import paper_2201_05413_b200 as p
    return p


def test_library_exports_every_declared_symbol(pcg):
    L = pcg.lib()
    names = _declared_functions()
    assert len(names) >= 17
    for nm in names:
        assert hasattr(L, nm), nm


def test_library_is_sm100a():
    import subprocess
    so = os.path.join(ROOT, "paper_2201_05413_b200", "libpcg_b200.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings_and_invalid_args(pcg):
    import ctypes as C
    L = pcg.lib()
    assert L.pcg_status_string(0) == b"PCG_OK"
    assert L.pcg_status_string(7) == b"PCG_ERR_NOT_SPD"
    h = C.c_void_p()
    # null arrays / negative sizes are rejected before any CUDA call
    assert L.csr_create(-1, 0, None, None, None, 0, None, C.byref(h)) == 2
    assert L.csr_create(3, 3, None, None, None, 0, None, C.byref(h)) == 2
    assert L.pcg_solve(None, None, None, 1e-10, 10, None, None) == 2
    assert L.pcg_solve_multi(None, 0, None, 0, None, 0, 1e-10, 10, None, None) == 2
    assert b"null" in L.pcg_last_error()


@pytest.mark.parametrize("G", [1, 2, 3, 4, 8])
def test_partition_rows_matches_oracle(pcg, G):
    """Row partition is bit-exact between product and oracle."""
    for name, c in [("C2", 32), ("C3", 16), ("C5", 12)]:
        A = O.build_problem(name, c=c)["A"]
        assert np.array_equal(pcg.partition_rows(A.row_ptr, G), O.partition(A, G))


@pytest.mark.parametrize("name,c", [("C1", 64), ("C2", 1024), ("C3", 1024), ("C4", 128), ("C5", 512), ("C5", 8)])
def test_fem_problem_size_closed_forms(pcg, name, c):
    from paper_2201_05413_b200.problems import fem_spec, problem_size
    n, nnz, _ = problem_size(fem_spec(name, c=c))
    if c <= 64:  # compare with the oracle's assembled system
        A = O.build_problem(name, c=c, k=1)["A"]
        assert (n, nnz) == (A.n, A.nnz)
    want = {"C1": (3969, 19593), "C2": (1046529, 7317521), "C3": (4190209, 48136245),
            "C4": (2048383, 14241907), "C5": (133432831, 932463091)}
    if c == O.configs()[name]["c"]:
        assert (n, nnz) == want[name]


def test_python_binding_has_the_abi_names():
    """The binding exposes the C ABI's entry points under their header names (no GPU needed)."""
    import paper_2201_05413_b200 as pcg
    for name in ("csr_create", "csr_create_dist", "csr_destroy", "pcg_spmv", "pcg_solve", "pcg_solve_multi",
                 "pcg_bicgstab", "pcg_partition_rows", "coo_to_csr", "csr_rcm_order", "pcg_solve_pipelined", "solve"):
        assert callable(getattr(pcg, name)), name
