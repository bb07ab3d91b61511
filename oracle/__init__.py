"""Oracle: plain fp64 CPU implementation of FEM assembly + Jacobi-PCG.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product (``paper_2201_05413_b200``) never imports it, and this
package imports nothing from the product.

The arithmetic lives in ``oracle.c`` (plain loops, single thread); this module
only marshals numpy arrays through ctypes.  Citations (P:n = PAPER.md line n,
§8(c).k = SURVEY.md §8(c) step k) are on the C functions.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

P1_TRI, P1_TET, P2_TRI = 1, 2, 3
FAMILY = {"P1_TRI": P1_TRI, "P1_TET": P1_TET, "P2_TRI": P2_TRI}
F_ZERO, F_CONST, F_SIN2D, F_SIN3D, F_BUMP3D, F_LINEAR = 0, 1, 2, 3, 4, 5
PAT_ELEMENT, PAT_AXIS = 0, 1
OK, NOT_CONVERGED, ERR_INVALID_ARG, ERR_ZERO_DIAGONAL, ERR_NOT_SPD, ERR_POLICY, ERR_OOM, ERR_INDEX = range(8)


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_LIB_OMP = os.path.join(_HERE, "liboracle_omp.so")
_lib_omp = None


def build_omp(force: bool = False) -> str:
    """TIMING-ONLY all-cores build of the same oracle.c (-fopenmp -DORC_OMP: OpenMP
    static loops, chunked Dot2).  Used by bench.py's CPU legs only, never for parity."""
    if force or not os.path.exists(_LIB_OMP) or os.path.getmtime(_LIB_OMP) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                               "-DORC_OMP", "-fPIC", "-shared", "-o", _LIB_OMP, _SRC, "-lm"])
    return _LIB_OMP


def pcg_all_cores(A, b, tol=1e-10, max_iter=50000):
    """Jacobi-PCG of the all-cores timing build (OMP_NUM_THREADS / all host cores).
    Returns (iterations, status, threads).  Timing only."""
    global _lib_omp
    if _lib_omp is None:
        L = C.CDLL(build_omp())
        L.orc_pcg.argtypes = [C.POINTER(_Csr), C.c_void_p, C.c_void_p, C.c_double, C.c_int64,
                              C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double),
                              C.c_void_p, C.c_void_p, C.c_int64]
        _lib_omp = L
    import numpy as _np
    b = _np.ascontiguousarray(b, dtype=_np.float64)
    x = _np.zeros(A.n)
    it, rr, rt = C.c_int64(0), C.c_double(0), C.c_double(0)
    Ac = A._c()
    st = _lib_omp.orc_pcg(C.byref(Ac), b.ctypes.data_as(C.c_void_p), x.ctypes.data_as(C.c_void_p), tol, max_iter,
                          C.byref(it), C.byref(rr), C.byref(rt), None, None, 0)
    threads = int(os.environ.get("OMP_NUM_THREADS", "0")) or len(os.sched_getaffinity(0))
    return it.value, st, threads


class _Mesh(C.Structure):
    _fields_ = [("dim", C.c_int), ("family", C.c_int), ("c", C.c_int),
                ("n_nodes", C.c_int64), ("n_elem", C.c_int64), ("npe", C.c_int),
                ("coord", C.POINTER(C.c_double)), ("elem", C.POINTER(C.c_int32)),
                ("boundary", C.POINTER(C.c_uint8)), ("n_reset", C.c_int64)]


class _Csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("row_ptr", C.POINTER(C.c_int64)),
                ("col", C.POINTER(C.c_int64)), ("val", C.POINTER(C.c_double))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        P = C.POINTER
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_uniform.restype = C.c_double
        L.orc_uniform.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_mesh_build.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, P(_Mesh)]
        L.orc_mesh_free.argtypes = [P(_Mesh)]
        L.orc_elem_stiffness.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        L.orc_elem_load.argtypes = [C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_assemble.argtypes = [P(_Mesh), C.c_int, C.c_void_p, P(_Csr), C.c_void_p]
        L.orc_assemble_load.argtypes = [P(_Mesh), C.c_int, C.c_void_p, C.c_void_p]
        L.orc_dirichlet.argtypes = [P(_Mesh), P(_Csr), C.c_void_p, C.c_void_p, C.c_int,
                                    P(_Csr), C.c_void_p, C.c_void_p]
        L.orc_csr_free.argtypes = [P(_Csr)]
        L.orc_spmv.argtypes = [P(_Csr), C.c_void_p, C.c_void_p]
        L.orc_dot.argtypes = [C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_dot.restype = C.c_double
        L.orc_pcg.argtypes = [P(_Csr), C.c_void_p, C.c_void_p, C.c_double, C.c_int64,
                              P(C.c_int64), P(C.c_double), P(C.c_double),
                              C.c_void_p, C.c_void_p, C.c_int64]
        L.orc_pcg_ex.argtypes = [P(_Csr), C.c_void_p, C.c_void_p, C.c_double, C.c_int64,
                                 P(C.c_int64), P(C.c_double), P(C.c_double),
                                 C.c_void_p, C.c_void_p, C.c_int64, P(C.c_int64), C.c_void_p, P(C.c_int64)]
        L.orc_assemble_free_lattice.argtypes = [P(_Mesh), C.c_int, C.c_void_p, P(_Csr), C.c_void_p]
        L.orc_partition.argtypes = [C.c_int64, C.c_void_p, C.c_int, C.c_void_p]
        L.orc_fd_cube.argtypes = [C.c_int64, C.c_int, P(_Csr), C.c_void_p]
        L.orc_bicgstab.argtypes = [P(_Csr), C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.c_int64,
                                   P(C.c_int64), P(C.c_double), P(C.c_double)]
        L.orc_bicgstab_pc.argtypes = [P(_Csr), C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.c_int, C.c_int64,
                                      P(C.c_int64), P(C.c_double), P(C.c_double)]
        L.orc_ilu0_factor.argtypes = [P(_Csr), C.c_int64, C.c_void_p]
        L.orc_ilu0_apply.argtypes = [P(_Csr), C.c_int64, C.c_void_p, C.c_void_p]
        L.orc_halo.restype = C.c_int64
        L.orc_coo_to_csr.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_pcg_pipelined.argtypes = [P(_Csr), C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.c_void_p,
                                        C.c_void_p, C.c_void_p]
        L.orc_halo.argtypes = [P(_Csr), C.c_int64, C.c_int64, C.c_void_p, C.c_int64]
        L.orc_rcm.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_block_cg.argtypes = [P(_Csr), C.c_int, C.c_void_p, C.c_void_p, C.c_double, C.c_int64, C.c_void_p,
                                   C.c_void_p]
        L.orc_fd_identity_rows_nnz.restype = C.c_int64
        L.orc_fd_identity_rows_nnz.argtypes = [C.c_int64]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# --------------------------------------------------------------------------
class Csr:
    """CSR with int64 row_ptr/col and float64 values (numpy-owned)."""

    def __init__(self, n, row_ptr, col, val):
        self.n = int(n)
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int64)
        self.val = np.ascontiguousarray(val, dtype=np.float64)
        self.nnz = int(self.row_ptr[-1]) if self.n >= 0 and len(self.row_ptr) else 0

    def _c(self):
        return _Csr(self.n, self.nnz, self.row_ptr.ctypes.data_as(C.POINTER(C.c_int64)),
                    self.col.ctypes.data_as(C.POINTER(C.c_int64)),
                    self.val.ctypes.data_as(C.POINTER(C.c_double)))

    @staticmethod
    def _adopt_c(s: _Csr) -> "Csr":
        """Wrap the C arrays without copying (for the largest systems); the C memory
        stays owned by the returned object and is freed with it."""
        n, nnz = s.n, s.nnz
        A = Csr.__new__(Csr)
        A.n, A.nnz = int(n), int(nnz)
        A.row_ptr = np.ctypeslib.as_array(s.row_ptr, shape=(n + 1,))
        A.col = np.ctypeslib.as_array(s.col, shape=(max(nnz, 1),))[:nnz]
        A.val = np.ctypeslib.as_array(s.val, shape=(max(nnz, 1),))[:nnz]
        A._owner = _CsrOwner(s)
        return A

    @staticmethod
    def _from_c(s: _Csr) -> "Csr":
        n, nnz = s.n, s.nnz
        rp = np.ctypeslib.as_array(s.row_ptr, shape=(n + 1,)).copy()
        col = np.ctypeslib.as_array(s.col, shape=(max(nnz, 1),))[:nnz].copy()
        val = np.ctypeslib.as_array(s.val, shape=(max(nnz, 1),))[:nnz].copy()
        lib().orc_csr_free(C.byref(s))
        return Csr(n, rp, col, val)

    def to_dense(self):
        A = np.zeros((self.n, self.n))
        for i in range(self.n):
            for k in range(self.row_ptr[i], self.row_ptr[i + 1]):
                A[i, self.col[k]] += self.val[k]
        return A

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.val, self.col, self.row_ptr), shape=(self.n, self.n))


class _CsrOwner:
    def __init__(self, s):
        self.s = s

    def __del__(self):
        try:
            lib().orc_csr_free(C.byref(self.s))
        except Exception:
            pass


class Mesh:
    def __init__(self, family: int, c: int, jitter: bool = False, seed: int = 0):
        self._m = _Mesh()
        st = lib().orc_mesh_build(family, c, int(jitter), seed, C.byref(self._m))
        if st != OK:
            raise ValueError(f"orc_mesh_build failed: {st}")
        m = self._m
        self.family, self.c, self.dim, self.npe = family, c, m.dim, m.npe
        self.n_nodes, self.n_elem, self.n_reset = m.n_nodes, m.n_elem, m.n_reset
        self.coord = np.ctypeslib.as_array(m.coord, shape=(m.n_nodes, m.dim))
        self.elem = np.ctypeslib.as_array(m.elem, shape=(m.n_elem, m.npe))
        self.boundary = np.ctypeslib.as_array(m.boundary, shape=(m.n_nodes,)).astype(bool)

    def __del__(self):
        try:
            lib().orc_mesh_free(C.byref(self._m))
        except Exception:
            pass


def splitmix64(seed: int, idx: int) -> int:
    return lib().orc_splitmix64(seed, idx)


def uniform(seed: int, idx: int) -> float:
    return lib().orc_uniform(seed, idx)


def elem_stiffness(family: int, xe) -> np.ndarray:
    xe = np.ascontiguousarray(xe, dtype=np.float64)
    npe = {P1_TRI: 3, P1_TET: 4, P2_TRI: 6}[family]
    K = np.zeros((npe, npe))
    lib().orc_elem_stiffness(family, _ptr(xe), _ptr(K))
    return K


def elem_load(family: int, xe, fkind: int, fparam=(0.0, 0.0, 0.0, 0.0)) -> np.ndarray:
    xe = np.ascontiguousarray(xe, dtype=np.float64)
    npe = {P1_TRI: 3, P1_TET: 4, P2_TRI: 6}[family]
    fp = np.ascontiguousarray(list(fparam) + [0.0] * (4 - len(fparam)), dtype=np.float64)
    fe = np.zeros(npe)
    lib().orc_elem_load(family, _ptr(xe), fkind, _ptr(fp), _ptr(fe))
    return fe


def assemble(mesh: Mesh, fkind: int, fparam=(0.0, 0.0, 0.0, 0.0)):
    """Neumann stiffness K (element-graph pattern) and load vector F over all nodes."""
    fp = np.ascontiguousarray(list(fparam) + [0.0] * (4 - len(fparam)), dtype=np.float64)
    F = np.zeros(mesh.n_nodes)
    s = _Csr()
    st = lib().orc_assemble(C.byref(mesh._m), fkind, _ptr(fp), C.byref(s), _ptr(F))
    if st != OK:
        raise RuntimeError(f"orc_assemble failed: {st}")
    return Csr._from_c(s), F


def assemble_load(mesh: Mesh, fkind: int, fparam=(0.0, 0.0, 0.0, 0.0)):
    fp = np.ascontiguousarray(list(fparam) + [0.0] * (4 - len(fparam)), dtype=np.float64)
    F = np.zeros(mesh.n_nodes)
    lib().orc_assemble_load(C.byref(mesh._m), fkind, _ptr(fp), _ptr(F))
    return F


def dirichlet(mesh: Mesh, K: Csr, F, g, policy: int):
    """K_FF (policy-filtered), b_F = F_F - K_FB g_B, and the free-node map."""
    F = np.ascontiguousarray(F, dtype=np.float64)
    g = np.ascontiguousarray(g, dtype=np.float64)
    nf = int((~mesh.boundary).sum())
    bF = np.zeros(nf)
    fmap = np.zeros(mesh.n_nodes, dtype=np.int64)
    s = _Csr()
    Kc = K._c()
    st = lib().orc_dirichlet(C.byref(mesh._m), C.byref(Kc), _ptr(F), _ptr(g), policy,
                             C.byref(s), _ptr(bF), _ptr(fmap))
    if st != OK:
        raise RuntimeError(f"orc_dirichlet failed: {st}")
    return Csr._from_c(s), bF, fmap


def spmv(A: Csr, x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros(A.n)
    Ac = A._c()
    lib().orc_spmv(C.byref(Ac), _ptr(x), _ptr(y))
    return y


def dot(a, b) -> float:
    """a.b as the oracle's PCG evaluates it (Dot2: as if in twice fp64 precision)."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    assert a.shape == b.shape
    return float(lib().orc_dot(a.size, _ptr(a), _ptr(b)))


class PcgResult(dict):
    __getattr__ = dict.__getitem__


def pcg(A: Csr, b, x0=None, tol=1e-10, max_iter=50000, hist: int = 0) -> PcgResult:
    """Jacobi-PCG (§8(c).8).  Returns x, iterations, recurrence/true relres, status."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it, rr, rt = C.c_int64(0), C.c_double(0), C.c_double(0)
    ah = np.zeros(hist) if hist else None
    bh = np.zeros(hist) if hist else None
    Ac = A._c()
    st = lib().orc_pcg(C.byref(Ac), _ptr(b), _ptr(x), tol, max_iter, C.byref(it), C.byref(rr),
                       C.byref(rt), _ptr(ah), _ptr(bh), hist)
    return PcgResult(x=x, iterations=it.value, relres_rec=rr.value, relres_true=rt.value,
                     status=st, alpha=ah, beta=bh)


def pcg_ex(A: Csr, b, x0=None, tol=1e-10, max_iter=50000) -> PcgResult:
    """pcg() plus the residual-replacement record (oracle.h orc_pcg_ex): the number of
    replacements, and the iterate / iteration count at the first one."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it, rr, rt = C.c_int64(0), C.c_double(0), C.c_double(0)
    nrep, kf = C.c_int64(0), C.c_int64(-1)
    xf = np.zeros(A.n)
    Ac = A._c()
    st = lib().orc_pcg_ex(C.byref(Ac), _ptr(b), _ptr(x), tol, max_iter, C.byref(it), C.byref(rr), C.byref(rt),
                          None, None, 0, C.byref(nrep), _ptr(xf), C.byref(kf))
    return PcgResult(x=x, iterations=it.value, relres_rec=rr.value, relres_true=rt.value, status=st,
                     replacements=nrep.value, x_first=xf if kf.value >= 0 else None, k_first=kf.value)


def assemble_free_lattice(mesh: Mesh, fkind: int, fparam=(0.0, 0.0, 0.0, 0.0), copy: bool = True):
    """K_FF and b_F of a lattice P1 mesh with g = 0 and the AXIS policy, without the
    Neumann K (oracle.h orc_assemble_free_lattice; bitwise assemble + dirichlet)."""
    fp = np.ascontiguousarray(list(fparam) + [0.0] * (4 - len(fparam)), dtype=np.float64)
    nf = int((~mesh.boundary).sum())
    bF = np.zeros(nf)
    s = _Csr()
    st = lib().orc_assemble_free_lattice(C.byref(mesh._m), fkind, _ptr(fp), C.byref(s), _ptr(bF))
    if st != OK:
        raise RuntimeError(f"orc_assemble_free_lattice failed: {st}")
    return (Csr._from_c(s) if copy else Csr._adopt_c(s)), bF


FD_X2MY2, FD_EXPSIN = 1, 2


def fd_cube(N: int, fkind: int = FD_X2MY2):
    """Table 1 system: FD Laplace on N^3 nodes, identity boundary rows
    with b = f (Dirichlet), b = 0 inside.  Returns (Csr, b)."""
    b = np.zeros(N ** 3)
    s = _Csr()
    st = lib().orc_fd_cube(N, fkind, C.byref(s), _ptr(b))
    if st != OK:
        raise RuntimeError(f"orc_fd_cube: {st}")
    return Csr._from_c(s), b


def bicgstab(A: Csr, b, x0=None, tol=1e-10, max_iter=50000, block=1) -> PcgResult:
    """Right-preconditioned BiCGSTAB with (block-)Jacobi (R2)."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it, rr, rt = C.c_int64(0), C.c_double(0), C.c_double(0)
    Ac = A._c()
    st = lib().orc_bicgstab(C.byref(Ac), _ptr(b), _ptr(x), tol, max_iter, block, C.byref(it), C.byref(rr),
                            C.byref(rt))
    return PcgResult(x=x, iterations=it.value, relres_rec=rr.value, relres_true=rt.value, status=st)


PC_BJ_LU, PC_BJ_ILU0 = 0, 1


def bicgstab_ilu(A: Csr, b, x0=None, tol=1e-10, max_iter=50000, block=None) -> PcgResult:
    """BiCGSTAB with Block-Jacobi ILU(0) blocks of `block` rows (default: one block, n rows),
    oracle.h orc_bicgstab_pc / DESIGN.md reading R6."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it, rr, rt = C.c_int64(0), C.c_double(0), C.c_double(0)
    Ac = A._c()
    st = lib().orc_bicgstab_pc(C.byref(Ac), _ptr(b), _ptr(x), tol, max_iter, PC_BJ_ILU0, int(block or max(A.n, 1)),
                               C.byref(it), C.byref(rr), C.byref(rt))
    return PcgResult(x=x, iterations=it.value, relres_rec=rr.value, relres_true=rt.value, status=st)


def ilu0_factor(A: Csr, block: int) -> np.ndarray:
    """ILU(0) factor values of the Block-Jacobi blocks in A's pattern (oracle.h orc_ilu0_factor)."""
    f = np.zeros(max(A.nnz, 1))
    Ac = A._c()
    st = lib().orc_ilu0_factor(C.byref(Ac), int(block), _ptr(f))
    if st != OK:
        raise RuntimeError(f"orc_ilu0_factor: {st}")
    return f[:A.nnz]


def ilu0_apply(A: Csr, block: int, v) -> np.ndarray:
    v = np.ascontiguousarray(v, dtype=np.float64)
    y = np.zeros(A.n)
    Ac = A._c()
    st = lib().orc_ilu0_apply(C.byref(Ac), int(block), _ptr(v), _ptr(y))
    if st != OK:
        raise RuntimeError(f"orc_ilu0_apply: {st}")
    return y


def coo_to_csr(n_rows: int, n_cols: int, row, col, val):
    """SPEC coo_to_csr: (row_ptr, col, val) numpy arrays; duplicates summed in
    input order.  Raises IndexError for an out-of-range index (SPEC IndexOutOfRange)."""
    row = np.ascontiguousarray(row, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    nnz = row.size
    rp = np.zeros(n_rows + 1, dtype=np.int64)
    co = np.zeros(max(nnz, 1), dtype=np.int64)
    vo = np.zeros(max(nnz, 1))
    u = C.c_int64(0)
    st = lib().orc_coo_to_csr(n_rows, n_cols, nnz, _ptr(row), _ptr(col), _ptr(val), _ptr(rp), _ptr(co), _ptr(vo),
                              C.byref(u))
    if st == ERR_INDEX:
        raise IndexError("orc_coo_to_csr: index out of range")
    if st != OK:
        raise RuntimeError(f"orc_coo_to_csr: {st}")
    return rp, co[:u.value].copy(), vo[:u.value].copy()


def block_cg(A: Csr, B, X0=None, tol=1e-10, max_iter=50000):
    """SURVEY §8(f) N3 (reading R5): block CG with the Jacobi M (oracle.h orc_block_cg).
    B: (n, k).  Returns (X (n, k), iterations, relres_true (k,), status)."""
    B = np.asarray(B, dtype=np.float64)
    n, k = B.shape
    Bc = np.asfortranarray(B)
    X = np.asfortranarray(np.zeros((n, k)) if X0 is None else np.array(X0, dtype=np.float64))
    it = C.c_int64(0)
    rt = np.zeros(k)
    Ac = A._c()
    st = lib().orc_block_cg(C.byref(Ac), k, Bc.ctypes.data_as(C.c_void_p), X.ctypes.data_as(C.c_void_p), tol,
                            max_iter, C.byref(it), rt.ctypes.data_as(C.c_void_p))
    return np.ascontiguousarray(X), it.value, rt, st


def rcm(A: Csr):
    """reverse Cuthill-McKee order of A's pattern (oracle.h orc_rcm);
    perm[k] = original index of the k-th node (new -> old)."""
    rp = np.ascontiguousarray(A.row_ptr, dtype=np.int64)
    col = np.ascontiguousarray(A.col, dtype=np.int64)
    perm = np.zeros(max(A.n, 1), dtype=np.int64)
    st = lib().orc_rcm(A.n, _ptr(rp), _ptr(col), _ptr(perm))
    if st != OK:
        raise RuntimeError(f"orc_rcm: {st}")
    return perm[:A.n].copy()


def pcg_pipelined(A: Csr, b, x0=None, tol=1e-10, max_iter=50000) -> PcgResult:
    """SURVEY §8(f) N3 (reading R4): preconditioned pipelined CG, one reduction per iteration."""
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.zeros(A.n) if x0 is None else np.array(x0, dtype=np.float64, copy=True)
    it, rr, rt = C.c_int64(0), C.c_double(0), C.c_double(0)
    Ac = A._c()
    st = lib().orc_pcg_pipelined(C.byref(Ac), _ptr(b), _ptr(x), tol, max_iter, C.byref(it), C.byref(rr), C.byref(rt))
    return PcgResult(x=x, iterations=it.value, relres_rec=rr.value, relres_true=rt.value, status=st)


def pcg_multi(A: Csr, B, X0=None, tol=1e-10, max_iter=50000):
    """§8(c).9: column j runs §8(c).8 independently (single r.h.s. terms)."""
    B = np.asarray(B, dtype=np.float64)
    k = B.shape[1]
    X0 = np.zeros_like(B) if X0 is None else X0
    res = [pcg(A, B[:, j], X0[:, j], tol, max_iter) for j in range(k)]
    X = np.stack([r.x for r in res], axis=1)
    return X, res


def partition(A: Csr, G: int) -> np.ndarray:
    bounds = np.zeros(G + 1, dtype=np.int64)
    lib().orc_partition(A.n, _ptr(A.row_ptr), G, _ptr(bounds))
    return bounds


def halo(A: Csr, r0: int, r1: int) -> np.ndarray:
    Ac = A._c()
    cnt = lib().orc_halo(C.byref(Ac), r0, r1, None, 0)
    out = np.zeros(max(cnt, 1), dtype=np.int64)
    lib().orc_halo(C.byref(Ac), r0, r1, _ptr(out), cnt)
    return out[:cnt]


def fd_identity_rows_nnz(N: int) -> int:
    return lib().orc_fd_identity_rows_nnz(N)


# --------------------------------------------------------------------------
# the five workloads (configs/configs.json; readings in DESIGN.md §3)
_CFG = os.path.join(os.path.dirname(_HERE), "configs", "configs.json")


def configs() -> dict:
    with open(_CFG) as fh:
        return {k: v for k, v in json.load(fh).items() if not k.startswith("_")}


def bump_centres(seed: int, k: int) -> np.ndarray:
    """C4 centres: c_s,axis = uniform(seed, 3s + axis)  (§8(c).11)."""
    return np.array([[uniform(seed, 3 * s + a) for a in range(3)] for s in range(k)])


def build_problem(name: str, c: int | None = None, k: int | None = None) -> dict:
    """Oracle pipeline for config `name` (optionally at another size c / RHS count k):
    mesh -> Neumann K, F -> Dirichlet elimination + policy -> (A, B)."""
    cfg = dict(configs()[name])
    if c is not None:
        cfg["c"] = c
    if k is not None:
        cfg["k"] = k
    fam = FAMILY[cfg["family"]]
    mesh = Mesh(fam, cfg["c"], cfg["jitter"], cfg["seed"])
    policy = {"AXIS": PAT_AXIS, "ELEMENT": PAT_ELEMENT}[cfg["policy"]]
    X = mesh.coord
    g = np.zeros(mesh.n_nodes)
    if cfg["g"] == "X2MY2":
        g = X[:, 0] * X[:, 0] - X[:, 1] * X[:, 1]
    elif cfg["g"] == "LINEAR3D":  # reading R3: harmonic and reproduced exactly by P1 (patch test)
        g = ((1.0 + 2.0 * X[:, 0]) - 3.0 * X[:, 1]) + 0.5 * X[:, 2]
    loads = []
    if cfg["f"] == "BUMP3D":
        for cs in bump_centres(cfg["seed"], cfg["k"]):
            loads.append((F_BUMP3D, (cs[0], cs[1], cs[2], cfg["sigma"])))
    else:
        fk = {"ZERO": F_ZERO, "ONE": F_CONST, "SIN2D": F_SIN2D, "SIN3D": F_SIN3D}[cfg["f"]]
        loads.append((fk, (1.0, 0.0, 0.0, 0.0)))
    A, cols, fmap, K = None, [], None, None
    for fk, fp in loads:
        if K is None:
            K, F = assemble(mesh, fk, fp)
        else:
            F = assemble_load(mesh, fk, fp)
        A_, bF, fmap = dirichlet(mesh, K, F, g, policy)
        if A is None:
            A = A_
        cols.append(bF)
    B = np.stack(cols, axis=1)
    free_nodes = np.nonzero(fmap >= 0)[0]
    return {"cfg": cfg, "mesh": mesh, "A": A, "B": B, "free_nodes": free_nodes, "g": g}
