"""Benchmark problems C1-C5 (BASELINE.json configs) built on the GPU by fem_gen.

configs/configs.json holds the parameters (plain data).  fem_build() calls the
library's device generator (include/fem_gen.h); nothing here computes values.
"""
from __future__ import annotations

import ctypes as C
import json
import os

from . import _lib
from ._lib import FemSpec, check, lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = os.path.join(ROOT, "configs", "configs.json")

_FAM = {"P1_TRI": 1, "P1_TET": 2, "P2_TRI": 3}
_F = {"ZERO": 0, "ONE": 1, "SIN2D": 2, "SIN3D": 3, "BUMP3D": 4}
_G = {"ZERO": 0, "X2MY2": 1, "LINEAR3D": 2}
_POL = {"ELEMENT": 0, "AXIS": 1}


def configs() -> dict:
    with open(CONFIGS) as fh:
        return {k: v for k, v in json.load(fh).items() if not k.startswith("_")}


def fem_spec(name: str, c: int | None = None, k: int | None = None) -> FemSpec:
    cfg = dict(configs()[name])
    if c is not None:
        cfg["c"] = c
    if k is not None:
        cfg["k"] = k
    return FemSpec(family=_FAM[cfg["family"]], c=cfg["c"], jitter=int(cfg["jitter"]), fkind=_F[cfg["f"]],
                   gkind=_G[cfg["g"]], policy=_POL[cfg["policy"]], k=cfg["k"] if cfg["f"] == "BUMP3D" else 1,
                   pad=0, seed=cfg["seed"], sigma=float(cfg.get("sigma", 0.0)))


def problem_size(spec: FemSpec):
    n, nnz, nodes = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().fem_problem_size(C.byref(spec), C.byref(n), C.byref(nnz), C.byref(nodes)), "fem_problem_size")
    return n.value, nnz.value, nodes.value


def fem_build(spec: FemSpec, row_begin: int = 0, row_end: int | None = None, device=None, stream=None):
    """Assemble rows [row_begin, row_end) of K_FF and B on the GPU.
    Returns dict(row_ptr, col, val, B) of torch CUDA tensors (col = global ids)."""
    import torch
    n, _, _ = problem_size(spec)
    row_end = n if row_end is None else row_end
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream if stream is None else stream.cuda_stream)
    rows = row_end - row_begin
    rp = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64()
    check(lib().fem_count(C.byref(spec), row_begin, row_end, C.c_void_p(rp.data_ptr()), C.byref(nnz), st),
          "fem_count")
    col = torch.empty(max(nnz.value, 1), dtype=torch.int64, device=dev)[:nnz.value]
    val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)[:nnz.value]
    k = spec.k
    B = torch.empty((k, max(rows, 1)), dtype=torch.float64, device=dev)[:, :rows]  # column-major (rows, k)
    check(lib().fem_assemble(C.byref(spec), row_begin, row_end, C.c_void_p(rp.data_ptr()),
                             C.c_void_p(col.data_ptr()), C.c_void_p(val.data_ptr()), C.c_void_p(B.data_ptr()),
                             max(rows, 1), st), "fem_assemble")
    return {"row_ptr": rp, "col": col, "val": val, "B": B.t(), "n_global": n, "row_begin": row_begin,
            "row_end": row_end}


FD_X2MY2, FD_EXPSIN = 1, 2


def fd_cube_build(N: int, fkind: int = FD_X2MY2, row_begin: int = 0, row_end: int | None = None, device=None,
                  stream=None):
    """The paper's Table 1 system (FD Laplace on N^3 nodes, identity boundary rows,
    b = f on the boundary; include/fem_gen.h fd_cube_*), rows [row_begin, row_end),
    assembled on the GPU.  Returns dict(row_ptr, col, val, b) of torch CUDA tensors."""
    import torch
    n = N ** 3
    row_end = n if row_end is None else row_end
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream if stream is None else stream.cuda_stream)
    rows = row_end - row_begin
    rp = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    nnz = C.c_int64()
    check(lib().fd_cube_count(N, row_begin, row_end, C.c_void_p(rp.data_ptr()), C.byref(nnz), st), "fd_cube_count")
    col = torch.empty(max(nnz.value, 1), dtype=torch.int64, device=dev)[:nnz.value]
    val = torch.empty(max(nnz.value, 1), dtype=torch.float64, device=dev)[:nnz.value]
    b = torch.empty(max(rows, 1), dtype=torch.float64, device=dev)[:rows]
    check(lib().fd_cube_assemble(N, fkind, row_begin, row_end, C.c_void_p(rp.data_ptr()), C.c_void_p(col.data_ptr()),
                                 C.c_void_p(val.data_ptr()), C.c_void_p(b.data_ptr()), st), "fd_cube_assemble")
    return {"row_ptr": rp, "col": col, "val": val, "b": b, "n": n}


def coo_to_csr(row, col, val, n_rows: int, n_cols: int | None = None, stream=None):
    """Generic COO -> CSR on the GPU (include/fem_gen.h coo_to_csr; SPEC coo_to_csr):
    (row, col) sorted, duplicates summed in input order.  row/col int64, val float64
    CUDA tensors.  Returns dict(row_ptr, col, val) of CUDA tensors (int64, int64, f64)."""
    import torch
    n_cols = n_rows if n_cols is None else n_cols
    dev = row.device
    row = row.to(torch.int64).contiguous()
    col = col.to(torch.int64).contiguous()
    val = val.to(torch.float64).contiguous()
    nnz = row.numel()
    if col.numel() != nnz or val.numel() != nnz:
        raise ValueError("coo_to_csr: row, col and val must have the same length")
    st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream if stream is None else stream.cuda_stream)
    rp = torch.empty(n_rows + 1, dtype=torch.int64, device=dev)
    co = torch.empty(max(nnz, 1), dtype=torch.int64, device=dev)
    vo = torch.empty(max(nnz, 1), dtype=torch.float64, device=dev)
    u = C.c_int64()
    check(lib().coo_to_csr(n_rows, n_cols, nnz, C.c_void_p(row.data_ptr()), C.c_void_p(col.data_ptr()),
                           C.c_void_p(val.data_ptr()), C.c_void_p(rp.data_ptr()), C.c_void_p(co.data_ptr()),
                           C.c_void_p(vo.data_ptr()), C.byref(u), st), "coo_to_csr")
    return {"row_ptr": rp, "col": co[:u.value], "val": vo[:u.value]}


def fem_element_triplets(spec, stream=None):
    """Element-by-element assembly, step 1 (include/fem_gen.h fem_element_coo): every
    element's stiffness K_e as (row, col, val) CUDA tensors over all lattice nodes,
    element-major.  Returns dict(row, col, val, n_nodes, npe)."""
    import torch
    ne, npe, nn = C.c_int64(), C.c_int32(), C.c_int64()
    check(lib().fem_element_count(C.byref(spec), C.byref(ne), C.byref(npe), C.byref(nn)), "fem_element_count")
    m = ne.value * npe.value * npe.value
    dev = torch.device("cuda", torch.cuda.current_device())
    st = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream if stream is None else stream.cuda_stream)
    r = torch.empty(max(m, 1), dtype=torch.int64, device=dev)[:m]
    c = torch.empty(max(m, 1), dtype=torch.int64, device=dev)[:m]
    v = torch.empty(max(m, 1), dtype=torch.float64, device=dev)[:m]
    check(lib().fem_element_coo(C.byref(spec), 0, ne.value, C.c_void_p(r.data_ptr()), C.c_void_p(c.data_ptr()),
                                C.c_void_p(v.data_ptr()), st), "fem_element_coo")
    return {"row": r, "col": c, "val": v, "n_nodes": nn.value, "npe": npe.value}


def fem_assemble_elements(spec, stream=None):
    """Element-by-element assembly on the GPU: fem_element_coo then coo_to_csr — the
    Neumann stiffness over all lattice nodes as dict(row_ptr, col, val)."""
    T = fem_element_triplets(spec, stream)
    return coo_to_csr(T["row"], T["col"], T["val"], T["n_nodes"], T["n_nodes"], stream)
