"""ctypes declarations of the C ABI in include/pcg.h and include/fem_gen.h.

Argument marshalling only: every step of the solve runs in libpcg_b200.so.
Importing fails loudly when the library is missing (no CPU fallback exists).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# PCG_LIB_VARIANT=<name> loads _variants/libpcg_<name>.so (scripts/build_variant.py: A/B builds
# of the same sources with -D knobs; development only, never the default)
LIB_PATH = (os.path.join(HERE, "_variants", f"libpcg_{os.environ['PCG_LIB_VARIANT']}.so")
            if os.environ.get("PCG_LIB_VARIANT") else os.path.join(HERE, "libpcg_b200.so"))

STATUS = ["PCG_OK", "PCG_NOT_CONVERGED", "PCG_ERR_INVALID_ARG", "PCG_ERR_INDEX_OUT_OF_RANGE",
          "PCG_ERR_UNSORTED_OR_DUPLICATE", "PCG_ERR_DIMENSION_MISMATCH", "PCG_ERR_ZERO_DIAGONAL",
          "PCG_ERR_NOT_SPD", "PCG_ERR_NONFINITE", "PCG_ERR_OOM", "PCG_ERR_CUDA", "PCG_ERR_NCCL", "PCG_ERR_BREAKDOWN"]
(PCG_OK, PCG_NOT_CONVERGED, PCG_ERR_INVALID_ARG, PCG_ERR_INDEX_OUT_OF_RANGE,
 PCG_ERR_UNSORTED_OR_DUPLICATE, PCG_ERR_DIMENSION_MISMATCH, PCG_ERR_ZERO_DIAGONAL, PCG_ERR_NOT_SPD,
 PCG_ERR_NONFINITE, PCG_ERR_OOM, PCG_ERR_CUDA, PCG_ERR_NCCL, PCG_ERR_BREAKDOWN) = range(13)
PCG_PTR_HOST, PCG_PTR_DEVICE = 0x0, 0x1
PCG_DROP_ZEROS = 0x100
PCG_REORDER_RCM = 0x200
PCG_FMT_AUTO, PCG_FMT_CSR, PCG_FMT_SELL, PCG_FMT_SELL_TMA, PCG_FMT_SELL_SIGMA = 0x00, 0x10, 0x20, 0x30, 0x40
PCG_FORMAT_CSR, PCG_FORMAT_SELL, PCG_FORMAT_SELL_TMA, PCG_FORMAT_SELL_SIGMA = 1, 2, 3, 4


class PcgInfo(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("relres_recurrence", C.c_double),
                ("relres_true", C.c_double), ("converged", C.c_int32), ("status", C.c_int32),
                ("replacements", C.c_int64), ("t_solve_s", C.c_double),
                ("bytes_algorithmic", C.c_double), ("flops", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class MatrixStats(C.Structure):
    _fields_ = [("n", C.c_int64), ("nnz", C.c_int64), ("format", C.c_int32),
                ("max_row_len", C.c_int32), ("sell_entries", C.c_int64), ("t_setup_s", C.c_double),
                ("device_bytes", C.c_double), ("spmv_us_csr", C.c_double),
                ("spmv_us_sell", C.c_double), ("n_ghost", C.c_int64), ("row_begin", C.c_int64),
                ("row_end", C.c_int64), ("n_global", C.c_int64), ("spmv_us_tma", C.c_double),
                ("stage_entries", C.c_int64), ("stages", C.c_int32), ("schedule", C.c_int32),
                ("spmv_us_sigma", C.c_double), ("sigma", C.c_int32), ("reorder", C.c_int32),
                ("overlap_rows", C.c_int64), ("d16_slices", C.c_int64),
                ("spmm_windowed", C.c_int32), ("short_rows", C.c_int32), ("dia_slices", C.c_int32),
                ("dia_positions", C.c_int64), ("dval_slices", C.c_int64), ("pat_slices", C.c_int64), ("npat", C.c_int32),
                ("aligned_slices", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


# host-callback communicator (include/pcg.h pcg_comm_ops)
ALLREDUCE_F64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.c_int64)
ALLREDUCE_MAX_I32 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int32), C.c_int64)
ALLGATHER_I64 = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int64), C.c_int64, C.POINTER(C.c_int64))
EXCHANGE = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p),
                       C.POINTER(C.c_int64), C.POINTER(C.c_void_p), C.POINTER(C.c_int64))


class CommOps(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allreduce_sum_f64", ALLREDUCE_F64), ("allreduce_max_i32", ALLREDUCE_MAX_I32),
                ("allgather_i64", ALLGATHER_I64), ("exchange", EXCHANGE)]


class FemSpec(C.Structure):
    _fields_ = [("family", C.c_int32), ("c", C.c_int32), ("jitter", C.c_int32),
                ("fkind", C.c_int32), ("gkind", C.c_int32), ("policy", C.c_int32),
                ("k", C.c_int32), ("pad", C.c_int32), ("seed", C.c_uint64), ("sigma", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2201_05413_b200.build` "
                          "(the product has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    P = C.POINTER
    sig = {
        "csr_create": [i64, i64, vp, vp, vp, C.c_int, vp, P(vp)],
        "csr_destroy": [vp],
        "pcg_matrix_get_stats": [vp, P(MatrixStats)],
        "pcg_spmv": [vp, vp, vp, vp],
        "pcg_solve": [vp, vp, vp, dbl, i64, vp, P(PcgInfo)],
        "pcg_solve_multi": [vp, i32, vp, i64, vp, i64, dbl, i64, vp, P(PcgInfo)],
        "pcg_solve_block": [vp, i32, vp, i64, vp, i64, dbl, i64, vp, P(PcgInfo)],
        "pcg_partition_rows": [i64, vp, i32, vp],
        "pcg_comm_unique_id": [vp],
        "pcg_halo_ghosts": [i64, i64, i64, vp, vp, i64, P(i64)],
        "pcg_halo_recv_plan": [i64, vp, i32, vp, vp, vp],
        "pcg_comm_init": [i32, i32, vp, P(vp)],
        "pcg_comm_init_ops": [i32, i32, P(CommOps), P(vp)],
        "pcg_comm_destroy": [vp],
        "pcg_comm_abort": [vp],
        "pcg_comm_set_timeout": [vp, dbl],
        "pcg_comm_get_info": [vp, P(i32), P(i32), P(i32)],
        "pcg_dar_emulate": [i32, i32, i32, vp, vp],
        "csr_create_dist": [vp, i64, i64, i64, i64, vp, vp, vp, C.c_int, vp, P(vp)],
        "pcg_profile_kernels": [vp, vp, i32, vp, vp, P(i32)],
        "pcg_profile_multi": [vp, i32, vp, i64, i32, vp, vp, P(i32)],
        "pcg_bicgstab": [vp, vp, vp, C.c_double, i64, i32, vp, P(PcgInfo)],
        "pcg_bicgstab_ilu": [vp, vp, vp, C.c_double, i64, i64, vp, P(PcgInfo)],
        "pcg_solve_pipelined": [vp, vp, vp, C.c_double, i64, vp, P(PcgInfo)],
        "fd_cube_count": [i64, i64, i64, vp, P(i64), vp],
        "fd_cube_assemble": [i64, i32, i64, i64, vp, vp, vp, vp, vp],
        "coo_to_csr": [i64, i64, i64, vp, vp, vp, vp, vp, vp, P(i64), vp],
        "csr_rcm_order": [i64, i64, vp, vp, C.c_int, vp, vp],
        "fem_element_count": [P(FemSpec), P(i64), P(i32), P(i64)],
        "fem_element_coo": [P(FemSpec), i64, i64, vp, vp, vp, vp],
        "fem_problem_size": [P(FemSpec), P(i64), P(i64), P(i64)],
        "fem_count": [P(FemSpec), i64, i64, vp, P(i64), vp],
        "fem_assemble": [P(FemSpec), i64, i64, vp, vp, vp, vp, i64, vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    L.pcg_last_error.restype = C.c_char_p
    L.pcg_last_error.argtypes = []
    L.pcg_status_string.restype = C.c_char_p
    L.pcg_status_string.argtypes = [C.c_int]
    L.pcg_kernel_launches.restype = C.c_int64
    L.pcg_kernel_launches.argtypes = []
    _lib = L
    return L


class PcgError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        msg = lib().pcg_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")


def check(status: int, where: str, ok=(PCG_OK,)):
    if status not in ok:
        raise PcgError(status, where)
    return status
