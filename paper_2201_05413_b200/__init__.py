"""B200-native Jacobi-preconditioned CG for FEM Laplace systems (arxiv 2201.05413 hot path).

Thin Python binding over the C ABI of ``libpcg_b200.so`` (include/pcg.h,
include/fem_gen.h): argument marshalling only.  torch supplies device memory,
streams and the process group used to broadcast the NCCL id; every step of the
solve runs in the library's sm_100a kernels.  There is no CPU fallback: if the
library or a GPU is missing, calls raise.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import (PCG_FMT_AUTO, PCG_FMT_CSR, PCG_FMT_SELL, PCG_FORMAT_CSR, PCG_FORMAT_SELL,  # noqa: F401
                   PCG_OK, PCG_NOT_CONVERGED, PcgError, check, lib)
from .problems import FemSpec, coo_to_csr, fem_spec, fem_build  # noqa: F401

__all__ = ["Matrix", "Comm", "partition_rows", "fem_spec", "fem_build", "coo_to_csr", "PcgError", "kernel_launches"]


def _torch():
    import torch
    return torch


def _stream_ptr(stream):
    torch = _torch()
    if stream is None:
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    return C.c_void_p(stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream))


def _as_tensor(a, dtype):
    """torch tensor (any device) or numpy array -> contiguous tensor of dtype (no copy if possible)."""
    torch = _torch()
    if isinstance(a, np.ndarray):
        a = torch.from_numpy(np.ascontiguousarray(a))
    if a.dtype != dtype:
        a = a.to(dtype)
    return a.contiguous()


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None and t.numel() > 0 else C.c_void_p(0 if t is None else t.data_ptr())


def _pin_host(b, x, out):
    """Host tensors are staged from pinned memory.  A non-pinned host `out` is replaced
    by a pinned copy for the call and written back afterwards (_copy_back), so `out`
    holds the solution on return as documented."""
    user_out = None
    if b.device.type == "cpu":
        if not b.is_pinned():
            b = b.pin_memory()
        if not x.is_pinned():
            if out is not None and x.data_ptr() == out.data_ptr():
                user_out = out
            x = x.pin_memory()
    return b, x, user_out


def _copy_back(x, user_out):
    if user_out is None:
        return x
    user_out.copy_(x)
    return user_out


def kernel_launches() -> int:
    """Kernels launched by the library in this process (host launches + graph-executed)."""
    return int(lib().pcg_kernel_launches())


class Matrix:
    """Device-resident SPD matrix (CSR + SELL-32) with solver workspace."""

    def __init__(self, handle, n: int, nnz: int, comm=None):
        self._h = C.c_void_p(handle)
        self.n, self.nnz, self.comm = n, nnz, comm

    # -------------------------------------------------------------- creation
    @classmethod
    def from_csr(cls, row_ptr, col, val, fmt: str = "auto", stream=None, drop_zeros: bool = False,
                 reorder: str | None = None) -> "Matrix":
        torch = _torch()
        rp, ci, va = _as_tensor(row_ptr, torch.int64), _as_tensor(col, torch.int64), _as_tensor(val, torch.float64)
        n = rp.numel() - 1
        nnz = ci.numel()
        dev = rp.is_cuda
        if dev != ci.is_cuda or dev != va.is_cuda:
            raise ValueError("row_ptr, col and val must live on the same device")
        flags = (_lib.PCG_PTR_DEVICE if dev else _lib.PCG_PTR_HOST) | {
            "auto": PCG_FMT_AUTO, "csr": PCG_FMT_CSR, "sell": PCG_FMT_SELL, "tma": _lib.PCG_FMT_SELL_TMA,
            "sigma": _lib.PCG_FMT_SELL_SIGMA}[fmt]
        if drop_zeros:
            flags |= _lib.PCG_DROP_ZEROS
        if reorder not in (None, "rcm"):
            raise ValueError(f"reorder must be None or 'rcm', not {reorder!r}")
        if reorder == "rcm":
            flags |= _lib.PCG_REORDER_RCM
        h = C.c_void_p()
        check(lib().csr_create(n, nnz, _ptr(rp), _ptr(ci), _ptr(va), flags, _stream_ptr(stream), C.byref(h)),
              "csr_create")
        m = cls(h.value, n, nnz)
        if drop_zeros:
            m.nnz = m.stats()["nnz"]
        return m

    @classmethod
    def from_csr_dist(cls, comm: "Comm", n_global: int, row_begin: int, row_end: int, row_ptr_local, col_global,
                      val, fmt: str = "auto", stream=None, drop_zeros: bool = False) -> "Matrix":
        torch = _torch()
        rp, ci, va = (_as_tensor(row_ptr_local, torch.int64), _as_tensor(col_global, torch.int64),
                      _as_tensor(val, torch.float64))
        flags = (_lib.PCG_PTR_DEVICE if rp.is_cuda else _lib.PCG_PTR_HOST) | {
            "auto": PCG_FMT_AUTO, "csr": PCG_FMT_CSR, "sell": PCG_FMT_SELL, "tma": _lib.PCG_FMT_SELL_TMA,
            "sigma": _lib.PCG_FMT_SELL_SIGMA}[fmt]
        if drop_zeros:
            flags |= _lib.PCG_DROP_ZEROS
        h = C.c_void_p()
        check(lib().csr_create_dist(comm._h, n_global, row_begin, row_end, ci.numel(), _ptr(rp), _ptr(ci), _ptr(va),
                                    flags, _stream_ptr(stream), C.byref(h)), "csr_create_dist")
        m = cls(h.value, row_end - row_begin, ci.numel(), comm=comm)
        if drop_zeros:
            m.nnz = m.stats()["nnz"]
        return m

    def close(self):
        if self._h and self._h.value:
            lib().csr_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def stats(self) -> dict:
        s = _lib.MatrixStats()
        check(lib().pcg_matrix_get_stats(self._h, C.byref(s)), "pcg_matrix_get_stats")
        return s.as_dict()

    # -------------------------------------------------------------- operations
    def spmv(self, x, y=None, stream=None):
        torch = _torch()
        x = _as_tensor(x, torch.float64)
        if y is None:
            y = torch.empty(self.n, dtype=torch.float64, device=x.device)
        check(lib().pcg_spmv(self._h, _ptr(x), _ptr(y), _stream_ptr(stream)), "pcg_spmv")
        return y

    def solve(self, b, x0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None, raise_on=("error",),
              out=None):
        """Jacobi-PCG.  Returns (x, info).  b/x0 may be host or device tensors.  x is a new
        tensor on b's device (x0 is not modified) unless `out` is given: then `out` (same
        device as b, float64, contiguous) holds x0 on entry and the solution on return."""
        torch = _torch()
        b = _as_tensor(b, torch.float64)
        if out is not None:
            x = out
        else:
            x = torch.zeros_like(b) if x0 is None else _as_tensor(x0, torch.float64).clone()
        b, x, user_out = _pin_host(b, x, out)
        info = _lib.PcgInfo()
        st = lib().pcg_solve(self._h, _ptr(b), _ptr(x), float(tol), int(max_iter), _stream_ptr(stream),
                             C.byref(info))
        if st not in (PCG_OK, PCG_NOT_CONVERGED) or ("not_converged" in raise_on and st == PCG_NOT_CONVERGED):
            raise PcgError(st, "pcg_solve")
        d = info.as_dict()
        d["status_name"] = _lib.STATUS[st]
        return _copy_back(x, user_out), d

    def solve_pipelined(self, b, x0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None,
                        raise_on=("error",), out=None):
        """Pipelined Jacobi-PCG (pcg_solve_pipelined): one reduction per
        iteration.  Same conventions as solve()."""
        torch = _torch()
        b = _as_tensor(b, torch.float64)
        if out is not None:
            x = out
        else:
            x = torch.zeros_like(b) if x0 is None else _as_tensor(x0, torch.float64).clone()
        b, x, user_out = _pin_host(b, x, out)
        info = _lib.PcgInfo()
        st = lib().pcg_solve_pipelined(self._h, _ptr(b), _ptr(x), float(tol), int(max_iter), _stream_ptr(stream),
                                       C.byref(info))
        if st not in (PCG_OK, PCG_NOT_CONVERGED) or ("not_converged" in raise_on and st == PCG_NOT_CONVERGED):
            raise PcgError(st, "pcg_solve_pipelined")
        d = info.as_dict()
        d["status_name"] = _lib.STATUS[st]
        return _copy_back(x, user_out), d

    def bicgstab(self, b, x0=None, tol: float = 1e-10, max_iter: int = 50000, block: int = 1, stream=None,
                 raise_on=("error",), out=None, precond: str = "bj"):
        """Right-preconditioned BiCGSTAB with (Block-)Jacobi (pcg_bicgstab).
        Same conventions as solve(); block = 1 (point Jacobi), 2, 4 or 8.  precond="ilu0":
        Block-Jacobi with ILU(0) blocks of `block` rows (pcg_bicgstab_ilu; block <= 0: one
        block per SM)."""
        if precond == "ilu0":
            return self._bicgstab_ilu(b, x0, tol, max_iter, block, stream, raise_on, out)
        if precond != "bj":
            raise ValueError(f"precond must be 'bj' or 'ilu0', not {precond!r}")
        torch = _torch()
        b = _as_tensor(b, torch.float64)
        if out is not None:
            x = out
        else:
            x = torch.zeros_like(b) if x0 is None else _as_tensor(x0, torch.float64).clone()
        b, x, user_out = _pin_host(b, x, out)
        info = _lib.PcgInfo()
        st = lib().pcg_bicgstab(self._h, _ptr(b), _ptr(x), float(tol), int(max_iter), int(block), _stream_ptr(stream),
                                C.byref(info))
        if st not in (PCG_OK, PCG_NOT_CONVERGED) or ("not_converged" in raise_on and st == PCG_NOT_CONVERGED):
            raise PcgError(st, "pcg_bicgstab")
        d = info.as_dict()
        d["status_name"] = _lib.STATUS[st]
        return _copy_back(x, user_out), d

    def _bicgstab_ilu(self, b, x0, tol, max_iter, block, stream, raise_on, out):
        torch = _torch()
        b = _as_tensor(b, torch.float64)
        if out is not None:
            x = out
        else:
            x = torch.zeros_like(b) if x0 is None else _as_tensor(x0, torch.float64).clone()
        b, x, user_out = _pin_host(b, x, out)
        info = _lib.PcgInfo()
        st = lib().pcg_bicgstab_ilu(self._h, _ptr(b), _ptr(x), float(tol), int(max_iter), int(block),
                                    _stream_ptr(stream), C.byref(info))
        if st not in (PCG_OK, PCG_NOT_CONVERGED) or ("not_converged" in raise_on and st == PCG_NOT_CONVERGED):
            raise PcgError(st, "pcg_bicgstab_ilu")
        d = info.as_dict()
        d["status_name"] = _lib.STATUS[st]
        return _copy_back(x, user_out), d

    def solve_multi(self, B, X0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None, out=None):
        """k right-hand sides, B an (n, k) tensor (column-major storage is used at the ABI:
        pass B as B.T.contiguous().T or let this wrapper arrange it).  With `out` (an (n, k)
        float64 column-major tensor on B's device, i.e. out.t() contiguous), out holds X0 on
        entry and the solutions on return, and no copies are made around the library call."""
        return self._solve_k("pcg_solve_multi", B, X0, tol, max_iter, stream, out)

    def solve_block(self, B, X0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None, out=None):
        """include/pcg.h pcg_solve_block: block CG over the k <= 32 columns of B (one shared
        Krylov space).  Arguments and results as solve_multi."""
        return self._solve_k("pcg_solve_block", B, X0, tol, max_iter, stream, out)

    def _solve_k(self, fname, B, X0, tol, max_iter, stream, out):
        torch = _torch()
        if not isinstance(B, torch.Tensor):
            B = _as_tensor(B, torch.float64)
        n, k = B.shape
        Bc = B.t().contiguous()  # (k, n) row-major == (n, k) column-major, ld = n
        if out is not None:
            if not out.t().is_contiguous() or out.shape != (n, k) or out.dtype != torch.float64:
                raise ValueError("out must be an (n, k) float64 column-major tensor")
            Xc = out.t()
        else:
            Xc = torch.zeros_like(Bc) if X0 is None else _as_tensor(X0, torch.float64).t().contiguous()
        Bc, Xc, user_out = _pin_host(Bc, Xc, out.t() if out is not None else None)
        infos = (_lib.PcgInfo * k)()
        st = getattr(lib(), fname)(self._h, k, _ptr(Bc), n, _ptr(Xc), n, float(tol), int(max_iter),
                                   _stream_ptr(stream), infos)
        if st not in (PCG_OK, PCG_NOT_CONVERGED):
            raise PcgError(st, fname)
        out = []
        for i in range(k):
            d = infos[i].as_dict()
            d["status_name"] = _lib.STATUS[infos[i].status]
            out.append(d)
        return _copy_back(Xc, user_out).t(), out


class Comm:
    """NCCL communicator owned by the library (bootstrap via torch.distributed)."""

    def __init__(self, rank: int, size: int, unique_id: bytes):
        self._h = C.c_void_p()
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().pcg_comm_init(rank, size, buf, C.byref(self._h)), "pcg_comm_init")
        self.rank, self.size = rank, size

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().pcg_comm_unique_id(buf), "pcg_comm_unique_id")
        return buf.raw

    @classmethod
    def from_process_group(cls, group=None) -> "Comm":
        """Rank 0 draws the NCCL id; torch.distributed broadcasts it."""
        import torch.distributed as dist
        rank, size = dist.get_rank(group), dist.get_world_size(group)
        obj = [cls.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        return cls(rank, size, obj[0])

    @classmethod
    def host_callbacks(cls, group=None) -> "Comm":
        """Communicator whose exchange steps run as host callbacks over a torch.distributed
        process group (e.g. gloo): the library's distributed path with device data staged
        through host memory.  For validating that path where ranks share one GPU; the
        product path is NCCL (from_process_group)."""
        import torch
        import torch.distributed as dist
        rank, size = dist.get_rank(group), dist.get_world_size(group)

        def _arr(ptr, count, dtype):
            return np.ctypeslib.as_array(ptr, shape=(count,)) if count > 0 else np.zeros(0, dtype)

        def allreduce_f64(ctx, buf, count):
            try:
                a = _arr(buf, count, np.float64)
                t = torch.from_numpy(a.copy())
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
                a[:] = t.numpy()
                return 0
            except Exception:
                return 1

        def allreduce_max(ctx, buf, count):
            try:
                a = _arr(buf, count, np.int32)
                t = torch.from_numpy(a.copy())
                dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
                a[:] = t.numpy()
                return 0
            except Exception:
                return 1

        def allgather(ctx, mine, count, out):
            try:
                m = torch.from_numpy(_arr(mine, count, np.int64).copy())
                parts = [torch.empty_like(m) for _ in range(size)]
                dist.all_gather(parts, m, group=group)
                _arr(out, count * size, np.int64)[:] = torch.cat(parts).numpy()
                return 0
            except Exception:
                return 1

        def exchange(ctx, n_peers, peers, send, send_bytes, recv, recv_bytes):
            try:
                reqs, outs = [], []
                for t in range(n_peers):
                    p = int(peers[t])
                    sb, rb = int(send_bytes[t]), int(recv_bytes[t])
                    if sb > 0:
                        buf = (C.c_uint8 * sb).from_address(send[t])
                        reqs.append(dist.isend(torch.frombuffer(bytearray(buf), dtype=torch.uint8), p, group=group))
                    if rb > 0:
                        r = torch.empty(rb, dtype=torch.uint8)
                        reqs.append(dist.irecv(r, p, group=group))
                        outs.append((recv[t], r))
                for q in reqs:
                    q.wait()
                for addr, r in outs:
                    C.memmove(addr, r.numpy().ctypes.data, r.numel())
                return 0
            except Exception:
                return 1

        ops = _lib.CommOps(None, _lib.ALLREDUCE_F64(allreduce_f64), _lib.ALLREDUCE_MAX_I32(allreduce_max),
                           _lib.ALLGATHER_I64(allgather), _lib.EXCHANGE(exchange))
        self = cls.__new__(cls)
        self._h = C.c_void_p()
        self._ops = ops  # keep the callbacks alive as long as the communicator
        check(lib().pcg_comm_init_ops(rank, size, C.byref(ops), C.byref(self._h)), "pcg_comm_init_ops")
        self.rank, self.size = rank, size
        return self

    def set_timeout(self, seconds: float):
        """Failure detection (pcg.h): a distributed call that sees no progress for
        `seconds` (or an asynchronous NCCL error) aborts the communicator and raises
        PcgError(PCG_ERR_NCCL) instead of blocking."""
        check(lib().pcg_comm_set_timeout(self._h, float(seconds)), "pcg_comm_set_timeout")

    def info(self) -> dict:
        r, n, d = C.c_int32(), C.c_int32(), C.c_int32()
        check(lib().pcg_comm_get_info(self._h, C.byref(r), C.byref(n), C.byref(d)), "pcg_comm_get_info")
        return {"rank": r.value, "size": n.value, "device_allreduce": bool(d.value)}

    def abort(self):
        """ncclCommAbort: pending and later calls on this communicator fail with PCG_ERR_NCCL."""
        check(lib().pcg_comm_abort(self._h), "pcg_comm_abort")

    def close(self):
        if self._h and self._h.value:
            lib().pcg_comm_destroy(self._h)
            self._h = C.c_void_p()


def partition_rows(row_ptr, G: int) -> np.ndarray:
    """SURVEY §8(c).10 rule, computed by the library (host arrays)."""
    rp = np.ascontiguousarray(np.asarray(row_ptr, dtype=np.int64))
    out = np.zeros(G + 1, dtype=np.int64)
    check(lib().pcg_partition_rows(len(rp) - 1, rp.ctypes.data_as(C.c_void_p), G,
                                   out.ctypes.data_as(C.c_void_p)), "pcg_partition_rows")
    return out


def csr_rcm_order(row_ptr, col, stream=None):
    """include/pcg.h csr_rcm_order: reverse Cuthill-McKee order of a symmetric CSR pattern,
    computed on the GPU.  row_ptr/col: int64 host arrays or CUDA tensors;
    returns perm (new -> old) on the same side (numpy int64 or CUDA int64 tensor)."""
    torch = _torch()
    rp, ci = _as_tensor(row_ptr, torch.int64), _as_tensor(col, torch.int64)
    n = rp.numel() - 1
    dev = rp.is_cuda
    if dev != ci.is_cuda:
        raise ValueError("row_ptr and col must live on the same device")
    perm = torch.empty(max(n, 0), dtype=torch.int64, device=rp.device)
    check(lib().csr_rcm_order(n, ci.numel(), _ptr(rp), _ptr(ci), _lib.PCG_PTR_DEVICE if dev else _lib.PCG_PTR_HOST,
                              _stream_ptr(stream), _ptr(perm)), "csr_rcm_order")
    return perm if dev else perm.numpy()


def halo_ghosts(row_begin: int, row_end: int, col_global) -> np.ndarray:
    """Sorted unique remote columns of a rank's rows (host logic of csr_create_dist)."""
    col = np.ascontiguousarray(np.asarray(col_global, dtype=np.int64))
    cnt = C.c_int64()
    check(lib().pcg_halo_ghosts(row_begin, row_end, len(col), col.ctypes.data_as(C.c_void_p), None, 0,
                                C.byref(cnt)), "pcg_halo_ghosts")
    out = np.zeros(max(cnt.value, 1), dtype=np.int64)
    check(lib().pcg_halo_ghosts(row_begin, row_end, len(col), col.ctypes.data_as(C.c_void_p),
                                out.ctypes.data_as(C.c_void_p), cnt.value, C.byref(cnt)), "pcg_halo_ghosts")
    return out[:cnt.value]


def halo_recv_plan(ghosts, bounds):
    """Per-rank ghost counts and offsets (host logic of csr_create_dist)."""
    g = np.ascontiguousarray(np.asarray(ghosts, dtype=np.int64))
    b = np.ascontiguousarray(np.asarray(bounds, dtype=np.int64))
    G = len(b) - 1
    need, off = np.zeros(G, dtype=np.int64), np.zeros(G, dtype=np.int64)
    check(lib().pcg_halo_recv_plan(len(g), g.ctypes.data_as(C.c_void_p), G, b.ctypes.data_as(C.c_void_p),
                                   need.ctypes.data_as(C.c_void_p), off.ctypes.data_as(C.c_void_p)),
          "pcg_halo_recv_plan")
    return need, off


# ---------------------------------------------------------------- the C ABI's names
# (include/pcg.h, include/fem_gen.h): thin aliases of the methods above, so a caller
# can follow the header entry point by entry point.  Argument marshalling only.
def csr_create(row_ptr, col, val, fmt: str = "auto", stream=None, drop_zeros: bool = False,
               reorder: str | None = None) -> Matrix:
    """include/pcg.h csr_create: validate, narrow and upload a CSR matrix (host or device tensors);
    drop_zeros -> PCG_DROP_ZEROS, reorder="rcm" -> PCG_REORDER_RCM."""
    return Matrix.from_csr(row_ptr, col, val, fmt=fmt, stream=stream, drop_zeros=drop_zeros, reorder=reorder)


def csr_create_dist(comm: Comm, n_global: int, row_begin: int, row_end: int, row_ptr_local, col_global, val,
                    fmt: str = "auto", stream=None, drop_zeros: bool = False) -> Matrix:
    """include/pcg.h csr_create_dist: this rank's rows [row_begin, row_end) with global column ids."""
    return Matrix.from_csr_dist(comm, n_global, row_begin, row_end, row_ptr_local, col_global, val, fmt=fmt,
                                stream=stream, drop_zeros=drop_zeros)


def csr_destroy(A: Matrix) -> None:
    """include/pcg.h csr_destroy."""
    A.close()


def pcg_spmv(A: Matrix, x, y=None, stream=None):
    """include/pcg.h pcg_spmv: y = A x."""
    return A.spmv(x, y, stream=stream)


def pcg_solve(A: Matrix, b, x0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None):
    """include/pcg.h pcg_solve: Jacobi-PCG from x0; returns (x, info)."""
    return A.solve(b, x0=x0, tol=tol, max_iter=max_iter, stream=stream)


def pcg_solve_multi(A: Matrix, B, X0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None):
    """include/pcg.h pcg_solve_multi: k independent Jacobi-PCG solves; returns (X, infos)."""
    return A.solve_multi(B, X0=X0, tol=tol, max_iter=max_iter, stream=stream)


def pcg_solve_block(A: Matrix, B, X0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None):
    """include/pcg.h pcg_solve_block: block CG, the k columns in one Krylov space; returns (X, infos)."""
    return A.solve_block(B, X0=X0, tol=tol, max_iter=max_iter, stream=stream)


def pcg_solve_pipelined(A: Matrix, b, x0=None, tol: float = 1e-10, max_iter: int = 50000, stream=None):
    """include/pcg.h pcg_solve_pipelined: pipelined Jacobi-PCG (one reduction per iteration)."""
    return A.solve_pipelined(b, x0=x0, tol=tol, max_iter=max_iter, stream=stream)


def pcg_bicgstab(A: Matrix, b, x0=None, tol: float = 1e-10, max_iter: int = 50000, block_size: int = 1,
                 stream=None):
    """include/pcg.h pcg_bicgstab: right-preconditioned BiCGSTAB with (Block-)Jacobi."""
    return A.bicgstab(b, x0=x0, tol=tol, max_iter=max_iter, block=block_size, stream=stream)


def pcg_bicgstab_ilu(A: Matrix, b, x0=None, tol: float = 1e-10, max_iter: int = 50000, block_rows: int = 0,
                     stream=None):
    """include/pcg.h pcg_bicgstab_ilu: BiCGSTAB with Block-Jacobi ILU(0) blocks of block_rows rows."""
    return A.bicgstab(b, x0=x0, tol=tol, max_iter=max_iter, block=block_rows, stream=stream, precond="ilu0")


pcg_partition_rows = partition_rows
solve = pcg_solve  # SURVEY §8(b) "Python: pcg.solve(A, b, x0, tol, max_iter)"

__all__ += ["csr_create", "csr_create_dist", "csr_destroy", "pcg_spmv", "pcg_solve", "pcg_solve_multi",
            "pcg_solve_pipelined", "pcg_bicgstab", "pcg_bicgstab_ilu", "pcg_partition_rows", "csr_rcm_order", "solve",
            "pcg_solve_block"]
