"""Seeded synthetic-input helpers shared by the tests and bench.py (no method arithmetic).

relabel: a mesh generator's node numbering is arbitrary (the paper's Sphere meshes come
from a mesher, Table 1); the lattice configs are generated in lexicographic
order, which is already banded.  A seeded random relabelling stands in for an unordered
mesher output: B = Q A Q^T with B[k, l] = A[q[k], q[l]],
q = argsort(SplitMix64(seed, i)) (stable), rows re-sorted by column.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def _splitmix64(seed: int, idx: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + (idx.astype(np.uint64) + np.uint64(1)) * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def relabel_order(n: int, seed: int) -> np.ndarray:
    """q[k] = the original node placed at new position k (int64)."""
    return np.argsort(_splitmix64(seed, np.arange(n, dtype=np.uint64)), kind="stable").astype(np.int64)


def relabel_csr_numpy(row_ptr, col, val, q):
    """B = Q A Q^T on host arrays (numpy); returns (row_ptr, col, val), rows sorted by column."""
    row_ptr, col, val, q = (np.asarray(a) for a in (row_ptr, col, val, q))
    n = len(row_ptr) - 1
    iq = np.empty(n, dtype=np.int64)
    iq[q] = np.arange(n)
    ln = np.diff(row_ptr)[q]
    rp = np.concatenate([[0], np.cumsum(ln)]).astype(np.int64)
    src = np.repeat(row_ptr[q], ln) + (np.arange(rp[-1]) - np.repeat(rp[:-1], ln))
    nr = np.repeat(np.arange(n, dtype=np.int64), ln)
    nc = iq[col[src]]
    o = np.lexsort((nc, nr))
    return rp, nc[o].astype(np.int64), np.asarray(val)[src][o]


def relabel_csr_torch(row_ptr, col, val, q):
    """The same relabelling on torch tensors (device-resident inputs for bench.py)."""
    import torch
    dev = row_ptr.device
    q = torch.as_tensor(q, device=dev, dtype=torch.int64)
    n = row_ptr.numel() - 1
    iq = torch.empty_like(q)
    iq[q] = torch.arange(n, device=dev, dtype=torch.int64)
    ln = (row_ptr[1:] - row_ptr[:-1])[q]
    rp = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    rp[1:] = torch.cumsum(ln, 0)
    nnz = int(rp[-1])
    nr = torch.repeat_interleave(torch.arange(n, device=dev, dtype=torch.int64), ln, output_size=nnz)
    src = row_ptr[:-1][q][nr] + (torch.arange(nnz, device=dev, dtype=torch.int64) - rp[:-1][nr])
    nc = iq[col[src]]
    o = torch.argsort(nr * n + nc)
    return rp, nc[o].contiguous(), val[src][o].contiguous()
