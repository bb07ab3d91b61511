"""Seeded COO triplet generator for the coo_to_csr tests (oracle pins and GPU parity).

Random numbers only: no arithmetic of the method lives here.  Both the oracle tests
and the GPU tests draw their inputs from this module.
"""
import numpy as np


def triplets(seed: int, n_rows: int, n_cols: int, nnz: int, n_keys: int | None = None):
    """nnz entries over (at most) n_keys distinct (row, col) positions, in random order,
    so that most positions repeat; values uniform in [-1, 1) with a few exact opposites
    (duplicate groups that cancel to an explicit zero)."""
    rng = np.random.default_rng(seed)
    if n_keys is None:
        n_keys = max(1, nnz // 3)
    kr = rng.integers(0, max(n_rows, 1), n_keys + 1)
    kc = rng.integers(0, max(n_cols, 1), n_keys + 1)
    pick = rng.integers(0, n_keys, nnz)
    val = rng.uniform(-1.0, 1.0, nnz)
    if nnz >= 4:  # an exact cancelling pair alone on one more position (kept as an explicit 0)
        hit = (kr[:n_keys] == kr[n_keys]) & (kc[:n_keys] == kc[n_keys])
        if not hit.any():
            pick[0] = pick[1] = n_keys
            val[1] = -val[0]
    return kr[pick].astype(np.int64), kc[pick].astype(np.int64), val
