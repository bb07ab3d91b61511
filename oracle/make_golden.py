"""Write tests/golden/oracle_full.json: oracle results at the full BASELINE.json sizes.

TEST INFRASTRUCTURE.  Calls only oracle/ (never the CUDA product).  The GPU
parity tests compare full-size GPU solves against these stored values on
sampled outputs (the oracle is too slow to run inside the test at full size).

  python -m oracle.make_golden [C1 C2 C3 C4 C5ladder]

Per config: n, nnz, iterations, relres_true, ||x||_2, ||b||_2 and x at 257 sampled
indices (seeded), per right-hand side.  "C5ladder" records the oracle's iteration
counts for the C5 construction at c = 32, 64, 128, 256 (C5 itself, c = 512, does
not fit the oracle's memory/time budget; its GPU count is checked against this
ladder's doubling ratio).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

import oracle as O

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                   "oracle_full.json")


def sample_idx(n, m=257, seed=12345):
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, n - 1, n // 2], rng.integers(0, n, m - 3)]))
    return idx


def run(name):
    t0 = time.time()
    P = O.build_problem(name)
    A, B = P["A"], P["B"]
    cfg = P["cfg"]
    idx = sample_idx(A.n)
    cols = []
    for j in range(B.shape[1]):
        r = O.pcg(A, B[:, j], tol=cfg["tol"], max_iter=cfg["max_iter"])
        cols.append({"iterations": r.iterations, "relres_true": r.relres_true, "status": r.status,
                     "x_norm": float(np.linalg.norm(r.x)), "b_norm": float(np.linalg.norm(B[:, j])),
                     "x_sample": r.x[idx].tolist()})
        print(name, j, r.iterations, f"{time.time() - t0:.0f}s", flush=True)
    return {"n": A.n, "nnz": A.nnz, "sample_idx": idx.tolist(), "rhs": cols,
            "row_ptr_sample": A.row_ptr[idx].tolist(), "seconds": time.time() - t0}


def ladder():
    out = {}
    for c in (32, 64, 128, 256):
        P = O.build_problem("C5", c=c)
        r = O.pcg(P["A"], P["B"][:, 0], tol=1e-10)
        out[str(c)] = {"n": P["A"].n, "iterations": r.iterations, "relres_true": r.relres_true}
        print("C5 ladder", c, r.iterations, flush=True)
    return out


def main(names):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    data["_doc"] = ("written by oracle/make_golden.py (oracle only); x_sample at sample_idx per RHS; "
                    "C5ladder = oracle iterations of the C5 construction at smaller c")
    for nm in names:
        data[nm] = ladder() if nm == "C5ladder" else run(nm)
        with open(OUT, "w") as fh:
            json.dump(data, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C4", "C5ladder", "C3"])
