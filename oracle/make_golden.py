"""Write tests/golden/oracle_full.json: oracle results at the full BASELINE.json sizes.

TEST INFRASTRUCTURE.  Calls only oracle/ (never the CUDA product).  The GPU
parity tests compare full-size GPU solves against these stored values on
sampled outputs (the oracle is too slow to run inside the test at full size).

  python -m oracle.make_golden [C1 C2 C3 C4 C5ladder C5c256 C5full]

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


def run(name, c=None):
    t0 = time.time()
    P = O.build_problem(name, c=c)
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


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def c5full():
    """C5 at full size: mesh -> free-lattice assembly -> Jacobi-PCG, all oracle."""
    cfg = O.configs()["C5"]
    t0 = time.time()
    mesh = O.Mesh(O.P1_TET, cfg["c"])
    A, b = O.assemble_free_lattice(mesh, O.F_SIN3D, (1.0, 0.0, 0.0, 0.0), copy=False)
    del mesh
    t_asm = time.time() - t0
    print("C5full assembled", A.n, A.nnz, f"{t_asm:.0f}s", flush=True)
    idx = sample_idx(A.n)
    t1 = time.time()
    r = O.pcg(A, b, tol=cfg["tol"], max_iter=cfg["max_iter"])
    t_solve = time.time() - t1
    print("C5full", r.iterations, f"{t_solve:.0f}s", flush=True)
    return {"n": A.n, "nnz": A.nnz, "sample_idx": idx.tolist(),
            "rhs": [{"iterations": r.iterations, "relres_true": r.relres_true, "status": r.status,
                     "x_norm": float(np.linalg.norm(r.x)), "b_norm": float(np.linalg.norm(b)),
                     "x_sample": r.x[idx].tolist()}],
            "row_ptr_sample": A.row_ptr[idx].tolist(), "seconds": time.time() - t0,
            "oracle_timing": {"assembly_s": t_asm, "solve_s": t_solve,
                              "solve_s_per_iteration": t_solve / max(r.iterations, 1), "threads": 1,
                              "cpu": _cpu_model(), "host": "development container (not the GPU box)"}}


def main(names):
    data = {}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            data = json.load(fh)
    data["_doc"] = ("written by oracle/make_golden.py (oracle only); x_sample at sample_idx per RHS; "
                    "C5ladder = oracle iterations of the C5 construction at smaller c")
    for nm in names:
        if nm == "C5ladder":
            data[nm] = ladder()
        elif nm == "C5full":
            data[nm] = c5full()
        elif nm == "C5c256":
            data[nm] = run("C5", c=256)
        else:
            data[nm] = run(nm)
        cur = {}
        if os.path.exists(OUT):
            with open(OUT) as fh:
                cur = json.load(fh)
        cur.update({"_doc": data["_doc"], nm: data[nm]})
        with open(OUT, "w") as fh:
            json.dump(cur, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C4", "C5ladder", "C3"])
