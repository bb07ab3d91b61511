"""Pipelined PCG vs PCG on the GPU and vs the oracle (development tool).

  python scripts/pipe_check.py [C1 C2 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_05413_b200 as pcg  # noqa: E402
from paper_2201_05413_b200.problems import configs, fem_build, fem_spec  # noqa: E402

for name in sys.argv[1:] or ["C1", "C2", "C3", "C4", "C6"]:
    cfg = configs()[name]
    P = fem_build(fem_spec(name))
    A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
    b = P["B"][:, 0].contiguous()
    out = {"config": name}
    for kind in ("pcg", "pipelined"):
        f = A.solve if kind == "pcg" else A.solve_pipelined
        ts = []
        for _ in range(4):
            x, info = f(b, tol=cfg["tol"], max_iter=cfg["max_iter"])
            ts.append(info["t_solve_s"])
        out[kind] = {"s": sorted(ts[1:])[1], "it": info["iterations"], "relres": info["relres_true"],
                     "status": info["status"]}
        out[kind + "_x"] = x
    xa, xb = out.pop("pcg_x"), out.pop("pipelined_x")
    out["relL2_pipe_vs_pcg"] = float(torch.linalg.norm(xa - xb) / torch.linalg.norm(xa))
    print(json.dumps(out), flush=True)
    A.close()
