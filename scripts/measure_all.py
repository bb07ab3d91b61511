"""One line per benchmark config (C1-C6, full size, one GPU): time-to-solution, iterations
against the oracle golden, rel-L2 on the golden's sampled entries, true relres,
standalone SpMV GB/s and the iteration's fraction of the byte roofline
(development tool; feeds BASELINE.md §7).

  python scripts/measure_all.py [C1 C2 ...]
"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2201_05413_b200 as pcg  # noqa: E402
from paper_2201_05413_b200.problems import configs, fem_build, fem_spec  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
gold = json.load(open(os.path.join(ROOT, "tests", "golden", "oracle_full.json")))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5", "C6"]
torch.cuda.set_device(0)
for name in names:
    cfg = configs()[name]
    P = fem_build(fem_spec(name))
    n = P["row_ptr"].numel() - 1
    nnz = P["col"].numel()
    A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
    B = P["B"]
    k = B.shape[1]
    del P
    times, infos, X = [], None, None
    for rep in range(4):
        if k > 1:
            X, infos = A.solve_multi(B, tol=cfg["tol"], max_iter=cfg["max_iter"])
        else:
            x, inf = A.solve(B[:, 0].contiguous(), tol=cfg["tol"], max_iter=cfg["max_iter"])
            X, infos = x[:, None], [inf]
        if rep:
            times.append(infos[0]["t_solve_s"])
    t = statistics.median(times)
    its = [i["iterations"] for i in infos]
    # standalone SpMV
    xs = torch.ones(n, dtype=torch.float64, device="cuda")
    ys = torch.empty_like(xs)
    for _ in range(3):
        A.spmv(xs, ys)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        A.spmv(xs, ys)
    e1.record()
    torch.cuda.synchronize()
    spmv_us = e0.elapsed_time(e1) * 1e3 / 20
    spmv_gbs = (12.0 * nnz + 4.0 * (n + 1) + 16.0 * n) / spmv_us / 1e3
    it_bytes = 12.0 * nnz + 4.0 * (n + 1) + 96.0 * k * n
    frac = it_bytes * max(its) / t / 1e9 / peak
    row = {"config": name, "n": n, "nnz": nnz, "k": k, "time_s": t, "iterations": its,
           "relres_true_max": max(i["relres_true"] for i in infos), "spmv_GBps": spmv_gbs,
           "spmv_frac": spmv_gbs / peak, "iteration_frac_96kn": frac, "format": A.stats()["format"]}
    g = gold.get("C5full" if name == "C5" else name)
    if g:
        idx = np.array(g["sample_idx"])
        Xc = X.cpu().numpy()
        row["oracle_iterations"] = [r["iterations"] for r in g["rhs"]]
        row["relL2_sampled_max"] = max(float(np.linalg.norm(Xc[idx, j] - np.array(r["x_sample"])) /
                                             np.linalg.norm(r["x_sample"])) for j, r in enumerate(g["rhs"]))
        row["oracle_seconds_1thread"] = g.get("seconds")
    print(json.dumps(row), flush=True)
    A.close()
    del B, X
    torch.cuda.empty_cache()
