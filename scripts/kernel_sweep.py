"""Per-kernel timing sweep (development tool): K1/K2 device time and GB/s for a config.

  python scripts/kernel_sweep.py --config C5 [--c 512] [--fmt auto] [--reps 20] [--solve]
"""
import argparse
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2201_05413_b200 as pcg  # noqa: E402
from paper_2201_05413_b200.problems import fem_build, fem_spec, problem_size  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--c", type=int, default=None)
ap.add_argument("--fmt", default="auto")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--solve", action="store_true")
ap.add_argument("--drop-zeros", action="store_true")
a = ap.parse_args()
spec = fem_spec(a.config, c=a.c)
n, nnz, _ = problem_size(spec)
P = fem_build(spec)
nnz = P["col"].numel()  # the 3D element pattern has no closed form (problem_size: -1)
A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"], fmt=a.fmt, drop_zeros=a.drop_zeros)
nnz = A.stats()["nnz"]  # stored entries (fewer with --drop-zeros)
b = P["B"][:, 0].contiguous()
del P
torch.cuda.synchronize()
us = (C.c_double * 3)()
done = C.c_int32()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    pcg.check(pcg.lib().pcg_profile_kernels(A._h, C.c_void_p(b.data_ptr()), a.reps, st, us, C.byref(done)), "profile")
stats = A.stats()
mat = 12.0 * nnz + 4.0 * (n + 1)
if stats["schedule"] == 3:  # K1a: mean over the deferral cycle (PCG_XDEFER: 4 default, 2, 0)
    xm = int(os.environ.get("PCG_XDEFER", "4"))
    byts = [{0: 40.0, 2: 36.0, 4: 34.0}.get(xm, 34.0) * n, mat + 16.0 * n, 40.0 * n]
else:
    byts = [0.0, mat + 48.0 * n, 40.0 * n]
out = {"config": a.config, "c": spec.c, "n": n, "nnz": nnz, "env": {k: v for k, v in os.environ.items() if k.startswith("PCG_")},
       "format": stats["format"], "schedule": stats["schedule"], "stages": stats["stages"],
       "us": list(us), "GBps": [b_ / u / 1e3 if u else 0 for b_, u in zip(byts, us)],
       "iter_us": sum(us), "iter_frac": sum(byts) / sum(us) / 1e3 / 6556.2,
       "iter_frac_vs_88n": (mat + 88.0 * n) / sum(us) / 1e3 / 6556.2,
       "spmv_us": {"csr": stats["spmv_us_csr"], "sell": stats["spmv_us_sell"], "tma": stats["spmv_us_tma"]},
       "sell_pad": stats["sell_entries"] / max(nnz, 1), "short_rows": stats["short_rows"], "max_row_len": stats["max_row_len"]}
if a.solve:
    x, info = A.solve(b)
    x, info = A.solve(b)
    out["solve_s"] = info["t_solve_s"]
    out["iterations"] = info["iterations"]
    out["us_per_iter"] = info["t_solve_s"] * 1e6 / max(1, info["iterations"])
print(json.dumps(out))
