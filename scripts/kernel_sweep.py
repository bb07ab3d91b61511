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
a = ap.parse_args()
spec = fem_spec(a.config, c=a.c)
n, nnz, _ = problem_size(spec)
P = fem_build(spec)
A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"], fmt=a.fmt)
b = P["B"][:, 0].contiguous()
del P
torch.cuda.synchronize()
us1, us2, done = C.c_double(), C.c_double(), C.c_int32()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    pcg.check(pcg.lib().pcg_profile_kernels(A._h, C.c_void_p(b.data_ptr()), a.reps, st, C.byref(us1), C.byref(us2),
                                             C.byref(done)), "profile")
k1 = 12.0 * nnz + 4.0 * (n + 1) + 48.0 * n
k2 = 40.0 * n
out = {"config": a.config, "c": spec.c, "n": n, "nnz": nnz, "env_chunk": os.environ.get("PCG_K1_CHUNK"),
       "stats": A.stats(), "k1_us": us1.value, "k1_GBps": k1 / us1.value / 1e3, "k2_us": us2.value,
       "k2_GBps": k2 / us2.value / 1e3, "iter_frac": (k1 + k2) / (us1.value + us2.value) / 1e3 / 6556.2}
if a.solve:
    x, info = A.solve(b)
    x, info = A.solve(b)
    out["solve_s"] = info["t_solve_s"]
    out["iterations"] = info["iterations"]
    out["us_per_iter"] = info["t_solve_s"] * 1e6 / max(1, info["iterations"])
print(json.dumps(out))
