"""Multi-RHS per-kernel timing (development tool): SpMM pass and R/Z pass of the
k-column PCG, device time and GB/s against SURVEY §8(d)'s per-iteration bytes.

  python scripts/multi_sweep.py --config C4 [--c 128] [--k 16] [--reps 20] [--solve]
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
ap.add_argument("--config", default="C4")
ap.add_argument("--c", type=int, default=None)
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--solve", action="store_true")
a = ap.parse_args()
spec = fem_spec(a.config, c=a.c, k=a.k)
n, nnz, _ = problem_size(spec)
P = fem_build(spec)
nnz = P["col"].numel()  # the 3D element pattern has no closed form (problem_size: -1)
A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
B = P["B"]  # (n, k) view of a column-major block
k = B.shape[1]
Bc = B.t().contiguous()
del P
torch.cuda.synchronize()
us = (C.c_double * 3)()
done = C.c_int32()
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    pcg.check(pcg.lib().pcg_profile_multi(A._h, k, C.c_void_p(Bc.data_ptr()), n, a.reps, st, us, C.byref(done)),
              "pcg_profile_multi")
Kp = 1
while Kp < k:
    Kp *= 2
mat = 12.0 * nnz + 4.0 * (n + 1)
byts = [{0: 40.0, 2: 36.0, 4: 34.0}.get(int(os.environ.get("PCG_XDEFER", "4")), 34.0) * k * n, mat + 16.0 * k * n,
        40.0 * k * n]
out = {"config": a.config, "c": spec.c, "n": n, "nnz": nnz, "k": k, "K": Kp,
       "env": {kk: v for kk, v in os.environ.items() if kk.startswith("PCG_")},
       "us": list(us), "GBps": [b_ / u / 1e3 if u else 0 for b_, u in zip(byts, us)],
       "iter_us": sum(us), "iter_frac": sum(byts) / sum(us) / 1e3 / 6549.1,
       "iter_frac_vs_88kn": (mat + 88.0 * k * n) / sum(us) / 1e3 / 6549.1, "reps": done.value}
if a.solve:
    X, infos = A.solve_multi(B)
    X, infos = A.solve_multi(B)
    out["solve_s"] = infos[0]["t_solve_s"]
    out["iterations"] = [i["iterations"] for i in infos]
    out["us_per_block_iter"] = infos[0]["t_solve_s"] * 1e6 / max(out["iterations"])
print(json.dumps(out))
