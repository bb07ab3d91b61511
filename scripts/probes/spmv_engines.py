"""Standalone SpMV time (pcg_spmv, CUDA events) of the one-chunk engines on the C5 matrix
and the Cube 3 FD grid: uniform-offset positions (default) vs ids everywhere (PCG_DIA=0)
vs the chunked engine (PCG_SHORT=0).  Development tool."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2201_05413_b200 as pcg  # noqa: E402
from paper_2201_05413_b200.problems import fd_cube_build, fem_build, fem_spec  # noqa: E402

for name in sys.argv[1:] or ["C5", "CUBE3"]:
    P = fd_cube_build(512) if name == "CUBE3" else fem_build(fem_spec(name))
    for env in ({}, {"PCG_DIA": "0"}, {"PCG_SHORT": "0"}):
        for k in ("PCG_DIA", "PCG_SHORT"):
            os.environ.pop(k, None)
        os.environ.update(env)
        A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
        st = A.stats()
        x = torch.rand(st["n"], dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            A.spmv(x, y)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            A.spmv(x, y)
        e1.record()
        torch.cuda.synchronize()
        print(name, env, "us", round(e0.elapsed_time(e1) * 100, 1), "dia_positions", st["dia_positions"], "dia_slices", st["dia_slices"], "slices", (st["n"] + 31) // 32,
              "positions", st["sell_entries"] // 32, flush=True)
        A.close()
