"""Small end-to-end run of every device path, for compute-sanitizer (development tool).

  compute-sanitizer --tool memcheck python scripts/sanitize_run.py
(compute-sanitizer is closed on this round's GPU pool; the plain run is the check.)

Exercises: FEM + FD generators, csr_create (CSR / SELL / SELL-C-sigma / TMA formats),
SpMV, CG through the conditional-graph loop and the persistent kernel, multi-RHS,
BiCGSTAB (point and block Jacobi) and a 1-rank NCCL-less callback communicator is
not included (multi-process).  Sizes are tiny so the instrumented run stays short.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2201_05413_b200 as pcg  # noqa: E402
from paper_2201_05413_b200.problems import fd_cube_build, fem_build, fem_spec  # noqa: E402

torch.cuda.set_device(0)
out = []
for name, c in (("C1", 16), ("C2", 24), ("C3", 12), ("C5", 16), ("C6", 8)):
    P = fem_build(fem_spec(name, c=c))
    for fmt in ("auto", "csr", "sell", "sigma", "tma"):
        try:
            A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"], fmt=fmt)
        except pcg.PcgError:
            continue  # e.g. TMA staging unavailable for the matrix
        b = P["B"][:, 0].contiguous()
        y = A.spmv(b)
        for persist in ("0", "1"):
            os.environ["PCG_PERSIST"] = persist
            x, info = A.solve(b, tol=1e-10)
            out.append((name, fmt, persist, info["iterations"], info["status"]))
        x, info = A.bicgstab(b, tol=1e-10)
        out.append((name, fmt, "bicg", info["iterations"], info["status"]))
        A.close()
P = fem_build(fem_spec("C4", c=16, k=5))
A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
X, infos = A.solve_multi(P["B"], tol=1e-10)
out.append(("C4", "multi", "", [i["iterations"] for i in infos], [i["status"] for i in infos]))
G = fd_cube_build(10)
A = pcg.Matrix.from_csr(G["row_ptr"], G["col"], G["val"])
for bs in (1, 2, 4, 8):
    x, info = A.bicgstab(G["b"], tol=1e-12, block=bs)
    out.append(("CUBE10", bs, "bicg", info["iterations"], info["status"]))
# round 2 paths: ILU(0) blocks (packed records and the cp.async ring), the deferred x
# update's cycles (graph loop), max_iter stops inside a cycle
for pk in ("1", "0"):
    os.environ["PCG_ILU_PACKED"] = pk
    for bs in (100, 0):
        A = pcg.Matrix.from_csr(G["row_ptr"], G["col"], G["val"], fmt="sell")
        x, info = A.bicgstab(G["b"], tol=1e-12, block=bs, precond="ilu0")
        out.append(("CUBE10-ilu0", pk, bs, info["iterations"], info["status"]))
        A.close()
os.environ["PCG_PERSIST"] = "0"
P = fem_build(fem_spec("C1", c=16))
for xd in ("4", "2", "0"):
    os.environ["PCG_XDEFER"] = xd
    A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"])
    b = P["B"][:, 0].contiguous()
    for mi in (5, 6, 7, 1000):
        x, info = A.solve(b, tol=1e-10, max_iter=mi)
        out.append(("C1-xdefer", xd, mi, info["iterations"], info["status"]))
    A.close()
torch.cuda.synchronize()
for o in out:
    print(o)
print("sanitize_run OK")
