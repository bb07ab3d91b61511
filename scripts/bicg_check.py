import sys, time, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import oracle as O, paper_2201_05413_b200 as pcg
from paper_2201_05413_b200.problems import fd_cube_build
for N in (16, 40, 64):
    A, b = O.fd_cube(N)
    G = fd_cube_build(N)
    assert np.array_equal(G["row_ptr"].cpu().numpy(), A.row_ptr) and np.array_equal(G["col"].cpu().numpy(), A.col)
    assert np.array_equal(G["val"].cpu().numpy(), A.val) and np.array_equal(G["b"].cpu().numpy(), b)
    M = pcg.Matrix.from_csr(G["row_ptr"], G["col"], G["val"])
    for bs in (1, 2, 4, 8):
        r = O.bicgstab(A, b, tol=1e-12, block=bs)
        x, info = M.bicgstab(G["b"], tol=1e-12, block=bs)
        x = x.cpu().numpy()
        print(N, bs, M.stats()["format"], "it gpu/orc", info["iterations"], r.iterations, info["status_name"], "%.1e" % info["relres_true"],
              "relL2 %.1e" % (np.linalg.norm(x - r.x) / np.linalg.norm(r.x)), "restarts", info["replacements"], "%.4fs" % info["t_solve_s"])
