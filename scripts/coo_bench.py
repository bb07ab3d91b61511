"""coo_to_csr throughput (development tool): entries/s and time for FEM-like triplet
counts (element-by-element assembly of a P1 tet mesh emits 16 triplets per element).

  python scripts/coo_bench.py [n_entries ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import torch  # noqa: E402

import paper_2201_05413_b200 as pcg  # noqa: E402
from coo_inputs import triplets  # noqa: E402

for nnz in [int(a) for a in sys.argv[1:]] or [8_000_000, 64_000_000]:
    n = nnz // 16
    r, c, v = triplets(2201, n, n, nnz, nnz // 7)
    r, c, v = torch.as_tensor(r).cuda(), torch.as_tensor(c).cuda(), torch.as_tensor(v).cuda()
    for _ in range(2):
        pcg.coo_to_csr(r, c, v, n, n)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 5
    for _ in range(reps):
        out = pcg.coo_to_csr(r, c, v, n, n)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"coo_to_csr nnz_in={nnz} n={n} unique={out['col'].numel()} {ms:.2f} ms "
          f"{nnz / ms / 1e6:.2f} G entries/s")
