"""The library's DISTRIBUTED path (csr_create_dist, halo plan, pack kernel, ghost
advance of p, distributed finishers, pcg_solve / pcg_spmv on local rows) run for
real on the GPU by 2-3 processes that share cuda:0.  This run has one GPU, and
NCCL refuses two ranks on one device, so the exchange steps go through the
library's host-callback communicator (pcg_comm_init_ops) over torch.distributed
gloo; every kernel and every line of host planning is the NCCL path's own.  The
per-rank results are gathered and compared with the oracle on the undivided
system (parity bars of DESIGN.md §5), and the plan with the oracle's halo lists.
"""
import os
import socket

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, c, use_generator, out_q, drop=False):
    import torch
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2201_05413_b200 as pcg
        P = O.build_problem(name, c=c, k=1)
        A, b = P["A"], P["B"][:, 0]
        bounds = pcg.partition_rows(A.row_ptr, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        comm = pcg.Comm.host_callbacks()
        if use_generator:  # bench.py's path: rows generated on the device
            spec = pcg.fem_spec(name, c=c)
            G = pcg.fem_build(spec, r0, r1)
            rp, col, val, bl = G["row_ptr"], G["col"], G["val"], G["B"][:, 0].contiguous()
        else:
            rp = torch.as_tensor(A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]).cuda()
            col = torch.as_tensor(A.col[A.row_ptr[r0]:A.row_ptr[r1]]).cuda()
            val = torch.as_tensor(A.val[A.row_ptr[r0]:A.row_ptr[r1]]).cuda()
            bl = torch.as_tensor(b[r0:r1]).cuda()
        M = pcg.Matrix.from_csr_dist(comm, A.n, r0, r1, rp, col, val, drop_zeros=drop)
        st = M.stats()
        x, info = M.solve(bl, tol=1e-10)
        # the every-iteration x update (PCG_XDEFER=0) on a second handle: bitwise the same
        os.environ["PCG_XDEFER"] = "0"
        M0 = pcg.Matrix.from_csr_dist(comm, A.n, r0, r1, rp, col, val, drop_zeros=drop)
        x0e, info0e = M0.solve(bl, tol=1e-10)
        del os.environ["PCG_XDEFER"]
        M0.close()
        xp, infop = M.solve_pipelined(bl, tol=1e-10)  # N3: one allreduce per iteration
        xr = np.random.default_rng(100 + rank).standard_normal(r1 - r0)
        y = M.spmv(torch.as_tensor(xr).cuda()).cpu().numpy()
        out_q.put((rank, dict(r0=r0, r1=r1, n_ghost=st["n_ghost"], overlap_rows=st["overlap_rows"], x=x.cpu().numpy(), info=info, xr=xr, y=y,
                              x_every=x0e.cpu().numpy(), it_every=info0e["iterations"],
                              b=bl.cpu().numpy(), xp=xp.cpu().numpy(), infop=infop)))
        M.close()
        comm.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        out_q.put((rank, {"error": f"{e!r}\n{traceback.format_exc()}"}))


def _run(world, name, c, use_generator=False, drop=False):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, c, use_generator, q, drop)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, d = q.get(timeout=600)
        res[r] = d
    for p in procs:
        p.join(timeout=120)
    for r, d in res.items():
        assert "error" not in d, d.get("error")
    return [res[r] for r in range(world)]


@pytest.mark.parametrize("world,name,c,gen,drop", [(2, "C2", 48, False, False), (3, "C3", 24, False, False),
                                                   (2, "C5", 32, True, False), (3, "C1", None, False, False),
                                                   (2, "C3", 24, False, True)])  # C3': explicit zeros dropped
def test_distributed_path_on_one_gpu(world, name, c, gen, drop):
    parts = _run(world, name, c, gen, drop)
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()[name]["tol"]
    # plan: contiguous row blocks of the partition rule, ghost counts == oracle halo lists
    bounds = O.partition(A, world)
    for g, d in enumerate(parts):
        assert (d["r0"], d["r1"]) == (bounds[g], bounds[g + 1])
        assert d["n_ghost"] == len(O.halo(A, d["r0"], d["r1"]))
    # the banded configs run the overlapped schedule (interior SpMV while the halo is in flight)
    assert all(d["overlap_rows"] > 0 for d in parts)
    bg = np.concatenate([d["b"] for d in parts])
    scale = np.max(np.abs(b))
    assert np.all(np.abs(bg - b) <= 1e-12 * scale)  # generator RHS (exact copy otherwise)
    # distributed SpMV == oracle SpMV rows, within the forward-error bound of any summation order
    xr = np.concatenate([d["xr"] for d in parts])
    y = np.concatenate([d["y"] for d in parts])
    yo = O.spmv(A, xr)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    mag = np.bincount(rows, weights=np.abs(A.val) * np.abs(xr)[A.col], minlength=A.n)
    assert np.all(np.abs(y - yo) <= 2 * np.diff(A.row_ptr) * U * mag * (1 + 1e-9) + (1e-13 * mag if gen else 0))
    # distributed PCG == oracle PCG (same recurrence, reduction order differs)
    r = O.pcg(A, bg, tol=tol)
    x = np.concatenate([d["x"] for d in parts])
    its = {d["info"]["iterations"] for d in parts}
    assert len(its) == 1  # every rank ran the same number of iterations
    it = its.pop()
    assert all(d["info"]["status"] == 0 and d["info"]["relres_true"] <= tol for d in parts)
    assert np.linalg.norm(x - r.x) / np.linalg.norm(r.x) <= 1e-9
    assert abs(it - r.iterations) <= max(1, 0.02 * r.iterations), (it, r.iterations)
    # x updated every second iteration (default) == every iteration, bitwise, on every rank
    assert all(d["it_every"] == it and np.array_equal(d["x"], d["x_every"]) for d in parts)


@pytest.mark.parametrize("world,name,c", [(2, "C1", None), (3, "C4", 24), (2, "C2", 48)])
def test_distributed_pipelined_on_one_gpu(world, name, c):
    """pcg_solve_pipelined on distributed handles (reading R4; one allreduce per
    iteration): every rank runs the same number of steps; the gathered solution
    matches the oracle's pipelined and standard PCG solutions; the count stays within
    max(2, 3 %) of the oracle's pipelined count (no restarts on these systems)."""
    parts = _run(world, name, c)
    P = O.build_problem(name, c=c, k=1)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()[name]["tol"]
    ro = O.pcg_pipelined(A, b, tol=tol)
    rc = O.pcg(A, b, tol=tol)
    x = np.concatenate([d["xp"] for d in parts])
    its = {d["infop"]["iterations"] for d in parts}
    assert len(its) == 1
    it = its.pop()
    assert all(d["infop"]["status"] == 0 and d["infop"]["relres_true"] <= tol for d in parts)
    assert np.linalg.norm(x - ro.x) <= 1e-8 * np.linalg.norm(ro.x)
    assert np.linalg.norm(x - rc.x) <= 1e-8 * np.linalg.norm(rc.x)
    assert abs(it - ro.iterations) <= max(2, 0.03 * ro.iterations), (it, ro.iterations)


def test_bench_multi_rank_flow_on_one_gpu():
    """bench.py's N>1 path (torchrun, row partition by the device generator, barriers, max
    over ranks, one JSON line from rank 0) with 2 ranks sharing cuda:0 (host-callback
    communicator).  The iteration count must match the oracle's C5 ladder at c = 64."""
    import json
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2", "--comm",
           "callbacks", "--config", "C5", "--c", "64", "--steps", "2", "--warmup", "1"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["steps"] == 2 and line["unit"] == "s" and line["value"] > 0
    r = O.pcg(*(lambda P: (P["A"], P["B"][:, 0]))(O.build_problem("C5", c=64)), tol=1e-10)
    it = line["config"]["iterations"]
    assert abs(it - r.iterations) <= max(1, 0.02 * r.iterations), (it, r.iterations)
    assert line["config"]["relres_true"] <= 1e-10


def test_bench_multi_rank_rcm_partition_on_one_gpu():
    """bench.py --relabel/--reorder rcm with 2 ranks (N4): the randomly numbered C6 is put in
    RCM order by csr_rcm_order on the global pattern before the partition; the halo per rank
    is then an interface (compare: the oracle's halo of the RCM-ordered matrix), and the
    solve meets the oracle's iteration count."""
    import json
    import subprocess
    import sys
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2201_05413_b200 import inputs as I
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(root, "bench.py"), "--gpus", "2", "--comm",
           "callbacks", "--config", "C6", "--c", "12", "--steps", "2", "--warmup", "1", "--relabel", "7",
           "--reorder", "rcm", "--no-cpu-baseline"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    P = O.build_problem("C6", c=12, k=1)
    A = P["A"]
    q = I.relabel_order(A.n, 7)
    Ar = O.Csr(A.n, *I.relabel_csr_numpy(A.row_ptr, A.col, A.val, q))
    Ao = O.Csr(A.n, *I.relabel_csr_numpy(Ar.row_ptr, Ar.col, Ar.val, O.rcm(Ar)))
    b = O.partition(Ao, 2)
    assert line["config"]["n_ghost"] == len(O.halo(Ao, int(b[0]), int(b[1])))  # rank 0's halo
    r = O.pcg(A, P["B"][:, 0], tol=1e-10)
    it = line["config"]["iterations"]
    assert abs(it - r.iterations) <= max(1, 0.02 * r.iterations), (it, r.iterations)


@pytest.mark.parametrize("force_overlap", [False, True])
def test_nccl_single_rank_distributed_handle(force_overlap, monkeypatch):
    """The NCCL backend end to end on one GPU: unique id broadcast through a
    torch.distributed group, ncclCommInitRank, csr_create_dist, and the distributed
    solve loop whose graph captures ncclAllReduce (a 1-rank communicator still issues
    every collective).  Against the oracle.  force_overlap: the split K1 schedule
    (side-stream fork/join captured in the NCCL loop graph, three row ranges)."""
    if force_overlap:
        monkeypatch.setenv("PCG_FORCE_OVERLAP", "1")
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_05413_b200 as pcg
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        P = O.build_problem("C2", c=48, k=1)
        A, b = P["A"], P["B"][:, 0]
        comm = pcg.Comm.from_process_group()
        M = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, torch.as_tensor(A.row_ptr).cuda(),
                                     torch.as_tensor(A.col).cuda(), torch.as_tensor(A.val).cuda())
        assert (M.stats()["overlap_rows"] > 0) == force_overlap
        x, info = M.solve(torch.as_tensor(b).cuda(), tol=1e-10)
        r = O.pcg(A, b, tol=1e-10)
        assert info["status"] == 0 and info["relres_true"] <= 1e-10
        assert np.linalg.norm(x.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-9
        assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
        # the loop graph with x updated every iteration: bitwise the same x
        monkeypatch.setenv("PCG_XDEFER", "0")
        M0 = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, torch.as_tensor(A.row_ptr).cuda(),
                                      torch.as_tensor(A.col).cuda(), torch.as_tensor(A.val).cuda())
        x0, i0 = M0.solve(torch.as_tensor(b).cuda(), tol=1e-10)
        monkeypatch.delenv("PCG_XDEFER")
        assert i0["iterations"] == info["iterations"] and bool((x0 == x).all())
        M0.close()
        # max_iter stops after hold and apply passes: bitwise too
        for mi in (5, 6):
            xa, _ = M.solve(torch.as_tensor(b).cuda(), tol=1e-10, max_iter=mi)
            monkeypatch.setenv("PCG_XDEFER", "0")
            M1 = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, torch.as_tensor(A.row_ptr).cuda(),
                                          torch.as_tensor(A.col).cuda(), torch.as_tensor(A.val).cuda())
            xb, _ = M1.solve(torch.as_tensor(b).cuda(), tol=1e-10, max_iter=mi)
            monkeypatch.delenv("PCG_XDEFER")
            M1.close()
            assert bool((xa == xb).all()), mi
        # the pipelined solver's distributed schedule through NCCL (one allreduce per step)
        xp, ip = M.solve_pipelined(torch.as_tensor(b).cuda(), tol=1e-10)
        rp = O.pcg_pipelined(A, b, tol=1e-10)
        assert ip["status"] == 0 and ip["relres_true"] <= 1e-10
        assert np.linalg.norm(xp.cpu().numpy() - rp.x) / np.linalg.norm(rp.x) <= 1e-8
        assert abs(ip["iterations"] - rp.iterations) <= max(2, 0.03 * rp.iterations)
        M.close()
        comm.close()
    finally:
        dist.destroy_process_group()


def _bicg_worker(rank, world, port, N, out_q):
    import torch
    import torch.distributed as dist
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        import paper_2201_05413_b200 as pcg
        from paper_2201_05413_b200.problems import fd_cube_build
        A, b = O.fd_cube(N)
        bounds = pcg.partition_rows(A.row_ptr, world)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        G = fd_cube_build(N, row_begin=r0, row_end=r1)  # this rank's rows, generated on the device
        comm = pcg.Comm.host_callbacks()
        M = pcg.Matrix.from_csr_dist(comm, A.n, r0, r1, G["row_ptr"], G["col"], G["val"])
        x, info = M.bicgstab(G["b"], tol=1e-12)
        out_q.put((rank, dict(x=x.cpu().numpy(), info=info)))
        M.close()
        comm.close()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        out_q.put((rank, {"error": f"{e!r}\n{traceback.format_exc()}"}))


@pytest.mark.parametrize("world,N", [(2, 20), (3, 32)])
def test_distributed_bicgstab_on_one_gpu(world, N):
    """pcg_bicgstab on distributed handles (N2 on the paper's own setting: the Table 1
    FD grid row-partitioned; point Jacobi; four allreduces and two halo exchanges per
    iteration) with 2-3 ranks sharing the GPU through the host-callback communicator.
    Same bars as the single-GPU BiCGSTAB test: x within 1e-9 of the oracle and of the
    closed form x^2 - y^2, iterations within max(2 %, 2) of the range the oracle spans
    under rounding-level perturbations of b."""
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bicg_worker, args=(r, world, port, N, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r, d = q.get(timeout=600)
        res[r] = d
    for p in procs:
        p.join(timeout=120)
    for d in res.values():
        assert "error" not in d, d.get("error")
    parts = [res[r] for r in range(world)]
    A, b = O.fd_cube(N)
    ro = O.bicgstab(A, b, tol=1e-12)
    rng = np.random.default_rng(2201)
    its = [ro.iterations] + [O.bicgstab(A, b * (1 + 1e-15 * rng.standard_normal(A.n)), tol=1e-12).iterations
                             for _ in range(8)]
    lo, hi = min(its), max(its)
    x = np.concatenate([d["x"] for d in parts])
    gits = {d["info"]["iterations"] for d in parts}
    assert len(gits) == 1
    it = gits.pop()
    assert all(d["info"]["status"] == 0 and d["info"]["relres_true"] <= 1e-12 for d in parts)
    assert np.linalg.norm(x - ro.x) <= 1e-9 * np.linalg.norm(ro.x)
    assert lo - max(2, 0.02 * lo) <= it <= hi + max(2, 0.02 * hi), (it, lo, hi)
    i = np.arange(N)
    X, Y = np.tile(i, N * N) / (N - 1), np.tile(np.repeat(i, N), N) / (N - 1)
    assert np.max(np.abs(x - (X * X - Y * Y))) <= 1e-9


def test_nccl_failure_detection_aborts_instead_of_blocking():
    """SURVEY §5 failure detection: every host wait of a distributed call polls the
    queued work and ncclCommGetAsyncError under the communicator's timeout.  With a
    timeout no real wait can meet, the solve must return PCG_ERR_NCCL (communicator
    aborted) instead of blocking, later calls must keep failing with PCG_ERR_NCCL, and
    the handles must still be destroyable.  A fresh communicator then solves normally."""
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_05413_b200 as pcg
    from paper_2201_05413_b200._lib import STATUS
    nccl_err = STATUS.index("PCG_ERR_NCCL")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        P = O.build_problem("C2", c=96, k=1)
        A, b = P["A"], P["B"][:, 0]
        dev = [torch.as_tensor(a).cuda() for a in (A.row_ptr, A.col, A.val)]
        comm = pcg.Comm.from_process_group()
        M = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, *dev)
        comm.set_timeout(1e-9)
        for _ in range(2):
            with pytest.raises(pcg.PcgError) as e:
                M.solve(torch.as_tensor(b).cuda(), tol=1e-10)
            assert e.value.status == nccl_err, e.value
        M.close()
        comm.close()
        comm = pcg.Comm.from_process_group()
        M = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, *dev)
        x, info = M.solve(torch.as_tensor(b).cuda(), tol=1e-10)
        r = O.pcg(A, b, tol=1e-10)
        assert info["status"] == 0
        assert np.linalg.norm(x.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-9
        M.close()
        comm.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("G,nv", [(1, 1), (2, 3), (3, 2), (8, 3)])
def test_device_allreduce_protocol_emulated(G, nv):
    """The device-initiated allreduce's protocol (csrc/dar.cu) with G
    ranks played by G co-resident blocks of one cooperative kernel, each with its own
    mailbox, over 64 successive rounds: every rank's result equals the rank-order sum
    of all ranks' inputs, bitwise, and all ranks agree (the parity-alternating mailbox
    slots and monotonic flags survive back-to-back rounds)."""
    import ctypes as C
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2201_05413_b200 import _lib
    rounds = 64
    rng = np.random.default_rng(G * 10 + nv)
    x = rng.standard_normal((rounds, G, nv)) * 10.0 ** rng.integers(-8, 8, (rounds, G, nv))
    out = np.zeros_like(x)
    st = _lib.lib().pcg_dar_emulate(G, rounds, nv, x.ctypes.data_as(C.c_void_p), out.ctypes.data_as(C.c_void_p))
    assert st == 0
    for r in range(rounds):
        for v in range(nv):
            s = 0.0
            for g in range(G):
                s += x[r, g, v]
            for g in range(G):
                assert out[r, g, v] == s, (r, g, v)


def test_device_allreduce_single_rank_nccl_solves(monkeypatch):
    """PCG_DEVICE_ALLREDUCE=1 on a 1-rank NCCL communicator: the mailbox is set up, the
    distributed PCG, pipelined PCG and BiCGSTAB loops run their scalar reductions
    through the device kernel (captured in the iteration graphs) and match the oracle."""
    import torch
    import torch.distributed as dist
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2201_05413_b200 as pcg
    monkeypatch.setenv("PCG_DEVICE_ALLREDUCE", "1")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        P = O.build_problem("C2", c=48, k=1)
        A, b = P["A"], P["B"][:, 0]
        comm = pcg.Comm.from_process_group()
        assert comm.info()["device_allreduce"]
        M = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, torch.as_tensor(A.row_ptr).cuda(),
                                     torch.as_tensor(A.col).cuda(), torch.as_tensor(A.val).cuda())
        x, info = M.solve(torch.as_tensor(b).cuda(), tol=1e-10)
        r = O.pcg(A, b, tol=1e-10)
        assert info["status"] == 0 and info["relres_true"] <= 1e-10
        assert np.linalg.norm(x.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-9
        assert abs(info["iterations"] - r.iterations) <= max(1, 0.02 * r.iterations)
        # the loop graph with x updated every iteration: bitwise the same x
        monkeypatch.setenv("PCG_XDEFER", "0")
        M0 = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, torch.as_tensor(A.row_ptr).cuda(),
                                      torch.as_tensor(A.col).cuda(), torch.as_tensor(A.val).cuda())
        x0, i0 = M0.solve(torch.as_tensor(b).cuda(), tol=1e-10)
        monkeypatch.delenv("PCG_XDEFER")
        assert i0["iterations"] == info["iterations"] and bool((x0 == x).all())
        M0.close()
        # max_iter stops after hold and apply passes: bitwise too
        for mi in (5, 6):
            xa, _ = M.solve(torch.as_tensor(b).cuda(), tol=1e-10, max_iter=mi)
            monkeypatch.setenv("PCG_XDEFER", "0")
            M1 = pcg.Matrix.from_csr_dist(comm, A.n, 0, A.n, torch.as_tensor(A.row_ptr).cuda(),
                                          torch.as_tensor(A.col).cuda(), torch.as_tensor(A.val).cuda())
            xb, _ = M1.solve(torch.as_tensor(b).cuda(), tol=1e-10, max_iter=mi)
            monkeypatch.delenv("PCG_XDEFER")
            M1.close()
            assert bool((xa == xb).all()), mi
        xp, ip = M.solve_pipelined(torch.as_tensor(b).cuda(), tol=1e-10)
        assert ip["status"] == 0 and np.linalg.norm(xp.cpu().numpy() - r.x) / np.linalg.norm(r.x) <= 1e-8
        M.close()
        Af, bf = O.fd_cube(16)
        Mf = pcg.Matrix.from_csr_dist(comm, Af.n, 0, Af.n, torch.as_tensor(Af.row_ptr).cuda(),
                                      torch.as_tensor(Af.col).cuda(), torch.as_tensor(Af.val).cuda())
        xb, ib = Mf.bicgstab(torch.as_tensor(bf).cuda(), tol=1e-12)
        rb = O.bicgstab(Af, bf, tol=1e-12)
        assert ib["status"] == 0 and np.linalg.norm(xb.cpu().numpy() - rb.x) <= 1e-9 * np.linalg.norm(rb.x)
        Mf.close()
        comm.close()
    finally:
        dist.destroy_process_group()
