"""Multi-GPU path, host logic, on CPU with world_size-2 gloo (no GPU).

Each rank runs the library's host planning functions exactly as csr_create_dist
does (partition rule, ghost list, per-rank receive plan), exchanges the plan with
gloo the way dist.cu does with NCCL (allgather of counts, send/recv of index
lists), and then emulates the distributed iteration schedule of the kernels (K1:
gathered p recomputed from z and p_old incl. locally advanced ghost copies; K2;
z halo exchange; two scalar allreduces) in numpy.  Checks: plan == oracle halo
lists (bit-exact), send lists == what the peer references, and the emulated
distributed solve == the oracle within the parity bars.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, c, out_q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2201_05413_b200 as pcg
        P = O.build_problem(name, c=c, k=1)
        A, b = P["A"], P["B"][:, 0]
        bounds = pcg.partition_rows(A.row_ptr, world)
        assert np.array_equal(bounds, O.partition(A, world))
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        n = r1 - r0
        rp = A.row_ptr[r0:r1 + 1] - A.row_ptr[r0]
        colg = A.col[A.row_ptr[r0]:A.row_ptr[r1]]
        val = A.val[A.row_ptr[r0]:A.row_ptr[r1]]
        ghosts = pcg.halo_ghosts(r0, r1, colg)
        assert np.array_equal(ghosts, O.halo(A, r0, r1))
        need, off = pcg.halo_recv_plan(ghosts, bounds)
        # counts matrix via allgather (dist.cu: ncclAllGather)
        M = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(M, torch.as_tensor(need))
        M = torch.stack(M).numpy()
        send = {}
        reqs = []
        for h in range(world):
            if h == rank:
                continue
            if need[h]:
                reqs.append(dist.isend(torch.as_tensor(ghosts[off[h]:off[h] + need[h]]), h))
            if M[h, rank]:
                buf = torch.zeros(int(M[h, rank]), dtype=torch.int64)
                dist.recv(buf, h)
                send[h] = buf.numpy() - r0  # local rows to pack for h
        for r in reqs:
            r.wait()
        # the send list for h is exactly my rows that h's rows reference
        for h, rows in send.items():
            hr0, hr1 = bounds[h], bounds[h + 1]
            ref = np.unique(A.col[A.row_ptr[hr0]:A.row_ptr[hr1]])
            ref = ref[(ref >= r0) & (ref < r1)] - r0
            assert np.array_equal(np.sort(rows), ref)
        # local column ids: owned -> j - r0, ghosts -> n + index
        loc = np.where((colg >= r0) & (colg < r1), colg - r0, n + np.searchsorted(ghosts, colg))
        dinv = np.array([1.0 / val[rp[i] + np.nonzero(colg[rp[i]:rp[i + 1]] == r0 + i)[0][0]] for i in range(n)])
        ng = len(ghosts)

        def halo(vec):  # pack + grouped send/recv (dist.cu halo_exchange)
            rq = []
            for h, rows in send.items():
                rq.append(dist.isend(torch.as_tensor(vec[rows].copy()), h))
            for h in range(world):
                if h != rank and need[h]:
                    buf = torch.zeros(int(need[h]), dtype=torch.float64)
                    dist.recv(buf, h)
                    vec[n + off[h]:n + off[h] + need[h]] = buf.numpy()
            for r in rq:
                r.wait()

        def allreduce(*vals):
            t = torch.tensor(vals, dtype=torch.float64)
            dist.all_reduce(t)
            return t.numpy()

        rows_of = np.repeat(np.arange(n), np.diff(rp))
        bl = b[r0:r1]
        tol = 1e-10
        x = np.zeros(n + ng)
        # init (resid_kernel + finisher): r = b - A x, z = dinv r, p = 0
        halo(x)
        w = bl - np.bincount(rows_of, weights=val * x[loc], minlength=n)
        z = np.zeros(n + ng)
        z[:n] = dinv * w
        r = w.copy()
        ww, wz, bb = allreduce(w @ w, w @ z[:n], bl @ bl)
        nb = np.sqrt(bb)
        rho, beta, alpha = wz, 0.0, 0.0
        p = [np.zeros(n + ng), np.zeros(n + ng)]
        par, k = 0, 0
        halo(z)
        while True:
            pold, pnew = p[par], p[par ^ 1]
            # K1: gathered p recomputed from (z, p_old), own p written, ghost p advanced
            g = beta * pold + z
            q = np.bincount(rows_of, weights=val * g[loc], minlength=n)
            pnew[:] = g
            x[:n] += alpha * pold[:n]
            (sigma,) = allreduce(pnew[:n] @ q)
            assert sigma > 0
            alpha = rho / sigma
            k += 1
            par ^= 1
            # K2
            r = r - alpha * q
            z[:n] = dinv * r
            rho_new, gamma = allreduce(r @ z[:n], r @ r)
            if np.sqrt(gamma) <= tol * nb:
                break
            beta = rho_new / rho
            rho = rho_new
            halo(z)
        x[:n] += alpha * p[par][:n]
        if rank == 0:
            parts = [x[:n].copy()]
            for h in range(1, world):
                buf = torch.zeros(int(bounds[h + 1] - bounds[h]), dtype=torch.float64)
                dist.recv(buf, h)
                parts.append(buf.numpy())
            out_q.put((rank, k, np.concatenate(parts), None))
        else:
            dist.send(torch.as_tensor(x[:n].copy()), 0)
            out_q.put((rank, k, None, None))
    except Exception as e:  # surface failures to the parent
        import traceback
        out_q.put((rank, None, None, traceback.format_exc()))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("name,c", [("C2", 24), ("C5", 10), ("C3", 10)])
def test_two_rank_plan_and_distributed_schedule(name, c):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, c, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, k, x, err in res:
        assert err is None, err
    x = [r for r in res if r[0] == 0][0][2]
    its = {r[1] for r in res}
    assert len(its) == 1
    P = O.build_problem(name, c=c, k=1)
    ro = O.pcg(P["A"], P["B"][:, 0], tol=1e-10)
    assert abs(its.pop() - ro.iterations) <= max(1, 0.02 * ro.iterations)
    assert np.linalg.norm(x - ro.x) / np.linalg.norm(ro.x) <= 1e-9
