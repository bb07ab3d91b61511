#!/usr/bin/env python
"""Benchmark: Jacobi-PCG time-to-solution at rel-res 1e-10 on the C5 workload
(3D P1 Kuhn cube, 512^3 cells, 133,432,831 unknowns, 932,463,091 nnz), on N GPUs.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU, NCCL)

One "step" = one full pcg_solve (init, all iterations, exit check) from x0 = 0 on
the device-resident system.  `value` is the device-timed time-to-solution (CUDA
events, max over ranks).  `e2e` repeats it through the same public API with
pinned HOST b and x (H2D of b, x0 and D2H of x inside the timed region).
The roofline object reports the dominant kernel (K1b: SpMV + sigma) against the
measured HBM copy bandwidth in MEASURED_PEAKS.json.

--config C4 (k = 16 right-hand sides) times pcg_solve_multi instead (a step = one
multi-RHS solve of all 16 columns; roofline = the SpMM pass).  The driver's
default line is C5.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# K1a bytes per row, averaged over the deferred x update's cycle (solver.cu k1a_hold / k1a_apply):
# every iteration 40; cycle 2: (24 + 48) / 2; cycle 4: (3 x 24 + 64) / 4
K1A_BYTES = {0: 40.0, 2: 36.0, 4: 34.0}


def xdefer_cycle():
    """the deferral cycle as the library reads PCG_XDEFER (solver.cu xdefer_m: atoi; 0 off,
    2 or 4, anything else the default 4)"""
    v = os.environ.get("PCG_XDEFER")
    if v is None:
        return 4
    import re
    mt = re.match(r"\s*([+-]?\d+)", v)
    m = int(mt.group(1)) if mt else 0  # atoi: no leading number -> 0
    return m if m in (0, 2, 4) else 4


def read_only_peak():
    """The read-only HBM stream rate measured on this GPU pool (scripts/probes/read_bw.cu,
    profiles/r02/read_bw.log): context for kernels whose traffic is mostly reads, whose
    DRAM rate can exceed the read+write copy figure of MEASURED_PEAKS.json."""
    p = os.path.join(ROOT, "profiles", "r02", "read_bw.log")
    if not os.path.exists(p):
        return None
    best = 0.0
    with open(p) as fh:
        for line in fh:
            if "read-only" in line:
                best = max(best, float(line.split("read-only")[1].split("GB/s")[0]))
    return {"GBps": best, "source": "profiles/r02/read_bw.log (scripts/probes/read_bw.cu: 8 GiB read-only stream, "
                                    "best over grid sizes; the same probe's copy: 6.3 TB/s)"} if best else None


HBM_FALLBACK_GBS = 6650.0  # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
BAD_REASONS = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK_GBS, "fallback"


class ClockSampler:
    """NVML sampling of SM clock + throttle reasons during the timed region."""

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
                for b, name in REASON_BITS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}

    def bad(self):
        if BAD_REASONS & self.reasons:
            return True
        if self.samples and self.max_mhz and statistics.median(self.samples) < 0.5 * self.max_mhz \
                and "sw_power_cap" not in self.reasons:
            return True
        return False


# ------------------------------------------------------------------------------ CPU oracle legs
# The oracle (oracle/oracle.c, plain C, one thread, "as it stands") is timed on this
# host's cores; nothing here loads the product library (libpcg_b200.so).
GOLD = os.path.join(ROOT, "tests", "golden", "oracle_full.json")


def host_cpu():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu": model, "host_cores": len(os.sched_getaffinity(0)), "logical_cpus": os.cpu_count()}


def closed_form_size(name, c):
    """n, nnz of the configs from SURVEY §8(c).7's closed forms (no library, no oracle);
    None for C6 (jittered element graph: no closed form)."""
    m = c - 1
    if name == "C1":
        return m * m, 5 * m * m - 4 * m
    if name == "C2":
        return m * m, 7 * m * m - 8 * m + 2
    if name == "C3":
        return (2 * c - 1) ** 2, 46 * c * c - 96 * c + 53
    if name in ("C4", "C5"):
        return m ** 3, 7 * m ** 3 - 6 * m * m
    return None


def oracle_golden(key):
    if os.path.exists(GOLD):
        with open(GOLD) as fh:
            return json.load(fh).get(key)
    return None


def oracle_sample(cfg_name: str, c_sample: int, reps: int = 1, all_cores: bool = True):
    """Time the oracle on the same construction at c_sample: the plain 1-thread build
    (as it stands) and, once, the all-cores timing build (oracle/__init__.py build_omp)."""
    import oracle as O
    P = O.build_problem(cfg_name, c=c_sample)
    A, b = P["A"], P["B"][:, 0]
    tol = O.configs()[cfg_name]["tol"]
    times, its = [], None
    for _ in range(reps):
        t0 = time.perf_counter()
        r = O.pcg(A, b, tol=tol)
        times.append(time.perf_counter() - t0)
        its = r.iterations
    out = {"n": A.n, "nnz": A.nnz, "iterations": its, "t_solve": times, "c": c_sample}
    if all_cores:
        t0 = time.perf_counter()
        it2, st2, threads = O.pcg_all_cores(A, b, tol=tol)
        out["all_cores"] = {"t_solve": time.perf_counter() - t0, "threads": threads, "iterations": it2}
    return out


def iter_bytes(n, nnz, k=1):
    return 12.0 * nnz + 4.0 * (n + 1) + 88.0 * k * n


def scale_to_workload(t_solve, sample, n, nnz, iters):
    """time-to-solution of the workload implied by the sample's measured per-iteration
    time (scaled by per-iteration bytes) and an iteration count for the workload."""
    per_iter = t_solve / sample["iterations"]
    return per_iter * iter_bytes(n, nnz) / iter_bytes(sample["n"], sample["nnz"]) * iters


def oracle_full_iterations(name, c):
    """The oracle's own iteration count on the workload, from its full-size golden run
    (tests/golden/oracle_full.json, written by oracle/make_golden.py), if present."""
    cfg_c = None
    try:
        import oracle as O
        cfg_c = O.configs()[name]["c"]
    except Exception:
        pass
    if c != cfg_c:
        return None, None
    g = oracle_golden("C5full" if name == "C5" else name)
    if not g:
        return None, None
    return max(r["iterations"] for r in g["rhs"]), g.get("oracle_timing")


def run_reference(args):
    """The reference arm of this tier: the oracle itself, timed on this host.  A step =
    one complete oracle time-to-solution (plain 1-thread build, as it stands) of the
    workload's construction at c = --ref-c (a bounded sample: the full C5 solve takes
    over an hour on one core); value = the measured median step.  The full-workload
    figure derived from it is reported separately and labelled as an estimate."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle as O
    cfg = O.configs()[args.config]
    c_full = args.c or cfg["c"]
    cs = args.ref_c
    P = O.build_problem(args.config, c=cs)
    A, b = P["A"], P["B"][:, 0]
    times, its = [], 0
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = O.pcg(A, b, tol=cfg["tol"])
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
        its = r.iterations
    value = statistics.median(times)
    sample = {"n": A.n, "nnz": A.nnz, "iterations": its, "c": cs}
    t0 = time.perf_counter()
    it2, _, threads = O.pcg_all_cores(A, b, tol=cfg["tol"])
    t_all = time.perf_counter() - t0
    size = closed_form_size(args.config, c_full)
    est = None
    if size:
        n, nnz = size
        iters_full, timing = oracle_full_iterations(args.config, c_full)
        if iters_full:
            est = {"value": scale_to_workload(value, sample, n, nnz, iters_full), "unit": "s",
                   "basis": (f"this run's per-iteration time x per-iteration bytes ({n} / {A.n} unknowns) x the "
                             f"oracle's own {iters_full} iterations on the full workload (tests/golden)"),
                   "oracle_measured_full_size": timing}
    hc = host_cpu()
    desc = (f"{args.config} construction at c={cs} ({A.n} unknowns, {A.nnz} nnz, {its} iterations): one complete "
            f"oracle Jacobi-PCG solve per step (oracle/oracle.c as it stands, 1 thread); measured, not scaled")
    wl = workload_config(args.config, c_full, *(size or (None, None)), args.gpus)
    wl["timed_sample"] = f"{args.config} construction at c={cs} (the reference arm's bounded sample)"
    line = {"impl": "reference", "metric": "pcg_time_to_solution", "value": value, "unit": "s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": wl,
            "cpu_baseline": {"value": value, "unit": "s", "cores": 1, "kind": "oracle", "sample": desc, **hc,
                             "all_cores": {"value": t_all, "unit": "s", "cores": threads, "iterations": it2,
                                           "build": "oracle.c -fopenmp -DORC_OMP (timing only)"}},
            "full_workload_estimate": est,
            "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(name, c, n, nnz, gpus):
    desc = {"C5": f"C5: 3D Laplace, P1 Kuhn tets on a {c}^3-cell unit cube, f=3pi^2 sin sin sin, u=0 on the "
                  f"boundary, Jacobi-PCG x0=0 to rel-res 1e-10",
            "C4": f"C4: 3D P1 Kuhn {c}^3 cells, 16 Gaussian-bump RHS", "C3": f"C3: 2D P2 {c}^2 cells, f=1",
            "C2": f"C2: 2D jittered P1 {c}^2 cells, harmonic x^2-y^2 boundary data",
            "C1": f"C1: 2D P1 {c}^2 cells, sin RHS",
            "C6": f"C6: 3D P1 Kuhn tets on a {c}^3-cell cube, interior nodes jittered by +-0.15h (irregular "
                  f"stand-in for the paper's Sphere meshes), f = 0, linear Dirichlet data"}[name]
    if n is None:
        return {"workload": desc, "config": name, "global_batch": 1, "tol": 1e-10}
    return {"workload": desc, "config": name, "n": n, "nnz": nnz, "global_batch": 1, "tol": 1e-10,
            "parallelism": f"row-partition over {gpus} GPU(s): halo of z + 2 scalar allreduces per iteration"
            if gpus > 1 else "1 GPU",
            "l2": (f"no flush needed: every iteration streams at least {iter_bytes(n, nnz) / 1e9:.1f} GB "
                   f"(>> 126 MB L2)") if iter_bytes(n, nnz) / gpus > 1e9 else
            f"no flush: an iteration moves {iter_bytes(n, nnz) / gpus / 1e6:.0f} MB per GPU, partly L2-resident "
            f"(126 MB L2); timed as the solve runs"}


# ------------------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5")
    ap.add_argument("--c", type=int, default=None, help="override cells per axis (testing)")
    ap.add_argument("--sample-c", type=int, default=96, help="oracle sample size of the GPU arm's cpu_baseline")
    ap.add_argument("--ref-c", type=int, default=64, help="oracle sample size of the reference arm's steps")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fmt", default="auto", choices=["auto", "csr", "sell", "sigma"])
    ap.add_argument("--relabel", type=int, default=None, metavar="SEED",
                    help="N4: number the mesh nodes in a seeded random order (an unordered mesher's output)")
    ap.add_argument("--reorder", default="none", choices=["none", "rcm"],
                    help="N4: reverse Cuthill-McKee (PCG_REORDER_RCM on one GPU; csr_rcm_order before the partition)")
    ap.add_argument("--drop-zeros", action="store_true",
                    help="store no explicit zero entries (PCG_DROP_ZEROS; C3' of SURVEY Q7, same iterates)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "callbacks"],
                    help="callbacks: exchange steps through host callbacks over gloo (validation of the N>1 "
                         "path when ranks share a GPU; not a performance number)")
    ap.add_argument("--block", type=int, default=1, help="Block-Jacobi block size for the CUBE* BiCGSTAB configs "
                    "(--precond ilu0: rows per ILU(0) block, 0 = one block per SM)")
    ap.add_argument("--precond", default="bj", choices=["bj", "ilu0"],
                    help="CUBE* BiCGSTAB: Block-Jacobi with dense LU blocks (bj) or ILU(0) blocks (ilu0, the "
                         "paper's PETSc default sub-solver)")
    ap.add_argument("--solver", default="pcg", choices=["pcg", "pipelined", "block"],
                    help="Jacobi-PCG (the benchmark), the pipelined variant (single RHS) or block CG (k RHS), "
                         "both SURVEY N3")
    args = ap.parse_args()
    if args.config.startswith("CUBE"):
        return run_bicgstab(args)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    import paper_2201_05413_b200 as pcg
    from paper_2201_05413_b200.problems import configs, fem_build, fem_spec, problem_size

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cb = args.comm == "callbacks"
    if cb:  # ranks may share a GPU
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if cb:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs()[args.config]
    c = args.c or cfg["c"]
    spec = fem_spec(args.config, c=c)
    n, nnz, _ = problem_size(spec)
    tol, max_iter = cfg["tol"], cfg["max_iter"]

    # ---- build the system on the device (setup, untimed)
    t_setup0 = time.perf_counter()
    comm = None
    reorder = "rcm" if args.reorder == "rcm" else None
    if args.relabel is not None or (reorder and world > 1):
        # the global system, numbered in a seeded random order (inputs.py) and/or
        # put in RCM order: inside csr_create on one GPU (PCG_REORDER_RCM), by csr_rcm_order on
        # the global pattern before the contiguous row partition on N GPUs
        from paper_2201_05413_b200.inputs import relabel_csr_torch, relabel_order
        P = fem_build(spec)
        nnz = P["col"].numel()
        rp, col, val, B = P["row_ptr"], P["col"], P["val"], P["B"]
        del P
        if args.relabel is not None:
            q = relabel_order(n, args.relabel)
            rp, col, val = relabel_csr_torch(rp, col, val, q)
            B = B[torch.as_tensor(q, device=B.device)]
        if reorder and world > 1:
            o = pcg.csr_rcm_order(rp, col)
            rp, col, val = relabel_csr_torch(rp, col, val, o)
            B = B[o]
        if world == 1:
            r0, r1 = 0, n
            A = pcg.Matrix.from_csr(rp, col, val, fmt=args.fmt, drop_zeros=args.drop_zeros, reorder=reorder)
        else:
            bounds = pcg.partition_rows(rp.cpu().numpy(), world)
            r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
            e0, e1 = int(rp[r0]), int(rp[r1])
            comm = pcg.Comm.host_callbacks() if cb else pcg.Comm.from_process_group()
            A = pcg.Matrix.from_csr_dist(comm, n, r0, r1, (rp[r0:r1 + 1] - e0).contiguous(), col[e0:e1].contiguous(),
                                         val[e0:e1].contiguous(), fmt=args.fmt, drop_zeros=args.drop_zeros)
        P = {"B": B[r0:r1]}
        del rp, col, val, B
    elif world == 1:
        P = fem_build(spec)
        nnz = P["col"].numel()  # (the 3D element pattern has no closed form: problem_size gives -1)
        A = pcg.Matrix.from_csr(P["row_ptr"], P["col"], P["val"], fmt=args.fmt, drop_zeros=args.drop_zeros,
                                reorder=reorder)
        r0, r1 = 0, n
    else:
        rp_full = fem_build_rowptr(spec, n)
        rp_full_nnz = rp_full[-1]
        bounds = pcg.partition_rows(rp_full, world)
        del rp_full
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        P = fem_build(spec, r0, r1)
        if nnz < 0:
            nnz = int(rp_full_nnz)
        comm = pcg.Comm.host_callbacks() if cb else pcg.Comm.from_process_group()
        A = pcg.Matrix.from_csr_dist(comm, n, r0, r1, P["row_ptr"], P["col"], P["val"], fmt=args.fmt,
                                     drop_zeros=args.drop_zeros)
    nnz_given = nnz
    if args.drop_zeros:  # the bytes an iteration moves are those of the stored pattern
        t = torch.tensor([float(A.stats()["nnz"])], dtype=torch.float64, device="cpu" if cb else "cuda")
        if world > 1:
            dist.all_reduce(t)
        nnz = int(t.item())
    kcols = P["B"].shape[1]
    multi = kcols > 1
    if multi and world > 1:
        raise SystemExit("bench.py: multi-RHS configs run on one GPU (pcg_solve_multi takes single-GPU handles)")
    b = P["B"][:, 0].contiguous() if not multi else None
    Bm = P["B"].t().contiguous().t() if multi else None  # (n, k) view of a column-major block
    del P
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    t_setup = time.perf_counter() - t_setup0
    stats = A.stats()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if cb else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step(bb, out):
        if multi:
            solve_k = A.solve_block if args.solver == "block" else A.solve_multi
            X, infos = solve_k(bb, tol=tol, max_iter=max_iter, out=out)
            return X, infos
        solve = A.solve_pipelined if args.solver == "pipelined" else A.solve
        x, inf = solve(bb, tol=tol, max_iter=max_iter, out=out)
        return x, [inf]

    # ---- warm-up
    for _ in range(args.warmup):
        step(Bm if multi else b, None)

    # ---- timed region (device-resident inputs); re-measured once if clocks were bad
    def timed(device_inputs: bool):
        st = torch.cuda.current_stream()
        src = Bm if multi else b
        if device_inputs:
            bb = src
            xx = torch.empty_like(src.t().contiguous()).t() if multi else torch.empty_like(src)
        else:  # pinned host buffers, allocated outside the timed region
            bb = (src.t().cpu().pin_memory().t()) if multi else src.cpu().pin_memory()
            xx = (torch.empty(src.shape[::-1], dtype=torch.float64).pin_memory().t() if multi
                  else torch.empty(src.shape, dtype=torch.float64).pin_memory())
        barrier()
        l0 = pcg.kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as cs:
            e0.record(st)
            infos = []
            for _ in range(args.steps):
                xx.zero_()  # x0 = 0 every step (host memset for the e2e leg)
                x, inf = step(bb, xx)  # host buffers: H2D b, x0 + D2H x inside the library call
                infos.append(inf)
            e1.record(st)
            barrier()
        ms = e0.elapsed_time(e1) / args.steps
        return max_over_ranks(ms), infos, pcg.kernel_launches() - l0, cs, x

    ms, infos, launches, cs, x = timed(True)
    remeasured = False
    if cs.bad():
        ms, infos, launches, cs, x = timed(True)
        remeasured = True
    iters = max(i["iterations"] for i in infos[-1])  # block iterations (max over columns)
    rank_iters = None
    if world > 1:  # every rank must report the same count (the recurrence scalars are global)
        t = torch.tensor([float(iters)], dtype=torch.float64, device="cpu" if cb else "cuda")
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        rank_iters = [int(g.item()) for g in gathered]
    ms_e2e, infos_e2e, _, _, _ = timed(False)

    # ---- roofline of the dominant kernel (K1) + standalone SpMV bandwidth
    hbm, peak_kind = peaks()
    roof = None
    spmv_gbs = None
    k_us = None
    if world == 1 and multi:
        import ctypes as C
        us = (C.c_double * 3)()
        done = C.c_int32()
        Bc = Bm.t().contiguous()
        pcg.check(pcg.lib().pcg_profile_multi(A._h, kcols, C.c_void_p(Bc.data_ptr()), n, 20,
                                               C.c_void_p(torch.cuda.current_stream().cuda_stream), us,
                                               C.byref(done)), "pcg_profile_multi")
        mat = 12.0 * nnz + 4.0 * (n + 1)
        xdm = xdefer_cycle()  # X deferred over the cycle (multi.cu mk1a_deferred): mean over a hold/apply cycle
        names = ["mk1a_kernel (X += alpha P, P = Z + beta P; streaming, per column" +
                 (f"; X every {xdm}th iteration: mean over a hold/apply cycle)" if xdm else ")"),
                 "mspmm_kernel (SpMM Q = A P over SELL-32, per-column sigma, grid finish -> alpha)",
                 "mk2_kernel (R -= alpha Q, Z = dinv R, rho', gamma per column, finish -> beta)"]
        byts = [K1A_BYTES[xdm] * kcols * n, mat + 16.0 * kcols * n, 40.0 * kcols * n]
        kern = [{"kernel": nm, "bytes_per_launch": bt, "us_per_launch": u, "achieved_GBps": bt / u / 1e3 if u else None}
                for nm, bt, u in zip(names, byts, us)]
        dom = max(kern, key=lambda d: d["us_per_launch"])
        it_us = sum(us)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r02", "traffic_c4.json")
        if args.config == "C4" and c == 128 and kcols == 16 and os.path.exists(tp):
            with open(tp) as fh:  # the dominant kernel's DRAM bytes per launch (ncu, steady-state launch)
                traffic = json.load(fh)["kernels"].get(dom["kernel"].split(" ")[0], {}).get("traffic_bytes")
        roof = {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["achieved_GBps"], "peak": hbm,
                "unit": "GB/s", "frac": dom["achieved_GBps"] / hbm, "peak_source": peak_kind, "traffic": traffic,
                "traffic_source": "profiles/r02/traffic_c4.json (ncu --set full, dram read+write per launch)"
                if traffic else None,
                "bytes_per_launch": dom["bytes_per_launch"], "us_per_launch": dom["us_per_launch"],
                "kernels": kern, "schedule": 3,
                "iteration": {"bytes": sum(byts), "us": it_us, "frac": sum(byts) / it_us / 1e3 / hbm,
                              "frac_vs_88n_ideal": (mat + 88.0 * kcols * n) / it_us / 1e3 / hbm}}
        k_us = list(us)
    elif world == 1:
        import ctypes as C
        us = (C.c_double * 3)()
        done = C.c_int32()
        pcg.check(pcg.lib().pcg_profile_kernels(A._h, C.c_void_p(b.data_ptr()), 20,
                                                 C.c_void_p(torch.cuda.current_stream().cuda_stream), us,
                                                 C.byref(done)), "pcg_profile_kernels")
        mat = 12.0 * nnz + 4.0 * (n + 1)
        if stats["schedule"] == 3:
            # x deferred (solver.cu k1a_deferred; PCG_XDEFER=0 turns it off): K1a alternates
            # hold (24n B) and apply (48n B) launches, timed as pairs: 36n per launch on average
            xdm = xdefer_cycle()
            names = ["k1a_kernel (p = z + beta p, x += alpha p_old; streaming" +
                     (f"; x every {xdm}th iteration: mean over a hold/apply cycle)" if xdm else ")"),
                     "k1b_kernel (SpMV q = A p + sigma = p.q, grid finish -> alpha)",
                     "k2_kernel (r -= alpha q, z = dinv r, rho', gamma, grid finish -> beta; bytes by the 40 n formula: it reads dinv once per 32-row slice where the slice shares one, and where every slice does it stores no z (K1a forms it from r): 24.25 n on a lattice)"]
            byts = [K1A_BYTES[xdm] * n, mat + 16.0 * n, 40.0 * n]
        else:
            names = ["-", "k1_kernel (fused SpMV + p/x updates + sigma)", "k2_kernel (r/z updates + dots)"]
            byts = [0.0, mat + 48.0 * n, 40.0 * n]
        kern = [{"kernel": nm, "bytes_per_launch": bt, "us_per_launch": u, "achieved_GBps": bt / u / 1e3 if u else None}
                for nm, bt, u in zip(names, byts, us) if bt]
        dom = max(kern, key=lambda d: d["us_per_launch"])
        it_us = sum(us)
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r02", "traffic_c5.json")
        if args.config == "C5" and c == 512 and stats["schedule"] == 3 and stats["format"] == 2 and os.path.exists(tp):
            with open(tp) as fh:
                tk = json.load(fh)["kernels"]
            key = dom["kernel"].split(" ")[0]
            traffic = tk.get(key, {}).get("traffic_bytes")
        roof = {"bound": "hbm", "kernel": dom["kernel"], "achieved": dom["achieved_GBps"], "peak": hbm,
                "unit": "GB/s", "frac": dom["achieved_GBps"] / hbm, "peak_source": peak_kind, "traffic": traffic,
                "traffic_source": "profiles/r02/traffic_c5.json (ncu --set full, dram read+write per launch)"
                if traffic else None,
                "bytes_per_launch": dom["bytes_per_launch"], "us_per_launch": dom["us_per_launch"],
                "kernels": kern, "schedule": stats["schedule"], "engine": "short" if stats["short_rows"] else None,
                "iteration": {"bytes": sum(byts), "us": it_us, "frac": sum(byts) / it_us / 1e3 / hbm,
                              "frac_vs_88n_ideal": (mat + 88.0 * n) / it_us / 1e3 / hbm}}
        ro = read_only_peak()
        if stats["schedule"] == 3 and stats["dia_positions"] > 0:
            # one-trip (uniform-offset) slices carry no column ids: the bytes this K1b moves are
            # fewer than §8(d)'s 12 per entry (values 8 per stored entry, ids 4 in the other
            # slices, per slice 8 offsets + a mask + its slice offset, p read once, q written)
            se = float(stats["sell_entries"])
            ns = (n + 31) // 32
            # ids are read by the slices that are not one-trip (an average slice's entries each)
            ids = 4.0 * se * (1.0 - stats["dia_slices"] / max(ns, 1))
            # values are read by the slices that are not value-uniform too (the others take
            # their 8 per-position values, 64 B + a mask, with their offsets)
            dv = stats.get("dval_slices", 0)
            vals = 8.0 * se * (1.0 - dv / max(ns, 1))
            # per slice its pattern index (1 B); a slice without a shared pattern also its
            # offset 8, offset mask 1, length + value mask 2, 8 offsets 32 and 8 values 64
            pat = stats.get("pat_slices", 0)
            meta = 1.0 * ns + 107.0 * (ns - pat)
            fb = vals + ids + meta + 8.0 + 16.0 * n
            k1b = kern[1]
            roof["format_bytes"] = {"kernel": "k1b_kernel", "bytes_per_launch": fb,
                                    "achieved_GBps": fb / k1b["us_per_launch"] / 1e3,
                                    "frac_vs_copy_peak": fb / k1b["us_per_launch"] / 1e3 / hbm,
                                    "one_trip_slices": stats["dia_slices"], "value_free_slices": dv,
                                    "pattern_slices": pat, "patterns": stats.get("npat", 0),
                                    "slices": ns,
                                    "note": "frac > 1 by the section 8(d) bytes (12 per entry, CSR ids) is "
                                            "the format moving fewer bytes than that ideal: no column ids in "
                                            "uniform-offset slices, one value per position in value-uniform "
                                            "ones (the same values and sums)"}
            if ro:
                roof["format_bytes"]["frac_vs_read_only_peak"] = fb / k1b["us_per_launch"] / 1e3 / ro["GBps"]
        if ro:  # the contract's peak is a copy (read + write); K1b's stream is ~93 % reads
            roof["read_only_stream_peak"] = dict(ro, frac=dom["achieved_GBps"] / ro["GBps"])
        k_us = list(us)
        xs = torch.ones(n, dtype=torch.float64, device="cuda")
        ys = torch.empty_like(xs)
        for _ in range(3):
            A.spmv(xs, ys)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 20
        e0.record()
        for _ in range(reps):
            A.spmv(xs, ys)
        e1.record()
        torch.cuda.synchronize()
        spmv_us = e0.elapsed_time(e1) * 1e3 / reps
        spmv_gbs = (12.0 * nnz + 4.0 * (n + 1) + 16.0 * n) / (spmv_us * 1e-6) / 1e9
    else:
        per_iter_us = ms * 1e3 / max(iters, 1)
        vb = 56.0 + K1A_BYTES[xdefer_cycle()]  # K1b 16n + K2 40n + K1a (x deferred over the cycle)
        achieved = (12.0 * nnz + 4.0 * (n + 1) + vb * n) / world / (per_iter_us * 1e-6) / 1e9
        roof = {"bound": "hbm", "kernel": f"whole iteration incl. halo + allreduces (per GPU, {vb:.0f}n schedule)",
                "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm, "peak_source": peak_kind,
                "traffic": None, "comm": args.comm}

    if args.solver == "pipelined" and not multi:  # the whole pipelined solve is one kernel
        inf = infos[-1][0]
        ach = inf["bytes_algorithmic"] / world / max(inf["t_solve_s"], 1e-12) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "peak_source": peak_kind, "traffic": None,
                "kernel": ("pipe_kernel (whole pipelined solve: per iteration one fused SpMV + 8 vector updates, "
                           "12 nnz + 4(n+1) + 160 n bytes, one grid barrier)" if world == 1 else
                           "pd_fused_kernel + one allreduce + halo per iteration (per GPU, 160n schedule)"),
                "pcg_kernels_for_comparison": roof}

    if args.solver == "block" and multi:  # block CG, one shared Krylov space for the k columns
        inf = infos[-1]
        tot = sum(f["bytes_algorithmic"] for f in inf)
        ach = tot / max(inf[0]["t_solve_s"], 1e-12) / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "peak_source": peak_kind, "traffic": None,
                "kernel": ("block CG iteration (bcg_spmm + 2 Gram passes + update + P update + 2 k x k solves: "
                           "12 nnz + 4(n+1) + 112 k n + 8 n bytes per iteration)"),
                "independent_solver_kernels_for_comparison": roof}

    # ---- CPU oracle baseline (rank 0, N = 1 only): measured on a bounded sample, scaled
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        smp = oracle_sample(args.config, args.sample_c)
        iters_full, timing = oracle_full_iterations(args.config, c)
        it_w = iters_full or iters
        t1 = statistics.median(smp["t_solve"])
        v = scale_to_workload(t1, smp, n, nnz_given, it_w) * kcols  # the oracle solves the k columns one by one
        ac = smp.get("all_cores")
        cpu = {"value": v, "unit": "s", "cores": 1, "kind": "oracle", **host_cpu(),
               "sample": (f"oracle/oracle.c Jacobi-PCG as it stands, 1 thread, on the {args.config} construction at "
                          f"c={args.sample_c} ({smp['n']} unknowns, {smp['nnz']} nnz, {smp['iterations']} "
                          f"iterations, measured {t1:.2f} s); scaled to the workload by per-iteration bytes x "
                          f"{it_w} iterations ({'the oracle own full-size count, tests/golden' if iters_full else 'the GPU count'})"),
               "all_cores": ({"value": scale_to_workload(ac["t_solve"], smp, n, nnz_given, it_w) * kcols,
                              "cores": ac["threads"], "measured_sample_s": ac["t_solve"],
                              "build": "oracle.c -fopenmp -DORC_OMP (timing only)"} if ac else None),
               "oracle_measured_full_size": timing}

    if rank == 0:
        h2d = 16 * (r1 - r0) * kcols  # b and x0 per column
        d2h = 8 * (r1 - r0) * kcols   # x per column
        line = {
            "metric": "pcg_time_to_solution", "value": ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": dict(workload_config(args.config, c, n, nnz, world), iterations=iters,
                           format={1: "csr", 2: "sell", 3: "sell_tma", 4: "sell_sigma"}[stats["format"]], setup_s=round(t_setup, 3),
                           d16_slices=A.stats()["d16_slices"], dval_slices=A.stats()["dval_slices"],
                           pat_slices=A.stats()["pat_slices"], spmm_windowed=A.stats()["spmm_windowed"],
                           relres_true=max(i["relres_true"] for i in infos[-1]), k_rhs=kcols,
                           solver={"pcg": "jacobi-pcg", "pipelined": "pipelined jacobi-pcg (N3)",
                                   "block": "block cg, jacobi (N3)"}[args.solver],
                           **({"drop_zeros": True, "nnz_given": nnz_given} if args.drop_zeros else {}),
                           **({"relabel_seed": args.relabel} if args.relabel is not None else {}),
                           **({"reorder": args.reorder, "n_ghost": stats["n_ghost"]} if reorder else {}),
                           **({"iterations_per_rank": rank_iters} if rank_iters else {})),
            "throughput": {"cg_iterations_per_s": iters / (ms / 1e3),
                           "effective_GBps": iter_bytes(n, nnz, kcols) * iters / (ms / 1e3) / 1e9,
                           "spmv_GBps": spmv_gbs, "spmv_frac_of_hbm": spmv_gbs / hbm if spmv_gbs else None},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": ms_e2e / 1e3, "unit": "s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": cs.summary(), "remeasured": remeasured,
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        A.close()
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


# ------------------------------------------------------------------------------ SURVEY §8(f) N2
CUBES = {"CUBE1": 128, "CUBE2": 256, "CUBE3": 512}  # the paper's Table 1 grids, nodes per axis


def run_bicgstab(args):
    """The paper's own iterative experiment on its own regular grids: BiCGSTAB + (Block-)
    Jacobi on the Table 1 identity-row FD systems, eps = 1e-12,
    boundary data x^2 - y^2 (reading R2).  A step = one pcg_bicgstab solve
    from x0 = 0 on one GPU; the iteration is one cooperative kernel, so the roofline is
    the whole iteration's algorithmic bytes over its time."""
    N = args.c or CUBES[args.config]
    tol, bs = 1e-12, args.block
    n = N ** 3
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return 0
        import oracle as O
        Ns = 48
        A, b = O.fd_cube(Ns)
        times, its = [], 0
        for s_ in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            r = O.bicgstab(A, b, tol=tol, block=bs)
            if s_ >= args.warmup:
                times.append(time.perf_counter() - t0)
            its = r.iterations
        value = statistics.median(times)
        iters = its * (N - 1) / (Ns - 1)  # BiCGSTAB+Jacobi steps grow ~linearly in N here (37/81/169 at 16/32/64)
        nnz = 7 * (N - 2) ** 3 + n - (N - 2) ** 3
        per_iter_bytes = lambda nn, zz: 2 * (12.0 * zz + 28.0 * nn) + 136.0 * nn  # noqa: E731
        est = value / its * per_iter_bytes(n, nnz) / per_iter_bytes(A.n, A.nnz) * iters
        desc = (f"oracle BiCGSTAB (1 thread, as it stands) on the {Ns}^3 Table 1 grid ({its} iterations), one "
                f"complete solve per step; measured, not scaled")
        line = {"impl": "reference", "metric": "bicgstab_time_to_solution", "value": value, "unit": "s",
                "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
                "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": f"{args.config}: Table 1 grid {N}^3 nodes, BiCGSTAB block={bs}", "n": n,
                           "timed_sample": f"{Ns}^3 nodes"},
                "cpu_baseline": {"value": value, "unit": "s", "cores": 1, "kind": "oracle", "sample": desc,
                                 **host_cpu()},
                "full_workload_estimate": {"value": est, "unit": "s",
                                           "basis": f"per-iteration bytes x {iters:.0f} estimated iterations"},
                "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0
    import ctypes as C

    import torch
    import torch.distributed as dist

    import paper_2201_05413_b200 as pcg
    from paper_2201_05413_b200._lib import check, lib
    from paper_2201_05413_b200.problems import fd_cube_build
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    cb = args.comm == "callbacks"
    if cb:  # ranks may share a GPU
        local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if bs != 1:
            raise SystemExit("bench.py: distributed BiCGSTAB takes point Jacobi (--block 1)")
        if cb:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    t0 = time.perf_counter()
    comm = None
    if world == 1:
        r0, r1 = 0, n
        G = fd_cube_build(N)
        fmt = "sell" if (args.precond == "ilu0" and args.fmt == "auto") else args.fmt  # ILU(0): caller's order
        A = pcg.Matrix.from_csr(G["row_ptr"], G["col"], G["val"], fmt=fmt)
        nnz = G["col"].numel()
    else:  # the partition rule on the full row pointer, then this rank's rows on its GPU
        rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
        tot = C.c_int64()
        check(lib().fd_cube_count(N, 0, n, C.c_void_p(rp.data_ptr()), C.byref(tot),
                                  C.c_void_p(torch.cuda.current_stream().cuda_stream)), "fd_cube_count")
        bounds = pcg.partition_rows(rp.cpu().numpy(), world)
        del rp
        nnz = tot.value
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        G = fd_cube_build(N, row_begin=r0, row_end=r1)
        comm = pcg.Comm.host_callbacks() if cb else pcg.Comm.from_process_group()
        A = pcg.Matrix.from_csr_dist(comm, n, r0, r1, G["row_ptr"], G["col"], G["val"], fmt=args.fmt)
    b = G["b"].contiguous()
    del G
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    for _ in range(args.warmup):
        A.bicgstab(b, tol=tol, block=bs, precond=args.precond)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def allreduce(v, op):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device="cpu" if cb else "cuda")
        dist.all_reduce(t, op=op)
        return float(t.item())

    def timed(device_inputs):
        bb = b if device_inputs else b.cpu().pin_memory()
        xx = torch.empty_like(bb) if device_inputs else torch.empty(bb.shape, dtype=torch.float64).pin_memory()
        barrier()
        l0 = pcg.kernel_launches()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.current_stream()
        infos = []
        with ClockSampler(local) as cs:
            e0.record(st)
            for _ in range(args.steps):
                xx.zero_()
                x, inf = A.bicgstab(bb, tol=tol, block=bs, out=xx, precond=args.precond)
                infos.append(inf)
            e1.record(st)
            barrier()
        ms = e0.elapsed_time(e1) / args.steps
        return allreduce(ms, dist.ReduceOp.MAX if world > 1 else None), infos, pcg.kernel_launches() - l0, cs, x

    ms, infos, launches, cs, x = timed(True)
    remeasured = False
    if cs.bad():
        ms, infos, launches, cs, x = timed(True)
        remeasured = True
    ms_e2e = timed(False)[0]
    inf = infos[-1]
    A_fmt = A.stats()["format"]
    iters = inf["iterations"]
    hbm, peak_kind = peaks()
    per_iter_bytes = inf["bytes_algorithmic"] / max(iters, 1)  # this rank's rows
    achieved = per_iter_bytes * iters / allreduce(inf["t_solve_s"], dist.ReduceOp.MAX if world > 1 else None) / 1e9
    # x_err of Eq. ERROR-METRIC: the discrete solution is x^2 - y^2 exactly
    h = 1.0 / (N - 1)
    idx = torch.arange(r0, r1, device=x.device, dtype=torch.float64)
    X = torch.remainder(idx, N) * h
    Y = torch.remainder(torch.div(idx, N, rounding_mode="floor"), N) * h
    xg = X * X - Y * Y
    e2 = allreduce(float(torch.sum((x.to(xg.device) - xg) ** 2)), dist.ReduceOp.SUM if world > 1 else None)
    g2 = allreduce(float(torch.sum(xg ** 2)), dist.ReduceOp.SUM if world > 1 else None)
    x_err = (e2 / g2) ** 0.5
    if comm is not None:
        A.close()
        comm.close()
    if world > 1:
        dist.destroy_process_group()
    if rank != 0:
        return 0
    if args.precond == "ilu0":
        pc_desc = f"Block-Jacobi ILU(0), {(bs if bs > 0 else -(-n // torch.cuda.get_device_properties(local).multi_processor_count))} rows per block"
    else:
        pc_desc = "Jacobi" if bs == 1 else f"Block-Jacobi({bs})"
    line = {"metric": "bicgstab_time_to_solution", "value": ms / 1e3, "unit": "s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: paper Table 1 grid, {N}^3 nodes, identity boundary rows, "
                                   f"b = x^2 - y^2 on the boundary; BiCGSTAB + "
                                   f"{pc_desc}, eps = 1e-12, x0 = 0",
                       "n": n, "nnz": nnz, "tol": tol, "block": bs, "iterations": iters, "relres_true": inf["relres_true"],
                       "x_err": x_err, "format": {1: "csr", 2: "sell", 3: "sell_tma", 4: "sell_sigma"}[A_fmt],
                       "setup_s": round(setup, 3),
                       "parallelism": "1 GPU" if world == 1 else f"{world} GPUs, rows partitioned ({args.comm})",
                       "paper_context": "Cube 1 (128^3): BiCGSTAB+BJacobi 17.4 s, 128 it. on 1 Broadwell core; "
                                        "0.34 s on 576 cores (P:211, P:220, eps 1e-12)"},
            "roofline": {"bound": "hbm",
                         "kernel": ("five kernels per BiCGSTAB iteration (graph schedule; bytes per iteration "
                                    "over its time)" if world == 1 else
                                    "five kernels + four allreduces + two halos per iteration (rank 0's rows)"),
                         "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "peak_source": peak_kind, "traffic": None, "bytes_per_iteration": per_iter_bytes},
            "cpu_baseline": None,
            "e2e": {"value": ms_e2e / 1e3, "unit": "s", "h2d_bytes_per_step": 16 * (r1 - r0),
                    "d2h_bytes_per_step": 8 * (r1 - r0)},
            "gpu_launches": launches, "clocks": cs.summary(), "remeasured": remeasured}
    print(json.dumps(line), flush=True)
    return 0


def fem_build_rowptr(spec, n):
    """Row pointer of the full system (device count pass), for the partition rule."""
    import ctypes as C

    import torch

    from paper_2201_05413_b200._lib import check, lib
    rp = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    nnz = C.c_int64()
    check(lib().fem_count(C.byref(spec), 0, n, C.c_void_p(rp.data_ptr()), C.byref(nnz),
                          C.c_void_p(torch.cuda.current_stream().cuda_stream)), "fem_count")
    return rp.cpu().numpy()


if __name__ == "__main__":
    sys.exit(main())
