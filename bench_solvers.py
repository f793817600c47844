"""Solver / power-law workloads for bench.py (``--workload c1|c3|c4b|c4g|c5``).

  c1   CG, 2-D 5-point Poisson 256^2 (65,536 rows), rhs ones, x0 = 0, RNR 1e-8
  c3   Csr load-balanced vs Hybrid SpMV, power law 4,194,304 rows (~16 nnz/row)
  c4b  BiCGSTAB + block-Jacobi(32), 3-D 7-point convection-diffusion 256^3
  c4g  GMRES(30) + block-Jacobi(32), same system
  c5   CG, 3-D 7-point Poisson 512^3 (134,217,728 rows) on one GPU

Solver workloads report ms per iteration of complete solves (device time,
CUDA events on the solve stream, inputs resident in HBM); one step = one
full solve from x0 = 0. e2e = the same solve through the public API with host
b / x (H2D of b and x0, D2H of x inside the timed region).
"""

from __future__ import annotations

import os

import statistics
import time

import numpy as np

from bench import METRIC, ClockSampler, Timer, allmax, barrier, bytes_csr, bytes_format, peaks


def _solve_timer(fn, steps):
    import torch

    times = []
    for _ in range(steps):
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e-3)
    return times, out


def bench_solver(args, world, rank, local, kind):
    import torch

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib, problems

    exc = b2.CudaExecutor(local)
    torch.cuda.set_device(local)
    peak, peak_src = peaks()
    if kind == "c1":
        a = problems.stencil(exc, "5pt", 256)
        fac = b2.Cg(exc, criteria=[b2.Iteration(10000), b2.ResidualNormReduction(1e-8)])
        wl = "C1: CG, 2-D 5-point Poisson 256^2 (65,536 rows), rhs ones, x0 = 0, RNR 1e-8, fp64"
        vec_passes = 8  # the cooperative kernel folds p = r + beta p into the SpMV
    elif kind == "c5":
        a = problems.stencil(exc, "7pt", args.grid or 512)
        fac = b2.Cg(exc, criteria=[b2.Iteration(20000), b2.ResidualNormReduction(1e-8)])
        wl = f"C5: CG, 3-D 7-point Poisson {args.grid or 512}^3, rhs ones, x0 = 0, RNR 1e-8, fp64, 1 GPU"
        # SpMV + p update (3n) + x, r update with r.r (6n)
        vec_passes = 9
    else:
        g = args.grid or 256
        a = problems.stencil(exc, "convdiff", g)
        pre = b2.Jacobi(exc, block_size=32)
        if kind == "c4b":
            fac = b2.Bicgstab(exc, criteria=[b2.Iteration(20000), b2.ResidualNormReduction(1e-8)],
                              preconditioner=pre)
            wl = f"C4: BiCGSTAB + block-Jacobi(32), 3-D 7-point conv-diff {g}^3, rhs ones, RNR 1e-8, fp64"
        else:
            fac = b2.Gmres(exc, criteria=[b2.Iteration(20000), b2.ResidualNormReduction(1e-8)],
                           preconditioner=pre, krylov_dim=30)
            wl = f"C4: GMRES(30) + block-Jacobi(32), 3-D 7-point conv-diff {g}^3, rhs ones, RNR 1e-8, fp64"
        vec_passes = None
    n = a.size.rows
    t0 = time.perf_counter()
    solver = fac.generate(a)
    generate_s = time.perf_counter() - t0
    b = b2.Dense(exc, np.ones((n, 1)))
    x = b2.Dense.zeros(exc, n, 1)

    def one():
        x.fill(0.0)
        solver.apply(b, x)
        return solver.last_status

    for _ in range(max(1, args.warmup // 3)):
        one()
    barrier(world)
    launches0 = _lib.launch_count()
    with ClockSampler(local) as clk:
        times, st = _solve_timer(one, args.steps)
    launches = (_lib.launch_count() - launches0) // max(1, args.steps)
    its = st.iterations
    t = allmax(world, statistics.mean(times))
    ms_iter = t / max(its, 1) * 1e3
    # e2e through the public API with host operands
    host = exc.master
    bh = b2.Dense(host, np.ones((n, 1)))
    xh = b2.Dense(host, np.zeros((n, 1)))
    e2e = []
    for _ in range(max(1, min(args.steps, 3))):
        xh.values[...] = 0.0
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        solver.apply(bh, xh)
        e2e.append(time.perf_counter() - s0)
    e2e_t = allmax(world, statistics.mean(e2e))
    out = {
        "metric": METRIC, "value": round(ms_iter, 4), "unit": "ms/iter", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": False,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated stencil, b = ones, x0 = 0)",
        "config": {"workload": wl, "rows": n, "nnz": a.nnz, "iterations": its,
                   "converged": bool(st.converged), "generate_s": round(generate_s, 3),
                   "l2": "working set larger than L2 (C4/C5); C1 is L2-resident (latency-bound)"},
        "e2e": {"value": round(e2e_t / max(its, 1) * 1e3, 4), "unit": "ms/iter",
                "h2d_bytes_per_step": 2 * n * 8, "d2h_bytes_per_step": n * 8,
                "ms_per_step": round(e2e_t * 1e3, 3)},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }
    # the paper-comparable figure: the reference's traffic model (src/model.py,
    # COO-unpreconditioned ledger) per iteration over the measured time
    from paper_2006_16852_b200.model import per_iteration_bytes

    sname = {"c1": "cg", "c5": "cg", "c4b": "bicgstab", "c4g": "gmres"}[kind]
    mb = per_iteration_bytes(sname, n, a.nnz, its, krylov_dim=30 if kind == "c4g" else 100)
    out["model_traffic"] = {"source": "src/model.py ledger (reference solver loop, COO, no preconditioner)",
                            "bytes_per_iter": int(mb), "GBps": round(mb / (t / its) / 1e9, 1),
                            "frac_of_peak": round(mb / (t / its) / 1e9 / peak, 4)}
    if vec_passes is None:  # C4: bytes per counted iteration from the kernels' traffic
        spmv = bytes_csr(n, a.nnz, 8)
        jac = int(solver.precond._storage.numel()) * solver.precond._storage.element_size() + 2 * n * 8
        if kind == "c4b":
            # one cycle = two counted half-iterations: 2 SpMV (+ the fused
            # second-vector reads) + 2 Jacobi applies + 19 vector passes
            by_it = (2 * spmv + 2 * jac + 19 * n * 8) / 2
            label = "BiCGSTAB half-iteration (2 SpMV + 2 block-Jacobi + 19n vector values per cycle)"
        else:
            # GMRES step j: SpMV + Jacobi + the reference ledger for m = 1
            # (src/solvers/gmres.py:238-242), averaged over the run's steps
            k = 30
            tot = 0.0
            for it in range(1, its + 1):
                j = (it - 1) % k + 1
                tot += ((7 * n + 5) + (j - 1) * (4 * n + 4)) * 8 + 8 + ((3 * n + 8) + (j - 1) * (n + 2)) * 8 + 8
            by_it = spmv + jac + tot / max(its, 1)
            label = "GMRES(30) step (SpMV + block-Jacobi + reference MGS ledger, run average)"
        out["roofline"] = {"bound": "hbm", "achieved": round(by_it / (t / its) / 1e9, 1), "peak": peak,
                           "unit": "GB/s", "frac": round(by_it / (t / its) / 1e9 / peak, 4), "traffic": None,
                           "peak_source": peak_src, "kernel": label, "bytes_per_launch": int(by_it)}
    if vec_passes is not None:
        by = bytes_csr(n, a.nnz, 8) + vec_passes * n * 8
        out["roofline"] = {"bound": "hbm", "achieved": round(by / (t / its) / 1e9, 1), "peak": peak,
                           "unit": "GB/s", "frac": round(by / (t / its) / 1e9 / peak, 4), "traffic": None,
                           "peak_source": peak_src, "kernel": f"whole CG iteration (Csr SpMV + {vec_passes}n values)",
                           "bytes_per_launch": by}
    return out


def bench_c3(args, world, rank, local):
    import torch

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib, problems

    exc = b2.CudaExecutor(local)
    peak, peak_src = peaks()
    a = problems.power_law(exc, 4194304, seed=0, lengths="rng")  # SURVEY 8(d) row lengths
    n, nnz = a.size.rows, a.nnz
    b = b2.Dense(exc, np.random.default_rng(0).standard_normal((n, 1)))
    x = b2.Dense.zeros(exc, n, 1)
    timer = Timer(exc)
    res = {}
    for name in ("csr_lb", "hybrid", "coo", "csr_stream"):
        m = b2.convert(a, name)
        m.apply(b, x)
        ms = timer.run(lambda: m.apply(b, x), max(5, args.steps), 3)
        t = statistics.mean(ms) * 1e-3
        by = bytes_format(m, 8)
        res[name] = {"us": round(t * 1e6, 1), "gbs": round(by / t / 1e9, 1),
                     "gbs_useful": round(bytes_csr(n, nnz, 8) / t / 1e9, 1), "frac": round(by / t / 1e9 / peak, 4)}
    head = res["csr_lb"]
    return {"metric": METRIC, "value": head["gbs"], "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["us"] / 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic power law: SURVEY 8(d) row lengths (default_rng(0)), stratified distinct columns and U(-1,1) values from the device hash generator",
            "config": {"workload": "C3: Csr load-balanced SpMV, power law 4,194,304 rows, mean 16, max 50k",
                       "rows": n, "nnz": nnz},
            "roofline": {"bound": "hbm", "achieved": head["gbs"], "peak": peak, "unit": "GB/s",
                         "frac": head["frac"], "traffic": None, "peak_source": peak_src},
            "formats": res, "gpu_launches": 2}


def _dist_breakdown(A, comm, solver, world, reps=30):
    """Per-iteration pieces of the distributed CG, each timed alone with CUDA
    events (max over ranks): the communication-free iteration (step1, owned
    and ghost SpMV, sigma, step2 on a criterion-free control block), one halo
    exchange, one 8-byte all-reduce. iteration - compute = the communication
    the overlap does not hide."""
    import ctypes

    import torch

    from paper_2006_16852_b200 import _lib
    from paper_2006_16852_b200.executor import ptr

    exc = A.exec
    nl, dt = A.n_local, torch.float64
    suf = "f64"
    pext = torch.ones(A.n_ext, dtype=dt, device=exc.device)
    p, q, r, x = pext[:nl], torch.zeros(nl, dtype=dt, device=exc.device), torch.ones(nl, dtype=dt, device=exc.device), \
        torch.zeros(nl, dtype=dt, device=exc.device)
    ctl = torch.zeros(int(_lib.query("krylov_ctl_bytes")), dtype=torch.uint8, device=exc.device)
    part = torch.zeros(int(_lib.query("krylov_part_elems")), dtype=torch.float64, device=exc.device)
    t0, p0 = (ctypes.c_int32 * 1)(), (ctypes.c_double * 1)()
    _lib.call("krylov_ctl_init", ptr(ctl), 0, ctypes.addressof(t0), ctypes.addressof(p0), 1, 0, 0, exc.stream)
    J = (0, 0, 0, 0, 0)

    class _NoHalo:  # the same kernels as the solve, without the exchange
        def __getattr__(self, k):
            return getattr(A, k)

        def start_halo(self, xext):
            class _W:
                def wait(self):
                    pass
            return _W()

    view = solver.__class__.__new__(solver.__class__)
    view.__dict__.update(solver.__dict__)
    view.a = _NoHalo()

    def compute():
        _lib.call("cg_step1_" + suf, nl, ptr(p), ptr(r), ptr(ctl), exc.stream)
        view._spmv_sigma(pext, p, q, ptr(ctl), part, suf)
        _lib.call("cg_step2_" + suf, nl, ptr(x), 1, ptr(r), ptr(p), ptr(q), ptr(r), *J, ptr(ctl), ptr(part), 0,
                  exc.stream)

    def halo():
        A.start_halo(pext).wait()

    red = torch.zeros(1, dtype=torch.float64, device=exc.device)

    def allreduce():
        comm.allreduce_(red)

    cases = [("compute_ms", compute), ("halo_ms", halo), ("allreduce_ms", allreduce)]
    peer = getattr(A, "_peer_halo", {}).get(torch.float64)
    if peer is not None:  # the halo the solve used: peer stores fused into step1 + the flag wait
        cases += [("step1_ms", lambda: _lib.call("cg_step1_" + suf, nl, ptr(p), ptr(r), ptr(ctl), exc.stream)),
                  ("step1_peer_put_wait_ms", lambda: (peer.step1(nl, p, r, ptr(ctl), suf, exc.stream),
                                                      peer.wait(ptr(ctl), exc.stream)))]
    pred = getattr(A, "_peer_reduce", None)
    if pred is not None:
        cases.append(("peer_allreduce_ms", lambda: pred.allreduce_(red, exc.stream)))
    out = {}
    for name, fn in cases:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        barrier(world)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        out[name] = round(allmax(world, s.elapsed_time(e) / reps), 4)
    return out


def bench_c5_distributed(args, world, rank, local):
    """C5 row-partitioned CG over NCCL (torchrun, one rank per GPU): strong
    scaling of the fixed 512^3 problem; ms per iteration, max over ranks."""
    import torch

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200.distributed import DistCg, DistCsr, make_comm

    exc = b2.CudaExecutor(local)
    torch.cuda.set_device(local)
    g = args.grid or 512
    comm = make_comm()
    t0 = time.perf_counter()
    A = DistCsr.stencil(exc, comm, "7pt", g)
    build_s = time.perf_counter() - t0
    b = torch.ones(A.n_local, dtype=torch.float64, device=exc.device)
    x = torch.zeros(A.n_local, dtype=torch.float64, device=exc.device)
    solver = DistCg(A, [b2.Iteration(20000), b2.ResidualNormReduction(1e-8)])
    for _ in range(max(1, args.warmup // 3)):
        x.zero_()
        solver.solve(b, x)
    barrier(world)
    with ClockSampler(local) as clk:
        times, st = _solve_timer(lambda: (x.zero_(), solver.solve(b, x))[1], args.steps)
    t = allmax(world, statistics.mean(times))
    its = st.iterations
    brk = _dist_breakdown(A, comm, solver, world)
    brk["iteration_ms"] = round(t / max(its, 1) * 1e3, 4)
    brk["exposed_comm_ms"] = round(brk["iteration_ms"] - brk["compute_ms"], 4)
    return {"metric": METRIC, "value": round(t / max(its, 1) * 1e3, 4), "unit": "ms/iter", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (device-generated 7-point Poisson, b = ones, x0 = 0)",
            "config": {"workload": f"C5: row-partitioned CG, 3-D 7-point Poisson {g}^3, RNR 1e-8, "
                                   f"{'peer-memory' if solver.halo == 'peer' else 'NCCL'} halo + {'peer-memory' if solver.reduce == 'peer' else 'NCCL'} all-reduce",
                       "halo": solver.halo, "iterations": its,
                       "converged": bool(st.converged), "parallelism": f"row partition x{world}",
                       "rows_per_rank": A.n_local, "build_s": round(build_s, 3), "breakdown": brk},
            "gpu_launches": None, "clocks": clk.summary()}


PAPER_OVERHEAD_V100_US = {"bicgstab": 1.26, "cg": 1.28, "cgs": 1.00, "fcg": 1.45, "gmres": 1.51}


def bench_overhead(args, world, rank, local):
    """The paper's framework-overhead microbenchmark: us per iteration on a 1x1
    Coo system with b = NaN and Iteration(1000) (reference src/bench.py:253-291)."""
    from paper_2006_16852_b200 import CudaExecutor
    from paper_2006_16852_b200.profile import run_overhead

    res = run_overhead(iters=1000, runs=max(3, min(args.steps, 20)), executor=CudaExecutor(local))
    per = {k: round(v["time_per_iteration_us"], 3) for k, v in res["solvers"].items()}
    return {"metric": "framework overhead per iteration (1x1 system, b = NaN)", "value": per["cg"],
            "unit": "us/iter", "n_gpus": 1, "steps": args.steps, "warmup": 1, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "1x1 Coo [[1.0]], b = NaN",
            "config": {"workload": "PAPER.md:1789-1816 overhead benchmark", "solvers_us_per_iter": per,
                       "paper_v100_us_per_iter": PAPER_OVERHEAD_V100_US},
            "gpu_launches": None}


def bench_workload(args, world, rank, local):
    if args.workload == "overhead":
        return bench_overhead(args, world, rank, local)
    if args.workload == "c3":
        return bench_c3(args, world, rank, local)
    if args.workload == "c5" and world > 1:
        return bench_c5_distributed(args, world, rank, local)
    if args.workload == "c5d":  # the distributed solver, also at one rank (NCCL world of 1)
        import torch
        import torch.distributed as dist

        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
        return bench_c5_distributed(args, world, rank, local)
    return bench_solver(args, world, rank, local, args.workload)
