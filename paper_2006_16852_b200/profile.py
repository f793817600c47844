"""SpMV performance-profile harness on the GPU formats + automatic format
choice (the paper's SpMV comparison methodology, PAPER.md
§6.3, and the reference's src/bench.py:186-248).

``run_profile`` reads every ``.mtx`` of a directory (native parser), assembles
each matrix on the device once, converts it to every requested format, and
times ``apply`` with CUDA events on the executor's stream (median of ``reps``
after a warm-up; optional L2 flush between reps). ``profile_curves`` /
``profile_csv`` are the reference's coverage curves and CSV verbatim.

``choose_format`` is the automatic choice: it times the candidate formats
on the matrix itself (one warm-up + ``reps`` device-timed applies each) and
returns the fastest, caching the decision on the matrix object.
"""

from __future__ import annotations

import os

import numpy as np

from .errors import OpalgError, ParseError, Unsupported
from .formats import Dense, convert, matrix_from_data
from .mmio import read_matrix_market_file

PROFILE_SCHEMA = "opalg-bench/profile/v1"

#: every device SpMV of this package (format / Csr strategy names accepted by convert)
GPU_FORMATS = ("csr", "csr_classical", "csr_lb", "csr_pipe", "coo", "ell", "sellp", "hybrid")


def profile_curves(runtimes, taus):
    """Coverage curves from a (format -> per-matrix runtime list) table: a
    format covers a matrix at slowdown tau when its runtime is within tau of
    the per-matrix best; ties at tau = 1 credit every tied format
    (src/bench.py:186-200)."""
    formats = sorted(runtimes)
    table = np.asarray([runtimes[f] for f in formats], dtype=float)
    best = table.min(axis=0)
    return {f: [(float(tau), float(np.mean(table[i] <= tau * best))) for tau in taus]
            for i, f in enumerate(formats)}


def profile_csv(result):
    """format,tau,fraction rows (src/bench.py:241-246)."""
    lines = ["format,tau,fraction"]
    for fmt, curve in sorted(result["curves"].items()):
        for tau, frac in curve:
            lines.append(f"{fmt},{tau:.6g},{frac:.6g}")
    return "\n".join(lines) + "\n"


class _Timer:
    def __init__(self, exc, flush_mib):
        import torch

        self.torch = torch
        self.exc = exc
        self.stream = torch.cuda.current_stream(exc.device)  # the executor launches on it
        self.flush = torch.empty(flush_mib << 20, dtype=torch.uint8, device=exc.device) if flush_mib else None

    def median_ns(self, fn, reps):
        torch = self.torch
        fn()  # warm-up (plans, workspaces)
        torch.cuda.synchronize()
        samples = []
        for _ in range(reps):
            if self.flush is not None:
                self.flush.fill_(1)
                self.flush.view(torch.int64).sum()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(self.stream)
            fn()
            e.record(self.stream)
            e.synchronize()
            samples.append(s.elapsed_time(e) * 1e6)
        return float(np.median(samples))


def time_formats(exc, a, formats, reps=10, flush_mib=0, rhs=None):
    """{format: median device ns per apply} of ``a`` converted to each format."""
    n, m = a.size
    b = Dense(exc, rhs if rhs is not None else np.random.default_rng(0).standard_normal((m, 1)))
    x = Dense.zeros(exc, n, 1)
    timer = _Timer(exc, flush_mib)
    out = {}
    for f in formats:
        mat = convert(a, f)
        out[f] = timer.median_ns(lambda: mat.apply(b, x), reps)
        del mat
    return out


def run_profile(matrix_dir, formats=GPU_FORMATS, reps=10, tau_max=4.0, tau_points=31, executor=None,
                flush_mib=0):
    """The reference's profile run (src/bench.py:203-238) on the GPU formats."""
    from .executor import CudaExecutor

    exc = executor or CudaExecutor()
    paths = sorted(p for p in os.listdir(matrix_dir) if p.endswith(".mtx"))
    runtimes = {f: [] for f in formats}
    used, skipped = [], []
    for name in paths:
        path = os.path.join(matrix_dir, name)
        try:
            data = read_matrix_market_file(path)
            a = matrix_from_data(exc, data, "csr")
        except (ParseError, Unsupported, OSError, OpalgError) as err:
            skipped.append({"matrix": name, "error": str(err)})
            continue
        used.append(name)
        for f, t in time_formats(exc, a, formats, reps, flush_mib).items():
            runtimes[f].append(t)
    taus = np.linspace(1.0, tau_max, tau_points)
    curves = profile_curves(runtimes, taus) if used else {}
    return {"schema": PROFILE_SCHEMA, "matrices": used, "skipped": skipped, "repetitions": reps,
            "runtimes_ns": runtimes, "curves": curves}


def choose_format(a, candidates=("csr", "csr_lb", "ell", "sellp", "hybrid", "coo"), reps=3):
    """Fastest of ``candidates`` for ``a`` by device timing on ``a`` itself;
    returns (format name, converted matrix, {format: ns}). Ell is skipped when
    its padding would more than double the stored entries (the Ell
    conversion alone could exceed memory on skewed matrices)."""
    cached = getattr(a, "_auto_format", None)
    if cached is not None:
        return cached
    exc = a.exec
    cands = list(candidates)
    csr = convert(a, "csr")
    if "ell" in cands and csr.nnz:
        n = csr.size.rows
        if csr._row_stats() * n > 2 * csr.nnz:
            cands.remove("ell")
    times = time_formats(exc, csr, cands, reps)
    best = min(times, key=times.get)
    res = (best, convert(csr, best), times)
    a._auto_format = res
    return res


OVERHEAD_SCHEMA = "opalg-bench/overhead/v1"
OVERHEAD_SOLVERS = ("bicgstab", "cg", "cgs", "fcg", "gmres")


def run_overhead(solvers=OVERHEAD_SOLVERS, iters=1000, runs=20, krylov_dim=100, executor=None):
    """The paper's framework-overhead microbenchmark (
    reference src/bench.py:253-291): time per iteration of each solver on a
    1x1 Coo system with b = NaN and only an Iteration criterion, so every
    control branch runs with negligible kernel work. Wall clock around the
    public apply (device-resident solvers: the device loop and its host
    batch synchronisations included)."""
    import time

    from .executor import CudaExecutor
    from .formats import Coo
    from .solvers import SOLVER_FACTORIES
    from .stop import Iteration

    exc = executor or CudaExecutor()
    results = {}
    for name in solvers:
        kw = {"krylov_dim": krylov_dim} if name == "gmres" else {}
        a = Coo(exc, (1, 1), [0], [0], [1.0])
        solver = SOLVER_FACTORIES[name](exc, criteria=[Iteration(iters)], **kw).generate(a)
        per_run = []
        for r in range(runs + 1):
            b = Dense(exc, [[float("nan")]])
            x = Dense.zeros(exc, 1, 1)
            t0 = time.perf_counter_ns()
            solver.apply(b, x)
            dt = (time.perf_counter_ns() - t0) / iters
            if solver.last_status.iterations != iters:
                raise OpalgError(f"{name}: expected {iters} iterations, got {solver.last_status.iterations}")
            if r:  # the first run captures the CUDA graphs
                per_run.append(dt)
        results[name] = {"iterations": iters, "runs": runs,
                         "time_per_iteration_us": float(np.mean(per_run)) / 1000.0}
    times = [v["time_per_iteration_us"] for v in results.values()]
    return {"schema": OVERHEAD_SCHEMA, "solvers": results,
            "max_over_min": float(max(times) / min(times)) if times else None}
