"""Benchmark: SpMV GB/s & GFLOP/s per format vs the HBM roofline (C2), and
Krylov ms/iteration (C1/C4/C5 workloads).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload c2|c3|c1|c4b|c4g|c5]

Default workload (N=1) is BASELINE.json config C2: the 3-D 27-point stencil
128^3 (2,097,152 rows, 55,742,968 entries), fp64. One *step* = one Csr
(automatic strategy) SpMV x = A b through the C ABI; inputs are larger than
L2 and L2 is additionally flushed (256 MiB write, then read) between timed steps, each
step timed with CUDA events on the launching stream. Every other format
(Csr classical / load-balanced, Coo, Ell, Sellp, Hybrid) in fp64 and fp32 is
timed the same way and reported under "formats". N>1: replicas (weak
scaling; C2 does not shard -- see DESIGN.md).

``--impl reference`` times the reference's CPU algorithm (oracle port of
ParallelExecutor + csr_row_sums) on all host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "SpMV GB/s & GFLOP/s per format vs HBM peak; CG ms/iter at 1/2/4/8 GPUs"


def peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# algorithmic bytes
# ---------------------------------------------------------------------------
def bytes_csr(n, nnz, vt, it=4):
    return nnz * (vt + it) + (n + 1) * it + 2 * n * vt


def bytes_format(m, vt, it=4):
    from paper_2006_16852_b200 import Coo, Csr, Ell, Hybrid, Sellp

    n = m.size.rows
    if isinstance(m, Csr):
        return bytes_csr(n, m.nnz, vt, it)
    if isinstance(m, Coo):
        return m.nnz * (vt + 2 * it) + 2 * n * vt
    if isinstance(m, Ell):
        return n * m.width * (vt + it) + 2 * n * vt
    if isinstance(m, Sellp):
        return m.num_stored_elements * (vt + it) + 2 * m._sl.numel() * it + 2 * n * vt
    if isinstance(m, Hybrid):
        return n * m.ell.width * (vt + it) + m.coo.nnz * (vt + 2 * it) + 2 * n * vt
    raise TypeError(type(m))


# ---------------------------------------------------------------------------
# clocks during the timed region (NVML, 5 ms sampling)
# ---------------------------------------------------------------------------
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons = [], set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ---------------------------------------------------------------------------
# distributed plumbing (torchrun: one process per GPU)
# ---------------------------------------------------------------------------
def self_launch(args):
    """`python bench.py --gpus N` (N > 1) outside torchrun: re-exec under
    torch.distributed.run with N ranks on 127.0.0.1, so the line reports the
    N-rank run it claims. Under torchrun, WORLD_SIZE must equal --gpus."""
    world = os.environ.get("WORLD_SIZE")
    if world is None:
        if args.gpus <= 1:
            return
        import socket

        sock = socket.socket()
        sock.bind(("127.0.0.1", 0))
        port = sock.getsockname()[1]
        sock.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    if int(world) != args.gpus and "--gpus" in " ".join(sys.argv):
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")


#: process-group backend of this run ("nccl": one GPU per rank; "gloo": more
#: ranks than visible GPUs -- ranks share devices, collectives staged on the host)
BACKEND = None


def dist_setup():
    """One process per rank (torchrun env). NCCL when every rank has its own
    GPU; with fewer visible GPUs than ranks (a 1-GPU box running --gpus 2)
    the ranks share devices round-robin over gloo and the distributed
    solver's halo / all-reduce run through peer memory (CUDA IPC on the
    shared device) -- the same kernels, flags and ordering as over NVLink."""
    global BACKEND
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        ndev = max(1, torch.cuda.device_count())
        local = local % ndev
        torch.cuda.set_device(local)
        if ndev >= world:
            BACKEND = "nccl"
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            BACKEND = "gloo"
            os.environ.setdefault("B200SP_PEER_HALO", "1")  # read at package import
            dist.init_process_group("gloo")
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def _reduce_scalar(value, op_name):
    import torch
    import torch.distributed as dist

    dev = "cuda" if BACKEND == "nccl" else "cpu"
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=getattr(dist.ReduceOp, op_name))
    return float(t.item())


def allmax(world, value):
    return value if world == 1 else _reduce_scalar(value, "MAX")


def allsum(world, value):
    return value if world == 1 else _reduce_scalar(value, "SUM")


# ---------------------------------------------------------------------------
# timing helpers
# ---------------------------------------------------------------------------
class Timer:
    """Per-step CUDA-event timing on the launching stream, L2 flushed between
    steps (outside the events)."""

    def __init__(self, exc):
        import torch

        self.torch = torch
        self.flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=exc.device)

    def flush(self):
        # write a buffer larger than L2, then read it: the read evicts the
        # dirty lines of the write here, so their write-back is not charged to
        # the next timed kernel (tools/flush_study.py: a write-only flush
        # adds 10-15 us of write-back to a 150 us SpMV); L2 holds none of the
        # step's operands either way
        self.flush_buf.fill_(1)
        self.flush_buf.view(self.torch.int64).sum()

    def run(self, fn, steps, warmup):
        torch = self.torch
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        stream = torch.cuda.current_stream()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(steps)]
        for s, e in ev:
            self.flush()
            s.record(stream)
            fn()
            e.record(stream)
        torch.cuda.synchronize()
        return [s.elapsed_time(e) for s, e in ev]  # ms


def traffic_from_profiles(kernel_key):
    path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel_key)
    except Exception:
        return None


# ---------------------------------------------------------------------------
# C2: SpMV format sweep
# ---------------------------------------------------------------------------
def bench_c2(args, world, rank, local):
    import torch

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib, problems

    peak, peak_src = peaks()
    exc = b2.CudaExecutor(local)
    torch.cuda.set_device(local)
    g = 128
    timer = Timer(exc)
    rng = np.random.default_rng(0)
    a64 = problems.stencil(exc, "27pt", g, value_dtype="float64")
    n, nnz = a64.size.rows, a64.nnz
    bvec = rng.standard_normal((n, 1))
    results = {}
    head = None
    for dt, vt in (("float64", 8), ("float32", 4)):
        base = a64 if dt == "float64" else problems.stencil(exc, "27pt", g, value_dtype=dt)
        b = b2.Dense(exc, bvec, value_dtype=dt)
        x = b2.Dense.zeros(exc, n, 1, value_dtype=dt)
        variants = [("csr", b2.convert(base, "csr")), ("csr_classical", b2.convert(base, "csr_classical")),
                    ("csr_lb", b2.convert(base, "csr_lb")), ("coo", b2.convert(base, "coo")),
                    ("ell", b2.convert(base, "ell")), ("sellp", b2.convert(base, "sellp")),
                    ("hybrid", b2.convert(base, "hybrid"))]
        for name, m in variants:
            key = f"{name}_{'f64' if vt == 8 else 'f32'}"
            m.apply(b, x)  # build plans/workspaces outside timing
            if name == "csr" and dt == "float64":
                head = (m, b, x)
                continue
            ms = timer.run(lambda: m.apply(b, x), max(5, min(args.steps, 50)), 3)
            t = statistics.mean(ms) * 1e-3
            by = bytes_format(m, vt)
            results[key] = {"us": round(t * 1e6, 2), "gbs": round(by / t / 1e9, 1),
                            "gbs_useful": round(bytes_csr(n, nnz, vt) / t / 1e9, 1),
                            "gflops": round(2 * nnz / t / 1e9, 1), "frac": round(by / t / 1e9 / peak, 4),
                            "bytes": by}
            if name == "csr":
                results[key]["strategy"] = m.strategy
            del m
        torch.cuda.empty_cache()

    # ---- headline: Csr (automatic) fp64, exactly K timed steps ------------
    m, b, x = head
    by = bytes_format(m, 8)
    with ClockSampler(local) as clk:  # sampling spans the warm-up and the timed steps
        for _ in range(args.warmup):
            m.apply(b, x)
        barrier(world)
        torch.cuda.synchronize()
        launches0 = _lib.launch_count()
        ms = timer.run(lambda: m.apply(b, x), args.steps, 0)
        launches = _lib.launch_count() - launches0
    barrier(world)
    t_step = allmax(world, statistics.mean(ms) * 1e-3)
    total_bytes = allsum(world, by)
    value = total_bytes / t_step / 1e9
    results["csr_f64"] = {"us": round(t_step * 1e6, 2), "gbs": round(by / t_step / 1e9, 1),
                          "gbs_useful": round(by / t_step / 1e9, 1),
                          "gflops": round(2 * nnz / t_step / 1e9, 1),
                          "frac": round(by / t_step / 1e9 / peak, 4), "bytes": by,
                          "strategy": m.strategy}
    kern = {"classical": "csr_classical_kernel",
            "stream": "csr_pipe_kernel" if m.stream_impl() == "tma" else "csr_stream_kernel",
            "load_balance": {2: "csr_lb2_kernel", 3: "csr_seg_kernel"}[m.lb_mode()]}[m.strategy]
    roofline = {"bound": "hbm", "achieved": round(by / t_step / 1e9, 1), "peak": peak, "unit": "GB/s",
                "frac": round(by / t_step / 1e9 / peak, 4), "traffic": traffic_from_profiles(kern),
                "peak_source": peak_src, "kernel": kern, "bytes_per_launch": by}

    # ---- e2e: public API with host (pinned) operands ------------------------
    host = exc.master
    bh = b2.Dense(host, bvec)
    xh = b2.Dense(host, np.zeros((n, 1)))
    for _ in range(max(1, args.warmup)):
        m.apply(bh, xh)
    torch.cuda.synchronize()
    e2e_t = []
    for _ in range(max(3, min(args.steps, 20))):
        t0 = time.perf_counter()
        m.apply(bh, xh)  # H2D b, SpMV, D2H x (synchronous on return)
        e2e_t.append(time.perf_counter() - t0)
    e2e_step = allmax(world, statistics.median(e2e_t))  # median: robust to host jitter
    e2e = {"value": round(total_bytes / e2e_step / 1e9, 1), "unit": "GB/s",
           "h2d_bytes_per_step": n * 8, "d2h_bytes_per_step": n * 8,
           "ms_per_step": round(e2e_step * 1e3, 3)}

    # ---- CPU baseline: reference algorithm on host cores (rank 0, N=1) ------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle.cpu_baseline import time_csr_spmv

        rp = m._rp.cpu().numpy()
        ci = m._ci.cpu().numpy()
        vals = m._v.cpu().numpy()
        reps = 3
        tc, cores, _ = time_csr_spmv(rp, ci, vals, bvec, reps=reps, warmup=1)
        cpu = {"value": round(by / tc / 1e9, 3), "unit": "GB/s", "cores": cores, "kind": "port",
               "sample": f"full C2 matrix, Csr SpMV (ParallelExecutor restatement, {cores} threads), "
                         f"median of {reps} after 1 warm-up; {tc * 1e3:.1f} ms/SpMV"}

    out = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated 27-point stencil, b ~ N(0,1) seed 0)",
        "config": {"workload": "C2: Csr SpMV x = A b, 3-D 27-point stencil 128^3 "
                               "(2,097,152 rows, 55,742,968 nnz), fp64 values / int32 indices",
                   "format": f"csr ({m.strategy})", "rows": n, "nnz": nnz,
                   "l2": "inputs larger than L2 and L2 flushed (256 MiB write, then read back) between steps",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "gflops": round(2 * nnz / t_step / 1e9, 1),
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk.summary(), "formats": results,
    }
    return out


# ---------------------------------------------------------------------------
# C2 at N > 1: distributed (row-partitioned) SpMV, weak scaling
# ---------------------------------------------------------------------------
def bench_c2_dist(args, world, rank, local):
    """The C2 SpMV on N GPUs as ONE row-partitioned operator: the 27-point
    stencil on 128 x 128 x (128 N) -- each rank owns exactly one C2-sized
    slab (2,097,152 rows, z-planes [128 r, 128 r + 128)) -- so per-GPU work
    is C2's and the curve measures the distributed path: the 2-plane halo
    (peer-memory puts gated by the neighbours' acks when every pair of GPUs
    has P2P access -- the whole step one CUDA graph; NCCL send/recv, or gloo
    host staging when ranks share a GPU without the peer path, otherwise)
    overlapped with the owned-block SpMV, then the ghost-block accumulate. value = all ranks' algorithmic Csr bytes / the
    max-over-ranks step time; e2e adds each rank's pinned H2D of its x slice
    and D2H of its y slice."""
    import torch

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import _lib
    from paper_2006_16852_b200.distributed import DistCsr, make_comm

    peak, peak_src = peaks()
    exc = b2.CudaExecutor(local)
    g = 128
    comm = make_comm()
    A = DistCsr.stencil(exc, comm, "27pt", g, nz=g * world)
    nl, lo = A.n_local, A.lo
    nnz_l = A.a_own.nnz + (A.a_ghost.nnz if A.a_ghost is not None else 0)
    # x ~ N(0,1): this rank's slice of one global seeded vector (per-plane seeds)
    xh = np.random.default_rng(rank).standard_normal(nl)
    y = torch.empty(nl, dtype=torch.float64, device=exc.device)
    timer = Timer(exc)
    peer = A.peer(torch.float64)  # collective: peer-memory halo when every pair of GPUs has P2P access
    if peer is not None:
        # put / owned SpMV / wait / ghost SpMV / ack: kernels only, one CUDA graph per step
        xext = peer.pext
        xext[:nl].copy_(torch.from_numpy(xh))
        peer.apply_spmv(y, exc.stream)  # eager once (plans, workspaces)
        torch.cuda.synchronize()
        barrier(world)
        graph = torch.cuda.CUDAGraph()
        l0 = _lib.launch_count()
        with torch.cuda.graph(graph, capture_error_mode="relaxed"):
            peer.apply_spmv(y, exc.stream)
        per_step_launches = _lib.launch_count() - l0  # kernels in the graph (replays bypass the counter)
        step = graph.replay
        halo = "peer memory (CUDA IPC over NVLink), CUDA graph per step"
    else:
        xext = torch.zeros(A.n_ext, dtype=torch.float64, device=exc.device)
        xext[:nl].copy_(torch.from_numpy(xh))
        step = lambda: A.apply_ext(xext, y)  # noqa: E731
        halo = "NCCL send/recv" if BACKEND == "nccl" else "gloo (host-staged)"
        per_step_launches = None
    # algorithmic bytes of this rank's rows (Csr formula) + the ghost x values it reads
    by = bytes_csr(nl, nnz_l, 8) + (A.n_ext - nl) * 8
    with ClockSampler(local) as clk:
        for _ in range(args.warmup):
            step()
        barrier(world)
        torch.cuda.synchronize()
        launches0 = _lib.launch_count()
        ms = timer.run(step, args.steps, 0)
        launches = _lib.launch_count() - launches0
        if per_step_launches is not None:
            launches = per_step_launches * args.steps
    barrier(world)
    t_step = allmax(world, statistics.mean(ms) * 1e-3)
    total_bytes = allsum(world, by)
    # the owned-block SpMV alone (no exchange): the kernel's roofline
    own_x = b2.Dense.wrap(exc, xext[:nl].view(-1, 1))
    own_y = b2.Dense.wrap(exc, y.view(-1, 1))
    ms_own = timer.run(lambda: A.a_own.apply(own_x, own_y), max(5, min(args.steps, 20)), 3)
    t_own = allmax(world, statistics.mean(ms_own) * 1e-3)
    by_own = bytes_csr(nl, A.a_own.nnz, 8)
    # e2e: pinned host x slice up, distributed SpMV, y slice down, every step
    xpin = torch.from_numpy(xh).pin_memory()
    ypin = torch.empty(nl, dtype=torch.float64).pin_memory()

    def e2e_step():
        xext[:nl].copy_(xpin, non_blocking=True)
        A.apply_ext(xext, y)
        ypin.copy_(y, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    for _ in range(2):
        e2e_step()
    barrier(world)
    e2e_t = []
    for _ in range(max(3, min(args.steps, 20))):
        t0 = time.perf_counter()
        e2e_step()
        e2e_t.append(time.perf_counter() - t0)
    e2e_step_t = allmax(world, statistics.median(e2e_t))
    halo_bytes = (A.n_ext - nl) * 8
    return {
        "metric": METRIC, "value": round(total_bytes / t_step / 1e9, 1), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (device-generated 27-point stencil, x ~ N(0,1))",
        "config": {"workload": f"C2 distributed: Csr SpMV y = A x, 3-D 27-point stencil 128 x 128 x {128 * world} "
                               f"row-partitioned over {world} ranks (one 128^3 C2 slab = 2,097,152 rows per rank), "
                               "fp64 values / int32 indices",
                   "format": "csr", "rows": nl * world, "rows_per_rank": nl,
                   "parallelism": f"row partition x{world} ({BACKEND}"
                                  f"{', ranks share GPUs' if BACKEND == 'gloo' else ''})",
                   "halo_bytes_per_rank": halo_bytes, "halo": halo,
                   "l2": "inputs larger than L2 and L2 flushed (256 MiB write, then read back) between steps"},
        "gflops": round(2 * allsum(world, nnz_l) / t_step / 1e9, 1),
        "roofline": {"bound": "hbm", "achieved": round(by_own / t_own / 1e9, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(by_own / t_own / 1e9 / peak, 4), "traffic": traffic_from_profiles(
                         "csr_classical_kernel"), "peak_source": peak_src, "kernel": "csr_classical_kernel",
                     "bytes_per_launch": by_own, "note": "owned-block SpMV per rank, max over ranks"},
        "distributed": {"step_ms": round(t_step * 1e3, 4), "owned_spmv_ms": round(t_own * 1e3, 4),
                        "exchange_and_ghost_ms": round((t_step - t_own) * 1e3, 4),
                        "per_rank_frac_of_peak": round(by / t_step / 1e9 / peak, 4)},
        "cpu_baseline": None,
        "e2e": {"value": round(total_bytes / e2e_step_t / 1e9, 1), "unit": "GB/s",
                "h2d_bytes_per_step": nl * 8 * world, "d2h_bytes_per_step": nl * 8 * world,
                "ms_per_step": round(e2e_step_t * 1e3, 3)},
        "gpu_launches": int(launches), "clocks": clk.summary(),
    }


# ---------------------------------------------------------------------------
# reference arm: the reference's CPU algorithm on host cores
# ---------------------------------------------------------------------------
def bench_reference(args):
    from oracle import problems as P
    from oracle.cpu_baseline import ParallelCsr

    n, r, c, v = P.stencil3d(128, "27pt")
    rp, ci, vals = P.to_csr(n, r, c, v)
    del r, c, v
    ci = ci.astype(np.int32)
    b = np.random.default_rng(0).standard_normal((n, 1))
    op = ParallelCsr(rp, ci, vals)
    out = np.empty((n, 1))
    for _ in range(args.warmup):
        op.apply(b, out)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        op.apply(b, out)
        ts.append(time.perf_counter() - t0)
    t = statistics.mean(ts)
    by = bytes_csr(n, int(rp[-1]), 8)
    val = by / t / 1e9
    cores = len(op.blocks)
    op.close()
    return {
        "impl": "reference", "metric": METRIC, "value": round(val, 3), "unit": "GB/s", "n_gpus": 0,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (oracle-generated 27-point stencil, b ~ N(0,1) seed 0)",
        "config": {"workload": "C2: Csr SpMV x = A b, 3-D 27-point stencil 128^3 "
                               "(2,097,152 rows, 55,742,968 nnz), fp64 values / int32 indices",
                   "format": "csr", "rows": n, "nnz": int(rp[-1])},
        "cpu_baseline": {"value": round(val, 3), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": "full C2 matrix per step: reference ParallelExecutor + csr_row_sums "
                                   "restated (oracle/cpu_baseline.py)"},
        "e2e": {"value": round(val, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def c5_sub(args, world, rank, local, head):
    """C5 (3-D 7-point Poisson 512^3, CG to 1e-8) alongside the C2 line, so a
    plain `bench.py --gpus N` run also records the CG ms/iteration at N GPUs:
    single-GPU CG at N = 1, the row-partitioned NCCL CG (strong scaling,
    with the exposed-communication breakdown) at N > 1. Guarded: an error
    is reported in the sub-object, and a watchdog prints the C2 line and
    exits if the sub-measurement does not finish in time."""
    import types

    sub_args = types.SimpleNamespace(**vars(args))
    sub_args.steps, sub_args.warmup, sub_args.grid = 2, 3, args.grid or 512
    timer = threading.Timer(float(os.environ.get("B200SP_C5_TIMEOUT", "300")), _c5_watchdog,
                            args=(rank, head))
    timer.daemon = True
    timer.start()
    try:
        from bench_solvers import bench_c5_distributed, bench_solver

        if world > 1:
            r = bench_c5_distributed(sub_args, world, rank, local)
        else:
            r = bench_solver(sub_args, world, rank, local, "c5")
        keep = {"workload": r["config"]["workload"], "n_gpus": world, "ms_per_iter": r["value"],
                "iterations": r["config"]["iterations"], "converged": r["config"]["converged"],
                "scaling": "strong", "timed_solves": sub_args.steps}
        if "breakdown" in r["config"]:
            keep["breakdown"] = r["config"]["breakdown"]
            keep["halo"] = r["config"].get("halo")
        if r.get("roofline"):
            keep["frac_of_hbm_peak"] = r["roofline"]["frac"]
        if world > 1:
            keep.update(_c5_single_reference(sub_args, world, rank, local, r))
        return keep
    except Exception as e:  # noqa: BLE001 -- the C2 line must still be printed
        return {"error": f"{type(e).__name__}: {e}"[:300]}
    finally:
        timer.cancel()


def _c5_single_reference(sub_args, world, rank, local, r):
    """N > 1: the same C5 solve on ONE GPU inside the same job (rank 0,
    the other ranks wait), for the strong-scaling parallel efficiency
    t_1 / (N t_N), plus each rank's roofline fraction of the distributed
    iteration (fused-minimum CG bytes of its rows)."""
    import torch

    from bench_solvers import bench_solver

    t1 = its1 = None
    if rank == 0:
        one = bench_solver(sub_args, 1, 0, local, "c5")
        t1, its1 = one["value"], one["config"]["iterations"]
    torch.cuda.synchronize()
    barrier(world)
    t1 = allmax(world, t1 if t1 is not None else 0.0)
    tn = r["value"]
    g = sub_args.grid
    n, nnz = g ** 3, 7 * g ** 3 - 6 * g * g
    peak, _ = peaks()
    per_rank_bytes = (bytes_csr(n, nnz, 8) + 9 * n * 8) / world
    out = {"single_gpu_ms_per_iter": round(t1, 4), "parallel_efficiency": round(t1 / (world * tn), 4),
           "per_rank_frac_of_peak": round(per_rank_bytes / (tn * 1e-3) / 1e9 / peak, 4),
           "efficiency_note": "strong scaling of the fixed problem, t_1 measured in this job on rank 0's GPU"}
    if its1 is not None:
        out["single_gpu_iterations"] = its1
    if BACKEND == "gloo":
        out["efficiency_note"] += "; ranks SHARE GPUs here (gloo), so the efficiency is not a scaling figure"
    return out


def _c5_watchdog(rank, head):
    if rank == 0:
        head = dict(head)
        head["c5_cg"] = {"error": "timeout"}
        print(json.dumps(head), flush=True)
    os._exit(0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--grid", type=int, default=0, help="override the stencil grid of c4/c5")
    ap.add_argument("--no-c5", action="store_true",
                    help="c2 only: skip the C5 CG sub-measurement (distributed at N > 1)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl != "reference":
        self_launch(args)

    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        if rank != 0:
            return
        print(json.dumps(bench_reference(args)))
        return

    world, rank, local = dist_setup()
    if args.workload == "c2":
        out = bench_c2(args, world, rank, local) if world == 1 else bench_c2_dist(args, world, rank, local)
        if not args.no_c5:
            out["c5_cg"] = c5_sub(args, world, rank, local, out)
    else:
        from bench_solvers import bench_workload  # solver workloads

        out = bench_workload(args, world, rank, local)
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
