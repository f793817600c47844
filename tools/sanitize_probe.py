"""Exercise every kernel family of libb200sp.so at small sizes, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_probe.py [--part spmv|solvers|misc|dist]

Each part checks its results against the oracle / a direct solve, so a run
that the sanitizer passes is also a correct run. `--part dist` spawns two
ranks sharing device 0 (gloo + the peer-memory halo and all-reduce through
CUDA IPC); run it with `--target-processes all`.
"""

from __future__ import annotations

import argparse
import os
import socket
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def spmv(b2, exc):
    from oracle import problems as P
    from oracle import spmv as OS
    from paper_2006_16852_b200 import problems

    cases = [("27pt", problems.stencil(exc, "27pt", 12), P.stencil3d(12, "27pt")),
             ("powerlaw", problems.power_law(exc, 5000, seed=3, max_len=900), P.power_law(5000, seed=3, max_len=900))]
    for name, a, (n, r, c, v) in cases:
        rp, ci, vals = P.to_csr(n, r, c, v)
        bv = np.random.default_rng(0).standard_normal((n, 1))
        ref = OS.csr_spmv(rp, ci, vals, bv)
        for dt in ("float64", "float32"):
            base = a if dt == "float64" else b2.convert(a, "csr")
            if dt == "float32":
                base = b2.Csr.from_data(exc, a.to_data(), value_dtype="float32")
            b = b2.Dense(exc, bv, value_dtype=dt)
            for fmt in ("csr_classical", "csr_lb", "csr_stream", "csr_pipe", "coo", "ell", "sellp", "hybrid"):
                m = b2.convert(base, fmt)
                modes = [None]
                if fmt == "csr_lb":
                    modes = [2, 3]
                for mode in modes:
                    if mode is not None:
                        m.set_strategy("load_balance", lb_mode=mode)
                        m._plan = None
                    x = b2.Dense.zeros(exc, n, 1, value_dtype=dt)
                    m.apply(b, x)
                    tol = 1e-13 if dt == "float64" else 1e-5
                    err = OS.rel_error_inf(np.asarray(x.data, dtype=np.float64), ref)
                    assert err <= tol, (name, dt, fmt, mode, err)
                    x0 = b2.Dense(exc, np.ones((n, 1)), value_dtype=dt)
                    m.apply_advanced(0.5, b, -1.0, x0)  # alpha/beta + x_in path
            print(f"spmv {name} {dt} ok", flush=True)


def solvers(b2, exc):
    from paper_2006_16852_b200 import problems

    crit = [b2.Iteration(400), b2.ResidualNormReduction(1e-8)]
    for kind, g in (("7pt", 10), ("convdiff", 14)):
        a = problems.stencil(exc, kind, g)
        n = a.size.rows
        dense = a.to_data().to_dense_array()
        bv = np.ones((n, 1))
        for name in (("cg", "fcg") if kind == "7pt" else ("bicgstab", "cgs", "gmres")):
            for pre in (None, 32, 64):
                kw = {"krylov_dim": 30} if name == "gmres" else {}
                p = b2.Jacobi(exc, block_size=pre) if pre else None
                s = b2.SOLVER_FACTORIES[name](exc, criteria=crit, preconditioner=p, **kw).generate(a)
                x = b2.Dense.zeros(exc, n, 1)
                s.apply(b2.Dense(exc, bv), x)
                res = np.linalg.norm(bv[:, 0] - dense @ np.asarray(x.data)[:, 0]) / np.linalg.norm(bv)
                assert s.last_status.converged and res < 1e-7, (name, pre, s.last_status, res)
                print(f"solver {name} {kind} pre={pre} it={s.last_status.iterations} ok", flush=True)
    # GMRES at <= 2048 rows: the single-block Arnoldi step (with block-Jacobi)
    # and the whole-cycle single-block kernel (unpreconditioned, basis on chip)
    a = problems.stencil(exc, "convdiff", 10)
    for pre in (None, 32):
        s = b2.Gmres(exc, criteria=crit, krylov_dim=25,
                     preconditioner=b2.Jacobi(exc, block_size=pre) if pre else None).generate(a)
        x = b2.Dense.zeros(exc, a.size.rows, 1)
        s.apply(b2.Dense(exc, np.ones((a.size.rows, 1))), x)
        assert s.last_status.converged, s.last_status
    a = problems.stencil(exc, "convdiff", 4)  # 64 rows: the one-warp on-chip cycle
    s = b2.Gmres(exc, criteria=crit, krylov_dim=10).generate(a)
    x = b2.Dense.zeros(exc, 64, 1)
    s.apply(b2.Dense(exc, np.ones((64, 1))), x)
    assert s.last_status.converged
        # GMRES above the single-block limit (batched Arnoldi kernels) and CG above the cooperative limit
    a = problems.stencil(exc, "convdiff", 24)
    s = b2.Gmres(exc, criteria=crit, krylov_dim=20).generate(a)
    x = b2.Dense.zeros(exc, a.size.rows, 1)
    s.apply(b2.Dense(exc, np.ones((a.size.rows, 1))), x)
    assert s.last_status.converged
    from paper_2006_16852_b200 import config

    old = config.CG_COOP_MAX_ROWS
    config.CG_COOP_MAX_ROWS = 0
    try:
        a = problems.stencil(exc, "7pt", 12)
        s = b2.Cg(exc, criteria=crit).generate(a)
        x = b2.Dense.zeros(exc, a.size.rows, 1)
        s.apply(b2.Dense(exc, np.ones((a.size.rows, 1))), x)
        assert s.last_status.converged
    finally:
        config.CG_COOP_MAX_ROWS = old
    # ILU + triangular solves, Ir, multi-column host loop
    a = problems.stencil(exc, "convdiff", 8)
    s = b2.Bicgstab(exc, criteria=crit, preconditioner=b2.Ilu(exc)).generate(a)
    x = b2.Dense.zeros(exc, a.size.rows, 1)
    s.apply(b2.Dense(exc, np.ones((a.size.rows, 1))), x)
    assert s.last_status.converged
    s = b2.Ir(exc, criteria=crit, inner=b2.Jacobi(exc, block_size=16)).generate(a)
    x = b2.Dense.zeros(exc, a.size.rows, 1)
    s.apply(b2.Dense(exc, np.ones((a.size.rows, 1))), x)
    s = b2.Cg(exc, criteria=crit).generate(problems.stencil(exc, "7pt", 6))
    x = b2.Dense.zeros(exc, 216, 2)
    s.apply(b2.Dense(exc, np.ones((216, 2))), x)
    assert s.last_status.converged
    print("solvers ok", flush=True)


def misc(b2, exc):
    from paper_2006_16852_b200.formats import assemble_device

    rng = np.random.default_rng(3)
    r = rng.integers(0, 300, 20000)
    c = rng.integers(0, 200, 20000)
    v = rng.standard_normal(20000)
    d = b2.MatrixData((300, 200), r, c, v)
    ro, co, vo = assemble_device(exc, d, np.float64)
    ref = d.canonicalize()
    assert np.array_equal(ro.cpu().numpy(), ref.rows) and np.array_equal(vo.cpu().numpy(), ref.vals)
    import io

    text = "%%MatrixMarket matrix coordinate real general\n3 3 4\n1 1 2.0\n2 2 3.0\n3 1 -1.0\n3 3 4.0\n"
    md = b2.read_matrix_market(io.StringIO(text))  # native parser (csrc/mmio.cu) + device assembly
    assert b2.matrix_from_data(exc, md, "csr").nnz == 4
    x = b2.Dense(exc, rng.standard_normal((50, 3)))
    y = b2.Dense(exc, rng.standard_normal((50, 3)))
    x.dot(y)
    x.norm2()
    y.add_scaled(0.5, x)
    y.scale(2.0)
    print("misc ok", flush=True)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _dist_worker(rank, world, port):
    os.environ["B200SP_PEER_HALO"] = "1"
    import torch
    import torch.distributed as dist

    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200.distributed import DistCsr, StagedComm

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        exc = b2.CudaExecutor(0)
        A = DistCsr.stencil(exc, StagedComm(), "7pt", 8)
        s = b2.Cg(exc, criteria=[b2.Iteration(200), b2.ResidualNormReduction(1e-8)]).generate(A)
        x = b2.Dense.zeros(exc, A.n_local, 1)
        s.apply(b2.Dense.wrap(exc, torch.ones((A.n_local, 1), dtype=torch.float64, device=exc.device)), x)
        assert s.last_status.converged, s.last_status
        print(f"dist rank {rank} it={s.last_status.iterations} ok", flush=True)
    finally:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", default="spmv,solvers,misc")
    args = ap.parse_args()
    parts = args.part.split(",")
    if "dist" in parts:
        import torch.multiprocessing as mp

        mp.spawn(_dist_worker, args=(2, _free_port()), nprocs=2, join=True)
        parts.remove("dist")
    if not parts:
        return
    import paper_2006_16852_b200 as b2

    exc = b2.CudaExecutor(0)
    for p in parts:
        {"spmv": spmv, "solvers": solvers, "misc": misc}[p](b2, exc)


if __name__ == "__main__":
    main()
