"""Row-partitioned CG on the device with 2 ranks sharing one GPU (gloo with
host staging stands in for NCCL, which needs one GPU per rank): the
distributed solve must reproduce the single-GPU CG iteration count (+-1)
and solution, and DistCsr must reproduce the global SpMV."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, g, out_dir, halo="0"):
    import sys

    os.environ["B200SP_PEER_HALO"] = halo  # read at package import

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    import torch
    import torch.distributed as dist

    import paper_2006_16852_b200 as b2
    from oracle import problems as P
    from oracle import spmv as OS
    from paper_2006_16852_b200.distributed import DistCg, DistCsr, StagedComm

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        exc = b2.CudaExecutor(0)
        comm = StagedComm()
        A = DistCsr.stencil(exc, comm, "7pt", g)
        lo, hi = A.lo, A.hi
        n = g ** 3
        # SpMV vs the oracle
        xg = np.random.default_rng(1).standard_normal(n)
        nn, r, c, v = P.stencil3d(g, "7pt")
        rp, ci, vals = P.to_csr(nn, r, c, v)
        yg = OS.csr_spmv(rp, ci, vals, xg[:, None])[:, 0]
        ext = torch.zeros(A.n_ext, dtype=torch.float64, device=exc.device)
        ext[:A.n_local] = torch.from_numpy(xg[lo:hi]).to(exc.device)
        y = torch.zeros(A.n_local, dtype=torch.float64, device=exc.device)
        A.apply_ext(ext, y)
        err = OS.rel_error_inf(y.cpu().numpy(), yg[lo:hi])
        # the public apply on this rank's slices: the peer-memory halo (put /
        # wait / ack kernels) when halo == "1"; repeated so the ack-gated reuse
        # of the ghost slots runs, with a different x each time
        for rep in range(3):
            xr = xg * (rep + 1.0)
            xd = b2.Dense.wrap(exc, torch.from_numpy(xr[lo:hi].copy()).to(exc.device).view(-1, 1))
            yd = b2.Dense.zeros(exc, A.n_local, 1)
            A.apply(xd, yd)
            err = max(err, OS.rel_error_inf(np.asarray(yd.data)[:, 0], (rep + 1.0) * yg[lo:hi]))
        # distributed CG
        b = torch.ones(A.n_local, dtype=torch.float64, device=exc.device)
        x = torch.zeros(A.n_local, dtype=torch.float64, device=exc.device)
        solver = DistCg(A, [b2.Iteration(1000), b2.ResidualNormReduction(1e-8)], batch=8)
        st = solver.solve(b, x)
        np.save(os.path.join(out_dir, f"x{rank}.npy"), x.cpu().numpy())
        x2 = torch.zeros(A.n_local, dtype=torch.float64, device=exc.device)
        st2 = solver.solve(b, x2)  # again: the peer buffers, flags and epochs are reused
        same = bool(torch.equal(x, x2)) and st2.iterations == st.iterations
        with open(os.path.join(out_dir, f"st{rank}"), "w") as f:
            f.write(f"{lo} {hi} {st.iterations} {int(st.converged)} {err} {solver.halo}/{solver.reduce} {int(same)}")
        # the reference factory path on the partitioned matrix (row N1):
        # Cg(exc, criteria, preconditioner=Jacobi(32)).generate(DistCsr)
        for tag, pre in (("none", None), ("bj32", b2.Jacobi(exc, block_size=32))):
            crit = [b2.Iteration(1000), b2.ResidualNormReduction(1e-8), b2.TimeLimit(3600.0)]
            fs = b2.Cg(exc, criteria=crit, preconditioner=pre).generate(A)
            rec = b2.RecordLogger()
            fs.attach(rec)
            xf = b2.Dense.zeros(exc, A.n_local, 1)
            fs.apply(b2.Dense.wrap(exc, b.view(-1, 1)), xf)
            stf = fs.last_status
            np.save(os.path.join(out_dir, f"xf_{tag}{rank}.npy"), np.asarray(xf.data)[:, 0])
            n_it = len(rec.query(b2.EventKind.ITERATION_COMPLETE))
            with open(os.path.join(out_dir, f"stf_{tag}{rank}"), "w") as f:
                f.write(f"{stf.iterations} {int(stf.converged)} {stf.stopping_id} {n_it}")
        # solvers without a partitioned variant refuse the DistCsr at generate time
        try:
            b2.Bicgstab(exc, criteria=[b2.Iteration(5)]).generate(A)
            refused = 0
        except b2.Unsupported:
            refused = 1
        assert refused == 1
        # TimeLimit consensus: every rank stops at the same iteration, by the time child
        ft = b2.Cg(exc, criteria=[b2.Iteration(10**6), b2.ResidualNormReduction(1e-300), b2.TimeLimit(0.005)])
        ts = ft.generate(A)
        xt = b2.Dense.zeros(exc, A.n_local, 1)
        ts.apply(b2.Dense.wrap(exc, b.view(-1, 1)), xt)
        with open(os.path.join(out_dir, f"stt{rank}"), "w") as f:
            f.write(f"{ts.last_status.iterations} {ts.last_status.stopping_id}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,halo", [(2, "0"), (2, "1"), (3, "1")], ids=["2rank-staged", "2rank-peer", "3rank-peer"])
def test_multi_rank_cg_matches_single_gpu(tmp_path, cuda, world, halo):
    """halo "1": the ghosts travel by peer stores fused into the p update
    (CUDA IPC between the ranks' processes; with one GPU they map the same
    device) and the ghost SpMV waits on the flags -- the NVLink path of a
    multi-GPU run, minus the link."""
    import paper_2006_16852_b200 as b2
    from paper_2006_16852_b200 import problems

    g = 16
    port = _free_port()
    mp.spawn(_worker, args=(world, port, g, str(tmp_path), halo), nprocs=world, join=True)
    parts, its = [], set()
    for rank in range(world):
        lo, hi, it, conv, err, used, same = (tmp_path / f"st{rank}").read_text().split()
        assert float(err) <= 1e-14
        assert int(conv) == 1
        assert used == ("peer/peer" if halo == "1" else "nccl/nccl")
        assert int(same) == 1
        its.add(int(it))
        parts.append(np.load(tmp_path / f"x{rank}.npy"))
    assert len(its) == 1  # every rank took the same decisions
    a = problems.stencil(cuda, "7pt", g)
    x1 = b2.Dense.zeros(cuda, g ** 3, 1)
    s = b2.Cg(cuda, criteria=[b2.Iteration(1000), b2.ResidualNormReduction(1e-8)]).generate(a)
    s.apply(b2.Dense(cuda, np.ones((g ** 3, 1))), x1)
    assert abs(its.pop() - s.last_status.iterations) <= 1
    xd = np.concatenate(parts)
    x1 = np.asarray(x1.data)[:, 0]
    assert np.linalg.norm(xd - x1) <= 1e-7 * np.linalg.norm(x1)
    # the factory path against the REFERENCE's own runs (tests/golden/solvers.npz:
    # cg_7pt_g16 / cg_bj32_7pt_g16, made by tests/golden/make_golden.py)
    from conftest import load_golden

    gold = load_golden("solvers.npz")
    for tag, key in (("none", "cg_7pt_g16"), ("bj32", "cg_bj32_7pt_g16")):
        ref = gold[key]
        stats = [(tmp_path / f"stf_{tag}{rank}").read_text().split() for rank in range(world)]
        assert len({st_[0] for st_ in stats}) == 1
        it, conv, sid, n_it = map(int, stats[0])
        assert conv == 1 and sid == int(ref["stopping_id"]) == 2
        assert abs(it - int(ref["iterations"])) <= 1, (tag, it, int(ref["iterations"]))
        assert n_it == it  # ITERATION_COMPLETE events replayed from the device history
        xf = np.concatenate([np.load(tmp_path / f"xf_{tag}{rank}.npy") for rank in range(world)])
        xr = ref["x"][:, 0]
        assert np.linalg.norm(xf - xr) <= 1e-7 * np.linalg.norm(xr), tag
    stt = [(tmp_path / f"stt{rank}").read_text().split() for rank in range(world)]
    assert len({st_[0] for st_ in stt}) == 1  # same stop iteration on every rank
    assert all(int(st_[1]) == 3 for st_ in stt)  # stopped by the TimeLimit child
