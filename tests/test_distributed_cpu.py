"""Multi-rank host logic on CPU: world_size-2 gloo process group.

Partition (plane-aligned row blocks), ghost discovery, the halo plan learned
via all_gather, the point-to-point exchange protocol (Comm.exchange) and the
all-reduce used by the distributed CG -- checked against the global oracle
SpMV of a 3-D stencil. No GPU needed (gloo, CPU tensors).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, g, kind, result_dir):
    import sys

    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, repo)
    import torch.distributed as dist

    from oracle import problems as P
    from oracle import spmv as OS
    from paper_2006_16852_b200.distributed import Comm, Partition, plan_halo

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        n, r, c, v = P.stencil3d(g, kind)
        rp, ci, vals = P.to_csr(n, r, c, v)
        xg = np.random.default_rng(0).standard_normal(n)
        yg = OS.csr_spmv(rp, ci, vals, xg[:, None])[:, 0]
        part = Partition(n, world, align=g * g)
        lo, hi = part.range(rank)
        comm = Comm()
        # local rows (global columns), ghost columns
        e0, e1 = rp[lo], rp[hi]
        lrp, lci, lv = rp[lo:hi + 1] - e0, ci[e0:e1], vals[e0:e1]
        ghosts = np.unique(lci[(lci < lo) | (lci >= hi)])
        plan = plan_halo(rank, part, ghosts, comm)
        nl = hi - lo
        # exchange the halo of x with CPU tensors
        ext = torch.zeros(nl + ghosts.size, dtype=torch.float64)
        ext[:nl] = torch.from_numpy(xg[lo:hi])
        sends = [(peer, ext[torch.from_numpy(idx)].clone()) for peer, idx in plan.send]
        recvs = [(peer, ext[nl + g0:nl + g1]) for peer, g0, g1 in plan.recv]
        comm.exchange(sends, recvs).wait()
        got = ext.numpy()
        assert np.array_equal(got[nl:], xg[ghosts]), "ghost values"
        # local SpMV on the renumbered columns equals the global rows
        mapped = np.where((lci >= lo) & (lci < hi), lci - lo, nl + np.searchsorted(ghosts, lci))
        yl = OS.csr_spmv(lrp, mapped, lv, got[:, None])[:, 0]
        assert np.array_equal(yl, yg[lo:hi]), "distributed SpMV"
        # the CG reductions: all-reduce of local partial sums
        t = torch.tensor([float(np.dot(yl, yl)), 1.0], dtype=torch.float64)
        comm.allreduce_(t)
        assert np.isclose(t[0].item(), float(np.dot(yg, yg)), rtol=1e-12) and t[1].item() == world
        # plane alignment and full coverage
        assert lo % (g * g) == 0 and part.offsets[-1] == n
        with open(os.path.join(result_dir, f"ok{rank}"), "w") as f:
            f.write(f"{lo} {hi} {ghosts.size} {len(plan.send)}")
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,g", [("7pt", 6), ("27pt", 5)])
def test_two_rank_halo_and_spmv(tmp_path, kind, g):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, g, kind, str(tmp_path)), nprocs=2, join=True)
    for rank in range(2):
        lo, hi, ng, nsend = map(int, (tmp_path / f"ok{rank}").read_text().split())
        assert ng == (g * g if kind == "7pt" else g * g) and nsend == 1


def test_partition_alignment_and_owner():
    from paper_2006_16852_b200.distributed import Partition

    p = Partition(512 ** 3, 8, align=512 * 512)
    assert list(p.offsets) == [k * 64 * 512 * 512 for k in range(9)]
    assert list(p.owner([0, 64 * 512 * 512 - 1, 64 * 512 * 512, 512 ** 3 - 1])) == [0, 0, 1, 7]
    q = Partition(10, 3)
    assert q.offsets[0] == 0 and q.offsets[-1] == 10 and np.all(np.diff(q.offsets) >= 3)


def test_peer_halo_eligibility(monkeypatch):
    """The peer-memory halo is used for row-range sends with few neighbours,
    automatically only under NCCL (gloo needs B200SP_PEER_HALO=1)."""
    import types

    import numpy as np

    from paper_2006_16852_b200 import config
    from paper_2006_16852_b200.distributed import HaloPlan, PeerHalo

    def fake(backend, sends, nrecv=2, size=3):
        dist = types.SimpleNamespace(get_backend=lambda group=None: backend)
        comm = types.SimpleNamespace(dist=dist, group=None, size=size, rank=1)
        plan = HaloPlan([(p, 0, 4) for p in range(nrecv)], [], 10, 8)
        return types.SimpleNamespace(comm=comm, plan=plan, _send=sends)

    ranges = [(0, 0, 4, None, None), (2, 6, 10, None, None)]
    indexed = [(0, 0, 0, np.arange(3), None)]
    monkeypatch.setattr(config, "PEER_HALO", "auto")
    assert PeerHalo.usable(fake("nccl", ranges))
    assert not PeerHalo.usable(fake("gloo", ranges))
    assert not PeerHalo.usable(fake("nccl", indexed))
    assert not PeerHalo.usable(fake("nccl", ranges * 3))  # more puts than b200sp_peer_max()
    assert not PeerHalo.usable(fake("nccl", ranges, size=1))
    monkeypatch.setattr(config, "PEER_HALO", "1")
    assert PeerHalo.usable(fake("gloo", ranges))
    monkeypatch.setattr(config, "PEER_HALO", "0")
    assert not PeerHalo.usable(fake("nccl", ranges))
