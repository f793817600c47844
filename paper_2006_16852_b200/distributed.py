"""Row-partitioned distributed matrix and CG (one process per GPU).

The reference has no distributed executor (cross-process memory
is a non-goal; its only parallelism is ParallelExecutor's contiguous row
blocks, src/executor.py:181-190). This module scales that same decomposition
across GPUs:

* ``Partition``  -- contiguous row blocks (plane-aligned for 3-D grids).
* ``plan_halo``  -- ghost columns grouped by owning rank; the send lists are
  learned with one all_gather of the (small) per-peer ghost requests.
* ``DistCsr``    -- the rank's rows with columns renumbered to the local
  vector layout [owned | ghosts], split into A_own and A_ghost so the
  interior product overlaps the halo exchange:
      halo(p) on the NCCL stream  ||  q = A_own p_own   (compute stream)
      wait;  q += A_ghost p_ghost
* ``DistCg``     -- the device-resident CG kernels with the reductions split
  as local sum -> NCCL all-reduce (8-16 bytes) -> control step, two
  all-reduces per iteration (sigma = p.q; rho = r.z with ||r||).
* ``PeerHalo``   -- the halo as peer-memory stores fused into the step that
  produces p (CUDA IPC over NVLink/NVSwitch), used instead of NCCL
  send/recv when the partition allows it.
Communication goes through ``Comm`` (torch.distributed; NCCL over
NVLink/NVSwitch in production, gloo for the CPU tests).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib, config
from .base import Dim2, LinOp
from .executor import ptr
from .formats import Csr, Dense, _scan
from .problems import STENCILS
from .solvers.common import BreakdownInfo, SolveStatus
from .stop import Combined


# ---------------------------------------------------------------------------
# partition + communication (host logic, CPU-testable)
# ---------------------------------------------------------------------------
class Partition:
    """Contiguous row blocks of n rows over ``size`` ranks, boundaries rounded
    to multiples of ``align`` (a grid plane) where possible."""

    def __init__(self, n, size, align=1):
        self.n, self.size = int(n), int(size)
        units = -(-self.n // align)
        cuts = [min(self.n, (units * p // self.size) * align) for p in range(self.size + 1)]
        cuts[-1] = self.n
        self.offsets = np.asarray(cuts, dtype=np.int64)

    def range(self, rank):
        return int(self.offsets[rank]), int(self.offsets[rank + 1])

    def owner(self, cols):
        return np.searchsorted(self.offsets, np.asarray(cols, dtype=np.int64), side="right") - 1


class Comm:
    """Collectives over torch.distributed (the default process group)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce_(self, t):
        self.dist.all_reduce(t, group=self.group)

    def allgather_object(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return out

    def exchange(self, sends, recvs):
        """Start point-to-point transfers; returns a handle with wait()."""
        ops = [self.dist.P2POp(self.dist.isend, t, peer, self.group) for peer, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, t, peer, self.group) for peer, t in recvs]
        works = self.dist.batch_isend_irecv(ops) if ops else []
        return _Works(works)


class StagedComm(Comm):
    """Comm for backends without device tensors (gloo): stage through host
    memory. Used to test the multi-rank path with several processes sharing
    one GPU; production runs use NCCL directly."""

    def allreduce_(self, t):
        h = t.detach().cpu()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h.to(t.device))

    def exchange(self, sends, recvs):
        host_recv = [(peer, torch.empty(t.shape, dtype=t.dtype)) for peer, t in recvs]
        ops = [self.dist.P2POp(self.dist.isend, t.detach().cpu(), peer, self.group) for peer, t in sends]
        ops += [self.dist.P2POp(self.dist.irecv, h, peer, self.group) for peer, h in host_recv]
        for w in (self.dist.batch_isend_irecv(ops) if ops else []):
            w.wait()
        for (peer, h), (_, t) in zip(host_recv, recvs):
            t.copy_(h.to(t.device))
        return _Works([])


def make_comm(group=None):
    """Comm for the process group's backend: NCCL collectives on device
    tensors directly; gloo (ranks sharing a GPU, CPU tests) staged through
    host memory."""
    import torch.distributed as dist

    backend = str(dist.get_backend(group)).lower()
    return Comm(group) if backend == "nccl" else StagedComm(group)


class _Works:
    def __init__(self, works):
        self.works = works

    def wait(self):
        for w in self.works:
            w.wait()


class HaloPlan:
    """recv: [(peer, g0, g1)] ghost segments per owning peer (sorted ghosts);
    send: [(peer, local_idx)] owned rows each peer needs."""

    def __init__(self, recv, send, n_local, n_ghost):
        self.recv, self.send = recv, send
        self.n_local, self.n_ghost = n_local, n_ghost

    def send_is_range(self, idx):
        return idx.size > 0 and bool(np.all(np.diff(idx) == 1))


def plan_halo(rank, part, ghost_cols, comm):
    """Group sorted ghost columns by owner and learn the send lists."""
    ghost_cols = np.asarray(ghost_cols, dtype=np.int64)
    lo, hi = part.range(rank)
    owners = part.owner(ghost_cols)
    recv, requests = [], {}
    for q in np.unique(owners):
        q = int(q)
        seg = np.flatnonzero(owners == q)
        recv.append((q, int(seg[0]), int(seg[-1]) + 1))
        requests[q] = ghost_cols[seg]
    gathered = comm.allgather_object(requests)
    send = []
    for p, req in enumerate(gathered):
        if p != rank and rank in req:
            send.append((p, np.asarray(req[rank], dtype=np.int64) - lo))
    return HaloPlan(recv, send, hi - lo, ghost_cols.size)


# ---------------------------------------------------------------------------
# distributed matrix
# ---------------------------------------------------------------------------
class DistCsr(LinOp):
    """This rank's rows of a row-partitioned matrix (global size n x n)."""

    def __init__(self, exc, comm, part, a_own, a_ghost, plan):
        super().__init__(exc, Dim2(part.n, part.n))
        self.comm, self.part = comm, part
        self.a_own, self.a_ghost, self.plan = a_own, a_ghost, plan
        self.lo, self.hi = part.range(comm.rank)
        dev = exc.device
        self._send = []
        for peer, idx in plan.send:
            if plan.send_is_range(idx):
                self._send.append((peer, int(idx[0]), int(idx[-1]) + 1, None, None))
            else:
                it = torch.from_numpy(idx.astype(np.int32)).to(dev)
                self._send.append((peer, 0, 0, it, None))

    @property
    def n_local(self):
        return self.plan.n_local

    def _operand_rows(self):
        """apply(b, x) takes this rank's rows: (n_local, m) slices."""
        return self.n_local, self.n_local

    @property
    def n_ext(self):
        return self.plan.n_local + self.plan.n_ghost

    @classmethod
    def stencil(cls, exc, comm, kind, grid, value_dtype="float64", convection=0.4, strategy="automatic", nz=None):
        """Generate this rank's rows of a stencil matrix directly on its GPU.
        3-D kinds: ``nz`` planes of grid x grid (default: the grid^3 cube;
        nz = size * grid stacks one cube-sized slab per rank, weak scaling)."""
        code = STENCILS[kind]
        nz = int(nz or grid)
        n = grid * grid if code == 0 else grid * grid * nz
        plane = grid if code == 0 else grid * grid
        part = Partition(n, comm.size, align=plane)
        lo, hi = part.range(comm.rank)
        nl = hi - lo
        dev = exc.device
        lens = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
        _lib.call("stencil_lengths", code, grid, nz, lo, nl, ptr(lens), exc.stream)
        rp = _scan(exc, lens[:nl])
        nnz = int(rp[-1].item())
        vt = torch.float64 if np.dtype(value_dtype) == np.float64 else torch.float32
        ci = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        v = torch.empty(max(nnz, 1), dtype=vt, device=dev)
        _lib.call("stencil_fill_" + _lib.suffix(vt), code, grid, nz, float(convection), lo, nl, ptr(rp), ptr(ci),
                  ptr(v), exc.stream)
        return cls.from_local_rows(exc, comm, part, rp, ci[:nnz], v[:nnz], strategy)

    @classmethod
    def from_local_rows(cls, exc, comm, part, rp, ci, v, strategy="automatic"):
        """Local rows with GLOBAL column indices -> renumbered, split, planned."""
        lo, hi = part.range(comm.rank)
        nl, nnz = hi - lo, int(ci.numel())
        dev = exc.device
        # ghost columns: flag, compact (device), unique (host, small)
        flag = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
        _lib.call("flag_out_of_range", nnz, ptr(ci), lo, hi, ptr(flag), exc.stream)
        pos = _scan(exc, flag[:nnz])
        ng_all = int(pos[-1].item())
        gcols = torch.empty(max(ng_all, 1), dtype=torch.int32, device=dev)
        _lib.call("compact_cols", nnz, ptr(ci), ptr(flag), ptr(pos), ptr(gcols), exc.stream)
        ghosts = np.unique(gcols[:ng_all].cpu().numpy().astype(np.int64))
        plan = plan_halo(comm.rank, part, ghosts, comm)
        gdev = torch.from_numpy(ghosts.astype(np.int32)).to(dev)
        ci = ci.clone()
        _lib.call("map_cols", nnz, ptr(ci), lo, hi, ptr(gdev), ghosts.size, exc.stream)
        # split into owned / ghost column blocks
        llo = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
        lhi = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
        _lib.call("split_count", nl, ptr(rp), ptr(ci), nl, ptr(llo), ptr(lhi), exc.stream)
        rp_lo, rp_hi = _scan(exc, llo[:nl]), _scan(exc, lhi[:nl])
        n_lo, n_hi = int(rp_lo[-1].item()), int(rp_hi[-1].item())
        ci_lo = torch.empty(max(n_lo, 1), dtype=torch.int32, device=dev)
        ci_hi = torch.empty(max(n_hi, 1), dtype=torch.int32, device=dev)
        v_lo = torch.empty(max(n_lo, 1), dtype=v.dtype, device=dev)
        v_hi = torch.empty(max(n_hi, 1), dtype=v.dtype, device=dev)
        _lib.call("split_fill_" + _lib.suffix(v.dtype), nl, ptr(rp), ptr(ci), ptr(v), nl, ptr(rp_lo), ptr(rp_hi),
                  ptr(ci_lo), ptr(v_lo), ptr(ci_hi), ptr(v_hi), exc.stream)
        a_own = Csr._from_device(exc, Dim2(nl, nl), rp_lo, ci_lo[:n_lo], v_lo[:n_lo], strategy=strategy)
        a_gh = None
        if ghosts.size:
            a_gh = Csr._from_device(exc, Dim2(nl, ghosts.size), rp_hi, ci_hi[:n_hi], v_hi[:n_hi],
                                    strategy="classical")
        return cls(exc, comm, part, a_own, a_gh, plan)

    # -- halo + product ----------------------------------------------------
    def start_halo(self, xext):
        """Send owned values peers need, receive ghosts into xext[n_local:]."""
        nl = self.n_local
        sends = []
        for peer, a, b, idx, _ in self._send:
            if idx is None:
                sends.append((peer, xext[a:b]))
            else:
                buf = torch.empty(idx.numel(), dtype=xext.dtype, device=xext.device)
                _lib.call("gather_" + _lib.suffix(xext.dtype), idx.numel(), ptr(idx), ptr(xext), ptr(buf),
                          self.exec.stream)
                sends.append((peer, buf))
        recvs = [(peer, xext[nl + g0:nl + g1]) for peer, g0, g1 in self.plan.recv]
        return self.comm.exchange(sends, recvs)

    def apply_ext(self, xext, y, alpha=1.0, beta=None, y_in=None):
        """y = alpha * A x + beta * y_in with x = xext[:n_local] plus ghosts."""
        nl = self.n_local
        exc = self.exec
        work = self.start_halo(xext)
        xd = Dense.wrap(exc, xext[:nl].view(-1, 1))
        yd = Dense.wrap(exc, y.view(-1, 1))
        if y_in is None:
            self.a_own.apply(xd, yd) if alpha == 1.0 else self.a_own.apply_advanced(alpha, xd, 0.0, yd)
        else:
            from .kernels import SpmvOp

            exc.run(SpmvOp(self.a_own, xd, yd, alpha=alpha, beta=beta, x_in=Dense.wrap(exc, y_in.view(-1, 1))))
        work.wait()
        if self.a_ghost is not None:
            gd = Dense.wrap(exc, xext[nl:].view(-1, 1))
            self.a_ghost.apply_advanced(alpha, gd, 1.0, yd)

    def peer(self, dtype):
        """This matrix's peer-memory halo for ``dtype`` (built collectively on
        the first call of every rank), or None when the peer path is not
        usable: non-range sends, too many neighbours, B200SP_PEER_HALO=0, or a
        pair of devices without P2P access (then every rank falls back to NCCL,
        with a warning)."""
        if not PeerHalo.usable(self):
            return None
        if self.__dict__.get("_peer_ok") is None:
            ok, _ = peer_capable(self.comm, self.exec.device)  # collective, once per matrix
            self.__dict__["_peer_ok"] = ok
            if not ok:
                import warnings

                warnings.warn("distributed solve: peer access between the ranks' GPUs is unavailable; "
                              "falling back to NCCL send/recv halo and NCCL all-reduce", RuntimeWarning)
        if not self.__dict__["_peer_ok"]:
            return None
        cache = self.__dict__.setdefault("_peer_halo", {})
        if dtype not in cache:
            cache[dtype] = PeerHalo(self, dtype)
        return cache[dtype]

    def _apply_impl(self, b, x):
        if b.size.cols == 1:
            peer = self.peer(b.values.dtype)
            if peer is not None:  # halo through peer memory (kernels only)
                peer.pext[:self.n_local].copy_(b.values[:, 0])
                y = x.values[:, 0]
                yc = y if y.is_contiguous() else torch.empty_like(y)
                peer.apply_spmv(yc, self.exec.stream)
                if yc is not y:
                    y.copy_(yc)
                return
        ext = torch.empty(self.n_ext, dtype=b.values.dtype, device=self.exec.device)
        ext[:self.n_local].copy_(b.values[:, 0])
        self.apply_ext(ext, x.values[:, 0])


# ---------------------------------------------------------------------------
# halo through peer memory
# ---------------------------------------------------------------------------
def ipc_export(t):
    """(allocation handle bytes, byte offset) of a device tensor's storage,
    for peers to open with ipc_open (csrc/dist.cu: b200sp_ipc_export)."""
    buf = ctypes.create_string_buffer(int(_lib.query("ipc_handle_bytes")))
    off = ctypes.c_int64()
    _lib.call("ipc_export", t.data_ptr(), ctypes.addressof(buf), ctypes.addressof(off))
    return bytes(buf.raw), int(off.value)


def ipc_open(handle, offset):
    """Map a peer's exported buffer into THIS process's current device
    context (lazy peer access): returns (pointer, allocation base)."""
    buf = ctypes.create_string_buffer(handle, len(handle))
    p, base = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.call("ipc_open", ctypes.addressof(buf), int(offset), ctypes.addressof(p), ctypes.addressof(base))
    return int(p.value), int(base.value)


def _close_mapped(bases):
    """Unmap peer allocations opened with ipc_open (weakref finalizer)."""
    for base in bases:
        try:
            _lib.call("ipc_close", base)
        except Exception:  # noqa: BLE001 -- interpreter / context teardown
            pass
    bases.clear()


def peer_capable(comm, dev):
    """Collective: True on every rank when every rank can reach every other
    rank's device with loads/stores (cudaDeviceCanAccessPeer, then
    cudaDeviceEnablePeerAccess -- explicit, so a topology without P2P falls
    back to NCCL instead of faulting in a kernel). Ranks sharing one device
    always qualify."""
    devices = comm.allgather_object(int(dev.index if dev.index is not None else torch.cuda.current_device()))
    ok = True
    can = ctypes.c_int32()
    for j, d in enumerate(devices):
        if j == comm.rank:
            continue
        _lib.call("peer_enable", d, ctypes.addressof(can))
        ok = ok and bool(can.value)
    return all(comm.allgather_object(ok)), devices


class PeerHalo:
    """The halo exchange as peer-memory stores fused into the CG step that
    produces the values (b200sp_cg_step1_put): every rank exports its
    extended vector [owned | ghosts] and a flag array through CUDA IPC (one
    all_gather of the handles), opens the buffers of the ranks it sends to
    in its own device context (peer access over NVLink / NVSwitch enabled
    explicitly first, see peer_capable), and then
    writes its boundary rows straight into their ghost slots while updating
    p, raising its flag in their flag arrays when the kernel's stores are
    out. The receiver orders its ghost SpMV after b200sp_peer_wait on the
    flags of the ranks it receives from. No NCCL call, no pack/unpack.

    Valid when every send is a row range (slab partitions) and at most
    b200sp_peer_max() peers are involved; the iteration's all-reduces order
    the reuse of the ghost slots from one exchange to the next."""

    def __init__(self, A, dtype):
        comm, exc = A.comm, A.exec
        dev = exc.device
        self.A = A
        self.pext = torch.zeros(A.n_ext, dtype=dtype, device=dev)
        w = max(comm.size, 1)
        self.flags = torch.zeros(w, dtype=torch.int32, device=dev)
        # the plain SpMV's own flags / acks (apply_spmv): [sources' flags | destinations' acks]
        self.flags_x = torch.zeros(2 * w, dtype=torch.int32, device=dev)
        self.ticket = torch.zeros(1, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        mine = {"pext": ipc_export(self.pext), "flags": ipc_export(self.flags), "flags_x": ipc_export(self.flags_x),
                "nl": A.n_local, "g0": {int(peer): int(g0) for peer, g0, _ in A.plan.recv}}
        every = comm.allgather_object(mine)
        self._bases = []  # mapped peer allocations (closed with the object)
        lo, hi, dst, flg, flg_x = [], [], [], [], []
        esz = self.pext.element_size()
        for peer, a, b, idx, _ in A._send:
            info = every[peer]
            rp_, b0 = ipc_open(*info["pext"])
            rf, b1 = ipc_open(*info["flags"])
            rx, b2 = ipc_open(*info["flags_x"])
            self._bases += [b0, b1, b2]
            g0 = info["g0"][comm.rank]
            lo.append(a)
            hi.append(b)
            dst.append(rp_ + (info["nl"] + g0) * esz)
            flg.append(rf + 4 * comm.rank)
            flg_x.append(rx + 4 * comm.rank)
        # plain-SpMV acks: a source's ack array gets this rank's ack at [w + rank];
        # before a put this rank waits on its own [w + destination] entries
        ack_out = []
        for peer, _, _ in A.plan.recv:
            rx, bx = ipc_open(*every[int(peer)]["flags_x"])
            self._bases.append(bx)
            ack_out.append(rx + 4 * (w + comm.rank))
        ack_in = [self.flags_x.data_ptr() + 4 * (w + int(peer)) for peer, _, _, _, _ in A._send]
        waits_x = [self.flags_x.data_ptr() + 4 * int(peer) for peer, _, _ in A.plan.recv]
        self.flag_x = (ctypes.c_void_p * max(len(flg_x), 1))(*flg_x)
        self.ack_in = (ctypes.c_void_p * max(len(ack_in), 1))(*ack_in)
        self.ack_out = (ctypes.c_void_p * max(len(ack_out), 1))(*ack_out)
        self.waits_x = (ctypes.c_void_p * max(len(waits_x), 1))(*waits_x)
        self.nack_in, self.nack_out = len(ack_in), len(ack_out)
        self.epoch_x = torch.zeros(1, dtype=torch.int32, device=dev)
        import weakref

        weakref.finalize(self, _close_mapped, self._bases)
        k = len(lo)
        self.nput = k
        self.lo = (ctypes.c_int64 * max(k, 1))(*lo)
        self.hi = (ctypes.c_int64 * max(k, 1))(*hi)
        self.dst = (ctypes.c_void_p * max(k, 1))(*dst)
        self.flag = (ctypes.c_void_p * max(k, 1))(*flg)
        waits = [self.flags.data_ptr() + 4 * int(peer) for peer, _, _ in A.plan.recv]
        self.nwait = len(waits)
        self.waits = (ctypes.c_void_p * max(self.nwait, 1))(*waits)
        # the halo epoch lives on the device: the put kernel advances it, so a
        # captured CUDA graph of the iteration replays with fresh epochs
        self.epoch_dev = torch.zeros(1, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)

    @staticmethod
    def usable(A):
        """Every send a row range, few enough peers, mode allows it."""
        mode = config.PEER_HALO
        if mode == "0" or A.comm.size < 2:
            return False
        if mode != "1" and str(A.comm.dist.get_backend(A.comm.group)).lower() != "nccl":
            return False
        pmax = int(_lib.query("peer_max"))
        ranges = all(idx is None for _, _, _, idx, _ in A._send)
        return ranges and len(A._send) <= pmax and len(A.plan.recv) <= 2 * pmax

    def step1(self, nl, p, z, ctl, suf, stream):
        """p = z + beta p, boundary rows stored into the peers' ghost slots."""
        _lib.call("cg_step1_put_" + suf, nl, ptr(p), ptr(z), ctl, self.nput, ctypes.addressof(self.lo),
                  ctypes.addressof(self.hi), ctypes.addressof(self.dst), ctypes.addressof(self.flag), 0,
                  ptr(self.ticket), ptr(self.epoch_dev), stream)

    def wait(self, ctl, stream):
        _lib.call("peer_wait", ctl, self.nwait, ctypes.addressof(self.waits), 0, ptr(self.epoch_dev), stream)

    def apply_spmv(self, y, stream):
        """y = A x with x in self.pext[:n_local]: the boundary rows go into the
        destinations' ghost slots by a copy kernel (gated by their acks of
        the previous exchange), the owned-block SpMV runs meanwhile, then the
        wait on the sources' flags, the ghost-block accumulate and this rank's
        acks. Kernels only -- capturable in a CUDA graph."""
        A, exc = self.A, self.A.exec
        nl = A.n_local
        suf = _lib.suffix(self.pext.dtype)
        _lib.call("peer_put_" + suf, ptr(self.pext), self.nput, ctypes.addressof(self.lo), ctypes.addressof(self.hi),
                  ctypes.addressof(self.dst), ctypes.addressof(self.flag_x), self.nack_in,
                  ctypes.addressof(self.ack_in), ptr(self.epoch_x), ptr(self.ticket), stream)
        yd = Dense.wrap(exc, y.view(-1, 1))
        A.a_own.apply(Dense.wrap(exc, self.pext[:nl].view(-1, 1)), yd)
        _lib.call("peer_wait_plain", self.nwait, ctypes.addressof(self.waits_x), ptr(self.epoch_x), stream)
        if A.a_ghost is not None:
            A.a_ghost.apply_advanced(1.0, Dense.wrap(exc, self.pext[nl:].view(-1, 1)), 1.0, yd)
        _lib.call("peer_ack", self.nack_out, ctypes.addressof(self.ack_out), ptr(self.epoch_x), stream)


class PeerReduce:
    """The CG's 8-32 byte all-reduces through peer memory
    (b200sp_peer_allreduce): every rank maps every other rank's slot and flag
    arrays once; a call is one single-thread kernel that stores the local sums
    into every rank's slots, raises its flags and sums the slots in rank
    order after every flag has arrived -- identical results on every rank,
    no NCCL launch."""

    def __init__(self, comm, dev):
        w = comm.size
        self.world, self.rank = w, comm.rank
        self.slots = torch.zeros(2 * w * 4, dtype=torch.float64, device=dev)
        self.flags = torch.zeros(w, dtype=torch.int32, device=dev)
        torch.cuda.synchronize(dev)
        every = comm.allgather_object({"slots": ipc_export(self.slots), "flags": ipc_export(self.flags)})
        self._bases, sl, fl = [], [], []
        for j, info in enumerate(every):
            if j == comm.rank:
                sl.append(self.slots.data_ptr())
                fl.append(self.flags.data_ptr())
                continue
            ts, b0 = ipc_open(*info["slots"])
            tf, b1 = ipc_open(*info["flags"])
            self._bases += [b0, b1]
            sl.append(ts)
            fl.append(tf)
        self.sl = (ctypes.c_void_p * w)(*sl)
        self.fl = (ctypes.c_void_p * w)(*fl)
        import weakref

        weakref.finalize(self, _close_mapped, self._bases)
        self.epoch_dev = torch.zeros(1, dtype=torch.int32, device=dev)  # advanced by the kernel
        torch.cuda.synchronize(dev)

    def allreduce_(self, t, stream):
        """Sum a float64 device tensor of 1..4 values across the ranks, in place."""
        _lib.call("peer_allreduce", ptr(t), t.numel(), self.world, self.rank, ctypes.addressof(self.sl),
                  ctypes.addressof(self.fl), 0, ptr(self.epoch_dev), stream)


# ---------------------------------------------------------------------------
# distributed CG
# ---------------------------------------------------------------------------
def is_distributed(a):
    return isinstance(a, DistCsr)


class DistCg:
    """Row-partitioned CG engine on DistCsr: the device-resident CG kernels
    with every reduction split as local sum -> all-reduce (NCCL, or peer
    memory) -> control step (b200sp_cg_finish), two all-reduces per
    iteration. Criteria: every device-evaluable child of Combined --
    Iteration and ResidualNormReduction from the all-reduced norms, and
    TimeLimit through a per-rank "limit reached" flag summed by the same
    all-reduce, so every rank stops at the same iteration. Preconditioner:
    none or block-Jacobi on this rank's rows (blocks fused into the steps).

    Reached through the reference API -- ``Cg(exc, criteria,
    preconditioner=Jacobi(...)).generate(dist_csr).apply(b_local, x_local)``
    (solvers/krylov.py routes a DistCsr system here) -- or standalone via
    ``solve(b, x)`` on this rank's (n_local,) tensors."""

    def __init__(self, a, criteria, batch=None, precond=None):
        from .errors import Unsupported

        self.a = a
        self.exec = a.exec
        if isinstance(criteria, Combined):
            self.factory = criteria
        else:
            self.factory = Combined(criteria if isinstance(criteria, (list, tuple)) else [criteria])
        spec = self.factory.device_spec()
        if spec is None:
            raise Unsupported("the distributed CG evaluates its criteria on the device: use Iteration, "
                              "ResidualNormReduction and TimeLimit")
        self.spec, self.timed = spec
        self.precond = precond
        self.batch = int(batch or config.SOLVER_BATCH)
        self.last_status = None
        dev = self.exec.device
        self.ctl = torch.zeros(int(_lib.query("krylov_ctl_bytes")), dtype=torch.uint8, device=dev)
        self.part = torch.zeros(int(_lib.query("krylov_part_elems")), dtype=torch.float64, device=dev)
        self._red_off = int(_lib.query("krylov_red_offset"))
        self.halo = self.reduce = None
        self._bufs = {}
        self._graphs = {}

    def _jac(self):
        return self.precond.jac_args() if self.precond is not None else (0, 0, 0, 0, 0)

    def _spmv_sigma_peer(self, peer, pext, p, q, c, pp, suf):
        """q = A p, sigma parked; the ghosts arrive by peer stores from the
        neighbours' step1: owned SpMV, wait for the flags, ghost SpMV."""
        from .solvers.krylov import fused_csr_ok

        A, exc = self.a, self.exec
        nl = A.n_local
        own, gh = A.a_own, A.a_ghost
        own.apply(Dense.wrap(exc, pext[:nl].view(-1, 1)), Dense.wrap(exc, q.view(-1, 1)))
        peer.wait(c, exc.stream)
        if gh is None:
            _lib.call("cg_sigma_" + suf, nl, ptr(p), ptr(q), c, ptr(pp), exc.stream)
        elif config.FUSED_SPMV_DOT and fused_csr_ok(gh):
            _lib.call("csr_spmv_dot_" + suf, nl, ptr(gh._rp), ptr(gh._ci), ptr(gh._v), ptr(pext[nl:]), ptr(q),
                      ptr(p), 4, gh.subwarp(), c, ptr(pp), exc.stream)
        else:
            gh.apply_advanced(1.0, Dense.wrap(exc, pext[nl:].view(-1, 1)), 1.0, Dense.wrap(exc, q.view(-1, 1)))
            _lib.call("cg_sigma_" + suf, nl, ptr(p), ptr(q), c, ptr(pp), exc.stream)

    def _spmv_sigma(self, pext, p, q, c, pp, suf):
        """q = A p with the local sigma = p.q parked for the all-reduce. With
        classical-strategy blocks the reduction rides in an SpMV epilogue
        (csr_spmv_dot): the owned block's when there are no ghosts, else the
        ghost block's accumulate-and-dot pass after the halo lands (the owned
        SpMV still overlaps the exchange); otherwise SpMV + cg_sigma."""
        from .solvers.krylov import fused_csr_ok

        A, exc = self.a, self.exec
        nl = A.n_local
        own, gh = A.a_own, A.a_ghost
        if not (config.FUSED_SPMV_DOT and fused_csr_ok(own) and (gh is None or fused_csr_ok(gh))):
            A.apply_ext(pext, q)
            _lib.call("cg_sigma_" + suf, nl, ptr(p), ptr(q), c, ptr(pp), exc.stream)
            return
        if gh is None:
            _lib.call("csr_spmv_dot_" + suf, nl, ptr(own._rp), ptr(own._ci), ptr(own._v), ptr(p), ptr(q), 0, 1,
                      own.subwarp(), c, ptr(pp), exc.stream)
            return
        work = A.start_halo(pext)
        own.apply(Dense.wrap(exc, pext[:nl].view(-1, 1)), Dense.wrap(exc, q.view(-1, 1)))
        work.wait()
        _lib.call("csr_spmv_dot_" + suf, nl, ptr(gh._rp), ptr(gh._ci), ptr(gh._v), ptr(pext[nl:]), ptr(q), ptr(p),
                  4, gh.subwarp(), c, ptr(pp), exc.stream)

    @staticmethod
    def _status(c, stream):
        iv, dv = (ctypes.c_int32 * 8)(), (ctypes.c_double * 8)()
        _lib.call("krylov_status", c, ctypes.addressof(iv), ctypes.addressof(dv), stream)
        return list(iv), list(dv)

    def _comm_paths(self, dt):
        """(peer halo or None, extended p vector, peer all-reduce or None)."""
        A, exc, comm = self.a, self.exec, self.a.comm
        peer = A.peer(dt)  # collective: every rank builds it on its first solve of this dtype
        if peer is not None:
            pext = peer.pext
        else:
            pext = torch.empty(A.n_ext, dtype=dt, device=exc.device)
        red = None  # the all-reduces ride on peer memory too when the halo does
        if peer is not None and comm.size <= 8:
            red = getattr(A, "_peer_reduce", None)
            if red is None:
                red = PeerReduce(comm, exc.device)
                A.__dict__["_peer_reduce"] = red
        self.halo = "peer" if peer is not None else "nccl"
        self.reduce = "peer" if red is not None else "nccl"
        return peer, pext, red

    def run(self, ctl, c, pp, hist, b, x):
        """The iteration loop on an initialised control block ``ctl`` (uint8
        device tensor, pointer ``c``): b, x are this rank's (n_local,) slices
        (x = initial guess, overwritten). Returns when the device reports done."""
        exc, A = self.exec, self.a
        nl, dt = A.n_local, x.dtype
        suf = _lib.suffix(dt)
        comm = A.comm
        _lib.call("krylov_set_dist", c, 1, exc.stream)
        red_t = ctl[self._red_off:self._red_off + 32].view(torch.float64)
        J = self._jac()
        bufs = self._bufs.get(dt)
        if bufs is None:  # kept across solves: a captured graph refers to them
            r = torch.empty(nl, dtype=dt, device=exc.device)
            q = torch.empty(nl, dtype=dt, device=exc.device)
            z = r if J[0] == 0 else torch.empty(nl, dtype=dt, device=exc.device)
            bufs = self._bufs[dt] = (r, q, z)
        r, q, z = bufs
        peer, pext, red = self._comm_paths(dt)
        k_check = 4 if self.timed else 2  # + the summed "time limit reached" flags

        def allreduce(k):
            if red is not None:
                red.allreduce_(red_t[:k], exc.stream)
            else:
                comm.allreduce_(red_t[:k])
        p = pext[:nl]
        # r = b - A x  (x staged in the extended vector for its halo)
        pext[:nl].copy_(x)
        A.apply_ext(pext, r, alpha=-1.0, beta=1.0, y_in=b)
        _lib.call("cg_init_" + suf, nl, ptr(r), ptr(z), ptr(p), *J, c, ptr(pp), hist, exc.stream)
        allreduce(k_check)
        _lib.call("cg_finish", c, hist, 0, exc.stream)
        guard = int(_lib.query("krylov_guard", c, 0))

        def iteration():
            if peer is not None:
                peer.step1(nl, p, z, c, suf, exc.stream)
                self._spmv_sigma_peer(peer, pext, p, q, c, pp, suf)
            else:
                _lib.call("cg_step1_" + suf, nl, ptr(p), ptr(z), c, exc.stream)
                self._spmv_sigma(pext, p, q, c, pp, suf)
            allreduce(1)
            _lib.call("cg_finish", c, hist, 1, exc.stream)
            _lib.call("cg_step2_" + suf, nl, ptr(x), 1, ptr(r), ptr(p), ptr(q), ptr(z), *J, c, ptr(pp),
                      hist, exc.stream)
            allreduce(k_check)
            _lib.call("cg_finish", c, hist, 2, exc.stream)

        # with the peer halo AND the peer all-reduce an iteration is kernels
        # only (device-managed epochs): a batch is captured once as a CUDA
        # graph and replayed -- no per-kernel Python launch cost per iteration
        graphed = peer is not None and red is not None and config.DIST_GRAPH
        _lib.query("set_guard", guard)
        try:
            if graphed:
                key = (dt, c, ptr(x), ptr(pp), hist, ptr(r))
                g = self._graphs.get(key)
                while True:
                    iv, _ = self._status(c, exc.stream)
                    if iv[4]:
                        break
                    if g is None:
                        iteration()  # eager first (lazily built plans); the graph starts after it
                        iv, _ = self._status(c, exc.stream)
                        if iv[4]:
                            break
                        g = torch.cuda.CUDAGraph()
                        torch.cuda.synchronize(exc.device)
                        with torch.cuda.graph(g, capture_error_mode="relaxed"):
                            for _ in range(self.batch):
                                iteration()
                        self._graphs = {key: g}
                    g.replay()
            else:
                while True:
                    iv, _ = self._status(c, exc.stream)
                    if iv[4]:
                        break
                    for _ in range(self.batch):
                        iteration()
        finally:
            _lib.query("set_guard", 0)

    def solve(self, b, x):
        """b, x: this rank's (n_local,) device tensors; x is the initial guess."""
        exc = self.exec
        types = (ctypes.c_int32 * max(len(self.spec), 1))(*[t for t, _ in self.spec])
        params = (ctypes.c_double * max(len(self.spec), 1))(*[p for _, p in self.spec])
        c = ptr(self.ctl)
        _lib.call("krylov_ctl_init", c, len(self.spec), ctypes.addressof(types), ctypes.addressof(params), 1, 0, 0,
                  exc.stream)
        self.run(self.ctl, c, self.part, 0, b, x)
        iv, dv = self._status(c, exc.stream)
        status = np.zeros(1, dtype=[("stopped", "?"), ("stopping_id", "u1"), ("finalized", "?")])
        status["stopped"][0], status["stopping_id"][0], status["finalized"][0] = bool(iv[1]), iv[2], bool(iv[3])
        bd = BreakdownInfo(iv[6], "non-positive p^T A p") if iv[5] else None
        self.last_status = SolveStatus(iv[0], status, bd, self.factory.residual_criterion_ids())
        return self.last_status


def solve_cg(solver, b, x):
    """CgSolver._apply_impl for a DistCsr system (the reference factory path,
    src/solvers/krylov.py:36-77): b and x are this rank's (n_local, 1) slices.
    Same observable contract as the single-GPU device path: last_status,
    breakdown as status, logger events replayed from the device history."""
    from .errors import Unsupported
    from .precond import JacobiOperator
    from .solvers.device import get_state
    from .solvers.krylov import finish_from_device

    A = solver.a
    if b.size.cols != 1:
        raise Unsupported("the distributed CG solves one right-hand side at a time")
    pre = solver.precond
    if not (isinstance(pre, JacobiOperator) or type(pre).__name__ == "Identity"):
        raise Unsupported("the distributed CG takes no preconditioner or block-Jacobi")
    if isinstance(pre, JacobiOperator) and not pre.fusable:
        raise Unsupported("the distributed CG fuses block-Jacobi blocks of at most 32 rows")
    eng = solver.__dict__.get("_dist_engine")
    if eng is None:
        eng = solver.__dict__["_dist_engine"] = DistCg(
            A, solver.criterion_factory, precond=pre if isinstance(pre, JacobiOperator) else None)
    S = get_state(solver, A.n_local, x.values.dtype)
    S.begin(b, x)
    eng.run(S.ctl, S.c, S.part, S.h, S.b[:, 0], S.x[:, 0])
    finish_from_device(solver, S, S.status(), x)


def iteration_criteria(max_iters, factor):
    from .stop import Iteration, ResidualNormReduction

    return [Iteration(max_iters), ResidualNormReduction(factor)]
