"""Block-Jacobi preconditioner (reference src/precond.py:28-208).

Generation runs on the device as one warp per diagonal block: the block is
extracted from Csr, inverted with Gauss-Jordan / partial pivoting in the
reference's exact arithmetic order (bit-identical inverses), kappa_inf is
computed with NumPy's pairwise row sums, and with ``adaptive_precision`` a
block whose kappa is below ``condition_threshold`` is stored in fp32. The
apply is a batched warp-per-block mat-vec; the solvers fuse it into their
update kernels. Blocks of up to 32 rows take the warp-per-block kernels
(fused into the solver steps); larger blocks (any block_size or explicit
boundaries up to 4096 rows, src/precond.py:155-197) take a CTA-per-block
generation with the same Gauss-Jordan arithmetic and a CTA-per-block apply,
and the solvers then apply the preconditioner as its own launch.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .base import LinOp, LinOpFactory
from .errors import DimensionMismatch, Singular, Unsupported
from .executor import ptr
from .formats import Csr, _require_cuda, convert

WARP_BLOCK = 32     # largest block the fused warp-per-block kernels take
MAX_BLOCK = 4096    # b200sp_jacobi_large_max_block()
LARGE_SCRATCH_BYTES = 1 << 30  # Gauss-Jordan [B | I] scratch of the large-block path


def gauss_jordan_inverse(block, exc=None):
    """Explicit inverse of a dense block by Gauss-Jordan elimination with
    partial pivoting (src/precond.py:28-46), computed by the device
    generation kernel -- bit-identical to the reference -- or None when a
    pivot vanishes. Blocks are limited to 4096 rows on this backend."""
    from .executor import CudaExecutor
    from .formats import MatrixData

    blk = np.asarray(block, dtype=np.float64)
    bs = blk.shape[0]
    if blk.ndim != 2 or blk.shape[1] != bs:
        raise DimensionMismatch("gauss_jordan_inverse needs a square block")
    if bs > MAX_BLOCK:
        raise Unsupported(f"blocks are limited to {MAX_BLOCK} rows on this backend")
    if bs == 0:
        return np.zeros((0, 0))
    exc = exc or CudaExecutor()
    a = Csr.from_data(exc, MatrixData.from_dense_array(blk))
    try:
        op = Jacobi(exc, block_size=bs).generate(a)
    except Singular:
        return None
    return op.stored_inverse(0).astype(np.float64)


def uniform_block_boundaries(n, block_size):
    """Block start rows for uniform blocks (last block may be smaller)."""
    return list(range(0, n, int(block_size)))


def _scan64(exc, counts):
    n = counts.numel()
    out = torch.empty(n + 1, dtype=torch.int64, device=exc.device)
    ws = torch.empty(max(1, int(_lib.query("scan_workspace_elems", n))), dtype=torch.int64, device=exc.device)
    _lib.call("exclusive_scan_i64", n, ptr(counts), ptr(out), ptr(ws), exc.stream)
    return out


class JacobiOperator(LinOp):
    """Block-diagonal preconditioner holding the inverted diagonal blocks."""

    def __init__(self, exc, size, starts, offs, prec, storage, cond, max_block=None):
        super().__init__(exc, size)
        self._starts, self._offs, self._prec = starts, offs, prec
        self._storage, self._cond = storage, cond
        if max_block is None:
            st = starts.cpu().numpy()
            max_block = int(np.diff(st).max()) if st.size > 1 else 0
        self.max_block = int(max_block)

    _local_rows = None  # set for the blocks of one rank of a row-partitioned matrix

    def _operand_rows(self):
        if self._local_rows is not None:
            return self._local_rows, self._local_rows
        return super()._operand_rows()

    @property
    def fusable(self):
        """True when the solvers can fuse the apply into their step kernels
        (warp-per-block: every block at most 32 rows)."""
        return self.max_block <= WARP_BLOCK

    @property
    def num_blocks(self):
        return int(self._starts.numel()) - 1

    def jac_args(self):
        """(nblocks, starts, offs, prec, storage) pointers for the C ABI."""
        return (self.num_blocks, ptr(self._starts), ptr(self._offs), ptr(self._prec), ptr(self._storage))

    @property
    def block_precisions(self):
        return ["reduced" if p else "full" for p in self._prec.cpu().numpy()]

    @property
    def block_conditions(self):
        return [float(c) for c in self._cond.cpu().numpy()]

    def stored_inverse(self, idx):
        """The stored inverse of block idx (float64 or float32, row-major)."""
        s = self._starts.cpu().numpy()
        bs = int(s[idx + 1] - s[idx])
        off = int(self._offs[idx].item())
        reduced = bool(self._prec[idx].item())
        nbytes = bs * bs * (4 if reduced else 8)
        raw = self._storage[off:off + nbytes].cpu().numpy()
        arr = raw.view(np.float32 if reduced else np.float64).reshape(bs, bs)
        return arr.T.copy()  # stored column-major

    def _apply_impl(self, b, x):
        bt, xt = b.values, x.values
        suf = _lib.suffix(xt.dtype)
        kern = "jacobi_apply_" if self.fusable else "jacobi_apply_large_"
        _lib.call(kern + suf, *self.jac_args(), xt.shape[1], ptr(bt), bt.stride(0), ptr(xt),
                  xt.stride(0), self.exec.stream)

    def clone_to(self, target):
        _require_cuda(target)
        dev = target.device
        return JacobiOperator(target, self.size, self._starts.clone().to(dev), self._offs.clone().to(dev),
                              self._prec.clone().to(dev), self._storage.clone().to(dev),
                              self._cond.clone().to(dev), self.max_block)


class Jacobi(LinOpFactory):
    """Block-Jacobi factory: uniform ``block_size`` (default 1) or explicit
    ``block_boundaries`` (start rows); optional adaptive fp32 storage."""

    def __init__(self, exc, block_size=1, block_boundaries=None, adaptive_precision=False,
                 condition_threshold=1e6):
        super().__init__(exc)
        self.block_size = block_size
        self.block_boundaries = block_boundaries
        self.adaptive_precision = adaptive_precision
        self.condition_threshold = condition_threshold

    def _starts(self, n):
        if self.block_boundaries is not None:
            return [int(s) for s in self.block_boundaries]
        return uniform_block_boundaries(n, self.block_size)

    def _validate(self, a):
        if not a.size.square:
            raise DimensionMismatch("block-Jacobi needs a square matrix")
        n = a.size.rows
        st = self._starts(n)
        if not st or st[0] != 0:
            raise DimensionMismatch("block boundaries must start at row 0")
        if any(b <= s for s, b in zip(st, st[1:])) or (n and st[-1] >= n):
            raise DimensionMismatch("invalid block boundaries")
        sizes = np.diff(st + [n])
        if sizes.size and sizes.max() > MAX_BLOCK:
            raise Unsupported(f"block-Jacobi blocks are limited to {MAX_BLOCK} rows on this backend")

    def _local_starts(self, a):
        """Blocks of a row-partitioned matrix (distributed.DistCsr): the
        global blocks that fall in this rank's rows, which must not straddle
        a rank boundary; generated from the rank's owned diagonal block."""
        lo, hi = a.lo, a.hi
        st = [s for s in self._starts(a.size.rows) if lo <= s < hi]
        if hi > lo and (not st or st[0] != lo):
            raise Unsupported("a block-Jacobi block straddles a rank boundary of the row partition "
                              "(align the partition to the block size)")
        return [s - lo for s in st], a.a_own

    def _generate(self, a):
        exc = a.exec
        _require_cuda(exc)
        local = None
        if getattr(a, "comm", None) is not None:  # row-partitioned (distributed.DistCsr)
            starts_l, csr = self._local_starts(a)
            local = csr.size.rows
        else:
            csr = a if isinstance(a, Csr) else convert(a, "csr")
        n = csr.size.rows
        host_starts = np.asarray((starts_l if local is not None else self._starts(n)) + [n], dtype=np.int32)
        nb = host_starts.size - 1
        dev = exc.device
        starts = torch.from_numpy(host_starts).to(dev)
        sq = torch.empty(max(nb, 1), dtype=torch.int32, device=dev)
        _lib.call("jacobi_block_sizes_sq", nb, ptr(starts), ptr(sq), exc.stream)
        off64 = _scan64(exc, sq[:nb])
        total = int(off64[-1].item())
        inv64 = torch.empty(max(total, 1), dtype=torch.float64, device=dev)
        cond = torch.empty(max(nb, 1), dtype=torch.float64, device=dev)
        prec = torch.zeros(max(nb, 1), dtype=torch.uint8, device=dev)
        nbytes = torch.empty(max(nb, 1), dtype=torch.int32, device=dev)
        singular = torch.full((1,), np.iinfo(np.int64).max, dtype=torch.int64, device=dev)
        suf = _lib.suffix(csr._v.dtype)
        max_bs = int(np.diff(host_starts).max()) if nb else 0
        args = (nb, ptr(starts), ptr(csr._rp), ptr(csr._ci), ptr(csr._v), ptr(off64), ptr(inv64), ptr(cond),
                ptr(prec), ptr(nbytes), int(bool(self.adaptive_precision)), float(self.condition_threshold),
                ptr(singular))
        if max_bs <= WARP_BLOCK:
            _lib.call("jacobi_invert_" + suf, *args, exc.stream)
        else:
            slot = 2 * max_bs * max_bs
            slots = max(1, min(nb, 2 * 148, LARGE_SCRATCH_BYTES // (8 * slot)))
            scratch = torch.empty(slots * slot, dtype=torch.float64, device=dev)
            _lib.call("jacobi_invert_large_" + suf, *args, max_bs, ptr(scratch), slots, exc.stream)
        bad = int(singular.item())
        if bad != np.iinfo(np.int64).max:
            raise Singular(f"diagonal block {bad} is singular")
        if self.adaptive_precision:
            offs = _scan64(exc, nbytes[:nb])
            storage = torch.empty(max(int(offs[-1].item()), 1), dtype=torch.uint8, device=dev)
            _lib.call("jacobi_pack", nb, ptr(starts), ptr(off64), ptr(inv64), ptr(prec), ptr(offs),
                      ptr(storage), exc.stream)
            offs = offs[:nb]
        else:
            offs = (off64[:nb] * 8).contiguous()
            storage = inv64.view(torch.uint8)
        op = JacobiOperator(exc, a.size, starts, offs, prec[:nb], storage, cond[:nb], max_bs)
        op._local_rows = local
        return op


# ---------------------------------------------------------------------------
# ParILU(0) + ILU preconditioner (reference src/precond.py:211-426)
# ---------------------------------------------------------------------------
class IluFactors:
    """Level-0 incomplete factors: unit-lower L and upper U, both Csr with the
    sparsity of tril / triu of A (diagonals stored explicitly)."""

    def __init__(self, l, u):  # noqa: E741 (reference field names)
        self.l, self.u = l, u

    def defect_on_pattern(self, a):
        """Frobenius norm of (L U - A) restricted to the sparsity of A."""
        lu = self.l.to_data().to_dense_array() @ self.u.to_data().to_dense_array()
        ad = a.to_data()
        return float(np.linalg.norm(lu[ad.rows, ad.cols] - ad.vals))


def parilu_generate(a, sweeps=5):
    """Approximate ILU(0) factors after ``sweeps`` Jacobi-style fixed-point
    sweeps (csrc/ilu.cu); ``sweeps=0`` returns the scaled triangles of A."""
    from .formats import _scan

    csr = a if isinstance(a, Csr) else convert(a, "csr")
    exc = csr.exec
    _require_cuda(exc)
    n = csr.size.rows
    dev = exc.device
    vt = csr._v.dtype
    suf = _lib.suffix(vt)
    from .solvers.triangular import INT_MAX, extract_diagonal

    diag, bad = extract_diagonal(csr)
    if bad != INT_MAX:
        raise Singular(f"zero diagonal at row {bad}")
    lcnt = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    ucnt = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    nodiag = torch.full((1,), INT_MAX, dtype=torch.int32, device=dev)
    _lib.call("ilu_counts", n, ptr(csr._rp), ptr(csr._ci), ptr(lcnt), ptr(ucnt), ptr(nodiag), exc.stream)
    lrp, urp = _scan(exc, lcnt[:n]), _scan(exc, ucnt[:n])
    nl, nu = int(lrp[-1].item()), int(urp[-1].item())
    lci = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
    uci = torch.empty(max(nu, 1), dtype=torch.int32, device=dev)
    al, lv, lv2 = (torch.empty(max(nl, 1), dtype=vt, device=dev) for _ in range(3))
    au, uv, uv2 = (torch.empty(max(nu, 1), dtype=vt, device=dev) for _ in range(3))
    _lib.call("ilu_fill_" + suf, n, ptr(csr._rp), ptr(csr._ci), ptr(csr._v), ptr(diag), ptr(lrp), ptr(urp),
              ptr(lci), ptr(al), ptr(lv), ptr(uci), ptr(au), ptr(uv), exc.stream)
    if sweeps:
        lrow = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
        urow = torch.empty(max(nu, 1), dtype=torch.int32, device=dev)
        _lib.call("csr_rows", n, ptr(lrp), ptr(lrow), exc.stream)
        _lib.call("csr_rows", n, ptr(urp), ptr(urow), exc.stream)
        for _ in range(int(sweeps)):
            _lib.call("parilu_sweep_" + suf, n, nl, nu, ptr(lrow), ptr(lrp), ptr(lci), ptr(al), ptr(lv), ptr(lv2),
                      ptr(urow), ptr(urp), ptr(uci), ptr(au), ptr(uv), ptr(uv2), exc.stream)
            lv, lv2 = lv2, lv
            uv, uv2 = uv2, uv
    lower = Csr._from_device(exc, csr.size, lrp, lci[:nl], lv[:nl])
    upper = Csr._from_device(exc, csr.size, urp, uci[:nu], uv[:nu])
    return IluFactors(lower, upper)


class ParIlu(LinOpFactory):
    """Factorization factory producing :class:`IluFactors`."""

    def __init__(self, exc, sweeps=5):
        super().__init__(exc)
        self.sweeps = sweeps

    def _validate(self, a):
        if not a.size.square:
            raise DimensionMismatch("factorization needs a square matrix")

    def _generate(self, a):
        return parilu_generate(a, self.sweeps)


class IluPreconditioner(LinOp):
    """z = U^-1 (L^-1 r) through the configured triangular solvers."""

    def __init__(self, l_solver, u_solver):
        super().__init__(l_solver.exec, l_solver.size)
        self.l_solver = l_solver
        self.u_solver = u_solver

    def _apply_impl(self, b, x):
        tmp = b.like(*b.values.shape)
        self.l_solver.apply(b, tmp)
        self.u_solver.apply(tmp, x)

    def clone_to(self, target):
        return IluPreconditioner(self.l_solver.clone_to(target), self.u_solver.clone_to(target))


class Ilu(LinOpFactory):
    """ILU preconditioner factory: ``generate`` takes the system matrix
    (factors via ParILU) or pre-generated :class:`IluFactors`; the factor
    solvers default to the direct triangular solvers."""

    def __init__(self, exc, l_solver_factory=None, u_solver_factory=None, sweeps=5):
        from .solvers.triangular import LowerTrs, UpperTrs

        super().__init__(exc)
        self.l_solver_factory = l_solver_factory or LowerTrs(exc, unit_diagonal=True)
        self.u_solver_factory = u_solver_factory or UpperTrs(exc)
        self.sweeps = sweeps

    def _validate(self, a):
        if isinstance(a, IluFactors):
            return
        if not a.size.square:
            raise DimensionMismatch("ILU needs a square matrix")

    def generate(self, system_matrix):
        if isinstance(system_matrix, IluFactors):
            f = system_matrix
            return IluPreconditioner(self.l_solver_factory.generate(f.l), self.u_solver_factory.generate(f.u))
        return super().generate(system_matrix)

    def _generate(self, a):
        f = parilu_generate(a, self.sweeps)
        return IluPreconditioner(self.l_solver_factory.generate(f.l), self.u_solver_factory.generate(f.u))
