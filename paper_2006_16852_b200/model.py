"""Closed-form solver memory traffic (reference src/model.py:50-123).

The paper's traffic model: exact integer byte volumes a
whole solve reads and writes as functions of n, nnz, the value / index widths,
the iteration count and (GMRES) the restart length, for the reference's COO,
unpreconditioned solver loops. ``bench.py`` divides the per-iteration volume
by the measured time to give the paper-comparable bandwidth figure of each
solver; instrumented measurement (``measure_traffic``) is replaced here by
ncu DRAM counters (profiles/).
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import OpalgError, Unsupported

DEFAULT_KRYLOV_DIM = 100


@dataclass(frozen=True)
class TrafficParams:
    n: int
    nnz: int
    iterations: int
    value_bytes: int = 8
    index_bytes: int = 4
    krylov_dim: int = DEFAULT_KRYLOV_DIM

    def __post_init__(self):
        if min(self.n, self.nnz, self.iterations) < 0:
            raise OpalgError("traffic parameters must be non-negative")
        if self.krylov_dim < 1:
            raise OpalgError("krylov_dim must be >= 1")


@dataclass(frozen=True)
class TrafficPrediction:
    bytes_read: int
    bytes_written: int


# Per solver: the setup volume and the per-iteration volume, each as
# (value-count terms in n, nnz, constant) -- value bytes -- plus 2 nnz index
# reads per SpMV. Two-phase solvers (CGS, BiCGSTAB) alternate odd / even
# half-iterations.
#           setup read (n, nnz), setup write (n, 1), per-iteration read (n, nnz), write (n, 1)
_ONE_PHASE = {
    "cg": ((4, 2), (5, 2), (15, 2), (5, 2)),
    "fcg": ((4, 2), (6, 3), (17, 2), (6, 3)),
}
#           setup read, setup write, odd read, odd write, even read, even write
_TWO_PHASE = {
    "cgs": ((5, 2), (10, 2), (14, 2), (6, 3), (6, 2), (4, 0)),
    "bicgstab": ((5, 2), (10, 6), (16, 2), (4, 2), (13, 2), (4, 3)),
}


def _vals(p, coef_n, coef_other, other):
    return (coef_n * p.n + coef_other * other) * p.value_bytes


def _one_phase(p, c):
    (rn, rz), (wn, wc), (irn, irz), (iwn, iwc) = c
    spmv_idx = 2 * p.nnz * p.index_bytes
    reads = _vals(p, rn, rz, p.nnz) + spmv_idx + p.iterations * (_vals(p, irn, irz, p.nnz) + spmv_idx)
    # the per-iteration write volume is also charged once at setup
    writes = _vals(p, iwn, iwc, 1) * (1 + p.iterations)
    return reads, writes


def _two_phase(p, c):
    (rn, rz), (wn, wc), (orn, orz), (own, owc), (ern, erz), (ewn, ewc) = c
    odd, even = (p.iterations + 1) // 2, p.iterations // 2
    spmv_idx = 2 * p.nnz * p.index_bytes
    reads = (_vals(p, rn, rz, p.nnz) + spmv_idx + odd * (_vals(p, orn, orz, p.nnz) + spmv_idx)
             + even * (_vals(p, ern, erz, p.nnz) + spmv_idx))
    writes = _vals(p, wn, wc, 1) + odd * _vals(p, own, owc, 1) + even * _vals(p, ewn, ewc, 1)
    return reads, writes


def _gmres(p):
    n, z, vt, it = p.n, p.nnz, p.value_bytes, p.index_bytes
    k, iters = p.krylov_dim, p.iterations
    cycles, tail = divmod(iters, k)
    # sum over all steps of (j - 1): the modified Gram-Schmidt passes
    mgs = cycles * (k - 1) * k // 2 + (tail - 1) * tail // 2
    spmv_idx = 2 * z * it
    reads = ((11 * n + 2 * z + tail * (tail + 5) // 2 + n * tail + 1) * vt + spmv_idx
             + cycles * ((1 + k * (k + 5) // 2 + 10 * n + 2 * z + k * n) * vt + spmv_idx)
             + iters * ((7 * n + 5 + 2 * z) * vt + spmv_idx + 8)
             + mgs * (4 * n + 4) * vt)
    writes = ((6 * n + tail + 2 * k + 3) * vt + 8 + cycles * ((k + 6 * n + 2) * vt + 8)
              + iters * ((4 * n + 8) * vt + 8) + mgs * (n + 2) * vt)
    return reads, writes


def predict_traffic(solver: str, params: TrafficParams) -> TrafficPrediction:
    """The solver's closed-form read / write volume (exact integers)."""
    key = solver.lower()
    if key in _ONE_PHASE:
        r, w = _one_phase(params, _ONE_PHASE[key])
    elif key in _TWO_PHASE:
        r, w = _two_phase(params, _TWO_PHASE[key])
    elif key == "gmres":
        r, w = _gmres(params)
    else:
        raise Unsupported(f"no traffic formula for solver {solver!r}")
    return TrafficPrediction(int(r), int(w))


def per_iteration_bytes(solver, n, nnz, iterations, value_bytes=8, index_bytes=4, krylov_dim=DEFAULT_KRYLOV_DIM):
    """(read + write) bytes per iteration of a run, setup excluded."""
    full = predict_traffic(solver, TrafficParams(n, nnz, iterations, value_bytes, index_bytes, krylov_dim))
    none = predict_traffic(solver, TrafficParams(n, nnz, 0, value_bytes, index_bytes, krylov_dim))
    return ((full.bytes_read + full.bytes_written) - (none.bytes_read + none.bytes_written)) / max(iterations, 1)
