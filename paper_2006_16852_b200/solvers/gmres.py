"""Restarted GMRES(k), right preconditioned (reference src/solvers/gmres.py).

Device path (one column, device-evaluable criteria, Identity or block-Jacobi):
each restart cycle -- k Arnoldi steps (preconditioner, SpMV, modified
Gram-Schmidt as j fused dot/axpy passes, normalisation), then back-solve,
x += M (V y), true residual and reset -- is captured once as a CUDA graph and
replayed until the device reports done. The Givens rotations, residual
estimate |gamma_j|, happy-breakdown detection and criteria run in the
reduction epilogue of the last MGS pass. Otherwise the host-controlled loop
of generic.py runs.
"""

from __future__ import annotations

import torch

from .. import _lib, config
from ..errors import ParameterError
from ..executor import ptr
from . import generic
from .common import IterativeSolver, IterativeSolverFactory
from .device import get_state
from .krylov import device_path_ok, finish_from_device, jac_args

DEFAULT_KRYLOV_DIM = 100
EXACT_CONVERGENCE_ID = 254


def _sparse(a):
    from ..formats import _Sparse

    return isinstance(a, _Sparse)


class GmresSolver(IterativeSolver):
    def _apply_impl(self, b, x):
        k = int(self.params.get("krylov_dim") or DEFAULT_KRYLOV_DIM)
        if k < 1:
            raise ParameterError("krylov_dim must be >= 1")
        if not device_path_ok(self, b):
            return generic.gmres(self, b, x, k, EXACT_CONVERGENCE_ID)
        n = self.size.rows
        S = get_state(self, n, x.values.dtype, kdim=k)
        suf = _lib.suffix(S.dtype)
        exc = self.exec
        J = jac_args(self)
        r, w = S.vec("r"), S.vec("w")
        V = S.vec("V", (k + 1, n))
        z = S.vec("z") if J[0] else None
        if "gm" not in S.vecs:
            S.vecs["gm"] = torch.zeros(int(_lib.query("gmres_workspace_elems", k)), dtype=torch.float64,
                                       device=exc.device)
        gm = S.vecs["gm"]
        rd, wd = S.dense(r), S.dense(w)
        zd = S.dense(z) if z is not None else None
        vdense = [S.dense(V[i]) for i in range(k + 1)]
        S.begin(b, x)
        self._residual(S.xd, S.bd, rd)
        _lib.call("gmres_reset_" + suf, n, ptr(r), S.c, S.p, ptr(gm), S.h, 1, exc.stream)
        _lib.call("gmres_scale_v0_" + suf, n, ptr(r), ptr(V), S.c, exc.stream)
        stopped_guard, done_guard = S.guard(1), S.guard(0)

        small = config.GMRES_SMALL and n <= int(_lib.query("gmres_small_rows"))
        whole = small and z is None and _sparse(self.a)
        if whole:
            from .krylov import CgSolver

            a = CgSolver._coop_csr(self)

        if whole and config.GMRES_TINY and n <= 4 and k <= 128:
            # tiny system: the whole restarted solve is one launch (cycles,
            # back-solve, commit, true residual, restart -- all on chip)
            _lib.call("gmres_solve_tiny_" + suf, n, ptr(a._rp), ptr(a._ci), ptr(a._v), ptr(S.x), ptr(S.b), ptr(V),
                      ptr(w), S.c, ptr(gm), S.h, k, exc.stream)
            return finish_from_device(self, S, S.status(), x)

        def cycle():
            _lib.query("set_guard", stopped_guard)
            if whole:  # the whole Arnoldi cycle in one single-block launch
                _lib.call("gmres_cycle_small_" + suf, n, ptr(a._rp), ptr(a._ci), ptr(a._v), ptr(V), ptr(w), S.c,
                          ptr(gm), S.h, exc.stream)
            for j in range(1, k + 1) if not whole else ():
                src = vdense[j - 1]
                if z is not None:
                    self.precond.apply(src, zd)
                    src = zd
                self.a.apply(src, wd)
                if small:  # the whole MGS + Givens + normalisation in one single-block launch
                    _lib.call("gmres_arnoldi_small_" + suf, n, j, ptr(V), ptr(w), S.c, ptr(gm), S.h, exc.stream)
                    continue
                _lib.call("gmres_dot0_" + suf, n, j, ptr(V), ptr(w), S.c, S.p, ptr(gm), exc.stream)
                for i in range(j):
                    _lib.call("gmres_mgs_" + suf, n, j, i, ptr(V), ptr(w), S.c, S.p, ptr(gm), S.h, exc.stream)
                _lib.call("gmres_normalize_" + suf, n, j, ptr(V), ptr(w), S.c, exc.stream)
            _lib.call("gmres_backsolve", S.c, ptr(gm), exc.stream)
            _lib.call("gmres_combine_" + suf, n, ptr(V), ptr(S.x), 1, *J, S.c, ptr(gm), exc.stream)
            _lib.call("gmres_after_commit", S.c, exc.stream)
            _lib.query("set_guard", done_guard)
            self._residual(S.xd, S.bd, rd)
            _lib.call("gmres_reset_" + suf, n, ptr(r), S.c, S.p, ptr(gm), S.h, 0, exc.stream)
            _lib.call("gmres_scale_v0_" + suf, n, ptr(r), ptr(V), S.c, exc.stream)

        st = S.run(cycle, 1, guard_which=1)
        finish_from_device(self, S, st, x)


class Gmres(IterativeSolverFactory):
    solver_cls = GmresSolver

    def __init__(self, exc, criteria, preconditioner=None, generated_preconditioner=None,
                 krylov_dim=DEFAULT_KRYLOV_DIM):
        super().__init__(exc, criteria, preconditioner, generated_preconditioner, krylov_dim=krylov_dim)

    def _validate(self, a):
        super()._validate(a)
        if int(self.params["krylov_dim"]) < 1:
            raise ParameterError("krylov_dim must be >= 1")
