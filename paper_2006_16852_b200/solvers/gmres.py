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

from .. import _lib
from ..errors import ParameterError
from ..executor import ptr
from . import generic
from .common import IterativeSolver, IterativeSolverFactory
from .device import DeviceRun
from .krylov import _dense, _vec, device_path_ok, finish_from_device, jac_args

DEFAULT_KRYLOV_DIM = 100
EXACT_CONVERGENCE_ID = 254


class GmresSolver(IterativeSolver):
    def _apply_impl(self, b, x):
        k = int(self.params.get("krylov_dim") or DEFAULT_KRYLOV_DIM)
        if k < 1:
            raise ParameterError("krylov_dim must be >= 1")
        if not device_path_ok(self, b):
            return generic.gmres(self, b, x, k, EXACT_CONVERGENCE_ID)
        exc, n = self.exec, self.size.rows
        xt = x.values
        dt = xt.dtype
        suf = _lib.suffix(dt)
        r, w = _vec(exc, n, dt), _vec(exc, n, dt)
        V = torch.empty((k + 1, n), dtype=dt, device=exc.device)
        J = jac_args(self)
        z = _vec(exc, n, dt) if J[0] else None
        gm = torch.zeros(int(_lib.query("gmres_workspace_elems", k)), dtype=torch.float64, device=exc.device)
        rd, wd = _dense(exc, r), _dense(exc, w)
        zd = _dense(exc, z) if z is not None else None
        vdense = [_dense(exc, V[i]) for i in range(k + 1)]
        run = DeviceRun(self, kdim=k)
        self._residual(x, b, rd)
        _lib.call("gmres_reset_" + suf, n, ptr(r), run.c, run.p, ptr(gm), run.h, 1, exc.stream)
        _lib.call("gmres_scale_v0_" + suf, n, ptr(r), ptr(V), run.c, exc.stream)
        xs = xt.stride(0)
        stopped_guard, done_guard = run.guard(1), run.guard(0)

        def cycle():
            _lib.query("set_guard", stopped_guard)
            for j in range(1, k + 1):
                src = vdense[j - 1]
                if z is not None:
                    self.precond.apply(src, zd)
                    src = zd
                self.a.apply(src, wd)
                _lib.call("gmres_dot0_" + suf, n, j, ptr(V), ptr(w), run.c, run.p, ptr(gm), exc.stream)
                for i in range(j):
                    _lib.call("gmres_mgs_" + suf, n, j, i, ptr(V), ptr(w), run.c, run.p, ptr(gm), run.h,
                              exc.stream)
                _lib.call("gmres_normalize_" + suf, n, j, ptr(V), ptr(w), run.c, exc.stream)
            _lib.call("gmres_backsolve", run.c, ptr(gm), exc.stream)
            _lib.call("gmres_combine_" + suf, n, ptr(V), ptr(xt), xs, *J, run.c, ptr(gm), exc.stream)
            _lib.call("gmres_after_commit", run.c, exc.stream)
            _lib.query("set_guard", done_guard)
            self._residual(x, b, rd)
            _lib.call("gmres_reset_" + suf, n, ptr(r), run.c, run.p, ptr(gm), run.h, 0, exc.stream)
            _lib.call("gmres_scale_v0_" + suf, n, ptr(r), ptr(V), run.c, exc.stream)

        st = run.run(cycle, 1, guard_which=1, gmres=True)
        finish_from_device(self, run, st)


class Gmres(IterativeSolverFactory):
    solver_cls = GmresSolver

    def __init__(self, exc, criteria, preconditioner=None, generated_preconditioner=None,
                 krylov_dim=DEFAULT_KRYLOV_DIM):
        super().__init__(exc, criteria, preconditioner, generated_preconditioner, krylov_dim=krylov_dim)

    def _validate(self, a):
        super()._validate(a)
        if int(self.params["krylov_dim"]) < 1:
            raise ParameterError("krylov_dim must be >= 1")
