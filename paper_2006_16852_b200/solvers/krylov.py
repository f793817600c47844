"""CG and BiCGSTAB (reference src/solvers/krylov.py:36-77, :190-271).

Single right-hand side with device-evaluable criteria (Iteration,
ResidualNormReduction, TimeLimit) and an Identity or block-Jacobi
preconditioner runs device-resident: fused step kernels (csrc/krylov.cu),
the matrix's own SpMV, batches of iterations replayed as CUDA graphs. Every
other case (several columns, user-defined criteria, other preconditioners)
runs the host-controlled loop in generic.py -- same kernels, host scalars.
"""

from __future__ import annotations

import torch

from .. import _lib
from ..base import Identity
from ..executor import CudaExecutor, ptr
from ..formats import Dense
from ..precond import JacobiOperator
from . import generic
from .common import BreakdownInfo, IterativeSolver, IterativeSolverFactory
from .device import DeviceRun, batch_size

_BD_REASONS = {1: "non-positive p^T A p", 2: "rho = 0", 3: "r_tld^T A p = 0", 4: "t^T t = 0",
               5: "singular Hessenberg system"}


def device_path_ok(solver, b):
    if b.size.cols != 1 or not isinstance(solver.exec, CudaExecutor):
        return False
    if solver.criterion_factory.device_spec() is None:
        return False
    if not isinstance(solver.precond, (Identity, JacobiOperator)):
        return False
    return str(b.values.dtype) in ("torch.float64", "torch.float32")


def jac_args(solver):
    if isinstance(solver.precond, JacobiOperator):
        return solver.precond.jac_args()
    return (0, 0, 0, 0, 0)


def finish_from_device(solver, run, st):
    status = solver._new_status(1)
    status.data["stopped"][0] = bool(st["stopped"])
    status.data["stopping_id"][0] = st["stopping_id"]
    status.data["finalized"][0] = bool(st["finalized"])
    bd = None
    if st["breakdown"]:
        bd = BreakdownInfo(st["breakdown_it"], _BD_REASONS.get(st["breakdown"], "breakdown"))
    run.replay_events(st)
    solver._finish(st["it"], status, bd)


def _vec(exc, n, dt):
    return torch.empty(n, dtype=dt, device=exc.device)


def _dense(exc, t):
    return Dense.wrap(exc, t.view(-1, 1))


class CgSolver(IterativeSolver):
    """Preconditioned conjugate gradients (SPD systems)."""

    def _apply_impl(self, b, x):
        if not device_path_ok(self, b):
            return generic.cg(self, b, x)
        exc, n = self.exec, self.size.rows
        xt = x.values
        dt = xt.dtype
        suf = _lib.suffix(dt)
        r, p, q = _vec(exc, n, dt), _vec(exc, n, dt), _vec(exc, n, dt)
        J = jac_args(self)
        z = r if J[0] == 0 else _vec(exc, n, dt)
        rd, pd, qd = _dense(exc, r), _dense(exc, p), _dense(exc, q)
        run = DeviceRun(self)
        self._residual(x, b, rd)
        _lib.call("cg_init_" + suf, n, ptr(r), ptr(z), ptr(p), *J, run.c, run.p, run.h, exc.stream)
        xs = xt.stride(0)

        def body():
            _lib.call("cg_step1_" + suf, n, ptr(p), ptr(z), run.c, exc.stream)
            self.a.apply(pd, qd)
            _lib.call("cg_sigma_" + suf, n, ptr(p), ptr(q), run.c, run.p, exc.stream)
            _lib.call("cg_step2_" + suf, n, ptr(xt), xs, ptr(r), ptr(p), ptr(q), ptr(z), *J, run.c, run.p,
                      run.h, exc.stream)

        st = run.run(body, batch_size())
        finish_from_device(self, run, st)


class BicgstabSolver(IterativeSolver):
    """BiCGSTAB with half-iteration counting and the mid-cycle check."""

    def _apply_impl(self, b, x):
        if not device_path_ok(self, b):
            return generic.bicgstab(self, b, x)
        exc, n = self.exec, self.size.rows
        xt, bt = x.values, b.values
        dt = xt.dtype
        suf = _lib.suffix(dt)
        r, rt, p, v, s, t = (_vec(exc, n, dt) for _ in range(6))
        J = jac_args(self)
        y = p if J[0] == 0 else _vec(exc, n, dt)
        z = s if J[0] == 0 else _vec(exc, n, dt)
        yd, vd, zd, td, rd = _dense(exc, y), _dense(exc, v), _dense(exc, z), _dense(exc, t), _dense(exc, r)
        run = DeviceRun(self)
        self._residual(x, b, rd)
        _lib.call("bicgstab_init_" + suf, n, ptr(bt), bt.stride(0), ptr(r), ptr(rt), ptr(p), ptr(v), ptr(s),
                  ptr(t), ptr(y), ptr(z), run.c, run.p, run.h, exc.stream)
        xs = xt.stride(0)

        def body():
            _lib.call("bicgstab_step1_" + suf, n, ptr(r), ptr(p), ptr(v), ptr(y), *J, run.c, exc.stream)
            self.a.apply(yd, vd)
            _lib.call("bicgstab_gamma_" + suf, n, ptr(rt), ptr(v), run.c, run.p, exc.stream)
            _lib.call("bicgstab_step2_" + suf, n, ptr(r), ptr(v), ptr(s), ptr(z), *J, run.c, run.p, run.h,
                      exc.stream)
            self.a.apply(zd, td)
            _lib.call("bicgstab_tst_" + suf, n, ptr(t), ptr(s), run.c, run.p, exc.stream)
            _lib.call("bicgstab_step3_" + suf, n, ptr(xt), xs, ptr(r), ptr(s), ptr(t), ptr(y), ptr(z), ptr(rt),
                      run.c, run.p, run.h, exc.stream)

        st = run.run(body, max(1, batch_size() // 2))
        finish_from_device(self, run, st)


class Cg(IterativeSolverFactory):
    solver_cls = CgSolver


class Bicgstab(IterativeSolverFactory):
    solver_cls = BicgstabSolver
