"""Iterative refinement (reference src/solvers/ir.py:13-72).

x <- x + S(b - A x) per iteration with S the generated inner operator (a
solver, a preconditioner or any LinOp). The residual is the matrix's fused
residual SpMV; the update is a device add_scaled; stopped columns freeze.
"""

from __future__ import annotations

from ..errors import ParameterError
from ..stop import Combined
from . import generic
from .common import IterativeSolver, IterativeSolverFactory


class IrSolver(IterativeSolver):
    def _apply_impl(self, b, x):
        return generic.ir(self, b, x)


class Ir(IterativeSolverFactory):
    """``inner`` is the factory of the correction operator, or pass an
    already generated ``generated_inner``; one of them is required."""

    solver_cls = IrSolver

    def __init__(self, exc, criteria, inner=None, generated_inner=None):
        super().__init__(exc, criteria)
        self.inner = inner
        self.generated_inner = generated_inner

    def _validate(self, a):
        super()._validate(a)
        if self.inner is None and self.generated_inner is None:
            raise ParameterError("iterative refinement requires an inner solver")

    def _generate(self, a):
        inner_op = self.generated_inner if self.generated_inner is not None else self.inner.generate(a)
        return IrSolver(a, self._build_preconditioner(a), Combined(self.criteria), {"inner_op": inner_op})
