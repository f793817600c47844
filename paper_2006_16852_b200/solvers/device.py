"""Device-resident solve driver: control block, batches as CUDA graphs.

One DeviceRun owns the KrylovCtl block (csrc/krylov.cuh), the reduction
partials and the optional residual-norm history of a single m = 1 solve.
``run`` captures ``iters`` iterations of the solver body once as a CUDA graph
(with the SpMV launch guard pointed at the solve's done/stopped flag) and
replays it until the device reports done: one host synchronisation per batch,
none per iteration. Iteration counts stay exact because the criteria are
evaluated on the device at every iteration; launches after the stop are
no-ops.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from .. import _lib, config
from ..executor import ptr
from ..loggers import EventKind
from ..stop import CRIT_ITERATION, CRIT_RNR, ResidualNormReduction


class DeviceRun:
    def __init__(self, solver, kdim=0):
        self.solver = solver
        exc = solver.exec
        self.exc = exc
        spec, self.time_child = solver.criterion_factory.device_spec()
        self.spec = spec
        dev = exc.device
        self.ctl = torch.zeros(int(_lib.query("krylov_ctl_bytes")), dtype=torch.uint8, device=dev)
        self.part = torch.zeros(int(_lib.query("krylov_part_elems")), dtype=torch.float64, device=dev)
        self.logging = bool(solver._log_channels)
        cap = 0
        if self.logging:
            iters = [int(p) for t, p in spec if t == CRIT_ITERATION]
            cap = (min(iters) + 2) if iters else (1 << 20)
        self.hist = torch.zeros(max(cap, 1), dtype=torch.float64, device=dev) if cap else None
        types = (ctypes.c_int32 * max(len(spec), 1))(*[t for t, _ in spec])
        params = (ctypes.c_double * max(len(spec), 1))(*[p for _, p in spec])
        needs_res = int(any(isinstance(f, ResidualNormReduction)
                            for f in solver.criterion_factory.factories))
        _lib.call("krylov_ctl_init", ptr(self.ctl), len(spec), ctypes.addressof(types),
                  ctypes.addressof(params), needs_res, cap, int(kdim), exc.stream)
        self._time_crit = None
        if self.time_child is not None:
            from ..stop import CriterionArgs

            self._time_crit = solver.criterion_factory.factories[self.time_child].generate(
                CriterionArgs(solver.a, None, None))

    # -- pointers -------------------------------------------------------------
    @property
    def c(self):
        return ptr(self.ctl)

    @property
    def p(self):
        return ptr(self.part)

    @property
    def h(self):
        return ptr(self.hist) if self.hist is not None else 0

    def guard(self, which):
        """Device address of the done (0) / stopped (1) flag."""
        return int(_lib.query("krylov_guard", self.c, which))

    # -- status -------------------------------------------------------------------
    def status(self):
        iv = (ctypes.c_int32 * 8)()
        dv = (ctypes.c_double * 8)()
        _lib.call("krylov_status", self.c, ctypes.addressof(iv), ctypes.addressof(dv), self.exc.stream)
        names_i = ("it", "stopped", "stopping_id", "finalized", "done", "breakdown", "breakdown_it", "jpos")
        names_d = ("baseline", "rnorm", "rho", "alpha", "omega", "snorm", "hnorm", "sigma")
        out = {k: int(v) for k, v in zip(names_i, iv)}
        out.update({k: float(v) for k, v in zip(names_d, dv)})
        return out

    # -- batches ---------------------------------------------------------------------
    def run(self, body, iters, guard_which=0, gmres=False):
        """Replay ``iters`` captured calls of ``body`` until the solve is done."""
        st = self.status()
        if st["done"]:
            return st
        guard = self.guard(guard_which)
        # one eager call to build lazily created plans/workspaces, then capture
        _lib.query("set_guard", guard)
        try:
            body()
            st = self.status()
            if st["done"] or self._time_expired(gmres):
                return self.status()
            graph = torch.cuda.CUDAGraph()
            torch.cuda.synchronize(self.exc.device)
            with torch.cuda.graph(graph):
                for _ in range(iters):
                    body()
        finally:
            _lib.query("set_guard", 0)
        while True:
            graph.replay()
            st = self.status()
            if st["done"]:
                return st
            if self._time_expired(gmres):
                graph.replay()  # let GMRES commit its partial segment
                return self.status()

    def _time_expired(self, gmres):
        if self._time_crit is None or not self._time_crit.expired():
            return False
        _lib.call("krylov_force_stop", self.c, self.time_child + 1, int(gmres), self.exc.stream)
        return True

    # -- logger replay ----------------------------------------------------------------
    def replay_events(self, st):
        if not self.logging:
            return
        solver = self.solver
        final = st["it"]
        hist = self.hist[:min(final + 1, self.hist.numel())].cpu().numpy()
        base = st["baseline"]
        names = [type(f).__name__ for f in solver.criterion_factory.factories]
        for it in range(hist.size):
            if it > 0:
                solver._log(EventKind.ITERATION_COMPLETE, {"iteration": it})
            with np.errstate(invalid="ignore", divide="ignore"):
                rel = float(hist[it] / base) if base > 0 else (0.0 if hist[it] == 0 else float("inf"))
            stopped = int(st["stopped"] and it == final)
            for (typ, _), name in zip(self.spec, names):
                solver._log(EventKind.CRITERION_CHECK_COMPLETED, {
                    "criterion": name.replace("ResidualNormReduction", "ResidualNormReductionCriterion")
                                     .replace("Iteration", "IterationCriterion"),
                    "num_iterations": it, "num_stopped": stopped,
                    "relative_norms": [rel] if typ == CRIT_RNR else None})


def batch_size(default=None):
    return int(default or config.SOLVER_BATCH)
