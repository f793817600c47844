"""Device-resident solve driver: control block, batches as CUDA graphs.

A ``DeviceSolve`` is cached on the generated solver per (rows, value type):
it owns the KrylovCtl block (csrc/krylov.cuh), the reduction partials, the
optional residual-norm history, the work vectors and private copies of x and
b. The solver body (``iters`` iterations, or one GMRES restart cycle) is
captured ONCE as a CUDA graph -- with the SpMV launch guard pointed at the
solve's done/stopped flag -- and replayed until the device reports done: one
host synchronisation per batch, none per iteration, no re-capture across
solves. Iteration counts stay exact because the criteria are evaluated on the
device at every iteration; launches after the stop are no-ops.
"""

from __future__ import annotations

import ctypes
import gc

import numpy as np
import torch

from .. import _lib, config
from ..executor import ptr
from ..formats import Dense
from ..loggers import EventKind
from ..stop import CRIT_ITERATION, CRIT_RNR, ResidualNormReduction

HIST_CAP = 1 << 16


class DeviceSolve:
    def __init__(self, solver, n, dtype, kdim=0):
        self.solver = solver
        self.exc = exc = solver.exec
        self.n, self.dtype, self.kdim = n, dtype, kdim
        dev = exc.device
        self.ctl = torch.zeros(int(_lib.query("krylov_ctl_bytes")), dtype=torch.uint8, device=dev)
        self.part = torch.zeros(int(_lib.query("krylov_part_elems")), dtype=torch.float64, device=dev)
        self.hist = torch.zeros(HIST_CAP, dtype=torch.float64, device=dev)
        self.x = torch.empty((n, 1), dtype=dtype, device=dev)
        self.b = torch.empty((n, 1), dtype=dtype, device=dev)
        self.xd, self.bd = Dense.wrap(exc, self.x), Dense.wrap(exc, self.b)
        self.vecs = {}
        self.graph = None
        self.graph_key = None

    # -- work vectors -----------------------------------------------------
    def vec(self, name, shape=None):
        t = self.vecs.get(name)
        if t is None:
            t = torch.empty(shape or (self.n,), dtype=self.dtype, device=self.exc.device)
            self.vecs[name] = t
        return t

    def dense(self, t):
        return Dense.wrap(self.exc, t.view(-1, 1))

    # -- pointers -----------------------------------------------------------
    @property
    def c(self):
        return ptr(self.ctl)

    @property
    def p(self):
        return ptr(self.part)

    @property
    def h(self):
        return ptr(self.hist)

    def guard(self, which):
        """Device address of the done (0) / stopped (1) flag."""
        return int(_lib.query("krylov_guard", self.c, which))

    # -- per-solve setup --------------------------------------------------------
    def begin(self, b, x):
        solver = self.solver
        fac = solver.criterion_factory
        self.spec, self.timed = fac.device_spec()
        self.logging = bool(solver._log_channels)
        iters = [int(p) for t, p in self.spec if t == CRIT_ITERATION]
        cap = (min(min(iters) + 2, HIST_CAP) if iters else HIST_CAP) if self.logging else 0
        types = (ctypes.c_int32 * max(len(self.spec), 1))(*[t for t, _ in self.spec])
        params = (ctypes.c_double * max(len(self.spec), 1))(*[p for _, p in self.spec])
        needs_res = int(any(isinstance(f, ResidualNormReduction) for f in fac.factories))
        _lib.call("krylov_ctl_init", self.c, len(self.spec), ctypes.addressof(types),
                  ctypes.addressof(params), needs_res, cap, int(self.kdim), self.exc.stream)
        self.xd.copy_from(x)
        self.bd.copy_from(b)

    def end(self, x):
        x.copy_from(self.xd)

    # -- status --------------------------------------------------------------------
    def status(self):
        iv = (ctypes.c_int32 * 8)()
        dv = (ctypes.c_double * 8)()
        _lib.call("krylov_status", self.c, ctypes.addressof(iv), ctypes.addressof(dv), self.exc.stream)
        names_i = ("it", "stopped", "stopping_id", "finalized", "done", "breakdown", "breakdown_it", "jpos")
        names_d = ("baseline", "rnorm", "rho", "alpha", "omega", "snorm", "hnorm", "sigma")
        out = {k: int(v) for k, v in zip(names_i, iv)}
        out.update({k: float(v) for k, v in zip(names_d, dv)})
        return out

    # -- batches -----------------------------------------------------------------------
    def run(self, body, iters, guard_which=0):
        """Replay the captured ``iters`` x ``body`` graph until done."""
        st = self.status()
        if st["done"]:
            return st
        if self.graph is None or self.graph_key != (iters, guard_which):
            _lib.query("set_guard", self.guard(guard_which))
            try:
                body()  # eager pass: builds lazily created plans / workspaces
                st = self.status()
                if st["done"]:
                    return st
                graph = torch.cuda.CUDAGraph()
                torch.cuda.synchronize(self.exc.device)
                # relaxed mode + no GC: a collector-triggered free of a pinned
                # host tensor (event query) must not invalidate the capture
                gc_on = gc.isenabled()
                gc.disable()
                try:
                    with torch.cuda.graph(graph, capture_error_mode="relaxed"):
                        for _ in range(iters):
                            body()
                finally:
                    if gc_on:
                        gc.enable()
            finally:
                _lib.query("set_guard", 0)
            self.graph, self.graph_key = graph, (iters, guard_which)
        while True:
            self.graph.replay()
            st = self.status()
            if st["done"]:
                return st

    # -- logger replay --------------------------------------------------------------------
    def replay_events(self, st):
        if not self.logging:
            return
        solver = self.solver
        final = st["it"]
        hist = self.hist[:min(final + 1, HIST_CAP)].cpu().numpy()
        base = st["baseline"]
        for it in range(hist.size):
            if it > 0:
                solver._log(EventKind.ITERATION_COMPLETE, {"iteration": it})
            with np.errstate(invalid="ignore", divide="ignore"):
                rel = float(hist[it] / base) if base > 0 else (0.0 if hist[it] == 0 else float("inf"))
            stopped = int(st["stopped"] and it == final)
            for (typ, _), f in zip(self.spec, solver.criterion_factory.factories):
                solver._log(EventKind.CRITERION_CHECK_COMPLETED, {
                    "criterion": type(f).__name__ + "Criterion", "num_iterations": it,
                    "num_stopped": stopped, "relative_norms": [rel] if typ == CRIT_RNR else None})


def get_state(solver, n, dtype, kdim=0):
    cache = solver.__dict__.setdefault("_device_states", {})
    key = (n, str(dtype), kdim)
    st = cache.get(key)
    if st is None:
        st = cache[key] = DeviceSolve(solver, n, dtype, kdim)
    return st


def batch_size(default=None):
    return int(default or config.SOLVER_BATCH)
