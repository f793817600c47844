"""CG, BiCGSTAB, FCG and CGS (reference src/solvers/krylov.py:36-271).

Single right-hand side with device-evaluable criteria (Iteration,
ResidualNormReduction, TimeLimit) and an Identity or block-Jacobi
preconditioner runs device-resident: fused step kernels (csrc/krylov.cu),
the matrix's own SpMV, batches of iterations replayed as a cached CUDA
graph. Every other case (several columns, user-defined criteria, other
preconditioners) runs the host-controlled loop in generic.py -- same
kernels, host scalars.
"""

from __future__ import annotations

from .. import _lib, config
from ..base import Identity
from ..executor import CudaExecutor, ptr
from ..precond import JacobiOperator
from . import generic
from .common import BreakdownInfo, IterativeSolver, IterativeSolverFactory
from .device import batch_size, get_state

_BD_REASONS = {1: "non-positive p^T A p", 2: "rho = 0", 3: "r_tld^T A p = 0", 4: "t^T t = 0",
               5: "singular Hessenberg system", 6: "a peer rank did not respond (peer_timeout_ms)"}


def device_path_ok(solver, b):
    if b.size.cols != 1 or not isinstance(solver.exec, CudaExecutor):
        return False
    if solver.criterion_factory.device_spec() is None:
        return False
    if not isinstance(solver.precond, (Identity, JacobiOperator)):
        return False
    if isinstance(solver.precond, JacobiOperator) and not solver.precond.fusable:
        return False  # blocks over 32 rows: host-sequenced loop, apply as its own launch
    return str(b.values.dtype) in ("torch.float64", "torch.float32")


def jac_args(solver):
    if isinstance(solver.precond, JacobiOperator):
        return solver.precond.jac_args()
    return (0, 0, 0, 0, 0)


def fused_csr_ok(a):
    """True when ``a``'s SpMV can carry a reduction in its epilogue
    (csr_spmv_dot: Csr with the classical strategy)."""
    from ..formats import Csr

    return isinstance(a, Csr) and a.strategy == "classical"


def fused_csr(solver):
    """The system matrix when its SpMV can carry the next reduction in its
    epilogue, else None."""
    a = solver.a
    return a if config.FUSED_SPMV_DOT and fused_csr_ok(a) else None


def spmv_dot(S, a, suf, p, q, u, phase):
    _lib.call("csr_spmv_dot_" + suf, a.size.rows, ptr(a._rp), ptr(a._ci), ptr(a._v), ptr(p), ptr(q),
              ptr(u) if u is not None else 0, phase, a._subwarp_arg(), S.c, S.p, a.exec.stream)


def finish_from_device(solver, state, st, x):
    state.end(x)
    status = solver._new_status(1)
    status.data["stopped"][0] = bool(st["stopped"])
    status.data["stopping_id"][0] = st["stopping_id"]
    status.data["finalized"][0] = bool(st["finalized"])
    bd = None
    if st["breakdown"]:
        bd = BreakdownInfo(st["breakdown_it"], _BD_REASONS.get(st["breakdown"], "breakdown"))
    state.replay_events(st)
    solver._finish(st["it"], status, bd)


class CgSolver(IterativeSolver):
    """Preconditioned conjugate gradients (SPD systems)."""

    supports_distributed = True

    def _coop_ok(self, J, S):
        from ..formats import _Sparse

        return (config.CG_COOP_MAX_ROWS > 0 and self.size.rows <= config.CG_COOP_MAX_ROWS and J[0] == 0
                and isinstance(self.a, _Sparse) and not S.timed)

    def _coop_csr(self):
        """The system as Csr for the cooperative kernel (other sparse formats
        are converted once; their row sums run in the same entry order)."""
        from ..formats import Csr, convert

        if isinstance(self.a, Csr):
            return self.a
        c = getattr(self, "_coop_csr_cache", None)
        if c is None:
            c = self._coop_csr_cache = convert(self.a, "csr")
        return c

    def _apply_impl(self, b, x):
        from .. import distributed

        if distributed.is_distributed(self.a):  # row-partitioned system: one rank's slice
            return distributed.solve_cg(self, b, x)
        if not device_path_ok(self, b):
            return generic.cg(self, b, x)
        n = self.size.rows
        S = get_state(self, n, x.values.dtype)
        suf = _lib.suffix(S.dtype)
        exc = self.exec
        J = jac_args(self)
        r, p, q = S.vec("r"), S.vec("p"), S.vec("q")
        z = r if J[0] == 0 else S.vec("z")
        rd, pd, qd = S.dense(r), S.dense(p), S.dense(q)
        S.begin(b, x)
        self._residual(S.xd, S.bd, rd)
        _lib.call("cg_init_" + suf, n, ptr(r), ptr(z), ptr(p), *J, S.c, S.p, S.h, exc.stream)

        if self._coop_ok(J, S):
            # small system: the whole solve is one persistent cooperative launch
            a = self._coop_csr()
            _lib.call("cg_coop_" + suf, n, ptr(a._rp), ptr(a._ci), ptr(a._v), ptr(S.x), ptr(r), ptr(p),
                      ptr(S.vec("p2")), ptr(q), S.c, S.p, S.h, exc.stream)
            return finish_from_device(self, S, S.status(), x)

        fa = fused_csr(self)
        def body():
            _lib.call("cg_step1_" + suf, n, ptr(p), ptr(z), S.c, exc.stream)
            if fa is not None:  # q = A p and sigma = p.q in one pass
                spmv_dot(S, fa, suf, p, q, None, 1)
            else:
                self.a.apply(pd, qd)
                _lib.call("cg_sigma_" + suf, n, ptr(p), ptr(q), S.c, S.p, exc.stream)
            _lib.call("cg_step2_" + suf, n, ptr(S.x), 1, ptr(r), ptr(p), ptr(q), ptr(z), *J, S.c, S.p, S.h,
                      exc.stream)

        st = S.run(body, batch_size())
        finish_from_device(self, S, st, x)


class BicgstabSolver(IterativeSolver):
    """BiCGSTAB with half-iteration counting and the mid-cycle check."""

    def _apply_impl(self, b, x):
        if not device_path_ok(self, b):
            return generic.bicgstab(self, b, x)
        n = self.size.rows
        S = get_state(self, n, x.values.dtype)
        suf = _lib.suffix(S.dtype)
        exc = self.exec
        J = jac_args(self)
        r, rt, p, v, s, t = (S.vec(k) for k in ("r", "rt", "p", "v", "s", "t"))
        y = p if J[0] == 0 else S.vec("y")
        z = s if J[0] == 0 else S.vec("z")
        yd, vd, zd, td, rd = S.dense(y), S.dense(v), S.dense(z), S.dense(t), S.dense(r)
        S.begin(b, x)
        self._residual(S.xd, S.bd, rd)
        _lib.call("bicgstab_init_" + suf, n, ptr(S.b), 1, ptr(r), ptr(rt), ptr(p), ptr(v), ptr(s), ptr(t),
                  ptr(y), ptr(z), S.c, S.p, S.h, exc.stream)

        if config.BICGSTAB_COOP and CgSolver._coop_ok(self, J, S):
            # small system: the whole solve is one persistent cooperative launch
            a = CgSolver._coop_csr(self)
            _lib.call("bicgstab_coop_" + suf, n, ptr(a._rp), ptr(a._ci), ptr(a._v), ptr(S.x), ptr(r), ptr(rt),
                      ptr(p), ptr(v), ptr(s), ptr(t), S.c, S.p, S.h, exc.stream)
            return finish_from_device(self, S, S.status(), x)

        fa = fused_csr(self)

        def body():
            _lib.call("bicgstab_step1_" + suf, n, ptr(r), ptr(p), ptr(v), ptr(y), *J, S.c, exc.stream)
            if fa is not None:  # v = A y with gamma = rt.v fused
                spmv_dot(S, fa, suf, y, v, rt, 2)
            else:
                self.a.apply(yd, vd)
                _lib.call("bicgstab_gamma_" + suf, n, ptr(rt), ptr(v), S.c, S.p, exc.stream)
            _lib.call("bicgstab_step2_" + suf, n, ptr(r), ptr(v), ptr(s), ptr(z), *J, S.c, S.p, S.h, exc.stream)
            if fa is not None:  # t = A z with (t.s, t.t) fused
                spmv_dot(S, fa, suf, z, t, s, 3)
            else:
                self.a.apply(zd, td)
                _lib.call("bicgstab_tst_" + suf, n, ptr(t), ptr(s), S.c, S.p, exc.stream)
            _lib.call("bicgstab_step3_" + suf, n, ptr(S.x), 1, ptr(r), ptr(s), ptr(t), ptr(y), ptr(z), ptr(rt),
                      S.c, S.p, S.h, exc.stream)

        st = S.run(body, max(1, batch_size() // 2))
        finish_from_device(self, S, st, x)


class FcgSolver(IterativeSolver):
    """Flexible CG (src/solvers/krylov.py:80-125). Device-resident like CG:
    cg_init + fcg_init_ctl, then batches of cg_step1 -> SpMV + sigma ->
    fcg_step2 (t = r_new - r_old, rho = r.z, rho_t = t.z, ||r||, check);
    the host-controlled loop (generic.fcg) otherwise."""

    def _apply_impl(self, b, x):
        if not device_path_ok(self, b):
            return generic.fcg(self, b, x)
        n = self.size.rows
        S = get_state(self, n, x.values.dtype)
        suf = _lib.suffix(S.dtype)
        exc = self.exec
        J = jac_args(self)
        r, p, q, t = S.vec("r"), S.vec("p"), S.vec("q"), S.vec("t")
        z = r if J[0] == 0 else S.vec("z")
        rd, pd, qd, td = S.dense(r), S.dense(p), S.dense(q), S.dense(t)
        S.begin(b, x)
        self._residual(S.xd, S.bd, rd)
        td.fill(0.0)
        _lib.call("cg_init_" + suf, n, ptr(r), ptr(z), ptr(p), *J, S.c, S.p, S.h, exc.stream)
        _lib.call("fcg_init_ctl", S.c, exc.stream)
        if config.BICGSTAB_COOP and CgSolver._coop_ok(self, J, S):
            a = CgSolver._coop_csr(self)  # small system: one persistent cooperative launch
            _lib.call("fcg_coop_" + suf, n, ptr(a._rp), ptr(a._ci), ptr(a._v), ptr(S.x), ptr(r), ptr(p), ptr(q),
                      ptr(t), S.c, S.p, S.h, exc.stream)
            return finish_from_device(self, S, S.status(), x)
        fa = fused_csr(self)

        def body():
            _lib.call("cg_step1_" + suf, n, ptr(p), ptr(z), S.c, exc.stream)
            if fa is not None:
                spmv_dot(S, fa, suf, p, q, None, 1)
            else:
                self.a.apply(pd, qd)
                _lib.call("cg_sigma_" + suf, n, ptr(p), ptr(q), S.c, S.p, exc.stream)
            _lib.call("fcg_step2_" + suf, n, ptr(S.x), 1, ptr(r), ptr(p), ptr(q), ptr(t), ptr(z), *J, S.c, S.p,
                      S.h, exc.stream)

        st = S.run(body, batch_size())
        finish_from_device(self, S, st, x)


class CgsSolver(IterativeSolver):
    """Conjugate gradient squared (src/solvers/krylov.py:128-187), two
    SpMVs per cycle and a check after each half. Device-resident: BiCGSTAB's
    init, cgs_step1 (u, p, ph = M p) -> SpMV + gamma -> cgs_step2 (q, w,
    uh = M w) -> mid check -> SpMV -> cgs_step3 (r, x, ||r||, next rho);
    the host-controlled loop (generic.cgs) otherwise."""

    def _apply_impl(self, b, x):
        if not device_path_ok(self, b):
            return generic.cgs(self, b, x)
        n = self.size.rows
        S = get_state(self, n, x.values.dtype)
        suf = _lib.suffix(S.dtype)
        exc = self.exec
        J = jac_args(self)
        r, rt, p, q, u, vh, t = (S.vec(k) for k in ("r", "rt", "p", "q", "u", "vh", "t"))
        w = S.vec("w")
        ph = p if J[0] == 0 else S.vec("ph")
        uh = w if J[0] == 0 else S.vec("uh")
        rd, phd, vhd, uhd, td = S.dense(r), S.dense(ph), S.dense(vh), S.dense(uh), S.dense(t)
        S.begin(b, x)
        self._residual(S.xd, S.bd, rd)
        # rt = b, p q u uh vh t = 0, baseline / check(0), rho = rt.r, beta
        _lib.call("bicgstab_init_" + suf, n, ptr(S.b), 1, ptr(r), ptr(rt), ptr(p), ptr(q), ptr(u), ptr(t),
                  ptr(uh), ptr(vh), S.c, S.p, S.h, exc.stream)
        if config.BICGSTAB_COOP and CgSolver._coop_ok(self, J, S):
            a = CgSolver._coop_csr(self)  # small system: one persistent cooperative launch
            _lib.call("cgs_coop_" + suf, n, ptr(a._rp), ptr(a._ci), ptr(a._v), ptr(S.x), ptr(r), ptr(rt), ptr(p),
                      ptr(q), ptr(u), ptr(vh), ptr(w), ptr(t), S.c, S.p, S.h, exc.stream)
            return finish_from_device(self, S, S.status(), x)
        fa = fused_csr(self)

        def body():
            _lib.call("cgs_step1_" + suf, n, ptr(r), ptr(q), ptr(u), ptr(p), ptr(ph), *J, S.c, exc.stream)
            if fa is not None:  # v_hat = A ph with gamma = rt.v_hat fused
                spmv_dot(S, fa, suf, ph, vh, rt, 2)
            else:
                self.a.apply(phd, vhd)
                _lib.call("bicgstab_gamma_" + suf, n, ptr(rt), ptr(vh), S.c, S.p, exc.stream)
            _lib.call("cgs_step2_" + suf, n, ptr(u), ptr(vh), ptr(q), ptr(w), ptr(uh), *J, S.c, exc.stream)
            _lib.call("cgs_mid", S.c, S.h, exc.stream)
            self.a.apply(uhd, td)
            _lib.call("cgs_step3_" + suf, n, ptr(S.x), 1, ptr(r), ptr(t), ptr(uh), ptr(rt), S.c, S.p, S.h,
                      exc.stream)

        st = S.run(body, max(1, batch_size() // 2))
        finish_from_device(self, S, st, x)


class Cg(IterativeSolverFactory):
    solver_cls = CgSolver


class Fcg(IterativeSolverFactory):
    solver_cls = FcgSolver


class Cgs(IterativeSolverFactory):
    solver_cls = CgsSolver


class Bicgstab(IterativeSolverFactory):
    solver_cls = BicgstabSolver
