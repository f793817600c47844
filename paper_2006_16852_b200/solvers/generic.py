"""Host-controlled solver loops (multi-column / user-defined criteria).

When a solve cannot run fully device-resident -- several right-hand-side
columns (per-column masks and freezes), or a user-defined Criterion /
TimeLimit that must see every iteration -- the loops below follow the
reference's control flow statement by statement (src/solvers/krylov.py:36-77,
:190-271; src/solvers/gmres.py:183-340). Every vector operation is still a
device kernel (Dense BLAS-1, SpMV, block-Jacobi); only the per-column scalar
recurrences (a few doubles) and the criterion calls are on the host.
"""

from __future__ import annotations

import numpy as np

from ..base import Identity
from ..stop import Updater
from .common import RELATIVE_STOPPING_ID, BreakdownInfo, active_mask


def safe_div(num, den):
    with np.errstate(divide="ignore", invalid="ignore"):
        out = np.asarray(num, dtype=np.float64) / np.asarray(den, dtype=np.float64)
    both = (np.asarray(den) == 0) & (np.asarray(num) == 0)
    return np.where(both, 0.0, out)


def _cols(status):
    act = active_mask(status)
    m = len(status.data)
    return list(range(m)) if act is None else [int(j) for j in np.flatnonzero(act)]


def _new(like, n, m):
    return like.like(n, m)


def _zero(d):
    d.fill(0.0)
    return d


def cg(s, b, x):
    n, m = s.size.rows, b.size.cols
    r, z, p, q = (_zero(_new(b, n, m)) for _ in range(4))
    s._residual(x, b, r)
    prev_rho = np.ones(m)
    s.precond.apply(r, z)
    rho = r.dot(z)
    crit = s._make_criterion(b, x, initial_residual=r)
    status = s._new_status(m)
    it, breakdown = 0, None
    while True:
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status, Updater(it, residual=r, solution=x))
        if all_stopped:
            break
        act = _cols(status)
        beta = safe_div(rho, prev_rho)
        for j in act:  # p = z + beta p
            pj = p.column(j)
            pj.scale(float(beta[j]))
            pj.add_scaled(1.0, z.column(j))
        s.a.apply(p, q)
        sigma = p.dot(q)
        running = ~status.data["stopped"]
        if ((sigma <= 0) & (rho != 0) & running).any():
            breakdown = BreakdownInfo(it + 1, "non-positive p^T A p")
            break
        alpha = safe_div(rho, sigma)
        for j in act:
            x.column(j).add_scaled(float(alpha[j]), p.column(j))
            r.column(j).add_scaled(-float(alpha[j]), q.column(j))
        prev_rho = rho
        s.precond.apply(r, z)
        rho = r.dot(z)
        it += 1
        s._log_iteration(it)
    s._finish(it, status, breakdown)


def fcg(s, b, x):
    """Flexible CG (src/solvers/krylov.py:80-125; steps FcgStep1/2, steps.py:161-199)."""
    n, m = s.size.rows, b.size.cols
    r, z, p, q, t = (_zero(_new(b, n, m)) for _ in range(5))
    s._residual(x, b, r)
    prev_rho, rho_t = np.ones(m), np.zeros(m)
    s.precond.apply(r, z)
    rho = r.dot(z)
    crit = s._make_criterion(b, x, initial_residual=r)
    status = s._new_status(m)
    it, breakdown = 0, None
    while True:
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status, Updater(it, residual=r, solution=x))
        if all_stopped:
            break
        act = _cols(status)
        beta = safe_div(rho_t, prev_rho)
        for j in act:  # p = z + (rho_t / prev_rho) p
            pj = p.column(j)
            pj.scale(float(beta[j]))
            pj.add_scaled(1.0, z.column(j))
        s.a.apply(p, q)
        sigma = p.dot(q)
        running = ~status.data["stopped"]
        if ((sigma <= 0) & (rho != 0) & running).any():
            breakdown = BreakdownInfo(it + 1, "non-positive p^T A p")
            break
        alpha = safe_div(rho, sigma)
        for j in act:  # x += alpha p; t = (r - alpha q) - r; r = r - alpha q
            x.column(j).add_scaled(float(alpha[j]), p.column(j))
            tj, rj = t.column(j), r.column(j)
            tj.copy_from(rj)
            rj.add_scaled(-float(alpha[j]), q.column(j))
            tj.scale(-1.0)
            tj.add_scaled(1.0, rj)
        prev_rho = rho
        s.precond.apply(r, z)
        rho = r.dot(z)
        rho_t = t.dot(z)
        it += 1
        s._log_iteration(it)
    s._finish(it, status, breakdown)


def _residual_nonzero(r, cols):
    return any(float(r.column(int(j)).norm2()[0]) != 0.0 for j in cols)


def cgs(s, b, x):
    """Conjugate gradient squared (src/solvers/krylov.py:128-187; steps
    CgsStep1/2/3, steps.py:246-345): two SpMVs per cycle, a criterion check
    after each half."""
    n, m = s.size.rows, b.size.cols
    r = _new(b, n, m)
    r.copy_from(b)
    rt = _new(b, n, m)
    rt.copy_from(b)
    p, q, u, u_hat, v_hat, t = (_zero(_new(b, n, m)) for _ in range(6))
    w = _zero(_new(b, n, m))
    prev_rho, alpha = np.ones(m), np.zeros(m)
    s.a.apply_advanced(-1.0, x, 1.0, r)
    crit = s._make_criterion(b, x, initial_residual=r)
    status = s._new_status(m)
    it, breakdown = 0, None
    while True:
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status, Updater(it, residual=r, solution=x))
        if all_stopped:
            break
        act = _cols(status)
        running = ~status.data["stopped"]
        rho = rt.dot(r)
        zero_rho = (rho == 0) & running
        if zero_rho.any() and _residual_nonzero(r, np.flatnonzero(zero_rho)):
            breakdown = BreakdownInfo(it + 1, "rho = 0")
            break
        beta = safe_div(rho, prev_rho)
        for j in act:  # u = r + beta q; p = u + beta (q + beta p)
            bj = float(beta[j])
            uj, pj = u.column(j), p.column(j)
            uj.copy_from(q.column(j))
            uj.scale(bj)
            uj.add_scaled(1.0, r.column(j))
            pj.scale(bj)
            pj.add_scaled(1.0, q.column(j))
            pj.scale(bj)
            pj.add_scaled(1.0, uj)
        s.precond.apply(p, t)
        s.a.apply(t, v_hat)
        gamma = rt.dot(v_hat)
        if ((gamma == 0) & (rho != 0) & running).any():
            breakdown = BreakdownInfo(it + 1, "r_tld^T A p = 0")
            break
        a_new = safe_div(rho, gamma)
        for j in act:  # q = u - alpha v_hat; w = u + q
            alpha[j] = a_new[j]
            qj, wj = q.column(j), w.column(j)
            qj.copy_from(u.column(j))
            qj.add_scaled(-float(alpha[j]), v_hat.column(j))
            wj.copy_from(u.column(j))
            wj.add_scaled(1.0, qj)
        it += 1
        s._log_iteration(it)
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status, Updater(it, residual=r, solution=x))
        if all_stopped:
            break
        act = _cols(status)
        s.precond.apply(w, u_hat)
        s.a.apply(u_hat, t)
        for j in act:  # r -= alpha t; x += alpha u_hat
            r.column(j).add_scaled(-float(alpha[j]), t.column(j))
            x.column(j).add_scaled(float(alpha[j]), u_hat.column(j))
        prev_rho = rho
        it += 1
        s._log_iteration(it)
    s._finish(it, status, breakdown)


def ir(s, b, x):
    """Iterative refinement x <- x + S(b - A x) (src/solvers/ir.py:13-46)."""
    n, m = s.size.rows, b.size.cols
    # d is the inner operator's initial guess: zero on the first iteration
    # (the reference's np.empty arena hands out zeroed pages here; verified
    # bitwise against a zero-filled run), the previous correction afterwards
    r, d = _new(b, n, m), _zero(_new(b, n, m))
    inner = s.params["inner_op"]
    s._residual(x, b, r)
    crit = s._make_criterion(b, x, initial_residual=r)
    status = s._new_status(m)
    it = 0
    while True:
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status, Updater(it, residual=r, solution=x))
        if all_stopped:
            break
        act = _cols(status)
        inner.apply(r, d)
        if len(act) == m:
            x.add_scaled(1.0, d)
        else:  # freeze stopped columns
            for j in act:
                x.column(j).add_scaled(1.0, d.column(j))
        s._residual(x, b, r)
        it += 1
        s._log_iteration(it)
    s._finish(it, status, None)


def bicgstab(s, b, x):
    n, m = s.size.rows, b.size.cols
    r = _new(b, n, m)
    r.copy_from(b)
    rt = _new(b, n, m)
    rt.copy_from(b)
    p, v, sv, t, y, z = (_zero(_new(b, n, m)) for _ in range(6))
    prev_rho, alpha, omega = np.ones(m), np.ones(m), np.ones(m)
    rho = np.zeros(m)
    s.a.apply_advanced(-1.0, x, 1.0, r)
    crit = s._make_criterion(b, x, initial_residual=r)
    status = s._new_status(m)
    it, breakdown = 0, None
    while True:
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status, Updater(it, residual=r, solution=x))
        if all_stopped:
            break
        act = _cols(status)
        running = ~status.data["stopped"]
        rho = rt.dot(r)
        zero_rho = (rho == 0) & running
        if zero_rho.any() and any(np.any(np.asarray(r.column(int(j)).data) != 0) for j in np.flatnonzero(zero_rho)):
            breakdown = BreakdownInfo(it + 1, "rho = 0")
            break
        beta = safe_div(rho, prev_rho) * safe_div(alpha, omega)
        for j in act:  # p = r + beta (p - omega v)
            pj = p.column(j)
            pj.add_scaled(-float(omega[j]), v.column(j))
            pj.scale(float(beta[j]))
            pj.add_scaled(1.0, r.column(j))
        s.precond.apply(p, y)
        s.a.apply(y, v)
        gamma = rt.dot(v)
        if ((gamma == 0) & (rho != 0) & running).any():
            breakdown = BreakdownInfo(it + 1, "r_tld^T A p = 0")
            break
        a_new = safe_div(rho, gamma)
        for j in act:
            alpha[j] = a_new[j]
            sj = sv.column(j)
            sj.copy_from(r.column(j))
            sj.add_scaled(-float(alpha[j]), v.column(j))
        it += 1
        s._log_iteration(it)
        before = status.data["stopped"].copy()
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status, Updater(it, residual=sv, solution=x))
        newly = status.data["stopped"] & ~before
        if newly.any() and crit.needs_residual:
            for j in np.flatnonzero(newly):
                x.column(int(j)).add_scaled(float(alpha[j]), y.column(int(j)))
        if all_stopped:
            break
        act = _cols(status)
        running = ~status.data["stopped"]
        s.precond.apply(sv, z)
        s.a.apply(z, t)
        ts, tt = t.dot(sv), t.dot(t)
        if ((tt == 0) & (ts != 0) & running).any():
            breakdown = BreakdownInfo(it + 1, "t^T t = 0")
            break
        w_new = safe_div(ts, tt)
        for j in act:
            omega[j] = w_new[j]
            xj = x.column(j)
            tmp = y.column(j).clone_to(y.exec)
            tmp.scale(float(alpha[j]))
            tmp.add_scaled(float(omega[j]), z.column(j))
            xj.add_scaled(1.0, tmp)
            rj = r.column(j)
            rj.copy_from(sv.column(j))
            rj.add_scaled(-float(omega[j]), t.column(j))
        prev_rho = rho
        it += 1
        s._log_iteration(it)
    s._finish(it, status, breakdown)


def gmres(s, b, x, k, exact_id=254):
    n, m = s.size.rows, b.size.cols
    use_precond = not isinstance(s.precond, Identity)
    r = _new(b, n, m)
    s._residual(x, b, r)
    V = [_zero(_new(b, n, m)) for _ in range(k + 1)]
    w = _new(b, n, m)
    zd = _new(b, n, m) if use_precond else None
    H = np.zeros((k + 1, k, m))
    cs, sn = np.zeros((k, m)), np.zeros((k, m))
    gamma = np.zeros((k + 1, m))
    res_est = np.zeros(m)
    jcol = np.zeros(m, dtype=int)

    def reset(cols):
        beta = r.norm2()
        for c in cols:
            gamma[:, c] = 0.0
            gamma[0, c] = beta[c]
            cs[:, c] = 0.0
            sn[:, c] = 0.0
            v0 = V[0].column(c)
            if beta[c] == 0:
                v0.fill(0.0)
            else:
                v0.copy_from(r.column(c))
                v0.scale(1.0 / float(beta[c]))
            res_est[c] = beta[c]
            jcol[c] = 0

    def back_solve(c, jc):
        y = np.zeros(jc)
        for i in reversed(range(jc)):
            d = H[i, i, c]
            if d == 0:
                return None
            y[i] = (gamma[i, c] - H[i, i + 1:jc, c] @ y[i + 1:jc]) / d
        return y

    def commit(cols_jc):
        for c, jc in cols_jc:
            if jc == 0:
                continue
            y = back_solve(c, jc)
            if y is None:
                return "singular Hessenberg system"
            u = _zero(_new(b, n, 1))
            for i in range(jc):
                u.add_scaled(float(y[i]), V[i].column(c))
            if use_precond:
                mu = _new(b, n, 1)
                s.precond.apply(u, mu)
                u = mu
            x.column(c).add_scaled(1.0, u)
        return None

    def declare_exact(cols):
        commit([(c, int(jcol[c])) for c in cols])
        status.data["stopped"][cols] = True
        status.data["stopping_id"][cols] = exact_id
        status.data["finalized"][cols] = True
        res_est[cols] = 0.0

    reset(range(m))
    crit = s._make_criterion(b, x, initial_residual=r)
    status = s._new_status(m)
    it, j, breakdown = 0, 0, None
    exact0 = [int(c) for c in np.flatnonzero(res_est == 0)]
    if exact0:
        declare_exact(exact0)
    while True:
        before = status.data["stopped"].copy()
        all_stopped, _ = crit.check(RELATIVE_STOPPING_ID, True, status,
                                    Updater(it, residual_norm=res_est.copy(), solution=x))
        newly = np.flatnonzero(status.data["stopped"] & ~before)
        if newly.size:
            err = commit([(int(c), int(jcol[c])) for c in newly])
            if err is not None:
                breakdown = BreakdownInfo(it, err)
                break
        if all_stopped:
            break
        running = [int(c) for c in np.flatnonzero(~status.data["stopped"])]
        j += 1
        if use_precond:
            s.precond.apply(V[j - 1], zd)
            s.a.apply(zd, w)
        else:
            s.a.apply(V[j - 1], w)
        for i in range(j):  # modified Gram-Schmidt
            hi = V[i].dot(w)
            for c in running:
                H[i, j - 1, c] = hi[c]
                w.column(c).add_scaled(-float(hi[c]), V[i].column(c))
        hj = w.norm2()
        happy = []
        for c in running:
            H[j, j - 1, c] = hj[c]
            vj = V[j].column(c)
            if hj[c] == 0:
                vj.fill(0.0)
                happy.append(c)
            else:
                vj.copy_from(w.column(c))
                vj.scale(1.0 / float(hj[c]))
            for i in range(j - 1):
                h1, h2 = H[i, j - 1, c], H[i + 1, j - 1, c]
                H[i, j - 1, c] = cs[i, c] * h1 + sn[i, c] * h2
                H[i + 1, j - 1, c] = -sn[i, c] * h1 + cs[i, c] * h2
            h1, h2 = H[j - 1, j - 1, c], H[j, j - 1, c]
            den = np.hypot(h1, h2)
            cc, ss = (h1 / den, h2 / den) if den != 0 else (1.0, 0.0)
            cs[j - 1, c], sn[j - 1, c] = cc, ss
            H[j - 1, j - 1, c], H[j, j - 1, c] = den, 0.0
            g = gamma[j - 1, c]
            gamma[j - 1, c], gamma[j, c] = cc * g, -ss * g
            res_est[c] = abs(gamma[j, c])
            jcol[c] = j
        it += 1
        s._log_iteration(it)
        if happy:
            declare_exact(happy)
            if status.data["stopped"].all():
                break
        if j == k:
            running = [int(c) for c in np.flatnonzero(~status.data["stopped"])]
            err = commit([(c, k) for c in running])
            if err is not None:
                breakdown = BreakdownInfo(it, err)
                break
            s._residual(x, b, r)
            prev = res_est.copy()
            reset(running)
            stopped = status.data["stopped"]
            res_est[stopped] = prev[stopped]
            j = 0
    s._finish(it, status, breakdown)
