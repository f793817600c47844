"""Generate the golden vectors by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py
The reference (`opalg`, pure Python + NumPy 2.3.5) is imported read-only from
/root/reference/pkg/src; its outputs on seeded inputs are written to
tests/golden/*.npz, which travel with the repo (the GPU box has no
/root/reference). Inputs for systems the reference cannot generate itself
(3-D stencils, power law) come from oracle/problems.py and are fed to the
reference's own MatrixData / Csr / Coo / solvers.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import opalg  # noqa: E402  (the reference)
from opalg import (Bicgstab, Cg, Coo, Csr, Dense, Dim2, Gmres, Iteration, Jacobi,  # noqa: E402
                   MatrixData, ResidualNormReduction)
from opalg.solvers import Cgs, Fcg, Ir  # noqa: E402
from opalg.problems import (convection_diffusion, five_point_poisson, random_sparse,  # noqa: E402
                            random_spd, tridiagonal)
from opalg.stop import Criterion, CriterionFactory  # noqa: E402

from oracle import problems as P  # noqa: E402

REF = opalg.ReferenceExecutor()


def triples(d):
    d = d.canonicalize()
    return d.size.rows, d.rows, d.cols, d.vals


def md(n, r, c, v):
    return MatrixData(Dim2(n, n), r, c, v)


# ---------------------------------------------------------------------------
def spmv_cases():
    out = {}

    def add(name, n, r, c, v, b, adv=None):
        data = md(n, r, c, v).canonicalize()
        b = np.asarray(b, dtype=np.float64)
        if b.ndim == 1:
            b = b[:, None]
        rec = {"n": n, "rows": data.rows, "cols": data.cols, "vals": data.vals, "b": b}
        for fmt in ("csr", "coo"):
            a = opalg.matrix_from_data(REF, data, fmt)
            x = Dense.zeros(REF, n, b.shape[1])
            a.apply(Dense(REF, b), x)
            rec["x_" + fmt] = x.data.copy()
            if adv is not None:
                alpha, beta, x0 = adv
                xa = Dense(REF, x0.copy())
                a.apply_advanced(Dense(REF, [[alpha]]), Dense(REF, b), Dense(REF, [[beta]]), xa)
                rec["xadv_" + fmt] = xa.data.copy()
                rec["adv"] = np.array([alpha, beta])
                rec["x0"] = x0
        out[name] = rec

    n, r, c, v = triples(tridiagonal(3))
    add("tri3", n, r, c, v, [1.0, 2.0, 3.0])
    for seed, n_, dens in ((5, 12, 0.3), (7, 24, 0.5), (11, 1, 1.0), (13, 64, 0.05)):
        n, r, c, v = triples(random_sparse(n_, density=dens, seed=seed, diag_dominant=False))
        b = np.random.default_rng(seed).standard_normal(n)
        x0 = np.random.default_rng(seed + 1).standard_normal((n, 1))
        add(f"rand{seed}", n, r, c, v, b, adv=(0.5, -2.0, x0))
    n, r, c, v = triples(five_point_poisson(31))
    add("poisson31", n, r, c, v, np.random.default_rng(0).standard_normal(n))
    n, r, c, v = P.stencil3d(8, "27pt")
    add("st27_g8", n, r, c, v, np.random.default_rng(0).standard_normal(n))
    n, r, c, v = P.stencil3d(10, "convdiff")
    add("convdiff_g10", n, r, c, v, np.random.default_rng(1).standard_normal(n))
    n, r, c, v = P.power_law(3000, seed=3, max_len=700)
    add("powerlaw3000", n, r, c, v, np.random.default_rng(2).standard_normal(n))
    # empty rows + multi-RHS
    rng = np.random.default_rng(17)
    n = 50
    dense = np.where(rng.random((n, n)) < 0.2, rng.uniform(-1, 1, (n, n)), 0.0)
    dense[[0, 7, 8, 9, 49]] = 0.0
    d = MatrixData.from_dense_array(dense)
    add("empty_rows", n, d.rows, d.cols, d.vals, rng.standard_normal((n, 3)))
    return out


# ---------------------------------------------------------------------------
class _History(Criterion):
    def __init__(self, sink):
        super().__init__()
        self.sink = sink

    def check(self, stopping_id, set_finalized, status, updater):
        if updater.residual_norm is not None:
            self.sink.append(np.asarray(updater.residual_norm, dtype=float).copy())
        elif updater.residual is not None:
            r = updater.residual.data
            self.sink.append(np.sqrt(np.einsum("ij,ij->j", r, r)))
        return False, False


class _HistoryFactory(CriterionFactory):
    def __init__(self):
        self.rows = []

    def generate(self, args):
        self.rows = []
        return _History(self.rows)


def solve_case(name, data, solver, precond, b, crit_iters, factor, **kw):
    a = Csr.from_data(REF, data)
    n = a.size.rows
    bd = Dense(REF, b.reshape(n, -1))
    x = Dense.zeros(REF, n, bd.size.cols)
    hist = _HistoryFactory()
    crits = [Iteration(crit_iters), ResidualNormReduction(factor), hist]
    fac = {"cg": Cg, "bicgstab": Bicgstab, "gmres": Gmres, "fcg": Fcg, "cgs": Cgs, "ir": Ir}[solver]
    pre = Jacobi(REF, block_size=precond) if precond else None
    if pre is not None:
        kw["preconditioner"] = pre
    s = fac(REF, criteria=crits, **kw).generate(a)
    s.apply(bd, x)
    st = s.last_status
    true_r = bd.data - data.to_dense_array() @ x.data if n <= 5000 else None
    if true_r is None:
        # sparse true residual via the reference's own Csr
        ax = Dense.zeros(REF, n, bd.size.cols)
        a.apply(x, ax)
        true_r = bd.data - ax.data
    rec = {
        "iterations": np.array(st.iterations),
        "stopping_id": np.array(st.stopping_id),
        "breakdown": np.array(st.breakdown is not None),
        "history": np.array(hist.rows),
        "x": x.data.copy(),
        "true_res": np.linalg.norm(true_r, axis=0),
        "b": b,
    }
    print(f"  {name}: iterations={st.iterations} stop_id={st.stopping_id} "
          f"breakdown={st.breakdown}")
    return rec


def solver_cases():
    out = {}
    n, r, c, v = triples(five_point_poisson(256))
    d = md(n, r, c, v)
    out["cg_c1"] = solve_case("cg_c1", d, "cg", 0, np.ones(n), 10000, 1e-8)
    for g in (16,):
        n, r, c, v = P.stencil3d(g, "7pt")
        d = md(n, r, c, v)
        out[f"cg_7pt_g{g}"] = solve_case(f"cg_7pt_g{g}", d, "cg", 0, np.ones(n), 10000, 1e-8)
        out[f"cg_bj32_7pt_g{g}"] = solve_case(f"cg_bj32_7pt_g{g}", d, "cg", 32, np.ones(n), 10000, 1e-8)
    for g in (12,):
        n, r, c, v = P.stencil3d(g, "convdiff")
        d = md(n, r, c, v)
        for pre in (0, 32):
            tag = "bj32" if pre else "none"
            out[f"bicgstab_{tag}_cd_g{g}"] = solve_case(f"bicgstab_{tag}_cd_g{g}", d, "bicgstab", pre,
                                                        np.ones(n), 10000, 1e-8)
            out[f"gmres30_{tag}_cd_g{g}"] = solve_case(f"gmres30_{tag}_cd_g{g}", d, "gmres", pre,
                                                       np.ones(n), 10000, 1e-8, krylov_dim=30)
    # larger systems (iteration counts / histories; SURVEY 8(c) probes)
    for g in (32, 64, 128):
        n, r, c, v = P.stencil3d(g, "7pt")
        rec = solve_case(f"cg_7pt_g{g}", md(n, r, c, v), "cg", 0, np.ones(n), 10000, 1e-8)
        if g > 32:
            rec.pop("x")
        out[f"cg_7pt_g{g}"] = rec
    n, r, c, v = P.stencil3d(32, "convdiff")
    d = md(n, r, c, v)
    for pre in (0, 32):
        tag = "bj32" if pre else "none"
        for name, solver, kw in (("bicgstab", "bicgstab", {}), ("gmres30", "gmres", {"krylov_dim": 30})):
            rec = solve_case(f"{name}_{tag}_cd_g32", d, solver, pre, np.ones(n), 10000, 1e-8, **kw)
            rec.pop("x")
            out[f"{name}_{tag}_cd_g32"] = rec
    # multi-column freeze (tests/test_solvers.py:218-248 pattern)
    data = random_spd(8, seed=11)
    dense = data.to_dense_array()
    w, vecs = np.linalg.eigh(dense)
    b2 = np.stack([dense @ vecs[:, 0], np.ones(8)], axis=1)
    out["cg_freeze"] = solve_case("cg_freeze", data.canonicalize(), "cg", 0, b2, 60, 1e-10)
    # nonsymmetric small system, restarted GMRES and BiCGSTAB
    data = random_sparse(100, density=0.1, seed=6)
    b = np.random.default_rng(6).standard_normal(100)
    out["gmres10_rand100"] = solve_case("gmres10_rand100", data.canonicalize(), "gmres", 0, b, 3000,
                                        1e-12, krylov_dim=10)
    out["bicgstab_rand100"] = solve_case("bicgstab_rand100", data.canonicalize(), "bicgstab", 0, b, 3000,
                                         1e-12)
    return out


def solver_ext_cases():
    """Fcg / Cgs / Ir: iteration counts, histories, x."""
    out = {}
    n, r, c, v = P.stencil3d(16, "7pt")
    d = md(n, r, c, v)
    for pre in (0, 32):
        tag = "bj32" if pre else "none"
        out[f"fcg_{tag}_7pt_g16"] = solve_case(f"fcg_{tag}_7pt_g16", d, "fcg", pre, np.ones(n), 10000, 1e-8)
    n, r, c, v = P.stencil3d(12, "convdiff")
    d = md(n, r, c, v)
    for pre in (0, 32):
        tag = "bj32" if pre else "none"
        out[f"cgs_{tag}_cd_g12"] = solve_case(f"cgs_{tag}_cd_g12", d, "cgs", pre, np.ones(n), 10000, 1e-8)
    # Ir with an inner CG of 4 iterations, and with a block-Jacobi inner operator
    n, r, c, v = P.stencil3d(12, "7pt")
    d = md(n, r, c, v)
    out["ir_cg4_7pt_g12"] = solve_case("ir_cg4_7pt_g12", d, "ir", 0, np.ones(n), 10000, 1e-8,
                                       inner=Cg(REF, criteria=[Iteration(4)]))
    n, r, c, v = P.stencil3d(12, "convdiff")
    d = md(n, r, c, v)
    out["ir_bj32_cd_g12"] = solve_case("ir_bj32_cd_g12", d, "ir", 0, np.ones(n), 10000, 1e-8,
                                       inner=Jacobi(REF, block_size=32))
    # multi-column freeze through Fcg and Cgs
    data = random_spd(8, seed=11)
    dense = data.to_dense_array()
    w, vecs = np.linalg.eigh(dense)
    b2 = np.stack([dense @ vecs[:, 0], np.ones(8)], axis=1)
    out["fcg_freeze"] = solve_case("fcg_freeze", data.canonicalize(), "fcg", 0, b2, 60, 1e-10)
    data = random_sparse(100, density=0.1, seed=6)
    b = np.random.default_rng(6).standard_normal(100)
    out["cgs_rand100"] = solve_case("cgs_rand100", data.canonicalize(), "cgs", 0, b, 3000, 1e-12)
    return out


def assemble_cases():
    """MatrixData.canonicalize on unsorted triples with duplicates (device
    assembly parity): several sizes, a lone -0.0, exact cancellations."""
    out = {}
    rng = np.random.default_rng(21)
    for name, (nr, nc, k) in {"small": (7, 5, 40), "mid": (300, 200, 20000), "wide": (3, 100000, 50000),
                              "tall": (70000, 3, 60000), "nodup": (1000, 1000, 0)}.items():
        if name == "nodup":
            idx = rng.choice(1000 * 1000, 5000, replace=False)
            r, c = idx // 1000, idx % 1000
        else:
            r = rng.integers(0, nr, k)
            c = rng.integers(0, nc, k)
        v = rng.standard_normal(r.size) * 10.0 ** rng.integers(-8, 8, r.size)
        v[::97] = -0.0
        if name == "mid":
            v[1::50] = -v[0::50][: v[1::50].size]  # exact cancellations where coordinates repeat
        d = MatrixData(Dim2(nr, nc), r, c, v).canonicalize()
        out[name] = {"size": np.array([nr, nc]), "rows_in": r, "cols_in": c, "vals_in": v,
                     "rows": d.rows, "cols": d.cols, "vals": d.vals}
    return out


def ilu_cases():
    """ParIlu factors (several sweep counts), triangular solves and
    ILU-preconditioned solves."""
    from opalg.precond import Ilu, ParIlu
    from opalg.solvers import LowerTrs, UpperTrs

    out = {}
    rng = np.random.default_rng(31)
    mats = {"cd5": P.stencil3d(5, "convdiff"), "p2d8": P.five_point(8)}
    d = random_sparse(40, density=0.15, seed=7).canonicalize()
    mats["rand40"] = (40, d.rows, d.cols, d.vals)
    for name, (n, r, c, v) in mats.items():
        a = Csr.from_data(REF, md(n, r, c, v))
        for sw in (0, 1, 3, 2 * n):
            f = ParIlu(REF, sweeps=sw).generate(a)
            out[f"parilu_{name}_s{sw}"] = {
                "l_rp": f.l.row_ptrs, "l_ci": f.l.col_idxs, "l_v": f.l.vals,
                "u_rp": f.u.row_ptrs, "u_ci": f.u.col_idxs, "u_v": f.u.vals,
                "defect": np.array(f.defect_on_pattern(a)), "sweeps": np.array(sw)}
        f = ParIlu(REF, sweeps=2 * n).generate(a)
        b = rng.standard_normal((n, 2))
        xl = Dense.zeros(REF, n, 2)
        LowerTrs(REF, unit_diagonal=True).generate(f.l).apply(Dense(REF, b), xl)
        xu = Dense.zeros(REF, n, 2)
        UpperTrs(REF).generate(f.u).apply(Dense(REF, b), xu)
        xz = Dense.zeros(REF, n, 2)
        Ilu(REF, sweeps=2 * n).generate(a).apply(Dense(REF, b), xz)
        out[f"trs_{name}"] = {"b": b, "xl": xl.data.copy(), "xu": xu.data.copy(), "xilu": xz.data.copy()}
    # ILU-preconditioned Krylov solves (5 sweeps, the default)
    for name, kind, solver in (("cg_ilu_7pt_g8", "7pt", "cg"), ("bicgstab_ilu_cd_g8", "convdiff", "bicgstab"),
                               ("gmres_ilu_cd_g8", "convdiff", "gmres")):
        n, r, c, v = P.stencil3d(8, kind)
        a = Csr.from_data(REF, md(n, r, c, v))
        fac = {"cg": Cg, "bicgstab": Bicgstab, "gmres": Gmres}[solver]
        hist = _HistoryFactory()
        s = fac(REF, criteria=[Iteration(1000), ResidualNormReduction(1e-10), hist],
                preconditioner=Ilu(REF)).generate(a)
        x = Dense.zeros(REF, n, 1)
        s.apply(Dense(REF, np.ones((n, 1))), x)
        st = s.last_status
        print(f"  {name}: iterations={st.iterations}")
        out[name] = {"iterations": np.array(st.iterations), "stopping_id": np.array(st.stopping_id),
                     "x": x.data.copy(), "history": np.array(hist.rows)}
    return out


def jacobi_cases():
    out = {}
    n, r, c, v = P.stencil3d(8, "convdiff")
    data = md(n, r, c, v)
    a = Csr.from_data(REF, data)
    for adaptive in (False, True):
        jac = Jacobi(REF, block_size=32, adaptive_precision=adaptive, condition_threshold=1e2).generate(a)
        out[f"convdiff_g8_bs32_adapt{int(adaptive)}"] = {
            "rows": data.canonicalize().rows, "cols": data.canonicalize().cols,
            "vals": data.canonicalize().vals, "n": n,
            "inv": np.stack([b.inv.astype(np.float64) for b in jac.blocks]),
            "reduced": np.array([b.inv.dtype == np.float32 for b in jac.blocks]),
            "cond": np.array(jac.block_conditions),
        }
    # pivoting-heavy random blocks, uneven last block
    d = random_sparse(60, density=0.4, seed=21, diag_dominant=False).canonicalize()
    a = Csr.from_data(REF, d)
    jac = Jacobi(REF, block_size=16).generate(a)
    rr = np.random.default_rng(4).standard_normal((60, 1))
    z = Dense.zeros(REF, 60, 1)
    jac.apply(Dense(REF, rr), z)
    out["rand60_bs16"] = {
        "rows": d.rows, "cols": d.cols, "vals": d.vals, "n": 60,
        "inv_flat": np.concatenate([b.inv.reshape(-1) for b in jac.blocks]),
        "cond": np.array(jac.block_conditions), "r": rr, "z": z.data.copy(),
    }
    return out


def jacobi_large_cases():
    """Blocks of more than 32 rows (uniform block_size and explicit
    boundaries, incl. a block over 128 rows for NumPy's recursive pairwise
    row sums), adaptive precision, the apply, and a preconditioned solve."""
    out = {}
    n, r, c, v = P.stencil3d(8, "convdiff")
    data = md(n, r, c, v)
    a = Csr.from_data(REF, data)
    d = data.canonicalize()
    rr = np.random.default_rng(8).standard_normal((n, 2))
    for name, kw in (("bs64", {"block_size": 64}), ("bs100", {"block_size": 100}),
                     ("bounds", {"block_boundaries": [0, 5, 37, 40, 240, 300, 301, 420]}),
                     ("bs64_adapt", {"block_size": 64, "adaptive_precision": True, "condition_threshold": 1e2})):
        jac = Jacobi(REF, **kw).generate(a)
        z = Dense.zeros(REF, n, 2)
        jac.apply(Dense(REF, rr), z)
        out[f"convdiff_g8_{name}"] = {
            "rows": d.rows, "cols": d.cols, "vals": d.vals, "n": n,
            "starts": np.array([b.start for b in jac.blocks]),
            "inv_flat": np.concatenate([b.inv.astype(np.float64).reshape(-1) for b in jac.blocks]),
            "reduced": np.array([b.inv.dtype == np.float32 for b in jac.blocks]),
            "cond": np.array(jac.block_conditions), "r": rr, "z": z.data.copy(),
        }
    # pivoting-heavy dense-ish random matrix, one 150-row block + a 50-row block
    dr = random_sparse(200, density=0.3, seed=23, diag_dominant=False).canonicalize()
    jac = Jacobi(REF, block_boundaries=[0, 150]).generate(Csr.from_data(REF, dr))
    out["rand200_b150"] = {
        "rows": dr.rows, "cols": dr.cols, "vals": dr.vals, "n": 200,
        "inv_flat": np.concatenate([b.inv.reshape(-1) for b in jac.blocks]),
        "cond": np.array(jac.block_conditions),
    }
    n, r, c, v = P.stencil3d(12, "convdiff")
    dd = md(n, r, c, v)
    out["bicgstab_bj64_cd_g12"] = solve_case("bicgstab_bj64_cd_g12", dd, "bicgstab", 64, np.ones(n), 10000, 1e-8)
    out["gmres30_bj144_cd_g12"] = solve_case("gmres30_bj144_cd_g12", dd, "gmres", 144, np.ones(n), 10000, 1e-8,
                                             krylov_dim=30)
    out["cg_bj64_7pt_g12"] = solve_case("cg_bj64_7pt_g12", md(*P.stencil3d(12, "7pt")), "cg", 64, np.ones(1728),
                                        10000, 1e-8)
    return out


def misc_cases():
    out = {}
    n, r, c, v = triples(convection_diffusion(20))
    out["convdiff1d_20"] = {"rows": r, "cols": c, "vals": v}
    n, r, c, v = triples(five_point_poisson(256))
    import hashlib
    h = hashlib.sha256()
    for arr in (r.astype(np.int64), c.astype(np.int64), v.astype(np.float64)):
        h.update(arr.tobytes())
    out["poisson256_sha256"] = {"digest": np.frombuffer(bytes.fromhex(h.hexdigest()), dtype=np.uint8)}
    return out


def save(name, cases):
    flat = {}
    for case, rec in cases.items():
        for k, val in rec.items():
            flat[f"{case}__{k}"] = np.asarray(val)
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **flat)
    print(f"wrote {path} ({os.path.getsize(path) // 1024} KiB)")


if __name__ == "__main__":
    if sys.argv[1:] == ["ext"]:
        save("solvers_ext.npz", solver_ext_cases())
        sys.exit(0)
    if sys.argv[1:] == ["ilu"]:
        save("ilu.npz", ilu_cases())
        sys.exit(0)
    if sys.argv[1:] == ["jacobi_large"]:
        save("jacobi_large.npz", jacobi_large_cases())
        sys.exit(0)
    if sys.argv[1:] == ["assemble"]:
        save("assemble.npz", assemble_cases())
        sys.exit(0)
    save("assemble.npz", assemble_cases())
    save("solvers_ext.npz", solver_ext_cases())
    save("spmv.npz", spmv_cases())
    save("misc.npz", misc_cases())
    save("jacobi.npz", jacobi_cases())
    save("solvers.npz", solver_cases())
