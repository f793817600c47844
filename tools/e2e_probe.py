"""Where the C2 e2e time goes (A.apply with pinned host b and x).

Times, with CUDA events around each variant (median of 20):
  * the production path (graph replay of the chunked H2D / SpMV / D2H pipeline),
  * the same issue sequence without the graph,
  * copy-engine transfers alone (H2D, D2H, both directions at once, in and out of a graph),
  * zero-copy alternatives: the SpMV writing x straight into the mapped pinned host
    buffer, and SM copy kernels (b200sp_copy) reading/writing host memory.

  python tools/e2e_probe.py
"""
import statistics
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2006_16852_b200 as b2  # noqa: E402
from paper_2006_16852_b200 import _lib, problems  # noqa: E402


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    out = []
    s = torch.cuda.current_stream()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


def make_plan(m, bounds):
    """Column chunks / waits for arbitrary row bounds (same rule as Csr._pipeline_plan)."""
    rp = m._rp.cpu().numpy()
    ci = m._ci
    k = len(bounds) - 1
    need = []
    for j in range(k):
        lo, hi = int(rp[bounds[j]]), int(rp[bounds[j + 1]])
        need.append(int(ci[lo:hi].max().item()) if hi > lo else -1)
    cb, hi = [0], 0
    ncol = m.size.cols
    for j in range(k - 1):
        hi = min(ncol, max(hi, need[j] + 1, cb[-1]))
        cb.append(hi)
    cb.append(ncol)
    wait = [next(i for i in range(k) if cb[i + 1] > nd) if nd >= 0 else -1 for nd in need]
    return {"rows": bounds, "cols": cb, "wait": wait}


def timeline(m, P, bt, xt, bd, xd, label, d2h_sm=False, reps=5, graph=False):
    """The pipeline with timing events after every copy and kernel (external
    event-record nodes when captured in a graph)."""
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    k = len(P["wait"])

    def issue(cur):
        E = lambda: torch.cuda.Event(enable_timing=True, external=graph)  # noqa: E731
        t0 = E()
        t0.record(cur)
        s_in.wait_stream(cur)
        s_out.wait_stream(cur)
        ein, eop, eout = [], [], []
        with torch.cuda.stream(s_in):
            for i in range(k):
                lo, hi = P["cols"][i], P["cols"][i + 1]
                bd[lo:hi].copy_(bt[lo:hi], non_blocking=True)
                e = E()
                e.record(s_in)
                ein.append(e)
        for j in range(k):
            r0, r1 = P["rows"][j], P["rows"][j + 1]
            cur.wait_event(ein[P["wait"][j]])
            _lib.call("csr_spmv_classical_f64", r1 - r0, m._rp.data_ptr() + 4 * r0, m._ci.data_ptr(),
                      m._v.data_ptr(), bd.data_ptr(), 1, xd.data_ptr() + 8 * r0, 1, 1.0, 0, 0.0, 0, 0, 0,
                      m.subwarp(), cur.cuda_stream)
            e = E()
            e.record(cur)
            eop.append(e)
            s_out.wait_event(e)
            if d2h_sm:
                _lib.call("copy_f64", r1 - r0, 1, xd.data_ptr() + 8 * r0, 1, xt.data_ptr() + 8 * r0, 1,
                          s_out.cuda_stream)
            else:
                with torch.cuda.stream(s_out):
                    xt[r0:r1].copy_(xd[r0:r1], non_blocking=True)
            e = E()
            e.record(s_out)
            eout.append(e)
        cur.wait_stream(s_in)
        cur.wait_stream(s_out)
        t1 = E()
        t1.record(cur)
        return t0, t1, ein, eop, eout

    best = None
    if graph:
        g = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            evs = issue(torch.cuda.current_stream())
    for _ in range(reps):
        if graph:
            g.replay()
        else:
            evs = issue(torch.cuda.current_stream())
        torch.cuda.synchronize()
        t0, t1, ein, eop, eout = evs
        tot = t0.elapsed_time(t1) * 1e3
        if best is None or tot < best[0]:
            best = (tot, [t0.elapsed_time(e) * 1e3 for e in ein], [t0.elapsed_time(e) * 1e3 for e in eop],
                    [t0.elapsed_time(e) * 1e3 for e in eout])
    tot, a, b, c = best
    print(f"[{label}{', graph' if graph else ''}] total {tot:.0f} us")
    print("   h2d  done:", " ".join(f"{v:.0f}" for v in a))
    print("   spmv done:", " ".join(f"{v:.0f}" for v in b))
    print("   d2h  done:", " ".join(f"{v:.0f}" for v in c))


def main():
    exc = b2.create_executor("cuda")
    a = problems.stencil(exc, "27pt", 128, value_dtype="float64")
    m = b2.convert(a, "csr")
    n = m.size.rows
    host = exc.master
    rng = np.random.default_rng(0)
    bh = b2.Dense(host, rng.standard_normal((n, 1)))
    xh = b2.Dense(host, np.zeros((n, 1)))
    bt = torch.from_numpy(np.asarray(bh.values).reshape(-1))
    xt = torch.from_numpy(np.asarray(xh.values).reshape(-1))
    print("pinned:", bt.is_pinned(), xt.is_pinned())
    bd = torch.empty(n, dtype=torch.float64, device="cuda")
    xd = torch.empty(n, dtype=torch.float64, device="cuda")
    cur = torch.cuda.current_stream()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def spmv(xp, r0=0, r1=n):
        _lib.call("csr_spmv_classical_f64", r1 - r0, m._rp.data_ptr() + 4 * r0, m._ci.data_ptr(), m._v.data_ptr(),
                  bd.data_ptr(), 1, xp + 8 * r0, 1, 1.0, 0, 0.0, 0, 0, 0, m.subwarp(), cur.cuda_stream)

    def copy_k(src, dst, cnt, st):
        _lib.call("copy_f64", cnt, 1, src, 1, dst, 1, st.cuda_stream)

    res = {}
    from paper_2006_16852_b200.formats import Csr
    for prod in (1, 2, 3, 4, 6):
        for per_sm in (1, 2, 3):
            _lib.set_tuning("hs_producers", prod)
            _lib.set_tuning("hs_per_sm", per_sm)
            res[f"host-stream kernel prod={prod} per_sm={per_sm}"] = timed(lambda: m.apply(bh, xh))
    # (a decomposition with probe-only kernel modes -- consumers not waiting, x
    # to device memory, no H2D -- measured 414 us H2D-only / 417 us D2H-only at 4
    # producers; profiles/r02_e2e_probe.txt)
    _lib.set_tuning("hs_producers", 32)
    _lib.set_tuning("hs_per_sm", 8)
    Csr.HOST_STREAM = "copies"
    for k in (4, 8, 16):
        m.HOST_PIPELINE_CHUNKS = k
        m._pplan = None
        res[f"apply graph k={k}"] = timed(lambda: m.apply(bh, xh))
    m.HOST_PIPELINE_CHUNKS = 8
    m._pplan = None
    P = m._pipeline_plan()
    res["issue (no graph) k=8"] = timed(lambda: m._pipeline_issue(P, bt, xt))
    res["spmv only"] = timed(lambda: spmv(xd.data_ptr()))
    res["h2d ce"] = timed(lambda: bd.copy_(bt, non_blocking=True))
    res["d2h ce"] = timed(lambda: xt.copy_(xd, non_blocking=True))

    def both_ce():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            bd.copy_(bt, non_blocking=True)
        with torch.cuda.stream(s2):
            xt.copy_(xd, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    res["both ce"] = timed(both_ce)
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g):
        both_ce()
    res["both ce (graph)"] = timed(g.replay)
    res["h2d sm copy"] = timed(lambda: copy_k(bt.data_ptr(), bd.data_ptr(), n, cur))
    res["d2h sm copy"] = timed(lambda: copy_k(xd.data_ptr(), xt.data_ptr(), n, cur))

    def both_sm():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        copy_k(bt.data_ptr(), bd.data_ptr(), n, s1)
        copy_k(xd.data_ptr(), xt.data_ptr(), n, s2)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    res["both sm copy"] = timed(both_sm)

    def h2d_ce_d2h_sm():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            bd.copy_(bt, non_blocking=True)
        copy_k(xd.data_ptr(), xt.data_ptr(), n, s2)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    res["h2d ce + d2h sm"] = timed(h2d_ce_d2h_sm)
    res["spmv -> host x (zero-copy)"] = timed(lambda: spmv(xt.data_ptr()))

    # pipeline variant: b up by copy engine in chunks, SpMV chunk writes x straight to host
    def zc_pipe(k=8):
        bounds = [n * j // k for j in range(k + 1)]
        cols, wait = P["cols"], P["wait"]
        kk = len(wait)
        s1.wait_stream(cur)
        evs = []
        with torch.cuda.stream(s1):
            for i in range(kk):
                lo, hi = cols[i], cols[i + 1]
                bd[lo:hi].copy_(bt[lo:hi], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
                evs.append(e)
        for j in range(kk):
            cur.wait_event(evs[wait[j]])
            spmv(xt.data_ptr(), P["rows"][j], P["rows"][j + 1])
        cur.wait_stream(s1)

    res["pipe: h2d ce, spmv writes host x"] = timed(zc_pipe)
    m.apply(bh, xh)
    torch.cuda.synchronize()
    ref = np.asarray(xh.values).copy()
    xt.zero_()
    zc_pipe()
    torch.cuda.synchronize()
    print("zero-copy pipe matches:", np.array_equal(np.asarray(xh.values), ref))
    # chunked copy-engine transfers: per-copy overhead alone and with the other direction busy
    def chunked(kc, dirs):
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        step = n // kc
        if "in" in dirs:
            with torch.cuda.stream(s1):
                for i in range(kc):
                    bd[i * step:(i + 1) * step].copy_(bt[i * step:(i + 1) * step], non_blocking=True)
        if "out" in dirs:
            with torch.cuda.stream(s2):
                for i in range(kc):
                    xt[i * step:(i + 1) * step].copy_(xd[i * step:(i + 1) * step], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    def graphed(fn):
        gg = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(gg):
            fn()
        return gg

    def mixed(kin, kout):
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            st = n // kin
            for i in range(kin):
                hi = n if i == kin - 1 else (i + 1) * st
                bd[i * st:hi].copy_(bt[i * st:hi], non_blocking=True)
        with torch.cuda.stream(s2):
            st = n // kout
            for i in range(kout):
                hi = n if i == kout - 1 else (i + 1) * st
                xt[i * st:hi].copy_(xd[i * st:hi], non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    for kin, kout in ((1, 1), (8, 1), (1, 8), (8, 8), (16, 1), (1, 16), (4, 4), (8, 2), (2, 8)):
        gg = graphed(lambda: mixed(kin, kout))
        print(f"mixed in={kin:2d} out={kout:2d}: graph {timed(gg.replay) * 1e3:6.1f} us")

    for kc in (1, 8, 16, 32, 64):
        row = []
        for dirs in (("in",), ("out",), ("in", "out")):
            gg = graphed(lambda: chunked(kc, dirs))
            row.append(timed(lambda: chunked(kc, dirs)) * 1e3)
            row.append(timed(gg.replay) * 1e3)
        print(f"chunks {kc:3d}: h2d {row[0]:6.1f} / graph {row[1]:6.1f} us  d2h {row[2]:6.1f} / {row[3]:6.1f} us  "
              f"both {row[4]:6.1f} / {row[5]:6.1f} us")

    # SpMV (full) while a big H2D / D2H is in flight on other streams
    def spmv_during(kind):
        s1.wait_stream(cur)
        with torch.cuda.stream(s1):
            if kind == "h2d":
                bd2.copy_(bt, non_blocking=True)
            else:
                xt.copy_(xd2, non_blocking=True)
        a, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(cur)
        spmv(xd.data_ptr())
        b_.record(cur)
        cur.wait_stream(s1)
        torch.cuda.synchronize()
        return a.elapsed_time(b_) * 1e3

    bd2 = torch.empty_like(bd)
    xd2 = torch.empty_like(xd)
    for kind in ("h2d", "d2h"):
        ts = [spmv_during(kind) for _ in range(6)]
        print(f"spmv during {kind}: {statistics.median(ts):.1f} us")
    r1 = n // 8
    print("spmv 1/8 chunk alone:", f"{timed(lambda: spmv(xd.data_ptr(), 0, r1)) * 1e3:.1f} us")
    print("plan k=8:", make_plan(m, [n * j // 8 for j in range(9)]))

    # timeline of the non-graph issue: event times relative to the start
    for k in (8, 16):
        timeline(m, make_plan(m, [n * j // k for j in range(k + 1)]), bt, xt, bd, xd, f"uniform k={k}")
    timeline(m, make_plan(m, [n * j // 8 for j in range(9)]), bt, xt, bd, xd, "uniform k=8, d2h sm", True)
    # small first / last chunks: the pipeline fill and drain are one small chunk each
    fr = [0, 1 / 32, 1 / 8, 1 / 4, 3 / 8, 1 / 2, 5 / 8, 3 / 4, 7 / 8, 15 / 16, 31 / 32, 1]
    nb = sorted(set(int(n * f) // 256 * 256 for f in fr[:-1])) + [n]
    timeline(m, make_plan(m, nb), bt, xt, bd, xd, "tapered")
    timeline(m, make_plan(m, nb), bt, xt, bd, xd, "tapered, d2h sm", True)
    for k in (8, 16):
        timeline(m, make_plan(m, [n * j // k for j in range(k + 1)]), bt, xt, bd, xd, f"uniform k={k}", graph=True)
    scheds = {"S2 1/8x6 1/16x4": [2] * 6 + [1] * 4, "S3 3/16x4 1/8 1/16x2": [3] * 4 + [2, 1, 1],
              "S4 1/16 1/8x7 1/16": [1] + [2] * 7 + [1], "S5 1/16 3/16x4 1/8 1/16": [1, 3, 3, 3, 3, 2, 1],
              "S6 1/16 3/16x5": [1] + [3] * 5, "S7 3/16x5 1/16": [3] * 5 + [1], "S8 1/8x7 1/16x2": [2] * 7 + [1] * 2,
              "S9 1/16x2 1/8x7": [1, 1] + [2] * 7, "S10 5/32 ... 3/32": [5] * 5 + [4, 3]}
    for name, w in scheds.items():
        tot = sum(w)
        acc = np.cumsum([0] + w)
        nb = [int(n * a // tot) // 256 * 256 for a in acc[:-1]] + [n]
        timeline(m, make_plan(m, nb), bt, xt, bd, xd, name, graph=True)
    timeline(m, make_plan(m, nb), bt, xt, bd, xd, "tapered", graph=True)
    timeline(m, make_plan(m, nb), bt, xt, bd, xd, "tapered, d2h sm", True, graph=True)
    by = n * 8
    for k, v in res.items():
        print(f"{k:40s} {v * 1e3:8.1f} us")
    print(f"(b and x are {by / 1e6:.1f} MB each)")


if __name__ == "__main__":
    main()
