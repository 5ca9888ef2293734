"""Lockstep Python emulation of warp_dtw (dtw_warp.cuh) for debugging on CPU."""
import math
import numpy as np

INF = math.inf


def warp_dtw(rows, cols, w, ub_fn, kill=False, rowthr=None, trace=False):
    lr, lc = len(rows), len(cols)
    qs = [0.0] + list(cols)
    rowbuf = [0.0] * (lc + 1)
    lo = hi = 0
    rowbuf[0] = 0.0
    result = INF
    ncell = 0
    i0 = 1
    while i0 <= lr:
        ub_strip = ub_fn()
        lanes = range(32)
        i = [i0 + L for L in lanes]
        active = [x <= lr for x in i]
        ub = [min(rowthr(ub_strip, i[L]) if rowthr else ub_strip, 1.7976931348623157e308) for L in lanes]
        c = [rows[i[L] - 1] if active[L] else 0.0 for L in lanes]
        last_lane = min(31, lr - i0)
        jb = max(lo, 1)
        bl = [max(max(1, i[L] - w), jb) for L in lanes]
        bh = [min(lc, i[L] + w) if active[L] else -1 for L in lanes]
        left = [INF] * 32
        v = [INF] * 32
        top_prev = [INF] * 32
        if jb - 1 >= lo and jb - 1 <= hi:
            top_prev[0] = rowbuf[jb - 1]
        fin = [not a for a in active]
        finmask = [f for f in fin]
        newlo = [10**9] * 32
        newhi = [-1] * 32
        j = [jb - L for L in lanes]
        while True:
            shfl = [INF] + v[:31]  # shfl_up: lane 0 keeps own value (irrelevant, replaced)
            shfl[0] = v[0]
            up_fin = [(j[0] > hi) if L == 0 else finmask[L - 1] for L in lanes]
            top = list(shfl)
            top[0] = rowbuf[j[0]] if (j[0] >= lo and j[0] <= hi) else INF
            diag = list(top_prev)
            top_prev = list(top)
            inb = [(not fin[L]) and j[L] >= bl[L] and j[L] <= bh[L] for L in lanes]
            nv = [INF] * 32
            for L in lanes:
                if inb[L]:
                    d = c[L] - qs[j[L]]
                    nv[L] = d * d + min(left[L], min(top[L], diag[L]))
            live = [nv[L] <= ub[L] for L in lanes]
            for L in lanes:
                if kill and not live[L]:
                    nv[L] = INF
                if live[L]:
                    newlo[L] = min(newlo[L], j[L])
                    newhi[L] = j[L]
                if L == last_lane and j[L] == lc and live[L] and i[L] == lr:
                    result = nv[L]
                if L == 31 and inb[L]:
                    rowbuf[j[L]] = nv[L]
            left = list(nv)
            v = list(nv)
            fin = [fin[L] or j[L] > bh[L] or (up_fin[L] and not live[L]) for L in lanes]
            ncell += sum(inb)
            finmask = list(fin)
            if all(fin):
                break
            j = [x + 1 for x in j]
        lo_n, hi_n = newlo[last_lane], newhi[last_lane]
        if trace:
            print("strip", i0, "lo,hi", lo_n, hi_n)
        if hi_n < 0:
            return INF, ncell
        lo, hi = lo_n, hi_n
        i0 += 32
    return result, ncell


if __name__ == "__main__":
    import sys
    sys.path.insert(0, "/root/repo")
    import oracle
    o = oracle.Oracle()
    rng = np.random.default_rng(1)
    bad = 0
    for it in range(300):
        la, lb = (int(x) for x in rng.integers(1, 70, 2))
        a = rng.uniform(-3, 3, la)
        b = rng.uniform(-3, 3, lb)
        w = int(rng.integers(0, 80)) if it % 3 else oracle.UNBOUNDED
        ub = rng.uniform(0, 60) if it % 2 else INF
        rows, cols = (a, b) if la >= lb else (b, a)
        lr, lc = len(rows), len(cols)
        if w != oracle.UNBOUNDED and lr - lc > w:
            continue
        weff = lr if (w == oracle.UNBOUNDED or w >= lc) else w
        got, _ = warp_dtw(rows, cols, weff, lambda: ub)
        want = o.ea_pruned_dtw_windowed(a, b, w, ub)
        if got != want:
            bad += 1
            if bad < 5:
                print("MISMATCH", it, la, lb, w, ub, got, want)
    print("bad", bad)
