"""Offline model of the leaf kernel's DtN op program (drop faces, engine orderings,
no interchanges): a Python mirror of ProgramBuilder (hps_leaf.cu) plus the
per-tile / per-warp chunk walk of gemm_t.  For every GEMM op it counts the k chunks
the CTA walks (tile start = the producer's bound) and the warp-chunk slots that
carry DMMAs (the warp's own bound), so tile geometries can be compared on CPU.

    python tools/r03/sim_program.py [p] [--geometries]

--geometries compares the wide tile's shape (rows x cols / warp grid / k granularity):
the fraction of the walked warp-chunk slots that carry DMMAs, edge waste included.
"""
import sys
import os
import collections

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2503_04033_b200.engine import interior_order, _first_nonzero, forward_prefix_rows  # noqa: E402

TN_SPLIT = 128
TRI = 64


def split16(w):
    A = TN_SPLIT
    half = w * 50 // 100
    if w > 2 * A:
        h = half // A * A
        return A if h < A else (w - A if h >= w else h)
    h = (half + 15) // 16 * 16
    return 16 if h < 16 else (w - 16 if h >= w else h)


class Geo:
    """tile geometry: TM x TN tile, warps WM x WN of (TM/WM) x (TN/WN), k chunk KC"""

    def __init__(self, name, TM, TN, KC, WM, WN):
        self.name, self.TM, self.TN, self.KC, self.WM, self.WN = name, TM, TN, KC, WM, WN


WIDE = Geo("wide64x128", 64, 128, 16, 2, 4)
NARROW = Geo("narrow256x32", 256, 32, 8, 8, 1)
TALL = Geo("tall128x64", 128, 64, 8, 4, 2)


def build(q, RW=256):
    n = q ** 3
    n_pad = (n + 15) // 16 * 16
    rowpos = interior_order(q, 3)
    g = _first_nonzero(rowpos, q, 3)
    gpos = np.arange(n_pad)
    gpos[rowpos] = g
    gmin16 = np.array([gpos[i:i + 16].min() for i in range(0, n_pad, 16)] + [1 << 30])
    f = forward_prefix_rows(q, 3)
    m = f.size
    m_pad = (m + 15) // 16 * 16
    fsort = np.full(m_pad, 1 << 30)
    fsort[:m] = np.sort(f, kind="stable")
    rhs_g = fsort.copy()  # suffix minima of a sorted array
    rhs_tab = np.array([int(np.searchsorted(fsort, 16 * e, side="left")) for e in range(n_pad // 16 + 1)])
    ops = []

    def gemm(kind, ar, ac, br, bc, cr, cc, M, N, K, dyn=0, kmode=-1, tag=""):
        if M <= 0 or N <= 0 or K <= 0:
            return
        ops.append(dict(kind=kind, ar=ar, ac=ac, br=br, bc=bc, cr=cr, cc=cc, M=M, N=N, K=K, dyn=dyn,
                        kmode=(kmode if kmode >= 0 else (1 if dyn else 0)), tag=tag))

    def small(c0, w):
        ops.append(dict(kind="small", a=c0, b=w))

    owner = {0: {}, 1: {}}

    def inv_cached(kind, r0, h):
        own = owner[kind]
        valid = all(own.get(gg) == (r0, h) for gg in range(r0 // 16, (r0 + h + 15) // 16))
        if valid:
            return
        for gg in range(r0 // 16, (r0 + h + 15) // 16):
            own[gg] = (r0, h)
        ops.append(dict(kind="inv", a=r0, b=h))

    st = dict(dyn_rhs=False)

    def trsm_lower(r0, h, lo, hi, colb=False, tag="lu_trsm"):
        if hi <= lo:
            return
        if h <= TRI:
            inv_cached(0, r0, h)
            gemm("set", r0, 0, r0, lo, r0, lo, h, hi - lo, h, r0 + h if st["dyn_rhs"] else 0, tag=tag + "_set")
            return
        h1 = split16(h)
        trsm_lower(r0, h1, lo, hi, colb, tag)
        gemm("sub", r0 + h1, r0, r0, lo, r0 + h1, lo, h - h1, hi - lo, h1, r0 + h1 if st["dyn_rhs"] else 0,
             (1 if st["dyn_rhs"] else 0) | 4 | (8 if colb else 0), tag=tag)
        trsm_lower(r0 + h1, h - h1, lo, hi, colb, tag)

    def trsm_right(c0, h, cst, M):
        if c0 + h <= cst:
            return
        if h <= TRI:
            inv_cached(1, c0, h)
            gemm("set_r", n_pad, c0, n_pad + c0, 0, n_pad, c0, M, h, h, 0, 2, tag="W_set")
            return
        h1 = split16(h)
        trsm_right(c0, h1, cst, M)
        k0 = max(c0, cst)
        if c0 + h1 > k0:
            gemm("sub", n_pad, k0, k0, c0 + h1, n_pad, c0 + h1, M, h - h1, c0 + h1 - k0, 0, 2 | 8, tag="W")
        trsm_right(c0 + h1, h - h1, cst, M)

    def lu(c0, w):
        if w <= 32:
            small(c0, w)
            return
        h = split16(w)
        lu(c0, h)
        trsm_lower(c0, h, c0 + h, c0 + w, True)
        gemm("sub", c0 + h, c0, c0, c0 + h, c0 + h, c0 + h, n_pad - c0 - h, w - h, h, 0, 12, tag="lu_update")
        lu(c0 + h, w - h)

    lu(0, n_pad)
    st["dyn_rhs"] = True
    trsm_lower(0, n_pad, n_pad, n_pad + m_pad, tag="forward")
    st["dyn_rhs"] = False
    for s0 in range(0, m, RW):
        R = min(RW, m - s0)
        cst = fsort[s0] // 16 * 16
        ops.append(dict(kind="wblock", a=s0, b=R))
        trsm_right(0, n_pad, cst, R)
        gemm("sub", n_pad, cst, cst, n_pad, n_pad, n_pad, R, m, n_pad - cst, 0, 3, tag="T")
        ops[-1]["s0"] = s0
    tabs = dict(n=n, n_pad=n_pad, m=m, m_pad=m_pad, gpos=gpos, gmin16=gmin16, fsort=fsort, rhs_g=rhs_g,
                rhs_tab=rhs_tab)
    return ops, tabs


def pick_geo(op):
    if op["kind"] == "sub" and op["N"] <= 64 and op["M"] >= 256 and op["K"] % 8 == 0:
        return NARROW
    if op["kind"] == "set_r" and op["N"] <= 64 and op["K"] % 8 == 0:
        return TALL
    return WIDE


def walk(op, T, G, wblock_s0=0):
    """(walked chunks x warps, active warp-chunks, executed flops, tiles) of one GEMM op"""
    n_pad = T["n_pad"]
    M, K = op["M"], op["K"]
    N = min(op["N"], T["rhs_tab"][op["dyn"] >> 4]) if op["dyn"] else op["N"]
    km, ar, ac, br, bc = op["kmode"], op["ar"], op["ac"], op["br"], op["bc"]
    TM, TN, KC, WM, WN = G.TM, G.TN, G.KC, G.WM, G.WN
    wr, wc = TM // WM, TN // WN
    kchunks = K // KC if K % KC == 0 else K // KC  # engine: K multiple of KC
    kchunks = max(kchunks, 1)
    gm16, gcol16, rhs_g = T["gmin16"], T["gmin16"], T["rhs_g"]
    fs = T["fsort"]

    def wf(r):  # W-block row r (slot row >= n_pad): first nonzero column
        i = r - n_pad
        return fs[wblock_s0 + i] if (wblock_s0 + i) < T["m"] else 1 << 30

    def bound(r0, r1, c0, c1):
        k = 0
        if km & 1:
            k = max(k, rhs_g[c0] - br)
        if km & 2:
            k = max(k, min(wf(r) for r in range(r0, r1)) - ac)
        if km & 4:
            k = max(k, min(gm16[r >> 4] for r in range(r0, r1, 16)) - ac)
        if km & 8:
            k = max(k, min(gcol16[c >> 4] for c in range(bc + c0, bc + c1, 16)) - br)
        return k

    walked = active = 0
    flops = 0.0
    ntiles = 0
    for tm in range((M + TM - 1) // TM):
        for tn in range((N + TN - 1) // TN):
            r0, r1 = ar + tm * TM, min(ar + tm * TM + TM, ar + M)
            c0, c1 = tn * TN, min(tn * TN + TN, N)
            kk = bound(r0, r1, c0, c1) if km else 0
            if (km & 4) and kk >= K:
                continue
            ntiles += 1
            kc0 = min(max(kk, 0) // KC, kchunks - 1)
            nch = kchunks - kc0
            walked += nch * WM * WN
            for wm in range(WM):
                for wn in range(WN):
                    rr0, rr1 = r0 + wm * wr, min(r0 + wm * wr + wr, ar + M)
                    cc0, cc1 = c0 + wn * wc, min(c0 + wn * wc + wc, N)
                    if rr1 <= rr0 or cc1 <= cc0:
                        continue
                    wk = bound(rr0, rr1, cc0, cc1) if km else 0
                    first = max(kc0, max(wk, 0) // KC)
                    if first < kchunks:
                        a = kchunks - first
                        active += a
                        flops += 2.0 * (rr1 - rr0) * (cc1 - cc0) * a * KC
    return walked, active, flops, ntiles


def geometries(p):
    ops, T = build(p - 2)
    geos = [Geo("64x128/2x4 k16", 64, 128, 16, 2, 4), Geo("64x128/2x4 k4", 64, 128, 4, 2, 4),
            Geo("128x64/4x2 k16", 128, 64, 16, 4, 2), Geo("32x256/1x8 k16", 32, 256, 16, 1, 8),
            Geo("128x128/4x4 k16", 128, 128, 16, 4, 4), Geo("128x256/4x8 k16", 128, 256, 16, 4, 8),
            Geo("64x64/2x2 k4", 64, 64, 4, 2, 2), Geo("256x32/8x1 k4", 256, 32, 4, 8, 1)]
    for G in geos:
        walked = fl_all = 0.0
        s0 = 0
        for o in ops:
            if o["kind"] == "wblock":
                s0 = o["a"]
            if o["kind"] not in ("sub", "set", "set_r"):
                continue
            g = pick_geo(o)
            if g is WIDE:
                g = G
            w, a, fl, nt = walk(o, T, g, s0)
            walked += w * (g.TM // g.WM) * (g.TN // g.WN) * g.KC * 2
            fl_all += fl
        print(f"{G.name:18s} executed {fl_all:.3e} flop/leaf, useful share of walked slots {fl_all / walked:.3f}")


def main():
    p = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    if "--geometries" in sys.argv:
        geometries(p)
        return
    ops, T = build(p - 2)
    cnt = collections.Counter(o["kind"] for o in ops)
    print(f"p={p}: {len(ops)} ops {dict(cnt)}")
    agg = collections.defaultdict(lambda: [0, 0, 0.0, 0, 0])
    s0 = 0
    for o in ops:
        if o["kind"] == "wblock":
            s0 = o["a"]
        if o["kind"] not in ("sub", "set", "set_r"):
            continue
        G = pick_geo(o)
        w, a, fl, nt = walk(o, T, G, s0)
        N = o["N"]
        key = (o["tag"], G.name)
        agg[key][0] += w
        agg[key][1] += a
        agg[key][2] += fl
        agg[key][3] += nt
        agg[key][4] += 1
    tw = ta = tf = 0
    for k, (w, a, fl, nt, no) in sorted(agg.items(), key=lambda kv: -kv[1][2]):
        print(f"{k[0]:14s} {k[1]:14s} ops {no:5d} tiles {nt:7d} exec {fl:.3e}  warp-slot use {a / max(w, 1):.3f}")
        tw += w
        ta += a
        tf += fl
    print(f"total exec {tf:.3e}, warp-slot use {ta / tw:.3f}")


if __name__ == "__main__":
    main()
