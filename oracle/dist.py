"""Distributed-scheme oracle (permuted partitions + reduced system).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Restates
/root/reference/pkg/src/btasel/{partition,dist}.py; every rank is simulated
in-process, in rank order, with a list standing in for the AllGather and a
rank-ordered sum for the AllReduce (collectives.py:149-158).
"""

from __future__ import annotations

import numpy as np

from .seq import Blocks, C128, OracleSingular, _Mul, backward, forward

_COST = {"si": (9, 20), "siq": (42, 94)}  # partition.py:19


def plan_partitions(n, parts, mode="si"):
    """partition.py:52-90 -> list of (lo, hi) and kinds."""
    if mode not in _COST:
        raise ValueError(mode)
    if parts < 2 or n < 2 * parts:
        raise ValueError("bad partition request")
    ce, cm = _COST[mode]
    nm = parts - 2
    if nm == 0:
        sizes = [(n + 1) // 2, n - (n + 1) // 2]
    else:
        mid = max(2, round(n * cm / (2 * cm + nm * ce) * ce / cm))
        while n - nm * mid < 4:
            mid -= 1
        rest = n - nm * mid
        sizes = [(rest + 1) // 2] + [mid] * nm + [rest - (rest + 1) // 2]
    bounds = np.concatenate([[0], np.cumsum(sizes)]).astype(int)
    ranges = [(int(bounds[p]), int(bounds[p + 1])) for p in range(parts)]
    kinds = ["first"] + ["middle"] * nm + ["last"]
    return ranges, kinds


class _Local:
    """Per-rank retained elimination data (dist.py:134-151)."""

    def __init__(self):
        self.s_a, self.s_b = {}, {}
        self.ar, self.ac, self.br, self.bc = {}, {}, {}, {}
        self.fr, self.fc, self.bfr, self.bfc = {}, {}, {}, {}


def _end_forward(A, B, lo, hi, downward, mul, st):
    """First (downward) / last (upward) partition elimination (dist.py:211-307).

    Downward eliminates lo..hi-2 into hi-1 (neighbour j = i+1, couplings
    L = lower[i] below, U = upper[i] above); upward eliminates hi-1..lo+1
    into lo (j = i-1, L = upper[i-1], U = lower[i-1]).
    """
    ad, ar, ac, bd, br, bc, tip_a, tip_b, fac = st
    fz = B is not None
    steps = range(lo, hi - 1) if downward else range(hi - 1, lo, -1)
    for i in steps:
        j = i + 1 if downward else i - 1
        e = i if downward else i - 1
        Lk, Uk = (A.lower[e], A.upper[e]) if downward else (A.upper[e], A.lower[e])
        S = mul.inv(ad[i], i)
        fac.s_a[i] = S
        fac.ar[i], fac.ac[i] = ar[i], ac[i]
        if fz:
            fac.br[i], fac.bc[i] = br[i], bc[i]
            BL, BU = (B.lower[e], B.upper[e]) if downward else (B.upper[e], B.lower[e])
            sb = mul(mul(S, bd[i]), S, hy=True)
            fac.s_b[i] = sb
            f = mul(Lk, S)
            g = mul(ar[i], S)
            p = mul(g, bd[i])
            k = mul(bd[i], g, hy=True)
            ad[j] = ad[j] - mul(f, Uk)
            ar[j] = ar[j] - mul(g, Uk)
            ac[j] = ac[j] - mul(f, ac[i])
            tip_a -= mul(g, ac[i])
            v = mul(Lk, sb)
            bd[j] = bd[j] + mul(v, Lk, hy=True) - mul(BL, f, hy=True) - mul(f, BU)
            br[j] = br[j] - mul(g, BU) + mul(p - br[i], f, hy=True)
            bc[j] = bc[j] - mul(f, bc[i]) - mul(BL, g, hy=True) + mul(f, k)
            tip_b += -mul(g, bc[i]) - mul(br[i], g, hy=True) + mul(p, g, hy=True)
        else:
            t1 = mul(S, Uk)
            t2 = mul(S, ac[i])
            ad[j] = ad[j] - mul(Lk, t1)
            ar[j] = ar[j] - mul(ar[i], t1)
            ac[j] = ac[j] - mul(Lk, t2)
            tip_a -= mul(ar[i], t2)


def _middle_forward(A, B, lo, hi, mul, st):
    """Middle partition elimination with fill-in to the top boundary lo
    (dist.py:309-397)."""
    ad, ar, ac, bd, br, bc, tip_a, tip_b, fac = st
    fz = B is not None
    fill_r, fill_c = A.upper[lo].copy(), A.lower[lo].copy()
    if fz:
        bfill_r, bfill_c = B.upper[lo].copy(), B.lower[lo].copy()
    for i in range(lo + 1, hi - 1):
        S = mul.inv(ad[i], i)
        fac.s_a[i] = S
        fac.ar[i], fac.ac[i] = ar[i], ac[i]
        if fz:
            fac.br[i], fac.bc[i] = br[i], bc[i]
        fac.fr[i], fac.fc[i] = fill_r, fill_c
        fn = mul(A.lower[i], S)
        fr = mul(fill_r, S)
        g = mul(ar[i], S)
        nfr = -mul(fr, A.upper[i])
        nfc = -mul(fn, fill_c)
        ad[i + 1] = ad[i + 1] - mul(fn, A.upper[i])
        ad[lo] = ad[lo] - mul(fr, fill_c)
        ar[i + 1] = ar[i + 1] - mul(g, A.upper[i])
        ar[lo] = ar[lo] - mul(g, fill_c)
        ac[i + 1] = ac[i + 1] - mul(fn, ac[i])
        ac[lo] = ac[lo] - mul(fr, ac[i])
        tip_a -= mul(g, ac[i])
        if fz:
            fac.bfr[i], fac.bfc[i] = bfill_r, bfill_c
            sb = mul(mul(S, bd[i]), S, hy=True)
            fac.s_b[i] = sb
            v0 = mul(fill_r, sb)
            vn = mul(A.lower[i], sb)
            p = mul(g, bd[i])
            BL, BU = B.lower[i], B.upper[i]
            bd[i + 1] = bd[i + 1] - mul(fn, BU) - mul(BL, fn, hy=True) + mul(vn, A.lower[i], hy=True)
            nbfc = -mul(fn, bfill_c) - mul(BL, fr, hy=True) + mul(vn, fill_r, hy=True)
            nbfr = -mul(fr, BU) - mul(bfill_r, fn, hy=True) + mul(v0, A.lower[i], hy=True)
            bd[lo] = bd[lo] - mul(fr, bfill_c) - mul(bfill_r, fr, hy=True) + mul(v0, fill_r, hy=True)
            bc[i + 1] = bc[i + 1] - mul(fn, bc[i]) - mul(BL, g, hy=True) + mul(vn, ar[i], hy=True)
            bc[lo] = bc[lo] - mul(fr, bc[i]) - mul(bfill_r, g, hy=True) + mul(v0, ar[i], hy=True)
            br[i + 1] = br[i + 1] - mul(g, BU) - mul(br[i], fn, hy=True) + mul(p, fn, hy=True)
            br[lo] = br[lo] - mul(g, bfill_c) - mul(br[i], fr, hy=True) + mul(p, fr, hy=True)
            tip_b += -mul(g, bc[i]) - mul(br[i], g, hy=True) + mul(p, g, hy=True)
            bfill_r, bfill_c = nbfr, nbfc
        fill_r, fill_c = nfr, nfc
    coupling = [fill_r, fill_c]
    bcoupling = [bfill_r, bfill_c] if fz else None
    return coupling, bcoupling


def local_forward(A, B, ranges, kinds, rank, mul):
    """dist.py:172-416 -> (payload dict, tip_delta [k,a,a], local factors)."""
    lo, hi = ranges[rank]
    kind = kinds[rank]
    fz = B is not None
    asz = A.a
    cp = lambda xs: {i: xs[i].copy() for i in range(lo, hi)}  # noqa: E731
    ad, ar, ac = cp(A.diag), cp(A.arrow_row), cp(A.arrow_col)
    bd = br = bc = None
    if fz:
        bd, br, bc = cp(B.diag), cp(B.arrow_row), cp(B.arrow_col)
    tip_a = np.zeros((asz, asz), C128)
    tip_b = np.zeros((asz, asz), C128)
    fac = _Local()
    st = (ad, ar, ac, bd, br, bc, tip_a, tip_b, fac)
    coupling = bcoupling = None
    if kind == "first":
        _end_forward(A, B, lo, hi, True, mul, st)
        bnd = [hi - 1]
    elif kind == "last":
        _end_forward(A, B, lo, hi, False, mul, st)
        bnd = [lo]
    else:
        coupling, bcoupling = _middle_forward(A, B, lo, hi, mul, st)
        bnd = [lo, hi - 1]
    pay = {
        "kind": kind,
        "diag": [ad[x] for x in bnd],
        "arrow_row": [ar[x] for x in bnd],
        "arrow_col": [ac[x] for x in bnd],
        "coupling": coupling,
    }
    if fz:
        pay.update(b_diag=[bd[x] for x in bnd], b_arrow_row=[br[x] for x in bnd],
                   b_arrow_col=[bc[x] for x in bnd], b_coupling=bcoupling)
    delta = np.stack([tip_a, tip_b]) if fz else np.stack([tip_a])
    return pay, delta, fac


def assemble(A, B, ranges, pays, delta_sum):
    """dist.py:419-504: reduced BT(A) system, provenance (rank, side)."""
    fz = B is not None
    prov, d, r, c, bd, br, bc = [], [], [], [], [], [], []
    for p, pay in enumerate(pays):
        sides = {"first": ("bottom",), "last": ("top",), "middle": ("top", "bottom")}[pay["kind"]]
        for j, side in enumerate(sides):
            prov.append((p, side))
            d.append(pay["diag"][j])
            r.append(pay["arrow_row"][j])
            c.append(pay["arrow_col"][j])
            if fz:
                bd.append(pay["b_diag"][j])
                br.append(pay["b_arrow_row"][j])
                bc.append(pay["b_arrow_col"][j])
    nr = len(d)
    up, lw, bup, blw = [], [], [], []
    for k in range(nr - 1):
        p1, p2 = prov[k][0], prov[k + 1][0]
        if p1 == p2:
            up.append(pays[p1]["coupling"][0])
            lw.append(pays[p1]["coupling"][1])
            if fz:
                bup.append(pays[p1]["b_coupling"][0])
                blw.append(pays[p1]["b_coupling"][1])
        else:
            s = ranges[p1][1] - 1
            up.append(A.upper[s].copy())
            lw.append(A.lower[s].copy())
            if fz:
                bup.append(B.upper[s].copy())
                blw.append(B.lower[s].copy())
    asz = A.a
    tip = A.tip + delta_sum[0] if asz else np.zeros((0, 0), C128)
    RA = Blocks(nr, A.b, asz, d, lw, up, r, c, tip)
    RB = None
    if fz:
        btip = B.tip + delta_sum[1] if asz else np.zeros((0, 0), C128)
        RB = Blocks(nr, A.b, asz, bd, blw, bup, br, bc, btip)
    return RA, RB, {key: k for k, key in enumerate(prov)}


def _bwd_step(mul, fac, i, rs, qs, ya, B, ss, ws, yb):
    from .seq import backstep

    if B is None:
        return backstep(mul, fac.s_a[i], rs, qs, ya)
    return backstep(mul, fac.s_a[i], rs, qs, ya, fac.s_b[i], ss, ws, yb)


def local_backward(A, B, ranges, kinds, rank, fac, index, XA_r, XB_r, XA, XB, mul):
    """dist.py:542-744, writing straight into the global outputs XA/XB."""
    lo, hi = ranges[rank]
    kind = kinds[rank]
    fz = B is not None
    ytt = XA_r.tip
    ztt = XB_r.tip if fz else None
    if rank == 0:
        XA.tip = ytt.copy()
        if fz:
            XB.tip = ztt.copy()

    def seed(side, g):
        k = index[(rank, side)]
        XA.diag[g], XA.arrow_col[g], XA.arrow_row[g] = XA_r.diag[k], XA_r.arrow_col[k], XA_r.arrow_row[k]
        ys = (XA_r.diag[k], XA_r.arrow_col[k], XA_r.arrow_row[k])
        zs = None
        if fz:
            XB.diag[g], XB.arrow_col[g], XB.arrow_row[g] = XB_r.diag[k], XB_r.arrow_col[k], XB_r.arrow_row[k]
            zs = (XB_r.diag[k], XB_r.arrow_col[k], XB_r.arrow_row[k])
        return k, ys, zs

    def separator(kb):
        s = hi - 1
        XA.lower[s], XA.upper[s] = XA_r.lower[kb].copy(), XA_r.upper[kb].copy()
        if fz:
            XB.lower[s], XB.upper[s] = XB_r.lower[kb].copy(), XB_r.upper[kb].copy()

    def store(out, which, blocks):
        for (kind_, idx), blk in zip(which, blocks):
            getattr(out, kind_)[idx] = blk

    if kind in ("first", "last"):
        down = kind == "first"
        kb, ys, zs = seed("bottom" if down else "top", hi - 1 if down else lo)
        if down:
            separator(kb)
        (ydd, ydt, ytd), zst = ys, zs
        steps = range(hi - 2, lo - 1, -1) if down else range(lo + 1, hi)
        for i in steps:
            e = i if down else i - 1
            rs = [A.upper[e] if down else A.lower[e], fac.ac[i]]
            qs = [A.lower[e] if down else A.upper[e], fac.ar[i]]
            ya = [[ydd, ydt], [ytd, ytt]]
            ss = ws = yb = None
            if fz:
                zdd, zdt, ztd = zst
                ss = [B.upper[e] if down else B.lower[e], fac.bc[i]]
                ws = [B.lower[e] if down else B.upper[e], fac.br[i]]
                yb = [[zdd, zdt], [ztd, ztt]]
            xa, xb = _bwd_step(mul, fac, i, rs, qs, ya, B if fz else None, ss, ws, yb)
            row, col, dia = xa
            off = ("upper", "lower") if down else ("lower", "upper")
            store(XA, [("diag", i), (off[0], e), (off[1], e), ("arrow_col", i), ("arrow_row", i)],
                  [dia, row[0], col[0], row[1], col[1]])
            ydd, ydt, ytd = dia, row[1], col[1]
            if fz:
                zr, zc, zd = xb
                store(XB, [("diag", i), (off[0], e), (off[1], e), ("arrow_col", i), ("arrow_row", i)],
                      [zd, zr[0], zc[0], zr[1], zc[1]])
                zst = (zd, zr[1], zc[1])
        return

    # middle (dist.py:678-742)
    kt, top, ztop = seed("top", lo)
    kb, bot, zbot = seed("bottom", hi - 1)
    separator(kb)
    y00, y0t, yt0 = top
    ydd, ydt, ytd = bot
    yfr, yfc = XA_r.upper[kt], XA_r.lower[kt]
    if fz:
        z00, z0t, zt0 = ztop
        zdd, zdt, ztd = zbot
        zfr, zfc = XB_r.upper[kt], XB_r.lower[kt]
    if hi - lo == 2:
        XA.upper[lo], XA.lower[lo] = yfr.copy(), yfc.copy()
        if fz:
            XB.upper[lo], XB.lower[lo] = zfr.copy(), zfc.copy()
    for i in range(hi - 2, lo, -1):
        rs = [fac.fc[i], A.upper[i], fac.ac[i]]
        qs = [fac.fr[i], A.lower[i], fac.ar[i]]
        ya = [[y00, yfr, y0t], [yfc, ydd, ydt], [yt0, ytd, ytt]]
        ss = ws = yb = None
        if fz:
            ss = [fac.bfc[i], B.upper[i], fac.bc[i]]
            ws = [fac.bfr[i], B.lower[i], fac.br[i]]
            yb = [[z00, zfr, z0t], [zfc, zdd, zdt], [zt0, ztd, ztt]]
        xa, xb = _bwd_step(mul, fac, i, rs, qs, ya, B if fz else None, ss, ws, yb)
        row, col, dia = xa
        store(XA, [("diag", i), ("upper", i), ("lower", i), ("arrow_col", i), ("arrow_row", i)],
              [dia, row[1], col[1], row[2], col[2]])
        if i == lo + 1:
            XA.upper[lo], XA.lower[lo] = col[0], row[0]
        ydd, ydt, ytd = dia, row[2], col[2]
        yfr, yfc = col[0], row[0]
        if fz:
            zr, zc, zd = xb
            store(XB, [("diag", i), ("upper", i), ("lower", i), ("arrow_col", i), ("arrow_row", i)],
                  [zd, zr[1], zc[1], zr[2], zc[2]])
            if i == lo + 1:
                XB.upper[lo], XB.lower[lo] = zc[0], zr[0]
            zdd, zdt, ztd = zd, zr[2], zc[2]
            zfr, zfc = zc[0], zr[0]


def dist_solve(a, b=None, num_parts=2, mode=None, counts=None, payload_log=None):
    """dist.py:804-896 with every rank simulated in rank order.

    Returns (X_A, X_B).  ``payload_log`` (list) receives per-rank payload
    dicts, for communication-contract checks.
    """
    from .seq import solve_selected

    if mode is None:
        mode = "si" if b is None else "siq"
    if mode == "siq" and b is None:
        raise ValueError("mode 'siq' requires a right-hand side")
    A = Blocks.of(a)
    B = Blocks.of(b) if mode == "siq" else None
    if num_parts == 1:
        return solve_selected(A, B, mode)
    ranges, kinds = plan_partitions(A.n, num_parts, mode)
    mul = _Mul(A.b, A.a)
    results = []
    for rank in range(num_parts):
        try:
            results.append(local_forward(A, B, ranges, kinds, rank, mul))
        except OracleSingular as exc:
            exc.rank = rank
            raise
    pays = [r[0] for r in results]
    if payload_log is not None:
        payload_log.extend(pays)
    total = results[0][1].copy()
    for r in results[1:]:
        total = total + r[1]
    RA, RB, index = assemble(A, B, ranges, pays, total)
    rmul = _Mul(A.b, A.a)
    F = forward(Blocks.of(RA), None if RB is None else Blocks.of(RB), rmul)
    XA_r, XB_r = backward(F, RA, RB, rmul)
    XA = Blocks.zeros(A.n, A.b, A.a)
    XB = Blocks.zeros(A.n, A.b, A.a) if B is not None else None
    for rank in range(num_parts):
        local_backward(A, B, ranges, kinds, rank, results[rank][2], index, XA_r, XB_r, XA, XB, mul)
    if counts is not None:
        counts.update(mul.counts)
        counts.update(rmul.counts)
    return XA, XB
