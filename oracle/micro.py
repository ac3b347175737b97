"""Pure-Python micro-oracle for tiny inputs -- TEST INFRASTRUCTURE ONLY.

An independent second implementation (no code shared with rf_oracle.c) used
to pin the C oracle:
  * its own Philox4x32-10 (pinned itself by the Random123 KAT vectors);
  * exact arithmetic: node sums, split quality and leaf means are Fractions;
    split quality is the two-pass SSE reduction  sum w (t - mean)^2  of the
    parent minus that of the children (the definition of the MSE criterion,
    P:215 / P:489) -- NOT the proxy G the C oracle evaluates;
  * ln via decimal (correctly rounded), not libm/libquadmath;
  * trees grown depth-first recursively, then renumbered breadth-first, so a
    match also pins that RNG addressing does not depend on growth order
    (R14).
Only usable for tiny inputs (n <= ~40).
"""
from __future__ import annotations

import decimal
from fractions import Fraction
import math

M0, M1, W0, W1 = 0xD2511F53, 0xCD9E8D57, 0x9E3779B9, 0xBB67AE85
MASK32 = 0xFFFFFFFF
TAG_FOLD, TAG_STRATUM, TAG_KEYDERIV, TAG_BOOT, TAG_FEAT = 0xD0, 0xD1, 0x4B, 0xB0, 0xF0
TAG_THR = 0xE7


def philox(ctr, key):
    c0, c1, c2, c3 = ctr
    k0, k1 = key
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        c0, c1, c2, c3 = ((p1 >> 32) ^ c1 ^ k0) & MASK32, p1 & MASK32, ((p0 >> 32) ^ c3 ^ k1) & MASK32, p0 & MASK32
        k0 = (k0 + W0) & MASK32
        k1 = (k1 + W1) & MASK32
    return [c0, c1, c2, c3]


def draw(key, c1, c2, c3, i):
    o = philox([(i >> 1) & MASK32, c1 & MASK32, c2 & MASK32, c3 & MASK32], key)
    return (o[1] << 32 | o[0]) if i % 2 == 0 else (o[3] << 32 | o[2])


def mulhi64(u, m):
    return (u * m) >> 64


def tree_key(seed, task, t):
    o = philox([t, task, 0, TAG_KEYDERIV], [seed & MASK32, seed >> 32])
    return [o[0], o[1]]


def ln_cr(y: float) -> float:
    """ln(y) correctly rounded to binary64 (60-digit decimal, then one rounding)."""
    with decimal.localcontext() as ctx:
        ctx.prec = 60
        return float(decimal.Decimal(y).ln())


def quantize(y, target, guard=0):
    t = [ln_cr(v) if target == 1 else float(v) for v in y]
    n = len(t)
    M = max(abs(v) for v in t)
    if M == 0:
        F = 0
    else:
        e = 0
        # smallest integer e with M <= 2^e, by exact comparison
        e = math.frexp(M)[1]
        while Fraction(M) <= Fraction(2) ** (e - 1):
            e -= 1
        while Fraction(M) > Fraction(2) ** e:
            e += 1
        F = 62 - (n - 1).bit_length() - e - guard  # guard = 2 under MAE (R32)
    tq = []
    for v in t:
        q = Fraction(v) * Fraction(2) ** F
        tq.append(round(q))  # Python round on Fraction: half to even
    return t, tq, F


def bootstrap(key, tr, n, boot=True):
    w = [0] * n
    if not boot:
        for r in tr:
            w[r] = 1
        return w
    ntr = len(tr)
    for j in range(ntr):
        w[tr[mulhi64(draw(key, 0, 0, TAG_BOOT, j), ntr)]] += 1
    return w


def draw_features(key, heap, p, m):
    perm = list(range(p))
    for j in range(m):
        u = draw(key, heap & MASK32, (heap >> 32) & MASK32, TAG_FEAT, j)
        r = j + mulhi64(u, p - j)
        perm[j], perm[r] = perm[r], perm[j]
    return perm[:m]


def canonical_gain(WL, SL, WR, SR):
    """fp64 proxy, used ONLY to reproduce the documented fp64 tie-break order."""
    a = float(SL) * float(SL)
    a = a / float(WL)
    b = float(SR) * float(SR)
    b = b / float(WR)
    return a + b


def sse(rows, w, tq):
    W = sum(w[r] for r in rows)
    if W == 0:
        return Fraction(0)
    mean = Fraction(sum(w[r] * tq[r] for r in rows), W)
    return sum(w[r] * (tq[r] - mean) ** 2 for r in rows)


def hist_cuts(col_vals_train):
    s = sorted(col_vals_train)
    u = sorted(set(s))
    if len(u) <= 256:
        return u[:-1]
    m = len(s)
    cuts = []
    for j in range(1, 256):
        q = -(-j * m // 256)
        v = s[q - 1]
        if v == u[-1] or (cuts and cuts[-1] == v):
            continue
        cuts.append(v)
    return cuts


class Node:
    __slots__ = ("rows", "depth", "heap", "feature", "thr_index", "thr_value", "value", "children",
                 "gain_exact_best", "gain_exact_chosen", "W", "S")


def extra_threshold(key, heap, j, lo, hi):
    """ExtraTrees threshold of drawn slot j (R29):
    uniform in [lo, hi) as scikit-learn's rand_uniform(lo, hi) = (hi - lo) u + lo,
    u = 53 random bits / 2^53 from stream (key; heap, TAG_THR)."""
    u = math.ldexp(draw(key, heap & MASK32, (heap >> 32) & MASK32, TAG_THR, j) >> 11, -53)
    thr = (hi - lo) * u + lo  # Python floats: IEEE binary64, round to nearest, no FMA
    return thr if thr < hi else lo


def wmedian(rows, w, tq):
    """Weighted median (scikit-learn's rule, R32): values ascending, k = first
    with cumulative weight >= W/2; exactly W/2 -> mean of t_k and the next value."""
    srt = sorted(rows, key=lambda r: (tq[r], r))
    W = sum(w[r] for r in srt)
    cum = 0
    for i, r in enumerate(srt):
        cum += w[r]
        if 2 * cum >= W:
            if 2 * cum == W and i + 1 < len(srt):
                return Fraction(tq[r] + tq[srt[i + 1]], 2)
            return Fraction(tq[r])
    return Fraction(0)


def sad(rows, w, tq):
    """Sum of weighted absolute deviations from the weighted median (MAE impurity x W)."""
    if not rows:
        return Fraction(0)
    m = wmedian(rows, w, tq)
    return sum(w[r] * abs(tq[r] - m) for r in rows)


def grow(X, tq, F, w, key, mtry, min_split=2, max_depth=-1, hist_cuts_per_f=None, extra=False, mae=False,
         tie_draw=False):
    """Depth-first recursive growth; returns the root Node.  mae: MAE criterion (R32) --
    cost = SAD_L + SAD_R minimised (candidates as for MSE), leaves = weighted medians.
    tie_draw: ties go to the first drawn feature (R9) instead of the lowest feature index
    (north_star's rule, the default)."""
    n, p = len(X), len(X[0])
    gvals = [sorted(set(X[i][f] for i in range(n))) for f in range(p)]

    def rec(rows, depth, heap):
        nd = Node()
        nd.rows, nd.depth, nd.heap = rows, depth, heap
        nd.W = sum(w[r] for r in rows)
        nd.S = sum(w[r] * tq[r] for r in rows)
        nd.children = None
        nd.gain_exact_best = nd.gain_exact_chosen = None
        leaf = (max_depth >= 0 and depth >= max_depth) or len(rows) < min_split or \
            len(set(tq[r] for r in rows)) == 1
        cands = []
        if not leaf:
            parent_sse = sse(rows, w, tq) if not mae else sad(rows, w, tq)
            imp_of = (lambda L, R: sse(L, w, tq) + sse(R, w, tq)) if not mae else \
                (lambda L, R: sad(L, w, tq) + sad(R, w, tq))
            for j, f in enumerate(draw_features(key, heap, p, mtry)):
                if extra:
                    vals = [X[r][f] for r in rows]
                    lo, hi = min(vals), max(vals)
                    if lo == hi:
                        continue
                    thr = extra_threshold(key, heap, j, lo, hi)
                    L = [r for r in rows if X[r][f] <= thr]
                    R = [r for r in rows if X[r][f] > thr]
                    WL = sum(w[r] for r in L)
                    SL = sum(w[r] * tq[r] for r in L)
                    a = max(X[r][f] for r in L)
                    red = parent_sse - imp_of(L, R)
                    score = canonical_gain(WL, SL, nd.W - WL, nd.S - SL) if not mae else -imp_of(L, R)
                    cands.append((score, f, gvals[f].index(a), thr, red, set(L), j))
                elif hist_cuts_per_f is None:
                    srt = sorted(rows, key=lambda r: (X[r][f], r))
                    for i in range(len(srt) - 1):
                        a, b = X[srt[i]][f], X[srt[i + 1]][f]
                        if not a < b:
                            continue
                        L, R = srt[:i + 1], srt[i + 1:]
                        WL = sum(w[r] for r in L)
                        SL = sum(w[r] * tq[r] for r in L)
                        red = parent_sse - imp_of(L, R)
                        thr = a / 2.0 + b / 2.0
                        if thr == b:
                            thr = a
                        score = canonical_gain(WL, SL, nd.W - WL, nd.S - SL) if not mae else -imp_of(L, R)
                        cands.append((score, f, gvals[f].index(a), thr, red, set(L), j))
                else:
                    cuts = hist_cuts_per_f[f]
                    for ci, c in enumerate(cuts):
                        L = [r for r in rows if X[r][f] <= c]
                        R = [r for r in rows if X[r][f] > c]
                        WL = sum(w[r] for r in L)
                        WR = nd.W - WL
                        if WL <= 0 or WR <= 0:
                            continue
                        SL = sum(w[r] * tq[r] for r in L)
                        red = parent_sse - sse(L, w, tq) - sse(R, w, tq)
                        cands.append((canonical_gain(WL, SL, WR, nd.S - SL), f, ci, c, red, set(L), j))
            if not cands:
                leaf = True
        if leaf:
            nd.feature = -1
            nd.thr_index, nd.thr_value = 0, 0.0
            v = wmedian(rows, w, tq) if mae else Fraction(nd.S, nd.W)  # R32 / R13
            nd.value = float(v * Fraction(2) ** (-F)) if F >= 0 else float(v / Fraction(2) ** F)
            return nd
        # tie-break (R9): lowest feature index (north_star) or, with tie_draw, first drawn
        # feature (slot j); then lowest threshold rank
        best = min(cands, key=lambda c: (-c[0], c[6] if tie_draw else c[1], c[2]))
        nd.feature, nd.thr_index, nd.thr_value = best[1], best[2], best[3]
        nd.gain_exact_best = max(c[4] for c in cands)
        nd.gain_exact_chosen = best[4]
        nd.value = 0.0
        Lset = best[5]
        left = [r for r in rows if r in Lset]
        right = [r for r in rows if r not in Lset]
        mask = (1 << 64) - 1
        nd.children = (rec(left, depth + 1, (2 * heap) & mask), rec(right, depth + 1, (2 * heap + 1) & mask))
        return nd

    root_rows = [i for i in range(n) if w[i] > 0]
    return rec(root_rows, 0, 1)


def to_bfs(root):
    """Breadth-first renumbering -> dict of lists (feature, thr_index, thr_value, left, leaf_value)."""
    order = [root]
    i = 0
    while i < len(order):
        if order[i].children is not None:
            order.extend(order[i].children)
        i += 1
    idx = {id(nd): k for k, nd in enumerate(order)}
    out = dict(feature=[], thr_index=[], thr_value=[], left=[], leaf_value=[], nodes=order)
    for nd in order:
        out["feature"].append(nd.feature)
        out["thr_index"].append(nd.thr_index if nd.feature >= 0 else 0)
        out["thr_value"].append(nd.thr_value if nd.feature >= 0 else 0.0)
        out["left"].append(idx[id(nd.children[0])] if nd.children else 0)
        out["leaf_value"].append(nd.value if nd.feature < 0 else 0.0)
    return out


def fit_tree(X, y, t, mtry, seed=0, boot=True, target=0, min_split=2, max_depth=-1, hist=False,
             task=0, train_rows=None, extra=False, mae=False, tie_draw=False):
    """Tree t of `task` over train_rows (default all rows).  extra=True grows an
    Extremely Randomized tree (split_mode 2)."""
    X = [[(0.0 if v == 0.0 else float(v)) for v in row] for row in X]
    _, tq, F = quantize(list(y), target, 2 if mae else 0)
    n = len(X)
    tr = list(range(n)) if train_rows is None else list(train_rows)
    key = tree_key(seed, task, t)
    w = bootstrap(key, tr, n, boot)
    cuts = None
    if hist:
        cuts = [hist_cuts([X[r][f] for r in tr]) for f in range(len(X[0]))]
    root = grow(X, tq, F, w, key, mtry, min_split, max_depth, cuts, extra, mae, tie_draw)
    out = to_bfs(root)
    # MDI (NEXT-3): per feature, the exact SSE reductions of its splits (the definition
    # W imp(node) - WL imp(L) - WR imp(R), two-pass sums) in target units (x 2^-2F)
    raw = [Fraction(0)] * len(X[0])
    for nd in out["nodes"]:
        if nd.children is not None:
            raw[nd.feature] += nd.gain_exact_chosen
    scale = Fraction(2) ** (-F if mae else -2 * F)  # SAD is linear in t, SSE quadratic
    out["imp_raw"] = [float(v * scale) for v in raw]
    return out, F


def mape_exact(y, yhat):
    """Eq. 1 in exact rationals, percent."""
    s = sum(abs(Fraction(a) - Fraction(b)) / Fraction(a) for a, b in zip(y, yhat))
    return 100 * s / len(y)
