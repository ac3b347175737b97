"""GPU tests of the C-ABI contract added in round 2:

* the tie-break rule is selectable (rf_params.tie_break, R9): RF_TIE_LOWEST_FEATURE (the
  default, BASELINE.json north_star: "lowest feature then lowest threshold") and
  RF_TIE_DRAW_ORDER (scikit-learn's first drawn feature); both bit-exact against the oracle in
  the same mode on the CTA-resident and the level-synchronous paths, in the exact, histogram
  and ExtraTrees split modes and under MAE; SURVEY.md Appendix C's Example A tree reproduced by
  the GPU in the default mode;
* rf_cross_validate / rf_cross_validate_dev (the problem statement's call, P:366-368,
  P:400-403) against the oracle: given folds, NULL folds (plain Philox folds from the seed),
  the library's mtry default, and its errors (tree_begin set -> RF_E_ARG, y <= 0, k < 2);
* the binding rejects device arguments of the wrong dtype or device instead of passing their
  pointers to the *_dev entry points.
"""
import json
import os

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2001_07104_b200 as rfg  # noqa: E402
from test_gpu_parity import RTOL, _compare_forest, _cuda  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ------------------------------------------------------------- tie-break ---
def test_example_A_lowest_feature_on_gpu():
    """SURVEY.md Appendix C Example A: both children tie across features; the default
    (north_star) rule takes f0 at both, for every seed (the draws do not matter)."""
    A = json.load(open(os.path.join(GOLD, "worked_examples.json")))["A"]
    E = A["tree_lowest_feature"]
    X, y = np.array(A["X"], float), np.array(A["y"], float)
    for seed in range(6):
        gf = rfg.fit(X, y, ntree=1, mtry=2, bootstrap=False, seed=seed, debug=True)
        e = gf.export()
        assert e["feature"].tolist() == E["feature"]
        assert e["thr_index"][:3].tolist() == E["thr_index"][:3]
        assert e["left"][:3].tolist() == E["left"][:3]
        internal = e["feature"] >= 0
        vals = np.where(internal, e["value"], 0.0)
        assert vals.tolist() == E["thr_value"]
        assert e["value"][~internal].tolist() == [v for v, f in zip(E["leaf_value"], E["feature"]) if f < 0]
        assert gf.leaf_rows()[0].tolist() == E["leaf_of_row"]
        assert rfg.predict(gf, np.array([A["query"]]))[0] == E["query_pred"]


TIE_CASES = [
    # name, data, kwargs: small (n_tr <= 255) and large paths, every split mode, MAE
    ("small_exact_ties", lambda: datagen.tiny(200, 5, 3, distinct=4), dict(mtry=5)),
    ("small_paper", lambda: datagen.paper_shaped(189, "K20", "time"), dict(mtry=12, target=1)),
    ("small_extra", lambda: datagen.tiny(180, 6, 4, distinct=5), dict(mtry=6, split_mode=2, bootstrap=False)),
    ("small_mae", lambda: datagen.tiny(150, 4, 5, distinct=4), dict(mtry=4, criterion=1)),
    ("large_exact_ties", lambda: datagen.tiny(3000, 6, 6, distinct=5), dict(mtry=6, max_depth=9)),
    ("large_scaled", lambda: datagen.scaled(4000, 64), dict(mtry=21, max_depth=8, target=1)),
    ("large_hist", lambda: datagen.tiny(2500, 5, 7, distinct=6), dict(mtry=5, split_mode=1)),
    ("large_extra", lambda: datagen.tiny(2000, 5, 8, distinct=7), dict(mtry=5, split_mode=2, max_depth=10)),
]


@pytest.mark.parametrize("tie", [0, 1])
@pytest.mark.parametrize("name,data,kw", TIE_CASES, ids=[c[0] for c in TIE_CASES])
def test_tie_break_modes_bit_exact(name, data, kw, tie):
    X, y = data()
    of = oracle.fit(X, y, ntree=6, seed=31, leaf_rows=True, tie_break=tie, **kw)
    gf = rfg.fit(X, y, ntree=6, seed=31, debug=True, tie_break=tie, **kw)
    _compare_forest(gf, of, X)


def test_tie_break_modes_differ():
    """Non-vacuous: on data with many exact cross-feature ties the two rules grow different
    trees (and each matches the oracle above)."""
    X, y = datagen.tiny(200, 5, 3, distinct=4)
    a = rfg.fit(X, y, ntree=6, seed=31, mtry=5, tie_break=0).export()
    b = rfg.fit(X, y, ntree=6, seed=31, mtry=5, tie_break=1).export()
    assert not (np.array_equal(a["feature"], b["feature"]) and np.array_equal(a["thr_index"], b["thr_index"]))
    with pytest.raises(rfg.RFError) as e:
        rfg.fit(X, y, ntree=1, tie_break=2)
    assert e.value.code == rfg.E_ARG


def test_tie_break_cv_both_modes():
    X, y = datagen.paper_shaped(189, "P100", "time")
    f = oracle.make_folds(y, 10, 2, seed=5, custom=True)
    for tie in (0, 1):
        fo = oracle.cv_grid(X, y, 10, 2, [16, 32], [12, 3], fold_ids=f, target=1, seed=5, tie_break=tie)
        fg = rfg.cross_validate_grid(X, y, 10, 2, [16, 32], [12, 3], fold_ids=f, target=1, seed=5, tie_break=tie)
        np.testing.assert_allclose(fg, fo, rtol=RTOL, atol=0)


# ----------------------------------------------------- rf_cross_validate ---
def test_cross_validate_single_point_host_and_device():
    X, y = datagen.paper_shaped(189, "V100", "time")
    folds = oracle.make_folds(y, 10, 3, seed=9, custom=True)
    want = oracle.cv_grid(X, y, 10, 3, [48], [4], fold_ids=folds, target=1, seed=9)[0, 0]
    got = rfg.cross_validate(X, y, 10, 3, folds, ntree=48, mtry=4, target=1, seed=9)
    assert got.shape == (3, 10)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)
    gd = rfg.cross_validate(_cuda(X), _cuda(y), 10, 3, _cuda(folds, torch.int32), ntree=48, mtry=4, target=1,
                            seed=9)
    np.testing.assert_allclose(gd.cpu().numpy(), want, rtol=RTOL, atol=0)


def test_cross_validate_null_folds_and_default_mtry():
    """fold_ids = NULL: plain Philox folds from prm->seed (R16); mtry = 0: the library's
    default max(1, floor(p/3)) (R5) -- both decided inside the library, not the binding."""
    X, y = datagen.paper_shaped(168, "TitanXp", "power")
    want = oracle.cv_grid(X, y, 10, 2, [20], [4], fold_ids=None, seed=13)[0, 0]  # p = 12 -> mtry 4
    got = rfg.cross_validate(X, y, 10, 2, None, ntree=20, mtry=0, seed=13)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)
    gd = rfg.cross_validate(_cuda(X), _cuda(y), 10, 2, None, ntree=20, seed=13)
    np.testing.assert_allclose(gd.cpu().numpy(), want, rtol=RTOL, atol=0)
    # large path (n_tr > 255) through the same call
    X, y = datagen.paper_shaped(600, "K20", "time")
    want = oracle.cv_grid(X, y, 3, 1, [6], [4], seed=2, target=1)[0, 0]
    np.testing.assert_allclose(rfg.cross_validate(X, y, 3, 1, None, ntree=6, seed=2, target=1), want,
                               rtol=RTOL, atol=0)


def test_cross_validate_errors():
    X, y = datagen.paper_shaped(189, "K20", "time")
    with pytest.raises(rfg.RFError) as e:  # a rank cannot score a partial forest
        rfg.cross_validate(X, y, 10, 1, None, ntree=8, tree_begin=0, tree_end=4)
    assert e.value.code == rfg.E_ARG
    with pytest.raises(rfg.RFError) as e:  # Eq. 1 divides by y
        rfg.cross_validate(X, np.where(np.arange(189) == 5, 0.0, y), 10, 1, None, ntree=4)
    assert e.value.code == rfg.E_NONPOSITIVE_Y
    with pytest.raises(rfg.RFError) as e:
        rfg.cross_validate(X, y, 1, 1, None, ntree=4)
    assert e.value.code == rfg.E_TOO_FEW
    with pytest.raises(rfg.RFError) as e:  # an empty test fold
        f = np.zeros((1, 189), np.int32)
        rfg.cross_validate(X, y, 2, 1, f, ntree=4)
    assert e.value.code == rfg.E_TOO_FEW


# ---------------------------------------------------- binding validation ---
def test_device_argument_validation():
    X, y = datagen.paper_shaped(189, "K20", "time")
    Xd, yd = _cuda(X), _cuda(y)
    with pytest.raises(TypeError):
        rfg.fit(Xd.float(), yd, ntree=2)
    with pytest.raises(TypeError):
        rfg.fit(Xd, torch.as_tensor(y), ntree=2)  # host tensor mixed with a device X
    f = rfg.fit(Xd, yd, ntree=2)
    with pytest.raises(TypeError):
        rfg.predict(f, Xd.float())
    with pytest.raises(TypeError):
        rfg.predict(f, Xd, out=torch.empty(189, dtype=torch.float32, device="cuda"))
    with pytest.raises(TypeError):
        rfg.cross_validate_grid(Xd, yd, 10, 1, [4], [3], fold_ids=torch.zeros((1, 189), dtype=torch.int64,
                                                                             device="cuda"))
    # non-contiguous inputs are made contiguous (same result as the contiguous copy)
    np.testing.assert_allclose(rfg.predict(f, Xd[::2]).cpu().numpy(), rfg.predict(f, X[::2]), rtol=RTOL, atol=0)


def test_forest_import_rejects_malformed():
    """rf_forest_import checks the structure on the host: a cyclic or out-of-range
    child, a bad feature or a non-increasing tree_off returns RF_E_ARG before any upload."""
    X, y = datagen.paper_shaped(189, "K20", "time")
    e = rfg.fit(X, y, ntree=3, mtry=4, target=1, seed=2).export()
    args = lambda **o: dict(dict(feature=e["feature"].copy(), left=e["left"].copy(), value=e["value"],
                                 thr_index=e["thr_index"], tree_off=e["tree_off"].copy(), p=12, F=e["F"],
                                 target=1), **o)
    ok = rfg.forest_import(**args())
    np.testing.assert_array_equal(rfg.predict(ok, X[:50]), rfg.predict(rfg.fit(X, y, ntree=3, mtry=4, target=1,
                                                                                seed=2), X[:50]))
    bad = []
    a = args(); i = int(np.nonzero(a["feature"] >= 0)[0][0]); a["left"][i] = 0; bad.append(a)        # cycle
    a = args(); a["left"][i] = 10 ** 6; bad.append(a)                                                # out of range
    a = args(); a["feature"][i] = 12; bad.append(a)                                                  # feature >= p
    a = args(); a["feature"][i] = -3; bad.append(a)
    a = args(); a["tree_off"][1] = a["tree_off"][0]; bad.append(a)                                   # empty tree
    a = args(p=0); bad.append(a)
    a = args(target=2); bad.append(a)
    for a in bad:
        with pytest.raises(rfg.RFError) as ex:
            rfg.forest_import(**a)
        assert ex.value.code == rfg.E_ARG


def test_ln_device_bit_exact_wide():
    """The device ln (double-double evaluation, R20) against the oracle's binary128 logq on 4M+
    values: uniform in the exponent over the whole normal range, the paper-shaped span (µs to
    seconds), dense neighbourhoods of 1 (tiny results, the hardest relative rounding), of powers of
    two and of e^k, and subnormals.  One disagreement would flip t_q and every tree on a LOG target."""
    rnd = np.random.default_rng(12)
    parts = [
        np.exp2(rnd.uniform(-1021, 1023, 1_500_000)),
        10 ** rnd.uniform(-3, 9, 1_000_000),
        1.0 + rnd.uniform(-2 ** -20, 2 ** -20, 500_000),
        np.nextafter(1.0, 2.0) ** 0 + np.arange(1, 200_001) * np.finfo(np.float64).eps,
        np.ldexp(1.0, rnd.integers(-1020, 1020, 400_000)) * (1.0 + rnd.integers(-64, 65, 400_000) * 2.0 ** -52),
        np.exp(rnd.integers(-700, 700, 300_000).astype(np.float64)) * (1.0 + rnd.normal(0, 1e-15, 300_000)),
        rnd.uniform(1e-310, 2.2e-308, 100_000),
    ]
    y = np.concatenate(parts)
    y = y[(y > 0) & np.isfinite(y)]
    got = rfg.debug_ln(_cuda(y)).cpu().numpy()
    want = oracle.quantize(y, 1)[0]
    bad = np.nonzero(got.view(np.int64) != want.view(np.int64))[0]
    assert bad.size == 0, (bad.size, y[bad[:5]], got[bad[:5]], want[bad[:5]])


def test_ln_uncertified_fails_loudly():
    """ln's rounding test (ddlog.cuh, R20): a value it cannot certify makes a LOG-target call fail
    with RF_E_INEXACT instead of quantising a possibly misrounded ln.  A widened margin (test switch)
    reaches the path; the default margin certifies the same data, and the near-1 hard cases
    (y = 1 - 2^-52, ...) certify and match the oracle."""
    X, y = datagen.paper_shaped(189, "K20", "time")
    rfg.debug_set_option("ln_cert_margin_log2", -20)
    try:
        with pytest.raises(rfg.RFError) as ex:
            rfg.fit(X, y, ntree=2, mtry=3, target=1, seed=1)
        assert ex.value.code == rfg.E_INEXACT
        rfg.fit(X, y, ntree=2, mtry=3, target=0, seed=1)  # the identity target takes no ln
    finally:
        rfg.debug_set_option("ln_cert_margin_log2", 0)
    rfg.fit(X, y, ntree=2, mtry=3, target=1, seed=1)
    hard = np.concatenate([1.0 + np.arange(1, 4000) * 2.0 ** -52, 1.0 - np.arange(1, 4000) * 2.0 ** -53])
    Xh = np.random.default_rng(5).uniform(0, 1, (hard.size, 3))
    f = rfg.fit(Xh, hard, ntree=1, mtry=3, target=1, seed=1)  # certified: no RF_E_INEXACT
    assert f is not None
    got = rfg.debug_ln(_cuda(hard)).cpu().numpy()
    want = oracle.quantize(hard, 1)[0]
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


def _swap_sibling_pairs(e):
    """Per tree with two internal nodes A, B on one level (depth >= 7 where there is one): swap the
    records of their child pairs and the two parents' child pointers -- the same trees, no longer in
    the BFS order the blocked compact layout assumes (its validation must fall back)."""
    feat, left = e["feature"].copy(), e["left"].copy()
    val, ti, off = e["value"].copy(), e["thr_index"].copy(), e["tree_off"]
    swapped = 0
    for t in range(len(off) - 1):
        o0, o1 = int(off[t]), int(off[t + 1])
        depth = np.zeros(o1 - o0, np.int64)
        for i in range(o1 - o0):
            if feat[o0 + i] >= 0:
                depth[left[o0 + i]] = depth[left[o0 + i] + 1] = depth[i] + 1
        internal = [i for i in range(o1 - o0) if feat[o0 + i] >= 0]
        for dmin in (7, 1):
            cand = [i for i in internal if depth[i] >= dmin]
            pair = next(((a, b) for a in cand for b in cand if a < b and depth[a] == depth[b]), None)
            if pair:
                break
        if not pair:
            continue
        a, b = pair
        ca, cb = int(left[o0 + a]), int(left[o0 + b])
        for arr in (feat, left, val, ti):
            x, y_ = arr[o0 + ca:o0 + ca + 2].copy(), arr[o0 + cb:o0 + cb + 2].copy()
            arr[o0 + ca:o0 + ca + 2], arr[o0 + cb:o0 + cb + 2] = y_, x
        left[o0 + a], left[o0 + b] = cb, ca
        swapped += 1
    return dict(feature=feat, left=left, value=val, thr_index=ti, tree_off=off), swapped


@pytest.mark.parametrize("max_depth", [12, -1])
def test_predict_blocked_layout_and_fallback(max_depth):
    """Batched inference through the compact copy in its blocked layout (shallow BFS forests:
    three-level 64-byte blocks below the 7-level prefix) and in the BFS-slot layout (deep forests,
    and forests whose trees are not BFS-ordered: sibling pairs swapped, imported) gives the same bits
    as the 16-byte node walk, at depth 12 (staged prefix, blocked) and unbounded depth (BFS slots)."""
    X, y = datagen.scaled(30_000, 16)
    f = rfg.fit(X, y, ntree=12, mtry=5, target=1, seed=4, max_depth=max_depth)
    Q = datagen.scaled(20_000, 16, seed=9)[0]
    blocked = rfg.predict(f, Q)
    rfg.debug_set_option("predict_node16", 1)
    try:
        ref = rfg.predict(f, Q)
    finally:
        rfg.debug_set_option("predict_node16", 0)
    assert np.array_equal(blocked.view(np.int64), ref.view(np.int64))
    e = f.export()
    d, swapped = _swap_sibling_pairs(e)
    assert swapped >= 6
    g = rfg.forest_import(d["feature"], d["left"], d["value"], d["thr_index"], d["tree_off"], e["p"], e["F"],
                          e["target"])
    assert np.array_equal(rfg.predict(g, Q).view(np.int64), ref.view(np.int64))
    imp = rfg.forest_import(e["feature"], e["left"], e["value"], e["thr_index"], e["tree_off"], e["p"], e["F"],
                            e["target"])  # an imported BFS forest takes the blocked layout too
    assert np.array_equal(rfg.predict(imp, Q).view(np.int64), ref.view(np.int64))


def test_predict_host_pipelined_chunks():
    """The host-pointer rf_predict streams large batches in chunks over two CUDA streams: with small
    chunks forced (test switch), an odd number of chunks and a ragged last one give the same bits as
    the device entry point; a non-finite value in a late chunk still fails with RF_E_NONFINITE."""
    X, y = datagen.paper_shaped(189, "K20", "time")
    f = rfg.fit(X, y, ntree=64, mtry=4, target=1, seed=3)
    Q = X[np.random.default_rng(2).integers(0, 189, 23_457)] * (1 + np.random.default_rng(3).normal(0, 1e-3, (23_457, 12)))
    want = rfg.predict(f, _cuda(Q)).cpu().numpy()
    rfg.debug_set_option("predict_chunk_rows", 5000)
    try:
        got = rfg.predict(f, np.ascontiguousarray(Q))
        assert np.array_equal(got.view(np.int64), want.view(np.int64))
        Qb = Q.copy()
        Qb[21_000, 3] = np.nan
        with pytest.raises(rfg.RFError) as ex:
            rfg.predict(f, Qb)
        assert ex.value.code == rfg.E_NONFINITE
    finally:
        rfg.debug_set_option("predict_chunk_rows", 0)
    assert np.array_equal(rfg.predict(f, np.ascontiguousarray(Q)).view(np.int64), want.view(np.int64))
