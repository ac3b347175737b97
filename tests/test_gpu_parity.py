"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bar: tree structures bit-exact (split feature,
threshold index, threshold value, child ids, leaf values, leaf row sets);
fold ids and ln bit-exact; predictions and fold MAPE within 1e-9 relative
(north_star), the summation order being the only difference.
"""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2001_07104_b200 as rfg  # noqa: E402

RTOL = 1e-9


def _cuda(a, dtype=torch.float64):
    return torch.as_tensor(np.ascontiguousarray(a)).to(device="cuda", dtype=dtype)


# ------------------------------------------------------------ primitives --
def test_philox_device_kat(golden_dir):
    rows = []
    for line in open(f"{golden_dir}/philox_kat.txt"):
        if line.startswith("#") or not line.strip():
            continue
        rows.append([int(x, 16) for x in line.split()])
    rnd = np.random.default_rng(0)
    extra = rnd.integers(0, 2 ** 32, size=(200, 6), dtype=np.uint64)
    inp = np.concatenate([np.array([r[:6] for r in rows], np.uint64), extra])
    out = rfg.debug_philox(torch.tensor(inp.astype(np.int64), device="cuda")).cpu().numpy()
    for i, r in enumerate(rows):
        assert out[i].tolist() == r[6:]
    for i in range(len(rows), len(inp)):
        c = inp[i]
        assert out[i].tolist() == [int(v) for v in oracle.philox(c[:4], c[4:])]


def test_ln_device_bit_exact():
    rnd = np.random.default_rng(1)
    y = np.concatenate([10 ** rnd.uniform(-5, 9, 20000), rnd.uniform(0.5, 2.0, 5000), [1.0, 2.0, np.e, 1e-310]])
    got = rfg.debug_ln(_cuda(y)).cpu().numpy()
    want = np.array([oracle.ln(v) for v in y])
    assert np.array_equal(got.view(np.int64), want.view(np.int64))


@pytest.mark.parametrize("n,k,custom", [(189, 10, False), (168, 10, False), (10, 10, False), (23, 4, False),
                                        (5000, 10, False), (189, 10, True), (95, 5, True)])
def test_folds_bit_exact(n, k, custom):
    if custom:
        y = datagen.paper_shaped(n, "K20", "time")[1] if n == 189 else 10 ** np.random.default_rng(3).uniform(1, 7, n)
    else:
        y = np.ones(n)
    g = rfg.make_folds(y, k, 5, seed=77, custom=custom)
    o = oracle.make_folds(y, k, 5, seed=77, custom=custom)
    assert np.array_equal(g, o)
    gd = rfg.make_folds(_cuda(y), k, 5, seed=77, custom=custom).cpu().numpy()
    assert np.array_equal(gd, o)


# ---------------------------------------------------------------- fit ---
def _compare_forest(gf, of, X):
    e = gf.export()
    off = e["tree_off"]
    assert e["ntree"] == len(of.trees)
    assert e["F"] == of.F
    lr = gf.leaf_rows() if of.trees and of.trees[0].leaf_of_row is not None else None
    for t, tr in enumerate(of.trees):
        a, b = int(off[t]), int(off[t + 1])
        feat = e["feature"][a:b]
        assert b - a == tr.n_nodes, f"tree {t}: {b - a} vs {tr.n_nodes} nodes"
        assert np.array_equal(feat, tr.feature), f"tree {t} features"
        internal = feat >= 0
        assert np.array_equal(e["left"][a:b][internal], tr.left[internal]), f"tree {t} children"
        assert np.array_equal(e["thr_index"][a:b][internal], tr.thr_index[internal]), f"tree {t} thr index"
        assert np.array_equal(e["value"][a:b][internal].view(np.int64), tr.thr_value[internal].view(np.int64))
        assert np.array_equal(e["value"][a:b][~internal].view(np.int64), tr.leaf_value[~internal].view(np.int64)), \
            f"tree {t} leaf values"
        if lr is not None and tr.leaf_of_row is not None:
            assert np.array_equal(lr[t], tr.leaf_of_row), f"tree {t} leaf rows"


FIT_CASES = [
    # name, data fn, kwargs
    ("paper_time_m12", lambda: datagen.paper_shaped(189, "K20", "time"), dict(mtry=12, target=1)),
    ("paper_time_m3", lambda: datagen.paper_shaped(189, "V100", "time"), dict(mtry=3, target=1)),
    ("paper_power", lambda: datagen.paper_shaped(168, "P100", "power"), dict(mtry=4)),
    ("ties", lambda: datagen.tiny(200, 5, 3, distinct=6), dict(mtry=2)),
    ("noboot", lambda: datagen.tiny(120, 4, 5), dict(mtry=4, bootstrap=False)),
    ("depth3", lambda: datagen.paper_shaped(189, "TitanXp", "time"), dict(mtry=5, max_depth=3, target=1)),
    ("mss5", lambda: datagen.tiny(150, 6, 8, distinct=20), dict(mtry=3, min_samples_split=5)),
    ("n255", lambda: datagen.tiny(255, 3, 9), dict(mtry=1)),
    ("n2", lambda: (np.array([[0.0], [1.0]]), np.array([1.0, 3.0])), dict(mtry=1)),
    ("const", lambda: (datagen.tiny(40, 3, 1)[0], np.full(40, 2.5)), dict(mtry=2)),
    ("negzero", lambda: (np.array([[-0.0, 1], [0.0, 2], [1, 3], [2, 1]]), np.array([1.0, 2, 3, 4])), dict(mtry=2)),
]


@pytest.mark.parametrize("name,data,kw", FIT_CASES, ids=[c[0] for c in FIT_CASES])
def test_fit_structures_bit_exact(name, data, kw):
    X, y = data()
    of = oracle.fit(X, y, ntree=24, seed=11, leaf_rows=True, **kw)
    gf = rfg.fit(X, y, ntree=24, seed=11, debug=True, **kw)
    _compare_forest(gf, of, X)


def test_fit_many_seeds_paper_shaped():
    X, y = datagen.paper_shaped(189, "GTX1650", "time")
    for seed in range(6):
        of = oracle.fit(X, y, ntree=64, seed=seed, mtry=3, target=1, leaf_rows=True)
        gf = rfg.fit(X, y, ntree=64, seed=seed, mtry=3, target=1, debug=True)
        _compare_forest(gf, of, X)


def test_fit_tree_shard_is_prefix():
    X, y = datagen.paper_shaped(189, "K20", "time")
    full = rfg.fit(X, y, ntree=32, seed=4, mtry=3, target=1).export()
    part = rfg.fit(X, y, ntree=32, seed=4, mtry=3, target=1, tree_begin=8, tree_end=20).export()
    a, b = int(full["tree_off"][8]), int(full["tree_off"][20])
    assert np.array_equal(part["feature"], full["feature"][a:b])
    assert np.array_equal(part["value"].view(np.int64), full["value"][a:b].view(np.int64))


def test_fit_device_path_matches_host():
    X, y = datagen.paper_shaped(168, "V100", "power")
    h = rfg.fit(X, y, ntree=16, seed=2, mtry=4).export()
    d = rfg.fit(_cuda(X), _cuda(y), ntree=16, seed=2, mtry=4)
    torch.cuda.synchronize()
    d = d.export()
    for key in ("feature", "left", "thr_index"):
        assert np.array_equal(h[key], d[key])
    assert np.array_equal(h["value"].view(np.int64), d["value"].view(np.int64))


# ------------------------------------------------------------ predict ---
@pytest.fixture(params=[0, 1], ids=["node8_bf16", "node16_fp32"])
def node_layout(request):
    """Batched inference through the compact 8-byte nodes with bf16 staging (default) and through
    the 16-byte nodes with fp32 staging (rf_debug_set_option "predict_node16")."""
    rfg.debug_set_option("predict_node16", request.param)
    yield request.param
    rfg.debug_set_option("predict_node16", 0)


@pytest.mark.parametrize("target", [0, 1])
def test_predict_parity(target, node_layout):
    X, y = datagen.paper_shaped(189, "P100", "time")
    Q = datagen.paper_shaped(500, "P100", "time", seed=123)[0]
    of = oracle.fit(X, y, ntree=50, seed=3, mtry=4, target=target)
    gf = rfg.fit(X, y, ntree=50, seed=3, mtry=4, target=target)
    want = oracle.predict(of, Q)
    got = rfg.predict(gf, Q)
    np.testing.assert_allclose(got, want, rtol=RTOL, atol=0)
    got_d = rfg.predict(gf, _cuda(Q)).cpu().numpy()
    np.testing.assert_allclose(got_d, want, rtol=RTOL, atol=0)
    # partial + finalize (tree-shard combine) equals predict
    part = rfg.predict_partial(gf, _cuda(Q))
    fin = rfg.predict_finalize(part, 50, target).cpu().numpy()
    np.testing.assert_allclose(fin, want, rtol=RTOL, atol=0)


@pytest.mark.parametrize("nq", [1, 7, 256, 257])
def test_predict_few_rows_latency_path(nq):
    X, y = datagen.paper_shaped(189, "K20", "time")
    of = oracle.fit(X, y, ntree=512, seed=3, mtry=12, target=1)
    gf = rfg.fit(X, y, ntree=512, seed=3, mtry=12, target=1)
    Q = datagen.paper_shaped(300, "K20", "time", seed=77)[0][:nq]
    np.testing.assert_allclose(rfg.predict(gf, Q), oracle.predict(of, Q), rtol=RTOL, atol=0)
    Qn = Q.copy()
    Qn[-1, 3] = np.inf
    with pytest.raises(rfg.RFError) as e:
        rfg.predict(gf, Qn)
    assert e.value.code == rfg.E_NONFINITE


def test_predict_fits_exactly():
    X, y = datagen.paper_shaped(189, "K20", "time")
    _, idx = np.unique(X, axis=0, return_index=True)
    X, y = X[np.sort(idx)], y[np.sort(idx)]
    gf = rfg.fit(X, y, ntree=1, mtry=12, bootstrap=False)
    _, tq, F = oracle.quantize(y, 0)
    assert np.array_equal(rfg.predict(gf, X), np.ldexp(tq.astype(np.float64), -F))


# ----------------------------------------------------------------- CV ---
CV_CASES = [
    ("c1_paper", lambda: datagen.paper_shaped(189, "K20", "time"), dict(k=10, reps=1, ntrees=[20], mtrys=[12], target=1)),
    ("grid_power", lambda: datagen.paper_shaped(168, "V100", "power"),
     dict(k=10, reps=2, ntrees=[8, 16, 32], mtrys=[12, 3, 3], target=0)),
    ("k2", lambda: datagen.tiny(90, 3, 4), dict(k=2, reps=2, ntrees=[5, 10], mtrys=[1, 3], target=0)),
    ("loo", lambda: datagen.tiny(30, 2, 5), dict(k=30, reps=1, ntrees=[6], mtrys=[2], target=1)),
    ("ties", lambda: datagen.tiny(150, 4, 6, distinct=5), dict(k=5, reps=3, ntrees=[12], mtrys=[2], target=1)),
]


@pytest.mark.parametrize("name,data,kw", CV_CASES, ids=[c[0] for c in CV_CASES])
def test_cv_parity(name, data, kw):
    X, y = data()
    fm_o, pr_o = oracle.cv_grid(X, y, kw["k"], kw["reps"], kw["ntrees"], kw["mtrys"], target=kw["target"],
                                seed=9, want_pred=True)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, kw["k"], kw["reps"], kw["ntrees"], kw["mtrys"], target=kw["target"],
                                         seed=9, want_pred=True)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)


def test_cv_custom_split_and_device_path():
    X, y = datagen.paper_shaped(189, "TitanXp", "time")
    f = oracle.make_folds(y, 10, 3, seed=5, custom=True)
    fm_o = oracle.cv_grid(X, y, 10, 3, [16, 32], [12, 3], fold_ids=f, target=1, seed=5)
    fm_g = rfg.cross_validate_grid(_cuda(X), _cuda(y), 10, 3, [16, 32], [12, 3],
                                   fold_ids=_cuda(f, torch.int32), target=1, seed=5).cpu().numpy()
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)


def test_cv_task_shard():
    X, y = datagen.paper_shaped(168, "K20", "power")
    full = rfg.cross_validate_grid(X, y, 10, 2, [8], [4], seed=1)
    part = rfg.cross_validate_grid(X, y, 10, 2, [8], [4], seed=1, task_begin=5, task_end=13)
    flat_f, flat_p = full.reshape(-1), part.reshape(-1)
    assert np.array_equal(flat_p[5:13], flat_f[5:13])
    assert np.isnan(flat_p[:5]).all() and np.isnan(flat_p[13:]).all()


def test_cv_tree_shard_partial_finalize():
    X, y = datagen.paper_shaped(189, "V100", "time")
    Xd, yd = _cuda(X), _cuda(y)
    folds = rfg.make_folds(yd, 10, 2, seed=3)
    ntrees, mtrys = [16, 32], [3, 12]
    tot = None
    for lo, hi in [(0, 8), (8, 16), (16, 32)]:
        part = rfg.cv_partial(Xd, yd, 10, 2, folds, ntrees, mtrys, tree_begin=lo, tree_end=hi, target=1, seed=3)
        tot = part if tot is None else tot + part
    fm = rfg.cv_finalize(yd, 10, 2, folds, ntrees, len(mtrys), tot, target=1).cpu().numpy()
    want = oracle.cv_grid(X, y, 10, 2, ntrees, mtrys, fold_ids=folds.cpu().numpy(), target=1, seed=3)
    np.testing.assert_allclose(fm, want, rtol=RTOL, atol=0)
    # host twins (rf_cv_partial / rf_cv_finalize / rf_predict_partial)
    fh = folds.cpu().numpy()
    toth = sum(rfg.cv_partial(X, y, 10, 2, fh, ntrees, mtrys, tree_begin=lo, tree_end=hi, target=1, seed=3)
               for lo, hi in [(0, 16), (16, 32)])
    np.testing.assert_allclose(rfg.cv_finalize(y, 10, 2, fh, ntrees, len(mtrys), toth, target=1), want,
                               rtol=RTOL, atol=0)
    f = rfg.fit(X, y, ntree=12, seed=3, mtry=3, target=1)
    ph = rfg.predict_partial(f, X[:50])
    np.testing.assert_allclose(np.exp(ph / 12), rfg.predict(f, X[:50]), rtol=1e-12, atol=0)


def test_cv_full_study_config_sampled():
    """Full study config (30 reps x 10 folds x 1024 trees x mtry {12,3,3}) on one dataset;
    the oracle recomputes a sample of tasks (trees are keyed by (task, tree), R15)."""
    X, y = datagen.paper_shaped(189, "K20", "time")
    folds = oracle.make_folds(y, 10, 30, seed=7104, custom=True)
    nt, mt = [128, 256, 512, 1024], [12, 3, 3]
    fm_g = rfg.cross_validate_grid(X, y, 10, 30, nt, mt, fold_ids=folds, target=1, seed=7104)
    assert np.isfinite(fm_g).all()
    for task in (0, 157, 299):
        fm_o = oracle.cv_grid(X, y, 10, 30, nt, [12, 3], fold_ids=folds, target=1, seed=7104,
                              task_begin=task, task_end=task + 1)
        rep, fold = divmod(task, 10)
        np.testing.assert_allclose(fm_g[[0, 1], :, rep, fold], fm_o[:, :, rep, fold], rtol=RTOL, atol=0)
    assert np.array_equal(fm_g[1], fm_g[2])


# ------------------------------------------------- large-n exact path ---
LARGE_FIT_CASES = [
    ("n256", lambda: datagen.tiny(256, 4, 21), dict(mtry=2)),
    ("n300_ties", lambda: datagen.tiny(300, 5, 22, distinct=7), dict(mtry=3)),
    ("paper1000", lambda: datagen.paper_shaped(1000, "V100", "time"), dict(mtry=4, target=1)),
    ("paper2000_noboot", lambda: datagen.paper_shaped(2000, "K20", "power"), dict(mtry=12, bootstrap=False)),
    ("scaled5000_depth", lambda: datagen.scaled(5000, 64), dict(mtry=21, max_depth=8, target=1)),
    ("mss7", lambda: datagen.tiny(900, 3, 23, distinct=50), dict(mtry=3, min_samples_split=7)),
]


@pytest.mark.parametrize("name,data,kw", LARGE_FIT_CASES, ids=[c[0] for c in LARGE_FIT_CASES])
def test_large_fit_structures_bit_exact(name, data, kw):
    X, y = data()
    of = oracle.fit(X, y, ntree=5, seed=31, leaf_rows=True, **kw)
    gf = rfg.fit(X, y, ntree=5, seed=31, debug=True, **kw)
    _compare_forest(gf, of, X)


def test_large_fit_scaled_100k_sampled():
    """Config 3 shape (100k x 64, mtry 21, unbounded depth): 2 trees vs the oracle."""
    X, y = datagen.scaled(100_000, 64)
    of = oracle.fit(X, y, ntree=2, seed=7, mtry=21, target=1)
    gf = rfg.fit(X, y, ntree=2, seed=7, mtry=21, target=1)
    _compare_forest(gf, of, X)
    Q = datagen.queries(2000, 64)
    np.testing.assert_allclose(rfg.predict(gf, Q), oracle.predict(of, Q), rtol=RTOL, atol=0)


def test_large_cv_parity():
    X, y = datagen.paper_shaped(700, "P100", "time")
    fm_o, pr_o = oracle.cv_grid(X, y, 3, 1, [4, 8], [3, 12], target=1, seed=3, want_pred=True)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, 3, 1, [4, 8], [3, 12], target=1, seed=3, want_pred=True)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)


# ------------------------------------------------ histogram split mode ---
HIST_CASES = [
    ("few_distinct", lambda: datagen.tiny(300, 5, 41, distinct=40), dict(mtry=3)),
    ("paper600", lambda: datagen.paper_shaped(600, "K20", "time"), dict(mtry=4, target=1)),
    ("scaled3000", lambda: datagen.scaled(3000, 64), dict(mtry=21, max_depth=6, target=1)),
    ("small_n", lambda: datagen.tiny(120, 3, 42), dict(mtry=2)),
    ("noboot_mss", lambda: datagen.tiny(800, 4, 43, distinct=300), dict(mtry=4, bootstrap=False, min_samples_split=5)),
]


@pytest.mark.parametrize("name,data,kw", HIST_CASES, ids=[c[0] for c in HIST_CASES])
def test_hist_fit_structures_bit_exact(name, data, kw):
    X, y = data()
    of = oracle.fit(X, y, ntree=4, seed=17, leaf_rows=True, split_mode=1, **kw)
    gf = rfg.fit(X, y, ntree=4, seed=17, debug=True, split_mode=1, **kw)
    _compare_forest(gf, of, X)


def test_hist_equals_exact_structure_when_few_distinct():
    """Cross-mode pin: with <= 256 distinct values per feature the histogram
    mode grows the same partitions as the exact mode."""
    X, y = datagen.tiny(2000, 6, 44, distinct=100)
    ge = rfg.fit(X, y, ntree=6, seed=2, mtry=3, debug=True).export()
    gh = rfg.fit(X, y, ntree=6, seed=2, mtry=3, debug=True, split_mode=1).export()
    for key in ("feature", "left", "thr_index"):
        assert np.array_equal(ge[key], gh[key]), key
    leaves = ge["feature"] < 0
    assert np.array_equal(ge["value"][leaves].view(np.int64), gh["value"][leaves].view(np.int64))


def test_hist_config4_shape_sampled():
    """Config 4 shape (x 64 features, mtry 21, max_depth 12, histogram mode) at 200k rows,
    2 trees vs the oracle; predictions on held-out rows."""
    X, y = datagen.scaled(200_000, 64)
    of = oracle.fit(X, y, ntree=2, seed=11, mtry=21, max_depth=12, split_mode=1, target=1)
    gf = rfg.fit(X, y, ntree=2, seed=11, mtry=21, max_depth=12, split_mode=1, target=1)
    _compare_forest(gf, of, X)
    Q = datagen.queries(5000, 64)
    np.testing.assert_allclose(rfg.predict(gf, Q), oracle.predict(of, Q), rtol=RTOL, atol=0)


def test_hist_cv_parity():
    X, y = datagen.paper_shaped(500, "V100", "power")
    fm_o, pr_o = oracle.cv_grid(X, y, 4, 1, [3, 6], [4], seed=5, split_mode=1, want_pred=True)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, 4, 1, [3, 6], [4], seed=5, split_mode=1, want_pred=True)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)


# ------------------------------------- ExtraTrees split mode (R29, NEXT-1) ---
EXTRA_CASES = [
    ("paper_time_m12_noboot", lambda: datagen.paper_shaped(189, "K20", "time"), dict(mtry=12, target=1, bootstrap=False)),
    ("paper_time_m3", lambda: datagen.paper_shaped(189, "V100", "time"), dict(mtry=3, target=1)),
    ("paper_power", lambda: datagen.paper_shaped(168, "P100", "power"), dict(mtry=4, bootstrap=False)),
    ("ties", lambda: datagen.tiny(200, 5, 3, distinct=6), dict(mtry=2)),
    ("depth3", lambda: datagen.paper_shaped(189, "TitanXp", "time"), dict(mtry=5, max_depth=3, target=1)),
    ("mss5", lambda: datagen.tiny(150, 6, 8, distinct=20), dict(mtry=3, min_samples_split=5, bootstrap=False)),
    ("n255", lambda: datagen.tiny(255, 3, 9), dict(mtry=1)),
    ("n2", lambda: (np.array([[0.0], [1.0]]), np.array([1.0, 3.0])), dict(mtry=1)),
    ("negzero", lambda: (np.array([[-0.0, 1], [0.0, 2], [1, 3], [2, 1]]), np.array([1.0, 2, 3, 4])), dict(mtry=2)),
    # large path (n_tr > 255)
    ("large_n256", lambda: datagen.tiny(256, 4, 21), dict(mtry=2)),
    ("large_paper1000", lambda: datagen.paper_shaped(1000, "V100", "time"), dict(mtry=12, target=1, bootstrap=False)),
    ("large_ties", lambda: datagen.tiny(900, 3, 23, distinct=50), dict(mtry=3, min_samples_split=7)),
    ("large_scaled5000_depth", lambda: datagen.scaled(5000, 64), dict(mtry=21, max_depth=8, target=1)),
]


@pytest.mark.parametrize("name,data,kw", EXTRA_CASES, ids=[c[0] for c in EXTRA_CASES])
def test_extra_fit_structures_bit_exact(name, data, kw):
    X, y = data()
    of = oracle.fit(X, y, ntree=12, seed=13, leaf_rows=True, split_mode=2, **kw)
    gf = rfg.fit(X, y, ntree=12, seed=13, debug=True, split_mode=rfg.SPLIT_EXTRA, **kw)
    _compare_forest(gf, of, X)


def test_extra_large_scaled_50k_sampled():
    X, y = datagen.scaled(50_000, 64)
    of = oracle.fit(X, y, ntree=2, seed=5, mtry=64, bootstrap=False, target=1, split_mode=2)
    gf = rfg.fit(X, y, ntree=2, seed=5, mtry=64, bootstrap=False, target=1, split_mode=rfg.SPLIT_EXTRA)
    _compare_forest(gf, of, X)
    Q = datagen.queries(2000, 64)
    np.testing.assert_allclose(rfg.predict(gf, Q), oracle.predict(of, Q), rtol=RTOL, atol=0)


@pytest.mark.parametrize("n,boot", [(189, False), (189, True), (600, False)])
def test_extra_cv_parity(n, boot):
    X, y = datagen.paper_shaped(n, "GTX1650", "time")
    f = oracle.make_folds(y, 10, 2, seed=8, custom=True)
    fm_o, pr_o = oracle.cv_grid(X, y, 10, 2, [8, 16], [12, 3], fold_ids=f, target=1, seed=8, bootstrap=boot,
                                split_mode=2, want_pred=True)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, 10, 2, [8, 16], [12, 3], fold_ids=f, target=1, seed=8,
                                         bootstrap=boot, split_mode=rfg.SPLIT_EXTRA, want_pred=True)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)


# ------------------------------------- feature importance (MDI, NEXT-3) ---
IMP_CASES = [
    ("small_exact", lambda: datagen.paper_shaped(189, "K20", "time"), dict(mtry=4, target=1)),
    ("small_exact_m12", lambda: datagen.paper_shaped(168, "P100", "power"), dict(mtry=12)),
    ("small_extra", lambda: datagen.paper_shaped(189, "V100", "time"), dict(mtry=12, target=1, bootstrap=False,
                                                                          split_mode=2)),
    ("large_exact", lambda: datagen.paper_shaped(1000, "TitanXp", "time"), dict(mtry=4, target=1)),
    ("large_extra", lambda: datagen.paper_shaped(800, "K20", "power"), dict(mtry=6, split_mode=2)),
    ("hist", lambda: datagen.paper_shaped(600, "GTX1650", "time"), dict(mtry=4, target=1, split_mode=1)),
    ("scaled_depth", lambda: datagen.scaled(5000, 64), dict(mtry=21, max_depth=8, target=1)),
]


@pytest.mark.parametrize("name,data,kw", IMP_CASES, ids=[c[0] for c in IMP_CASES])
def test_importance_parity(name, data, kw):
    """Per-tree split-decrease sums within 1e-12 relative (order of the atomic sums and
    one rounding of the int128 numerator differ), importance vector within 1e-12."""
    X, y = data()
    of = oracle.fit(X, y, ntree=8, seed=21, **kw)
    gf = rfg.fit(X, y, ntree=8, seed=21, **kw)
    _compare_forest(gf, of, X)
    imp, raw = gf.importance(raw=True)
    want_raw = np.stack([t.imp_raw for t in of.trees])
    np.testing.assert_allclose(raw, want_raw, rtol=1e-12, atol=0)
    np.testing.assert_allclose(imp, of.importance(), rtol=0, atol=1e-12)
    assert abs(imp.sum() - 1.0) < 1e-12
    # tree shards: the combined raw arrays give the same vector (multi-GPU assembly)
    a = rfg.fit(X, y, ntree=8, seed=21, tree_begin=0, tree_end=3, **kw).importance(raw=True)[1]
    b = rfg.fit(X, y, ntree=8, seed=21, tree_begin=3, tree_end=8, **kw).importance(raw=True)[1]
    comb = rfg.importance_dev(_cuda(np.concatenate([a, b]))).cpu().numpy()
    np.testing.assert_allclose(comb, imp, rtol=0, atol=1e-14)


def test_importance_imported_forest_unsupported():
    X, y = datagen.paper_shaped(189, "K20", "time")
    e = rfg.fit(X, y, ntree=2, seed=1, mtry=3).export()
    f = rfg.forest_import(e["feature"], e["left"], e["value"], e["thr_index"], e["tree_off"], 12, e["F"], 0)
    with pytest.raises(rfg.RFError) as err:
        f.importance()
    assert err.value.code == rfg.E_UNSUPPORTED


# ----------------------------------------- nested CV, LOO, buckets (NEXT-2) ---
@pytest.mark.parametrize("custom", [False, True])
def test_masked_folds_bit_exact(custom):
    y = datagen.paper_shaped(189, "K20", "time")[1]
    rnd = np.random.default_rng(8)
    mask = (rnd.random((12, 189)) < 0.8).astype(np.uint8)
    want = oracle.make_folds_masked(y, 6, mask, seed=13, custom=custom)
    got = rfg.make_folds_masked(_cuda(y), 6, _cuda(mask, torch.uint8), seed=13, custom=custom).cpu().numpy()
    assert np.array_equal(got, want)


def test_cv_excluded_rows_parity():
    X, y = datagen.paper_shaped(189, "P100", "time")
    f = oracle.make_folds(y, 5, 3, seed=6, custom=True)
    f[:, ::7] = -2
    fm_o, pr_o = oracle.cv_grid(X, y, 5, 3, [8, 16], [12, 3], fold_ids=f, target=1, seed=6, want_pred=True)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, 5, 3, [8, 16], [12, 3], fold_ids=f, target=1, seed=6, want_pred=True)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)
    assert np.isnan(pr_g[:, :, :, ::7]).all()


@pytest.mark.parametrize("custom,split_mode", [(True, 0), (False, 0), (True, 2)])
def test_nested_cv_parity(custom, split_mode):
    """Inner scores and outer fold MAPEs <= 1e-9 relative; the selected grid point equal
    wherever the oracle's best beats the runner-up by more than 1e-8 relative (else both
    tied candidates are valid and the outer MAPE must be that candidate's)."""
    X, y = datagen.paper_shaped(189, "GTX1650", "time")
    kw = dict(custom=custom, seed=17, target=1, split_mode=split_mode,
              bootstrap=split_mode != 2)
    b_o, om_o, sc_o = oracle.nested_cv(X, y, 5, 4, 3, [8, 24], [12, 3], **kw)
    b_g, om_g, sc_g = rfg.nested_cv(X, y, 5, 4, 3, [8, 24], [12, 3], **kw)
    np.testing.assert_allclose(sc_g, sc_o, rtol=RTOL, atol=0)
    flat = sc_o.reshape(3, 5, -1)
    for it in range(3):
        for o in range(5):
            s = np.sort(flat[it, o])
            if s[1] - s[0] > 1e-8 * s[0]:
                assert b_g[it, o] == b_o[it, o]
            else:
                assert abs(flat[it, o, b_g[it, o]] - s[0]) <= 1e-8 * s[0]
    f = oracle.make_folds(y, 5, 3, seed=17, custom=custom)
    fm = oracle.cv_grid(X, y, 5, 3, [8, 24], [12, 3], fold_ids=f, seed=17, target=1, split_mode=split_mode,
                        bootstrap=split_mode != 2)
    for it in range(3):
        for o in range(5):
            mi, ti = divmod(int(b_g[it, o]), 2)
            np.testing.assert_allclose(om_g[it, o], fm[mi, ti, it, o], rtol=RTOL)
    # device twin
    bd, omd, _ = rfg.nested_cv(_cuda(X), _cuda(y), 5, 4, 3, [8, 24], [12, 3], **kw)
    assert np.array_equal(bd.cpu().numpy(), b_g) and np.array_equal(omd.cpu().numpy(), om_g)


def test_loo_and_error_buckets_parity():
    X, y = datagen.paper_shaped(189, "K20", "time")
    fm_o, pr_o = oracle.cv_grid(X, y, 189, 1, [64], [12], target=1, seed=2, want_pred=True)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, 189, 1, [64], [12], target=1, seed=2, want_pred=True)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    want = oracle.error_buckets(y, pr_o[0, 0, 0])
    assert rfg.error_buckets(y, pr_g[0, 0, 0]).tolist() == want.tolist()
    assert rfg.error_buckets(_cuda(y), _cuda(pr_g[0, 0, 0])).cpu().numpy().tolist() == want.tolist()
    # with ties at the bucket edges: y = 100, yhat on the edges
    ye = np.full(6, 100.0)
    yh = np.array([90.0, 110.0, 75.0, 150.0, 200.0, np.nan])
    assert rfg.error_buckets(ye, yh).tolist() == oracle.error_buckets(ye, yh).tolist() == [0, 2, 1, 1, 1]


# -------------------------------------------------------------- errors ---
def test_errors():
    X, y = datagen.tiny(20, 3, 1)
    with pytest.raises(rfg.RFError) as e:
        rfg.fit(np.zeros((0, 3)), np.zeros(0))
    assert e.value.code == rfg.E_EMPTY
    Xn = X.copy()
    Xn[3, 1] = np.nan
    with pytest.raises(rfg.RFError) as e:
        rfg.fit(Xn, y, ntree=2)
    assert e.value.code == rfg.E_NONFINITE
    with pytest.raises(rfg.RFError) as e:
        rfg.fit(X, y - 10, ntree=2, target=1)
    assert e.value.code == rfg.E_NONPOSITIVE_Y
    f = rfg.fit(X, y, ntree=2)
    with pytest.raises(rfg.RFError) as e:
        rfg.predict(f, np.zeros((3, 4)))
    assert e.value.code == rfg.E_ARITY
    with pytest.raises(rfg.RFError) as e:
        rfg.cross_validate_grid(X, y, 25, 1, [2], [1])
    assert e.value.code == rfg.E_TOO_FEW
    with pytest.raises(rfg.RFError) as e:
        rfg.cross_validate_grid(X, y - 10, 4, 1, [2], [1])
    assert e.value.code == rfg.E_NONPOSITIVE_Y


# ------------------------------------------------ MAE criterion (NEXT-4, R32) ---
MAE_CASES = [
    ("paper_time_m12", lambda: datagen.paper_shaped(189, "K20", "time"), dict(mtry=12, target=1)),
    ("paper_time_m3", lambda: datagen.paper_shaped(189, "V100", "time"), dict(mtry=3, target=1)),
    ("paper_power", lambda: datagen.paper_shaped(168, "P100", "power"), dict(mtry=4)),
    ("ties", lambda: datagen.tiny(200, 5, 3, distinct=6), dict(mtry=2)),
    ("target_ties", lambda: (datagen.tiny(150, 4, 4)[0], np.round(datagen.tiny(150, 4, 4)[1], 0)), dict(mtry=3)),
    ("noboot", lambda: datagen.tiny(120, 4, 5), dict(mtry=4, bootstrap=False)),
    ("depth3", lambda: datagen.paper_shaped(189, "TitanXp", "time"), dict(mtry=5, max_depth=3, target=1)),
    ("mss5", lambda: datagen.tiny(150, 6, 8, distinct=20), dict(mtry=3, min_samples_split=5)),
    ("n255", lambda: datagen.tiny(255, 3, 9), dict(mtry=1)),
    ("n2", lambda: (np.array([[0.0], [1.0]]), np.array([1.0, 3.0])), dict(mtry=1)),
    ("const", lambda: (datagen.tiny(40, 3, 1)[0], np.full(40, 2.5)), dict(mtry=2)),
    ("p40", lambda: datagen.tiny(90, 40, 6, distinct=30), dict(mtry=13)),
    # ExtraTrees + MAE: the paper's best models (T4/T5 P:858-861)
    ("extra_time_m12", lambda: datagen.paper_shaped(189, "K20", "time"), dict(mtry=12, target=1, bootstrap=False,
                                                                             split_mode=2)),
    ("extra_power_boot", lambda: datagen.paper_shaped(168, "GTX1650", "power"), dict(mtry=4, split_mode=2)),
    ("extra_ties", lambda: datagen.tiny(200, 5, 3, distinct=6), dict(mtry=2, split_mode=2, bootstrap=False)),
    # ExtraTrees + MAE candidate ring (mae_flush): 12 candidates per node, several nodes and
    # flushes per level, equal costs across candidates (ties in x and y) -> the R9 tie-break
    ("extra_ring_ties", lambda: (datagen.tiny(240, 12, 4, distinct=4)[0],
                                 np.round(datagen.tiny(240, 12, 4)[1], 0) + 1.0),
     dict(mtry=12, split_mode=2)),
]


@pytest.mark.parametrize("name,data,kw", MAE_CASES, ids=[c[0] for c in MAE_CASES])
def test_mae_fit_structures_bit_exact(name, data, kw):
    """Structures, medians (leaf values) and leaf row sets bit-exact; the MAE costs are exact
    integers on both sides, so the chosen splits cannot differ."""
    X, y = data()
    of = oracle.fit(X, y, ntree=16, seed=31, leaf_rows=True, criterion=1, **kw)
    gf = rfg.fit(X, y, ntree=16, seed=31, debug=True, criterion=rfg.CRITERION_MAE, **kw)
    _compare_forest(gf, of, X)
    Q = np.random.default_rng(1).permuted(np.concatenate([X, X]), axis=0)  # columns shuffled independently
    np.testing.assert_allclose(rfg.predict(gf, Q), oracle.predict(of, Q), rtol=RTOL, atol=0)


def test_mae_fit_many_seeds_paper_shaped():
    X, y = datagen.paper_shaped(189, "GTX1650", "time")
    for seed in range(4):
        for sm in (0, 2):
            of = oracle.fit(X, y, ntree=32, seed=seed, mtry=3, target=1, split_mode=sm, criterion=1)
            gf = rfg.fit(X, y, ntree=32, seed=seed, mtry=3, target=1, split_mode=sm, criterion=1)
            _compare_forest(gf, of, X)


@pytest.mark.parametrize("custom,split_mode,boot", [(True, 0, True), (False, 0, True), (True, 2, False)])
def test_mae_cv_parity(custom, split_mode, boot):
    X, y = datagen.paper_shaped(189 if custom else 168, "V100", "time" if custom else "power")
    f = oracle.make_folds(y, 10, 2, seed=9, custom=custom)
    kw = dict(fold_ids=f, target=1 if custom else 0, seed=9, bootstrap=boot, split_mode=split_mode,
              want_pred=True, criterion=1)
    fm_o, pr_o = oracle.cv_grid(X, y, 10, 2, [4, 12], [12, 3], **kw)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, 10, 2, [4, 12], [12, 3], **kw)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)
    # device twin
    fm_d = rfg.cross_validate_grid(_cuda(X), _cuda(y), 10, 2, [4, 12], [12, 3], fold_ids=_cuda(f, torch.int32),
                                   target=kw["target"], seed=9, bootstrap=boot, split_mode=split_mode,
                                   criterion=1)
    np.testing.assert_allclose(fm_d.cpu().numpy(), fm_o, rtol=RTOL, atol=0)


@pytest.mark.parametrize("split_mode", [0, 2])
def test_mae_importance_parity(split_mode):
    X, y = datagen.paper_shaped(189, "K20", "time")
    kw = dict(mtry=6, target=1, split_mode=split_mode, bootstrap=split_mode == 0, criterion=1)
    of = oracle.fit(X, y, ntree=8, seed=23, **kw)
    gf = rfg.fit(X, y, ntree=8, seed=23, **kw)
    _compare_forest(gf, of, X)
    imp, raw = gf.importance(raw=True)
    np.testing.assert_allclose(raw, np.stack([t.imp_raw for t in of.trees]), rtol=1e-12, atol=0)
    np.testing.assert_allclose(imp, of.importance(), rtol=0, atol=1e-12)


def test_mae_unsupported_shapes():
    X, y = datagen.scaled(13_000, 16)
    with pytest.raises(rfg.RFError) as e:  # beyond the level-synchronous MAE path (12,288 rows)
        rfg.fit(X, y, ntree=2, mtry=3, target=1, criterion=1)
    assert e.value.code == rfg.E_UNSUPPORTED
    with pytest.raises(rfg.RFError) as e:  # histogram mode has no MAE variant (R32)
        rfg.fit(X[:100], y[:100], ntree=2, mtry=3, target=1, split_mode=rfg.SPLIT_HIST256, criterion=1)
    assert e.value.code == rfg.E_UNSUPPORTED


MAE_LARGE_CASES = [
    # n_tr > 255: the level-synchronous MAE path (R32), exact and ExtraTrees, ties, no bootstrap
    ("paper600", lambda: datagen.paper_shaped(600, "K20", "time"), dict(mtry=4, target=1)),
    ("ties", lambda: datagen.tiny(700, 5, 51, distinct=7), dict(mtry=3)),
    ("extra_noboot", lambda: datagen.paper_shaped(500, "V100", "power"), dict(mtry=6, split_mode=2, bootstrap=False)),
    ("depth_mss", lambda: datagen.tiny(900, 6, 52, distinct=40), dict(mtry=6, max_depth=7, min_samples_split=4)),
    ("scaled_p64", lambda: datagen.scaled(1500, 64), dict(mtry=21, target=1, max_depth=10)),
    ("tie_draw", lambda: datagen.tiny(400, 4, 53, distinct=5), dict(mtry=4, tie_break=1)),
]


@pytest.mark.parametrize("name,data,kw", MAE_LARGE_CASES, ids=[c[0] for c in MAE_LARGE_CASES])
def test_mae_large_fit_bit_exact(name, data, kw):
    """MAE on the level-synchronous path: structures, medians and leaf row sets bit-exact; MAE
    importance (SAD2(node) - D) within 1e-12."""
    X, y = data()
    of = oracle.fit(X, y, ntree=4, seed=61, leaf_rows=True, criterion=1, **kw)
    gf = rfg.fit(X, y, ntree=4, seed=61, debug=True, criterion=1, **kw)
    _compare_forest(gf, of, X)
    imp, raw = gf.importance(raw=True)
    np.testing.assert_allclose(raw, np.stack([t.imp_raw for t in of.trees]), rtol=1e-12, atol=0)


def test_mae_large_cv_parity():
    X, y = datagen.paper_shaped(700, "P100", "time")
    fm_o, pr_o = oracle.cv_grid(X, y, 3, 1, [3, 6], [4], target=1, seed=8, criterion=1, want_pred=True)
    fm_g, pr_g = rfg.cross_validate_grid(X, y, 3, 1, [3, 6], [4], target=1, seed=8, criterion=1, want_pred=True)
    np.testing.assert_allclose(fm_g, fm_o, rtol=RTOL, atol=0)
    np.testing.assert_allclose(pr_g, pr_o, rtol=RTOL, atol=0)


# ------------------------------------------- alternative large-path kernels ---
def test_large_partition_paths_agree():
    """The fused multi-list partition (default for n <= 2^20) and the tiled count/scan/scatter
    partition (histogram mode, n > 2^20) grow identical forests; the tiled one also matches the
    oracle, leaf row sets included."""
    X, y = datagen.scaled(20_000, 64)
    a = rfg.fit(X, y, ntree=4, mtry=21, target=1, seed=3).export()
    rfg.debug_set_option("large_tiled_partition", 1)
    try:
        b = rfg.fit(X, y, ntree=4, mtry=21, target=1, seed=3).export()
        Xs, ys = datagen.tiny(600, 5, 17, distinct=40)
        of = oracle.fit(Xs, ys, ntree=4, seed=5, mtry=3, leaf_rows=True)
        gf = rfg.fit(Xs, ys, ntree=4, seed=5, mtry=3, debug=True)
        _compare_forest(gf, of, Xs)
    finally:
        rfg.debug_set_option("large_tiled_partition", 0)
    for key in ("feature", "left", "thr_index", "tree_off"):
        assert np.array_equal(a[key], b[key]), key
    assert np.array_equal(a["value"].view(np.int64), b["value"].view(np.int64))
    with pytest.raises(rfg.RFError):
        rfg.debug_set_option("no_such_option", 1)


def test_predict_c5_shape(node_layout):
    """Config 5 shape: forest grown on scaled(20k, 64) with max_depth 12 (30 trees: two
    12-tree groups of the batched kernel plus a remainder), 200k query rows through the
    batched kernel (device and host entry points) vs the oracle, <= 1e-9 relative."""
    X, y = datagen.scaled(20_000, 64)
    of = oracle.fit(X, y, ntree=30, seed=9, mtry=21, target=1, max_depth=12)
    gf = rfg.fit(X, y, ntree=30, seed=9, mtry=21, target=1, max_depth=12)
    _compare_forest(gf, of, X)
    Q = datagen.queries(200_000, 64)
    want = oracle.predict(of, Q)
    np.testing.assert_allclose(rfg.predict(gf, _cuda(Q)).cpu().numpy(), want, rtol=RTOL, atol=0)
    np.testing.assert_allclose(rfg.predict(gf, Q[:777]), want[:777], rtol=RTOL, atol=0)


def test_predict_threshold_ties(node_layout):
    """Batched inference on query values at and next to the split thresholds (x == thr goes
    left; neighbours one ulp away, which share the threshold's fp32 rounding, must be decided
    in fp64) -- thresholds taken from the oracle's forest."""
    X, y = datagen.paper_shaped(189, "K20", "time")
    of = oracle.fit(X, y, ntree=40, seed=4, mtry=4, target=1)
    gf = rfg.fit(X, y, ntree=40, seed=4, mtry=4, target=1)
    _compare_forest(gf, of, X)
    rnd = np.random.default_rng(0)
    feats = np.concatenate([t.feature[t.feature >= 0] for t in of.trees])
    thrs = np.concatenate([t.thr_value[t.feature >= 0] for t in of.trees])
    Q = np.repeat(X[rnd.integers(0, len(X), 2000)], 1, axis=0).copy()
    for r in range(len(Q)):
        for _ in range(6):
            k = rnd.integers(0, len(feats))
            Q[r, feats[k]] = [thrs[k], np.nextafter(thrs[k], np.inf), np.nextafter(thrs[k], -np.inf)][r % 3]
    np.testing.assert_allclose(rfg.predict(gf, _cuda(Q)).cpu().numpy(), oracle.predict(of, Q), rtol=RTOL, atol=0)


def test_predict_quantised_ties(node_layout):
    """Query values that round to the threshold's bf16 (and, some, fp32) value but differ from it
    in fp64 -- thr * (1 +- 2^-k) for k = 9 .. 30 -- so the staged comparison ties and the decision
    must come from the fp64 row and threshold; every internal node's threshold is hit."""
    X, y = datagen.scaled(3_000, 16)
    of = oracle.fit(X, y, ntree=24, seed=5, mtry=5, target=1, max_depth=10)
    gf = rfg.fit(X, y, ntree=24, seed=5, mtry=5, target=1, max_depth=10)
    _compare_forest(gf, of, X)
    rnd = np.random.default_rng(1)
    feats = np.concatenate([t.feature[t.feature >= 0] for t in of.trees])
    thrs = np.concatenate([t.thr_value[t.feature >= 0] for t in of.trees])
    Q = X[rnd.integers(0, len(X), 3000)].copy()
    for r in range(len(Q)):
        for _ in range(8):
            k = rnd.integers(0, len(feats))
            e = int(rnd.integers(9, 31))
            Q[r, feats[k]] = thrs[k] * (1.0 + (1 if r % 2 else -1) * 2.0 ** -e)
    np.testing.assert_allclose(rfg.predict(gf, _cuda(Q)).cpu().numpy(), oracle.predict(of, Q), rtol=RTOL, atol=0)


def test_large_packed_rank_collisions():
    """The large path packs the low 15 bits of a row's x rank into its list entry (n <= 2^17)
    and gathers full ranks only when two neighbours' low bits agree.  Here feature 1 pairs
    rows i and i + 32768, so nodes end up holding such pairs whose x0 ranks differ by exactly
    2^15 (equal low bits, different values): the split between them must still be found."""
    n = 40_000
    i = np.arange(n)
    X = np.stack([i.astype(np.float64), (i % 32768).astype(np.float64)], 1)
    y = np.random.default_rng(5).normal(size=n) * 3 + 10
    of = oracle.fit(X, y, ntree=2, seed=1, mtry=2, bootstrap=False, leaf_rows=True)
    gf = rfg.fit(X, y, ntree=2, seed=1, mtry=2, bootstrap=False, debug=True)
    _compare_forest(gf, of, X)


def test_large_unpacked_rows_150k():
    """Exact mode above 2^17 rows: list entries are plain row ids (no rank bits), ranks are
    gathered for every boundary test; 150k rows, ExtraTrees and exact, vs the oracle."""
    X, y = datagen.scaled(150_000, 16)
    for kw in (dict(mtry=5), dict(mtry=8, split_mode=2, bootstrap=False)):
        of = oracle.fit(X, y, ntree=1, seed=4, target=1, **kw)
        gf = rfg.fit(X, y, ntree=1, seed=4, target=1, **kw)
        _compare_forest(gf, of, X)


@pytest.mark.gpu
def test_large_path_row_level_counter():
    """rf_debug_row_levels: the large-n path's unit of work equals
    sum over rows of the depth of the row's leaf when every node with >= 2 distinct rows splits
    (no bootstrap, mtry = p, continuous x and y) -- the figure bench_configs.py's C3 roofline uses."""
    X, y = datagen.tiny(400, 3, 5)
    rfg.row_levels(reset=True)
    gf = rfg.fit(X, y, ntree=3, seed=4, mtry=3, bootstrap=False, debug=True)
    got = rfg.row_levels(reset=True)
    e = gf.export()
    lr = gf.leaf_rows()
    want = 0
    for t in range(3):
        a, b = int(e["tree_off"][t]), int(e["tree_off"][t + 1])
        feat, left = e["feature"][a:b], e["left"][a:b]
        depth = np.zeros(b - a, np.int64)
        for i in range(b - a):  # BFS order: parents precede children
            if feat[i] >= 0:
                depth[left[i]] = depth[left[i] + 1] = depth[i] + 1
        want += int(depth[lr[t]].sum())
    assert got == want > 0
