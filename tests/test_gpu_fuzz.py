"""Randomised parity sweep of the CUDA path against the oracle: many small shapes across every
kernel variant (CTA-resident and level-synchronous paths, exact / histogram / ExtraTrees split
modes, MSE / MAE, bootstrap on/off, depth caps, min_samples_split, ties in x and in y,
IDENTITY / LOG targets); structures bit-exact, predictions <= 1e-9 relative, and a CV grid
per configuration family.  Seeds are fixed, so a failure is reproducible."""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2001_07104_b200 as rfg  # noqa: E402
from test_gpu_parity import RTOL, _compare_forest  # noqa: E402


def _config(i):
    rng = np.random.default_rng([2001, 7104, i])
    large = i % 4 == 3
    n = int(rng.integers(256, 700)) if large else int(rng.integers(2, 256))
    p = int(rng.integers(1, 13))
    mode = int(rng.choice([0, 0, 1, 2]))
    crit = int(rng.random() < 0.25) if (not large and mode != 1) else 0
    kw = dict(mtry=int(rng.integers(1, p + 1)), bootstrap=bool(rng.random() < 0.7),
              max_depth=int(rng.choice([-1, -1, 2, 5])), min_samples_split=int(rng.choice([2, 2, 3, 7])),
              split_mode=mode, criterion=crit, target=int(rng.random() < 0.5), seed=int(rng.integers(0, 1 << 30)))
    distinct = int(rng.choice([0, 3, 20])) or None
    X, y = datagen.tiny(n, p, i, distinct=distinct)
    if rng.random() < 0.2:
        y = np.round(y, 1) + 0.5  # ties in the target
    return X, y, kw


@pytest.mark.parametrize("i", range(48))
def test_fuzz_fit_parity(i):
    X, y, kw = _config(i)
    of = oracle.fit(X, y, ntree=4, leaf_rows=True, **kw)
    gf = rfg.fit(X, y, ntree=4, debug=True, **kw)
    _compare_forest(gf, of, X)
    Q = np.random.default_rng(i).permuted(np.concatenate([X, X + 0.25]), axis=0)
    np.testing.assert_allclose(rfg.predict(gf, Q), oracle.predict(of, Q), rtol=RTOL, atol=0)


@pytest.mark.parametrize("i", range(8))
def test_fuzz_cv_parity(i):
    X, y, kw = _config(100 + i)
    n = len(y)
    k = int(min(max(2, n // 8), 10))
    if n < 2 * k or kw["split_mode"] == 1 and n > 255:
        pytest.skip("shape too small for CV")
    kw = dict(kw)
    m = kw.pop("mtry")
    seed = kw.pop("seed")
    f = oracle.make_folds(y, k, 2, seed=seed)
    fo = oracle.cv_grid(X, y, k, 2, [2, 4], [m, max(1, m // 2)], fold_ids=f, seed=seed, **kw)
    fg = rfg.cross_validate_grid(X, y, k, 2, [2, 4], [m, max(1, m // 2)], fold_ids=f, seed=seed, **kw)
    np.testing.assert_allclose(fg, fo, rtol=RTOL, atol=0)
