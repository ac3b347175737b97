"""The product's double-double ln (csrc/ddlog.cuh, R20) built for the host and pinned
against 200-bit mpmath: the evaluation's relative error stays far inside the 2^-95 bound the
rounding test assumes, every certified result is the correctly rounded ln, and the rounding test
rejects double-double values near a rounding boundary.  The device runs the same operation
sequence (IEEE intrinsics, no contraction); tests/test_gpu_parity.py and test_gpu_boundary.py
compare the device bits with the oracle, and test_gpu_boundary.py reaches RF_E_INEXACT."""
import math
import os
import struct
import subprocess

import numpy as np
import pytest

mpmath = pytest.importorskip("mpmath")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2001_07104_b200", "csrc")
HARNESS = os.path.join(ROOT, "tests", "ddlog_host.cpp")


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("ddlog") / "ddlog_host")
    subprocess.run(["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-I" + CSRC, HARNESS, "-o", out],
                   check=True, capture_output=True)
    return out


def run(exe, data, mode, margin=None):
    args = [exe, str(mode)] + ([str(margin)] if margin is not None else [])
    r = subprocess.run(args, input=np.ascontiguousarray(data, dtype=np.float64).tobytes(),
                       capture_output=True, check=True)
    return np.frombuffer(r.stdout, dtype=np.float64).reshape(-1, 4 if mode == 0 else 2)


def inputs():
    rng = np.random.default_rng(2001_07104)
    bits = rng.integers(1, 0x7FEFFFFFFFFFFFFF, size=20000, dtype=np.int64)  # positive finite, subnormals incl.
    vals = [bits.view(np.float64)]
    vals.append(10.0 ** rng.uniform(-3, 9, 20000))  # the paper's measurement range (ms, W)
    vals.append(1.0 + rng.uniform(-0.3, 0.42, 5000))  # e = 0: ln m alone, no e ln2 term
    k = np.arange(1, 600, dtype=np.float64)
    # the structured hard cases (ln y within ~2^-105 of a midpoint, e.g. y = 1 - 2^-52): the
    # |y - 1| <= 2^-26 branch; and both sides of that branch's bound
    vals += [1.0 + k * 2.0 ** -52, 1.0 - k * 2.0 ** -53, 1.0 + rng.integers(1, 2 ** 20, 2000) * 2.0 ** -46,
             1.0 + rng.uniform(-2.0 ** -26, 2.0 ** -26, 2000),
             np.array([1 + 2.0 ** -26, 1 - 2.0 ** -26, np.nextafter(1 + 2.0 ** -26, 2), np.nextafter(1 - 2.0 ** -26, 0)])]
    s2 = math.sqrt(2.0)
    vals.append(np.array([np.nextafter(s2, 0), s2, np.nextafter(s2, 3), np.nextafter(s2 / 2, 0), s2 / 2,
                          np.nextafter(s2 / 2, 3)]) * 2.0 ** rng.integers(-60, 60, 6))  # range-split edges
    vals.append(2.0 ** np.arange(-1074, 1024, 7, dtype=np.float64))  # exact powers of two
    vals.append(np.array([5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, 1.0, 2.0, math.e]))
    return np.concatenate(vals)


def test_ln_dd_error_bound_and_correct_rounding(exe):
    y = inputs()
    out = run(exe, y, 0)
    mpmath.mp.prec = 200
    worst = 0.0
    for yi, (hi, lo, d, ok) in zip(y, out):
        ref = mpmath.log(mpmath.mpf(float(yi)))
        if yi == 1.0:
            assert hi == 0.0 and lo == 0.0 and d == 0.0 and ok == 1.0
            continue
        err = abs((mpmath.mpf(hi) + mpmath.mpf(lo) - ref) / ref)  # ln_dd (the general branch)
        worst = max(worst, float(err))
        assert ok == 1.0, yi.hex()  # certified: no value of the sample is left undecided
        assert d == float(ref), yi.hex()  # and correctly rounded (mpmath float() rounds to nearest)
    # the rounding test assumes < 2^-95; the evaluation stays at least 2^4 below it
    assert worst < 2.0 ** -99, math.log2(worst)


def test_rounding_test_rejects_near_boundaries(exe):
    rng = np.random.default_rng(7)
    hi = np.concatenate([rng.uniform(0.35, 745.0, 300), -rng.uniform(0.35, 745.0, 300),
                         rng.uniform(2.0 ** -52, 0.3, 300)])
    ulp = np.spacing(np.abs(hi))
    cases, expect = [], []
    for h, u in zip(hi, ulp):
        for frac, certified in ((0.25, True), (-0.25, True), (0.0, True), (0.4999, True),
                                (0.5, False), (-0.5, False)):
            cases.append((h, frac * u)); expect.append(certified)
        for sgn in (1, -1):  # within 2^-96 |hi| of the midpoint: must be rejected
            cases.append((h, sgn * (0.5 * u - abs(h) * 2.0 ** -96))); expect.append(False)
            cases.append((h, sgn * (0.5 * u + abs(h) * 2.0 ** -96))); expect.append(False)
    out = run(exe, np.array(cases), 1)
    for (h, lo), (d, ok), e in zip(cases, out, expect):
        assert bool(ok) == e, (h, lo)
        if ok:  # a certified value is RN(hi + lo)
            assert d == float(mpmath.mpf(h) + mpmath.mpf(lo))


def test_rounding_test_margin_switch(exe):
    # a wide margin (the rf_debug_set_option "ln_cert_margin_log2" path) rejects ordinary values
    y = 10.0 ** np.random.default_rng(3).uniform(-3, 9, 2000)
    out = run(exe, y, 0, margin=-20)
    assert (out[:, 3] == 0.0).mean() > 0.5
    assert np.array_equal(out[:, 2], run(exe, y, 0)[:, 2])  # the value does not depend on the margin
