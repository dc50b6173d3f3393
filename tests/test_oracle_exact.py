"""Pins for the oracle's exact-sum definition (reading R20, SURVEY.md
8(f) row 3): each bin's sum is the exact real sum of its values rounded once
to nearest-even.  Pinned against Python's exact rational arithmetic
(fractions.Fraction; float() of a Fraction rounds correctly, ties to even),
math.fsum (Shewchuk's correctly rounded sum), closed forms and IEEE rounding
cases worked by hand -- none of which shares code with the C oracle.
"""
import math
import struct
import sys
from fractions import Fraction

import numpy as np
import pytest

import oracle

DMAX = sys.float_info.max
TINY = 5e-324  # 2^-1074


def bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def frac_sum(vals):
    s = sum((Fraction(v) for v in vals), Fraction(0))
    try:
        return float(s)
    except OverflowError:
        return math.inf if s > 0 else -math.inf


def random_doubles(rng, n, lo_exp=-1074, hi_exp=1000):
    e = rng.integers(lo_exp, hi_exp, n)
    m = rng.random(n) + 0.5
    v = np.ldexp(m, e) * rng.choice([-1.0, 1.0], n)
    return v


@pytest.mark.parametrize("seed", range(120))
def test_exact_sum_matches_fractions(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(0, 60))
    kind = seed % 4
    if kind == 0:    # every binade, both signs (subnormals included)
        v = random_doubles(rng, n)
    elif kind == 1:  # narrow range with heavy cancellation
        v = rng.normal(0, 1, n)
        v = np.concatenate([v, -v[: n // 2]])
    elif kind == 2:  # subnormal / smallest-normal neighbourhood
        v = random_doubles(rng, n, -1080, -1015)
    else:            # near overflow (exact intermediates beyond DBL_MAX)
        v = random_doubles(rng, n, 1000, 1024)
    v = v[np.isfinite(v)]
    got = oracle.exact_sum(v)
    want = frac_sum(v.tolist())
    assert bits(got) == bits(want if want != 0 else 0.0), (got, want)


@pytest.mark.parametrize("seed", range(8))
def test_exact_sum_matches_fsum_large(seed):
    rng = np.random.default_rng(1000 + seed)
    v = rng.normal(0, 1, 20000) * np.ldexp(1.0, rng.integers(-60, 60, 20000))
    assert bits(oracle.exact_sum(v)) == bits(math.fsum(v))


def test_exact_sum_hand_cases():
    e = 2.0 ** -53
    assert oracle.exact_sum([]) == 0.0 and bits(oracle.exact_sum([])) == bits(0.0)
    assert bits(oracle.exact_sum([-0.0])) == bits(0.0)              # zero results are +0.0
    assert bits(oracle.exact_sum([1.0, -1.0])) == bits(0.0)
    assert oracle.exact_sum([1.0, e]) == 1.0                        # tie -> even (1.0)
    assert oracle.exact_sum([1.0, e, e]) == 1.0 + 2 * e             # exact 1 + 2^-52: no tie at all
    assert oracle.exact_sum([1.0, 2 * e, e]) == 1.0 + 4 * e         # 1 + 3*2^-53: tie -> even mantissa
    assert oracle.exact_sum([TINY] * 3) == 3 * TINY                 # subnormal, exact
    assert oracle.exact_sum([2.0 ** -1022, -TINY]) == 2.0 ** -1022 - TINY
    assert oracle.exact_sum([DMAX, DMAX]) == math.inf
    assert oracle.exact_sum([-DMAX, -DMAX]) == -math.inf
    assert oracle.exact_sum([DMAX, DMAX, -DMAX]) == DMAX            # intermediate beyond DBL_MAX
    # half an ulp above DBL_MAX rounds to inf (ties to even: DBL_MAX's mantissa is odd)
    assert oracle.exact_sum([DMAX, 2.0 ** 970]) == math.inf
    assert oracle.exact_sum([DMAX, 2.0 ** 969]) == DMAX
    # closed form: 1..n in any order
    for n in (1, 1000, 100000):
        v = np.random.default_rng(n).permutation(np.arange(1, n + 1, dtype=np.float64))
        assert oracle.exact_sum(v) == n * (n + 1) / 2


def test_binned_exact_sums():
    """Per bin: exact sum == fsum of the rows numpy puts in that bin (rows kept off
    the edges); == the row-order sum when every partial sum is exact."""
    rng = np.random.default_rng(5)
    n, res = 50000, (16, 8)
    x = (rng.integers(0, 16, n) + rng.uniform(0.05, 0.95, n)) / 16.0
    y = (rng.integers(0, 8, n) + rng.uniform(0.05, 0.95, n)) / 8.0
    v = rng.normal(0, 1, n) * np.ldexp(1.0, rng.integers(-40, 40, n))
    w = rng.integers(-1000, 1000, n).astype(np.float64)
    r = oracle.databin([x, y], [v, w], res, (0, 0), (1, 1), exact=True)
    b = np.floor(x * 16).astype(int) + 16 * np.floor(y * 8).astype(int)
    for k in range(128):
        sel = b == k
        assert bits(r["sum_exact"][0, k]) == bits(math.fsum(v[sel]) if sel.any() else 0.0)
        assert r["count"][k] == sel.sum()
    assert np.array_equal(r["sum_exact"][1], r["sum"][1])           # integers: every order exact
    occ = r["count"] > 0
    assert np.array_equal(r["avg_exact"][0][occ], r["sum_exact"][0][occ] / r["count"][occ])
    assert np.all(np.isnan(r["avg_exact"][0][~occ]))
    # within Higham's bound of the row-order fold (the two differ only by rounding)
    err = np.abs(r["sum_exact"][0] - r["sum"][0])
    assert np.all(err <= 1e-12 * r["sumabs"][0])
