"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by
element, on seeded inputs (-m gpu).  Sizes span many CTAs/tiles with ragged
tails; the full BASELINE.json sizes (C2, C3) run in the launch configuration
bench.py times."""
import math

import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALL_OPS, bits, compare, run_gpu, workload_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_available):
    if not cuda_available:
        pytest.fail("GPU tests need a CUDA device (run on the B200 box)")


def both(db, axes, attrs, res, lo=None, hi=None, ops=ALL_OPS, bounds_auto=False, exact=False, det_too=True, **kw):
    ref = oracle.databin(axes, attrs, res, lo, hi, bounds_auto=bounds_auto)
    out = run_gpu(db, axes, attrs, res, lo, hi, ops=ops, bounds_auto=bounds_auto, **kw)
    compare(out, ref, ops, exact=exact)
    if bounds_auto:
        assert np.array_equal(bits(out["lo"]), bits(ref["lo"])) and np.array_equal(bits(out["hi"]), bits(ref["hi"]))
    if det_too:
        outd = run_gpu(db, axes, attrs, res, lo, hi, ops=ops, bounds_auto=bounds_auto, deterministic=True, **kw)
        compare(outd, ref, ops, exact=True)
    return out, ref


# ---------------------------------------------------------------- worked examples
def test_we1_we3_we4_we6_we7_on_gpu(db):
    both(db, [[0.1], [0.1]], [[2.0]], [2, 2], [-1, -1], [1, 1], exact=True)                 # WE1
    xs = [0.0, 0.25, 0.5, 0.75, 1.0, -2.0 ** -52, 1.0 + 2.0 ** -52]
    out, _ = both(db, [xs, [0.5] * 7], [[1.0] * 7], [4, 4], [0, 0], [1, 1], exact=True)     # WE2
    assert out["count"][11] == 2 and (out["n_in"], out["n_out"]) == (5, 2)
    out, _ = both(db, [[0.0], [0.0]], [[1000.0]], [32, 32], [-1, -1], [1, 1], exact=True)   # WE3
    assert np.flatnonzero(out["count"]).tolist() == [528]
    m = np.arange(1, 1001, dtype=np.float64)                                                 # WE4: contention
    out, _ = both(db, [np.full(1000, 0.3), np.full(1000, 0.3)], [m], [8, 8], [0, 0], [1, 1], exact=True)
    assert out["sum"][0][18] == 500500.0 and out["avg"][0][18] == 500.5
    both(db, [[0.5] * 3], [[0.1] * 3], [1], [0], [1], exact=True)                            # WE6
    out, _ = both(db, [[0.5] * 2], [[-0.0, 0.0]], [1], [0], [1], exact=True)                 # WE7
    assert bits(out["min"][0][0]) == bits(-0.0) and bits(out["max"][0][0]) == bits(0.0)


def test_we5_order_sensitive_sum(db):
    e = 2.0 ** -53
    ref = oracle.databin([[0.5] * 3], [[1.0, e, e]], [1], [0], [1])
    out = run_gpu(db, [[0.5] * 3], [[1.0, e, e]], [1], [0], [1])
    assert out["sum"][0][0] in (1.0, 1.0 + 2.0 ** -52)                # atomic: any order, within tolerance
    compare(out, ref)
    outd = run_gpu(db, [[0.5] * 3], [[1.0, e, e]], [1], [0], [1], deterministic=True)
    assert outd["sum"][0][0] == 1.0                                    # deterministic: row order
    compare(outd, ref, exact=True)


def test_upper_clamp_and_nonfinite_axes(db):
    rng = np.random.default_rng(2)
    xs = []
    for _ in range(3000):
        lo, hi = np.sort(rng.uniform(-10, 10, 2))
        res = int(rng.integers(2, 5000))
        x = np.nextafter(hi, -np.inf)
        if math.floor((x - lo) * (res / (hi - lo))) >= res:
            xs.append((lo, hi, res, x))
        if len(xs) == 5:
            break
    for lo, hi, res, x in xs:
        out, _ = both(db, [[x, hi, lo, np.nan, np.inf, -np.inf]], [[1.0] * 6], [res], [lo], [hi], exact=True)
        assert out["count"][res - 1] == 2 and out["n_out"] == 3


# ---------------------------------------------------------------- configs[0]
@pytest.mark.parametrize("bounds_auto", [False, True])
def test_c1_uniform_1k_32x32(db, bounds_auto):
    w = synth.CONFIGS["c1"]
    axes, attrs = workload_inputs(w)
    lo, hi = (None, None) if bounds_auto else (w.lo, w.hi)
    out, ref = both(db, axes, attrs, w.res, lo, hi, bounds_auto=bounds_auto)
    assert out["n_in"] + out["n_out"] == 1000
    if bounds_auto:
        assert out["n_out"] == 0


# ---------------------------------------------------------------- randomized property cases
def _random_case(rng):
    ndim = int(rng.integers(1, 4))
    res = [int(rng.integers(1, 65)) for _ in range(ndim)]
    n = int(rng.integers(0, 10001))
    kind = rng.integers(0, 3)
    if kind == 0:
        axes = [rng.uniform(-1.3, 1.3, n) for _ in range(ndim)]
    elif kind == 1:
        axes = [rng.standard_normal(n) * 0.3 for _ in range(ndim)]
    else:  # duplicates and lattice points (exact edges)
        axes = [rng.integers(-4, 5, n) / 4.0 for _ in range(ndim)]
    if n and rng.random() < 0.2:
        axes[0][rng.integers(0, n, max(1, n // 50))] = np.nan
    nattr = int(rng.choice([0, 1, 2, 3, 4, 5, 16], p=[.1, .35, .15, .1, .15, .1, .05]))
    attrs = []
    for _ in range(nattr):
        if rng.random() < 0.3:
            attrs.append(rng.integers(-8, 9, n).astype(np.float64))
        else:
            attrs.append(rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3))
    ops = []
    for _ in range(nattr):
        o = tuple(op for op in ALL_OPS if rng.random() < 0.6)
        ops.append(o)
    auto = bool(rng.random() < 0.35) and n > 0
    lo = [-1.0] * ndim
    hi = [float(rng.choice([1.0, 0.7, 1.25]))] * ndim
    return axes, attrs, res, lo, hi, ops, auto


def test_200_random_cases(db):
    # SPEC.md:525 acceptance 3 on the GPU path; half the cases deterministic mode
    rng = np.random.default_rng(2026)
    for case in range(200):
        axes, attrs, res, lo, hi, ops, auto = _random_case(rng)
        det = case % 2 == 1
        off = int(rng.integers(0, 2))
        ref = oracle.databin(axes, attrs, res, None if auto else lo, None if auto else hi, bounds_auto=auto)
        out = run_gpu(db, axes, attrs, res, None if auto else lo, None if auto else hi, ops=list(ops) if attrs else (),
                      bounds_auto=auto, deterministic=det, offset=off)
        try:
            compare(out, ref, list(ops) if attrs else (), exact=det, nattr=len(attrs))
        except AssertionError as e:
            raise AssertionError(f"case {case}: ndim={len(res)} res={res} n={len(axes[0])} nattr={len(attrs)} "
                                 f"auto={auto} det={det} off={off}: {e}") from e


# ---------------------------------------------------------------- sizes, alignment, variants
@pytest.mark.parametrize("n", [1, 2, 3, 31, 33, 1023, 1025, 4097, 300001])
@pytest.mark.parametrize("offset", [0, 1])
def test_ragged_sizes_and_alignment(db, n, offset):
    rng = np.random.default_rng(n)
    axes = [rng.uniform(-1.1, 1.1, n), rng.uniform(-1.1, 1.1, n)]
    attrs = [rng.uniform(0.5, 1.5, n)]
    both(db, axes, attrs, [16, 16], [-1, -1], [1, 1], offset=offset, det_too=(n < 5000))   # full-grid window
    for route in ("window", "partition"):       # 512^2: hot window + L2, and the partition route
        both(db, axes, attrs, [512, 512], [-1, -1], [1, 1], offset=offset, det_too=False, route=route)


def test_mixed_alignment_falls_back_to_scalar(db):
    import torch
    rng = np.random.default_rng(9)
    n = 100001
    x, y, m = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), rng.uniform(0.5, 1.5, n)
    ref = oracle.databin([x, y], [m], [64, 64], [-1, -1], [1, 1])
    dev = torch.device("cuda:0")
    tx = torch.zeros(n + 1, dtype=torch.float64, device=dev)
    tx[1:] = torch.from_numpy(x).to(dev)
    ty = torch.from_numpy(y).to(dev)
    tm = torch.from_numpy(m).to(dev)
    hs = [db.wrap_tensor(tx[1:]), db.wrap_tensor(ty), db.wrap_tensor(tm)]
    spec = db.make_spec([64, 64], [-1, -1], [1, 1], nattr=1)
    h = db.bin_init(spec, db.make_placement(device_id=0))
    t = db.bin_execute(h, hs[:2], hs[2:])
    compare(db.result_to_numpy(h, t, spec), ref)
    db.bin_finalize(h)
    for a in hs:
        db.bin_array_release(a)


def test_3d_global_path_and_window(db):
    rng = np.random.default_rng(33)
    n = 200000
    axes = [rng.uniform(-1, 1, n) for _ in range(3)]
    attrs = [rng.uniform(0.5, 1.5, n)]
    both(db, axes, attrs, [64, 64, 64], [-1] * 3, [1] * 3, det_too=True)
    both(db, axes, attrs, [64, 64, 64], [-1] * 3, [1] * 3, det_too=False, route="window")
    axes = [rng.standard_normal(n) * 0.1 for _ in range(3)]       # clustered: window catches most rows
    out, _ = both(db, axes, attrs, [128, 128, 128], [-1] * 3, [1] * 3, det_too=False, route="window")
    assert out["profile"].variant & 15 == 1
    both(db, axes, attrs, [128, 128, 128], [-1] * 3, [1] * 3, det_too=False)   # auto (either route)


def test_zero_rows_and_degenerate_bounds(db):
    out, _ = both(db, [np.zeros(0), np.zeros(0)], [np.zeros(0)], [8, 8], [0, 0], [1, 1], exact=True)
    assert out["count"].sum() == 0 and np.all(np.isinf(out["min"][0]))
    with pytest.raises(db.BinError) as e:
        run_gpu(db, [np.zeros(0)], [np.zeros(0)], [8], bounds_auto=True)
    assert e.value.code == db.capi.BIN_EDEGENERATE
    with pytest.raises(db.BinError) as e:
        run_gpu(db, [np.full(5, np.nan)], [np.ones(5)], [8], bounds_auto=True)
    assert e.value.code == db.capi.BIN_EDEGENERATE
    out, ref = both(db, [[5.0, 5.0, 5.0]], [[1.0, 2.0, 3.0]], [4], bounds_auto=True, exact=True)
    assert (out["lo"][0], out["hi"][0]) == (4.5, 5.5)


def test_dyadic_masses_bit_exact_under_atomics(db):
    # partial sums of j * 2^-20 (j < 2^20, < 2^33 terms) are exact in any order
    rng = np.random.default_rng(12)
    n = 2_000_000
    axes = [rng.standard_normal(n) * 3, rng.standard_normal(n) * 3]
    attrs = [rng.integers(1, 2 ** 20, n) * 2.0 ** -20]
    both(db, axes, attrs, [512, 512], [-16, -16], [16, 16], exact=True, det_too=False)


# ---------------------------------------------------------------- full sizes (BASELINE.json configs[1], [2])
@pytest.mark.slow
def test_c2_full_10M_uniform_256x256_4attr(db):
    w = synth.CONFIGS["c2"]
    axes, attrs = workload_inputs(w)
    both(db, axes, attrs, w.res, w.lo, w.hi, det_too=True)


@pytest.mark.slow
def test_c3_full_100M_plummer_512x512(db):
    w = synth.CONFIGS["c3"]
    axes, attrs = workload_inputs(w)
    out, ref = both(db, axes, attrs, w.res, w.lo, w.hi, det_too=True)
    assert out["profile"].variant == 1 | 16                 # window + k_bin_fast: the bench's launch configuration
    tot = float(np.sum(attrs[0]))
    inside_mass = float(np.sum(out["sum"][0]))
    assert 0 < out["n_out"] < w.n // 100                    # ~0.1% outside the +-16 a box
    assert inside_mass < tot


# ---------------------------------------------------------------- unusable bounds (reading R4)
@pytest.mark.parametrize("route", ["window", "partition"])
@pytest.mark.parametrize("deterministic", [False, True])
def test_unusable_auto_bounds_are_degenerate(db, route, deterministic):
    # the oracle's pins (test_oracle.py) and the library agree: no mesh, BIN_EDEGENERATE
    big = np.finfo(np.float64).max
    cases = [[[0.0, 1.0, np.inf]], [[-np.inf, 0.0, 1.0]], [[-big, big]], [[0.0, 5e-324]], [[1e300, 1e300]],
             [[0.0, 1.0], [0.0, np.inf]]]
    for axes in cases:
        with pytest.raises(oracle.Degenerate):
            oracle.databin(axes, [np.ones(len(axes[0]))], [4] * len(axes), bounds_auto=True)
        with pytest.raises(db.BinError) as e:
            run_gpu(db, axes, [np.ones(len(axes[0]))], [4] * len(axes), bounds_auto=True, route=route,
                    deterministic=deterministic)
        assert e.value.code == db.capi.BIN_EDEGENERATE, axes
    # NaN rows alone do not spoil the bounds (R4): same result as the oracle
    both(db, [[0.0, np.nan, 1.0, 0.25]], [[1.0, 2.0, 3.0, 4.0]], [2], bounds_auto=True, exact=True, route=route)


def test_unusable_manual_bounds_are_invalid(db):
    big = np.finfo(np.float64).max
    for lo, hi in ((0.0, np.inf), (-np.inf, 0.0), (np.nan, 1.0), (1.0, 1.0), (2.0, 1.0), (-big, big), (0.0, 5e-324)):
        with pytest.raises(oracle.InvalidArgument):
            oracle.databin([[0.5]], [[1.0]], [4], [lo], [hi])
        with pytest.raises(db.BinError) as e:
            run_gpu(db, [[0.5]], [[1.0]], [4], [lo], [hi])
        assert e.value.code == db.capi.BIN_EINVAL, (lo, hi)
    both(db, [[-big / 2, big / 4, big / 2]], [[1.0, 2.0, 3.0]], [2], [-big / 2], [big / 2], exact=True)
