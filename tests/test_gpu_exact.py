"""BIN_SUM_EXACT (reading R20): every bin's sum
is its exact real sum rounded once -- bit-exact against the oracle's
``sum_exact`` (itself pinned by fractions.Fraction / math.fsum in
test_oracle_exact.py), on both accumulate routes, both kernels, at full
configuration sizes, and identical across routes and repeated executes.
"""
import zlib

import numpy as np
import pytest

import oracle
from tests.gpu_util import bits, run_gpu, workload_inputs

pytestmark = pytest.mark.gpu
ALL = ("sum", "min", "max", "avg")


def check_exact(out, ref, nattr, ops=ALL):
    assert (out["n_in"], out["n_out"]) == (ref["n_in"], ref["n_out"])
    assert np.array_equal(out["count"], ref["count"])
    for a in range(nattr):
        if "sum" in ops:
            bad = np.flatnonzero(bits(out["sum"][a]) != bits(ref["sum_exact"][a]))
            assert bad.size == 0, f"sum[{a}] at {bad[:8]}: {out['sum'][a][bad[:3]]} vs {ref['sum_exact'][a][bad[:3]]}"
        if "avg" in ops:
            g, r = out["avg"][a], ref["avg_exact"][a]
            assert np.array_equal(np.isnan(g), np.isnan(r))
            ok = ~np.isnan(r)
            assert np.array_equal(bits(g[ok]), bits(r[ok]))
        for k in ("min", "max"):
            if k in ops:
                assert np.array_equal(bits(out[k][a]), bits(ref[k][a]))


def hard_values(rng, n, kind):
    if kind == "mixed":       # 40 binades, both signs: cancellation inside every bin
        return rng.normal(0, 1, n) * np.ldexp(1.0, rng.integers(-20, 20, n))
    if kind == "wide":        # 1e-300 .. 1e300: far outside any window's fixed range
        return rng.choice([-1.0, 1.0], n) * np.ldexp(rng.random(n) + 0.5, rng.integers(-1000, 1000, n))
    if kind == "subnormal":
        return rng.choice([-1.0, 1.0], n) * np.ldexp(rng.random(n) + 0.5, rng.integers(-1074, -1015, n))
    if kind == "mass":        # the generators' masses plus a heavy body
        v = rng.uniform(0.5, 1.5, n)
        v[0] = 1000.0
        return v
    raise ValueError(kind)


@pytest.mark.parametrize("route", ["window", "partition"])
@pytest.mark.parametrize("kind", ["mixed", "wide", "subnormal", "mass"])
@pytest.mark.parametrize("nattr", [1, 3])
def test_exact_random(db, route, kind, nattr):
    rng = np.random.default_rng(zlib.crc32(f"{route}{kind}{nattr}".encode()))
    n = 400_001
    x = rng.normal(0, 0.6, n)
    y = rng.normal(0, 0.6, n)
    attrs = [hard_values(rng, n, kind) for _ in range(nattr)]
    ref = oracle.databin([x, y], attrs, (64, 48), (-2, -2), (2, 2), exact=True)
    out = run_gpu(db, [x, y], attrs, (64, 48), (-2, -2), (2, 2), route=route, exact=True)
    check_exact(out, ref, nattr)


def test_exact_overflow_and_zero(db):
    big = np.finfo(np.float64).max
    x = np.array([0.1, 0.1, 0.1, 0.6, 0.6, 0.9, 0.9, 0.9])
    v = np.array([big, big, -big, 1.0, -1.0, big, big, 1.0])
    ref = oracle.databin([x], [v], (4,), (0,), (1,), exact=True)
    out = run_gpu(db, [x], [v], (4,), (0,), (1,), exact=True)
    check_exact(out, ref, 1)
    assert out["sum"][0][0] == big and out["sum"][0][3] == np.inf
    assert bits(out["sum"][0][2]) == bits(0.0)                       # exact zero -> +0.0


def test_exact_fast_kernel_and_general_kernel_agree(db):
    """One attribute runs k_bin_fast, several run k_bin: same exact sums."""
    rng = np.random.default_rng(3)
    n = 1_000_000
    x, y = rng.normal(0, 1, n), rng.normal(0, 1, n)
    v = hard_values(rng, n, "mixed")
    one = run_gpu(db, [x, y], [v], (100, 100), (-3, -3), (3, 3), exact=True, route="window")
    two = run_gpu(db, [x, y], [v, v], (100, 100), (-3, -3), (3, 3), exact=True, route="window")
    part = run_gpu(db, [x, y], [v], (100, 100), (-3, -3), (3, 3), exact=True, route="partition")
    assert one["profile"].variant & 16 and not two["profile"].variant & 16
    for o in (two, part):
        assert np.array_equal(bits(one["sum"][0]), bits(o["sum"][0]))
    ref = oracle.databin([x, y], [v], (100, 100), (-3, -3), (3, 3), exact=True)
    check_exact(one, ref, 1)


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_exact_full_configs(db, name):
    import synth
    w = synth.CONFIGS[name]
    axes, attrs = workload_inputs(w)
    ref = oracle.databin(axes, attrs, w.res, w.lo, w.hi, exact=True)
    out = run_gpu(db, axes, attrs, w.res, w.lo, w.hi, exact=True)
    check_exact(out, ref, len(attrs))


def test_exact_repeatable_across_executes(db):
    """Back-to-back executes on one handle (both slots, digit ranges cleared by init)."""
    import torch
    rng = np.random.default_rng(9)
    n = 300_000
    cols = [rng.uniform(-1, 1, n), rng.uniform(-1, 1, n), hard_values(rng, n, "wide")]
    cols2 = [cols[0], cols[1], hard_values(rng, n, "mixed")]
    dev = torch.device("cuda:0")
    spec = db.make_spec((32, 32), (-1, -1), (1, 1), nattr=1, exact=True)
    h = db.bin_init(spec, db.make_placement(device_id=0))
    ts = [torch.from_numpy(c).to(dev) for c in cols]
    ts2 = [torch.from_numpy(c).to(dev) for c in cols2]
    hs = [db.wrap_tensor(t) for t in ts]
    hs2 = [db.wrap_tensor(t) for t in ts2]
    torch.cuda.synchronize()
    try:
        outs = []
        for k in range(5):
            src = hs if k % 2 == 0 else hs2
            t = db.bin_execute(h, src[:2], src[2:])
            outs.append(db.result_to_numpy(h, t, spec))
    finally:
        db.bin_finalize(h)
        for a in hs + hs2:
            db.bin_array_release(a)
    r1 = oracle.databin(cols[:2], cols[2:], (32, 32), (-1, -1), (1, 1), exact=True)
    r2 = oracle.databin(cols2[:2], cols2[2:], (32, 32), (-1, -1), (1, 1), exact=True)
    for k, o in enumerate(outs):
        check_exact(o, r1 if k % 2 == 0 else r2, 1)


def test_exact_spec_validation(db):
    with pytest.raises(db.BinError) as e:
        db.bin_init(db.make_spec((4,), (0,), (1,), nattr=1, exact=True, deterministic=True))
    assert e.value.code == 1
