"""Fused multi-operator binning (bin_multi_*, SURVEY.md 8(f) row 1;
PAPER.md:511-514: 10 variables over 9 coordinate systems per in situ step).

Every instance of a fused set must give what the single-instance definition
gives: each is compared element by element with the oracle run on that
instance's own columns (counts / n_in / n_out / min / max bit-exact, sums
within reading R8), and with a separate bin_init/bin_execute of the same spec.
Host-side validation (no GPU compute) runs with -m "not gpu".
"""
import numpy as np
import pytest

import oracle
from tests.gpu_util import compare

ALL = ("sum", "min", "max", "avg")


# ---------------------------------------------------------------- host-side validation (no GPU)
def test_multi_init_validation(db):
    sp = db.make_spec((4, 4), (0, 0), (1, 1), nattr=1)
    ok = db.make_multi_op(sp, (0, 1), (2,))
    with pytest.raises(db.BinError) as e:
        db.bin_multi_init([], 3)
    assert e.value.code == 1
    with pytest.raises(db.BinError) as e:
        db.bin_multi_init([ok], 17)                         # > BIN_MULTI_MAX_COLS
    assert e.value.code == 1
    with pytest.raises(db.BinError) as e:
        db.bin_multi_init([ok, db.make_multi_op(sp, (0, 3), (2,))], 3)   # axis column out of range
    assert e.value.code == 1 and "instance 1" in str(e.value)
    with pytest.raises(db.BinError) as e:
        db.bin_multi_init([db.make_multi_op(sp, (0, 1), (-1,))], 3)      # attribute column out of range
    assert e.value.code == 1
    det = db.make_spec((4, 4), (0, 0), (1, 1), nattr=1, deterministic=True)
    with pytest.raises(db.BinError) as e:
        db.bin_multi_init([db.make_multi_op(det, (0, 1), (2,))], 3)
    assert e.value.code == 7                                # BIN_ENOTSUP
    bad = db.make_spec((4, 4), (0, 1), (1, 1), nattr=1)     # lo == hi on axis 1
    with pytest.raises(db.BinError) as e:
        db.bin_multi_init([db.make_multi_op(bad, (0, 1), (2,))], 3)
    assert e.value.code == 1
    with pytest.raises(db.BinError):
        db.bin_multi_init([ok] * 33, 3)                     # > BIN_MULTI_MAX_OPS


# ---------------------------------------------------------------- GPU parity
def run_multi(db, cols, insts, offset=0, placement=None, profile=False):
    """insts: list of dict(res, lo, hi, axes=(col idx..), attrs=(col idx..), ops, bounds_auto)."""
    import torch
    dev = torch.device("cuda:0")
    keep, hs = [], []
    for c in cols:
        t = torch.empty(len(c) + offset, dtype=torch.float64, device=dev)
        t[offset:] = torch.from_numpy(np.ascontiguousarray(c)).to(dev)
        t = t[offset:]
        keep.append(t)
        hs.append(db.wrap_tensor(t))
    torch.cuda.synchronize()
    specs, ops = [], []
    for d in insts:
        sp = db.make_spec(d["res"], d.get("lo"), d.get("hi"), nattr=len(d["attrs"]), ops=d.get("ops", ALL),
                          bounds_auto=d.get("bounds_auto", False))
        specs.append(sp)
        ops.append(db.make_multi_op(sp, d["axes"], d["attrs"]))
    m = db.bin_multi_init(ops, len(cols), placement if placement is not None else db.make_placement(device_id=0))
    try:
        if profile:
            db.bin_multi_profile_enable(m, True)
        t = db.bin_multi_execute(m, hs)
        outs = [db.result_to_numpy(m, t, sp, op=k) for k, sp in enumerate(specs)]
        prof = db.bin_multi_profile_read(m) if profile else None
    finally:
        db.bin_multi_finalize(m)
        for a in hs:
            db.bin_array_release(a)
    return outs, prof


def oracle_of(cols, d):
    return oracle.databin([cols[i] for i in d["axes"]], [cols[i] for i in d["attrs"]], d["res"], d.get("lo"),
                          d.get("hi"), bounds_auto=d.get("bounds_auto", False))


def paper_step_instances(res=256):
    """9 coordinate systems x 7 variables (x, y, z, mass, vx, vy, vz = columns 0..6), R19."""
    systems = [(0, 1), (0, 2), (1, 2), (4, 5), (4, 6), (5, 6), (0, 4), (1, 5), (2, 6)]
    return [dict(res=(res, res), lo=(-1.0, -1.0), hi=(1.0, 1.0), axes=s, attrs=tuple(range(7))) for s in systems]


def synth_cols(n, seed=6, dist=0):
    import synth
    return [synth.fill_host(dist, 1, seed, c, 0, n) for c in range(7)]


@pytest.mark.gpu
def test_multi_paper_step_vs_oracle(db):
    cols = synth_cols(200_003)
    insts = paper_step_instances(64)
    outs, prof = run_multi(db, cols, insts, profile=True)
    for d, out in zip(insts, outs):
        compare(out, oracle_of(cols, d))
    assert prof.kernel_launches == 3 and prof.executes == 1       # init + bin + finalize for all 9


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(12))
def test_multi_random_sets_vs_oracle(db, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.choice([0, 1, 31, 1000, 77_777, 300_001]))
    ncols = int(rng.integers(2, 17))
    cols = [rng.normal(0, 1.5, n) for _ in range(ncols)]
    if n > 10:  # NaN / inf coordinates (column 0: axis only, reading R7), duplicates, signed zeros
        cols[0][rng.integers(0, n, 5)] = np.nan
        cols[0][rng.integers(0, n, 3)] = np.inf
        cols[1][: n // 10] = cols[1][0]
        cols[ncols - 1][rng.integers(0, n, 7)] = -0.0
    insts = []
    for _ in range(int(rng.integers(1, 9))):
        nd = int(rng.integers(1, 4))
        axes = tuple(int(c) for c in rng.choice(ncols, nd, replace=False))
        res = tuple(int(r) for r in rng.integers(1, 48, nd))
        na = int(rng.integers(0, 6))
        attrs = tuple(int(c) for c in rng.integers(1, ncols, na))
        ops = [tuple(o for o in ALL if rng.random() < 0.6) or ("sum",) for _ in range(na)]
        auto = bool(rng.random() < 0.3) and n > 0
        d = dict(res=res, axes=axes, attrs=attrs, ops=ops, bounds_auto=auto)
        if not auto:
            d["lo"] = tuple(-2.0 + rng.random() for _ in range(nd))
            d["hi"] = tuple(1.0 + rng.random() for _ in range(nd))
        insts.append(d)
    if any(d["bounds_auto"] for d in insts):  # auto bounds over columns with +inf are degenerate: finite only
        for c in cols:
            c[~np.isfinite(c) & ~np.isnan(c)] = 0.5
    outs, _ = run_multi(db, cols, insts, offset=int(rng.integers(0, 2)))
    for d, out in zip(insts, outs):
        compare(out, oracle_of(cols, d), ops=d["ops"], nattr=len(d["attrs"]))


@pytest.mark.gpu
def test_multi_matches_separate_instances(db):
    from tests.gpu_util import run_gpu
    cols = synth_cols(500_000, seed=9, dist=1)
    insts = [dict(res=(128, 128), lo=(-8.0, -8.0), hi=(8.0, 8.0), axes=(0, 1), attrs=(3,)),
             dict(res=(32, 32, 32), lo=(-4.0,) * 3, hi=(4.0,) * 3, axes=(0, 1, 2), attrs=(3, 4), ops=[ALL, ("sum",)]),
             dict(res=(100,), bounds_auto=True, axes=(4,), attrs=(3, 5, 6)),
             dict(res=(64, 64), bounds_auto=True, axes=(4, 5), attrs=())]
    outs, _ = run_multi(db, cols, insts)
    for d, out in zip(insts, outs):
        single = run_gpu(db, [cols[i] for i in d["axes"]], [cols[i] for i in d["attrs"]], d["res"], d.get("lo"),
                         d.get("hi"), ops=d.get("ops", ALL), bounds_auto=d.get("bounds_auto", False))
        ref = oracle_of(cols, d)
        compare(out, ref, ops=d.get("ops", ALL), nattr=len(d["attrs"]))
        assert np.array_equal(out["count"], single["count"])
        assert (out["n_in"], out["n_out"]) == (single["n_in"], single["n_out"])
        assert np.array_equal(out["lo"].view(np.uint64), single["lo"].view(np.uint64))


@pytest.mark.gpu
def test_multi_exact_instances(db):
    """BIN_SUM_EXACT instances inside a fused set: sums bit-exact vs the oracle's exact sums."""
    rng = np.random.default_rng(12)
    n = 250_001
    cols = [rng.normal(0, 1, n), rng.normal(0, 1, n),
            rng.normal(0, 1, n) * np.ldexp(1.0, rng.integers(-30, 30, n)), rng.uniform(0.5, 1.5, n)]
    insts = [dict(res=(40, 30), lo=(-3.0, -3.0), hi=(3.0, 3.0), axes=(0, 1), attrs=(2, 3), exact=True),
             dict(res=(64,), lo=(-3.0,), hi=(3.0,), axes=(1,), attrs=(2,), exact=False),
             dict(res=(16, 16), bounds_auto=True, axes=(0, 3), attrs=(2,), exact=True)]
    import torch
    dev = torch.device("cuda:0")
    ts = [torch.from_numpy(c).to(dev) for c in cols]
    hs = [db.wrap_tensor(t) for t in ts]
    torch.cuda.synchronize()
    specs = [db.make_spec(d["res"], d.get("lo"), d.get("hi"), nattr=len(d["attrs"]),
                          bounds_auto=d.get("bounds_auto", False), exact=d["exact"]) for d in insts]
    m = db.bin_multi_init([db.make_multi_op(sp, d["axes"], d["attrs"]) for sp, d in zip(specs, insts)], len(cols),
                          db.make_placement(device_id=0))
    try:
        outs = []
        for _ in range(3):  # repeated executes: digit ranges cleared between them
            t = db.bin_multi_execute(m, hs)
            outs.append([db.result_to_numpy(m, t, sp, op=k) for k, sp in enumerate(specs)])
    finally:
        db.bin_multi_finalize(m)
        for a in hs:
            db.bin_array_release(a)
    for d, out in zip(insts, outs[-1]):
        ref = oracle.databin([cols[i] for i in d["axes"]], [cols[i] for i in d["attrs"]], d["res"], d.get("lo"),
                             d.get("hi"), bounds_auto=d.get("bounds_auto", False), exact=True)
        compare(out, ref)
        if d["exact"]:
            for a in range(len(d["attrs"])):
                assert np.array_equal(out["sum"][a].view(np.uint64), ref["sum_exact"][a].view(np.uint64))
    for k in range(len(insts)):
        assert np.array_equal(outs[0][k]["sum"][0].view(np.uint64), outs[2][k]["sum"][0].view(np.uint64)) \
            or not insts[k]["exact"]


@pytest.mark.gpu
def test_multi_degenerate_auto_bounds(db):
    cols = [np.full(10, np.nan), np.linspace(0, 1, 10), np.ones(10)]
    insts = [dict(res=(4,), bounds_auto=True, axes=(0,), attrs=(2,)),
             dict(res=(4,), lo=(0.0,), hi=(1.0,), axes=(1,), attrs=(2,))]
    with pytest.raises(db.BinError) as e:
        run_multi(db, cols, insts)
    assert e.value.code == 5                                # BIN_EDEGENERATE


@pytest.mark.gpu
def test_multi_max_instances_and_columns(db):
    rng = np.random.default_rng(7)
    cols = [rng.uniform(-1, 1, 65_537) for _ in range(16)]
    insts = [dict(res=(16, 8), lo=(-1.0, -1.0), hi=(1.0, 1.0), axes=(k % 16, (k + 1) % 16),
                  attrs=tuple((k + j) % 16 for j in range(16)), ops=ALL) for k in range(32)]
    outs, _ = run_multi(db, cols, insts)
    for d, out in zip(insts, outs):
        compare(out, oracle_of(cols, d))


@pytest.mark.gpu
def test_multi_repeated_executes_and_host_columns(db):
    """Back-to-back executes on both slots (results of ticket t valid until t+2) and staged host columns."""
    import torch
    cols = synth_cols(100_000, seed=11)
    insts = paper_step_instances(32)[:3]
    specs = [db.make_spec(d["res"], d["lo"], d["hi"], nattr=7) for d in insts]
    ops = [db.make_multi_op(sp, d["axes"], d["attrs"]) for sp, d in zip(specs, insts)]
    pinned = []
    for c in cols:
        t = torch.from_numpy(c).pin_memory()
        pinned.append(t)
    hs = [db.wrap_tensor(t) for t in pinned]
    m = db.bin_multi_init(ops, 7, db.make_placement(device_id=0))
    try:
        t1 = db.bin_multi_execute(m, hs)
        t2 = db.bin_multi_execute(m, hs)
        for t in (t1, t2):
            for k, (d, sp) in enumerate(zip(insts, specs)):
                compare(db.result_to_numpy(m, t, sp, op=k), oracle_of(cols, d))
        t3 = db.bin_multi_execute(m, hs)
        with pytest.raises(db.BinError):
            db.bin_multi_result(m, t1, 0)                   # recycled by t3
        db.bin_multi_wait(m, t3)
    finally:
        db.bin_multi_finalize(m)
        for a in hs:
            db.bin_array_release(a)


@pytest.mark.gpu
def test_multi_filter_on_off_across_executes(db):
    """The min/max filter lines (C6) are used only from 8 rows per bin
    on: executes alternating below / above that (filter lines skipped, then
    cleared and used, then skipped) on one handle all match the oracle."""
    import torch
    insts = paper_step_instances(64)[:4]  # 4096 bins: filter from 32,768 rows on
    specs = [db.make_spec(d["res"], d["lo"], d["hi"], nattr=7) for d in insts]
    m = db.bin_multi_init([db.make_multi_op(sp, d["axes"], d["attrs"]) for sp, d in zip(specs, insts)], 7,
                          db.make_placement(device_id=0))
    try:
        for i, n in enumerate((20_000, 150_001, 3_000, 400_000, 150_001)):
            cols = synth_cols(n, seed=40 + i, dist=i % 2)
            ts = [torch.from_numpy(c).to("cuda:0") for c in cols]
            hs = [db.wrap_tensor(t) for t in ts]
            torch.cuda.synchronize()
            try:
                t = db.bin_multi_execute(m, hs)
                for k, (d, sp) in enumerate(zip(insts, specs)):
                    compare(db.result_to_numpy(m, t, sp, op=k), oracle_of(cols, d))
            finally:
                torch.cuda.synchronize()
                for a in hs:
                    db.bin_array_release(a)
    finally:
        db.bin_multi_finalize(m)


@pytest.mark.gpu
def test_multi_filter_hi32_ties(db):
    """Values sharing their top 32 encoded bits (1 + k 2^-40, -(1 + k 2^-40))
    in random order, 16 bins: the filter word ties on every row, so the exact
    extremum must still reach the slot; min / max bit-exact vs the oracle."""
    rng = np.random.default_rng(77)
    n = 200_000
    x = rng.uniform(-1, 1, n)
    y = rng.uniform(-1, 1, n)
    k = rng.permutation(n).astype(np.float64)
    a = 1.0 + k * 2.0 ** -40
    b = -(1.0 + rng.permutation(n) * 2.0 ** -40)
    cols = [x, y, a, b]
    insts = [dict(res=(4, 4), lo=(-1.0, -1.0), hi=(1.0, 1.0), axes=(0, 1), attrs=(2, 3)),
             dict(res=(2, 2), lo=(-1.0, -1.0), hi=(1.0, 1.0), axes=(1, 0), attrs=(3, 2, 2))]
    outs, _ = run_multi(db, cols, insts)
    for d, out in zip(insts, outs):
        ref = oracle_of(cols, d)
        compare(out, ref)
        for j in range(len(d["attrs"])):
            assert np.array_equal(out["min"][j].view(np.uint64), ref["min"][j].view(np.uint64))
            assert np.array_equal(out["max"][j].view(np.uint64), ref["max"][j].view(np.uint64))
