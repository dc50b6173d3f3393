"""GPU parity of the partition route (bin_part.cu; DESIGN.md "Partition
route"): rows grouped by bin tile, then accumulated tile by tile in shared
memory.  Forced with route="partition" and compared element by element with
the oracle at sizes spanning many tiles, CTAs and batches with ragged tails;
plus the auto route's choice on clustered vs spread-out data."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import ALL_OPS, compare, run_gpu, workload_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_available):
    if not cuda_available:
        pytest.fail("GPU tests need a CUDA device (run on the B200 box)")


def part(db, axes, attrs, res, lo=None, hi=None, ops=ALL_OPS, exact=False, bounds_auto=False, **kw):
    ref = oracle.databin(axes, attrs, res, lo, hi, bounds_auto=bounds_auto)
    out = run_gpu(db, axes, attrs, res, lo, hi, ops=ops, bounds_auto=bounds_auto, route="partition", **kw)
    assert out["profile"].variant & 15 == 4, out["profile"].variant
    compare(out, ref, ops, exact=exact)
    return out, ref


@pytest.mark.parametrize("offset", [0, 1])
@pytest.mark.parametrize("n", [3, 4, 1001, 2_000_003])
def test_2d_one_attr_ragged(db, n, offset):
    rng = np.random.default_rng(n + offset)
    axes = [rng.uniform(-1.05, 1.05, n), rng.uniform(-1.05, 1.05, n)]        # ~9% outside
    attrs = [rng.uniform(0.5, 1.5, n)]
    part(db, axes, attrs, (512, 512), (-1, -1), (1, 1), offset=offset)


def test_3d_many_tiles(db):
    w = synth.CONFIGS["c4"]
    axes, attrs = workload_inputs(w, n=6_000_001)
    out, _ = part(db, axes, attrs, w.res, w.lo, w.hi)
    assert out["n_out"] == 0


def test_c2_four_attrs_full_size(db):
    w = synth.CONFIGS["c2"]
    axes, attrs = workload_inputs(w)
    part(db, axes, attrs, w.res, w.lo, w.hi)


def test_c5_full_size(db):
    w = synth.CONFIGS["c5"]
    axes, attrs = workload_inputs(w)
    part(db, axes, attrs, w.res, w.lo, w.hi)


@pytest.mark.parametrize("ops", [("sum",), ("min", "max"), ("avg",), ("max",)])
def test_op_subsets(db, ops):
    rng = np.random.default_rng(5)
    n = 300_001
    axes = [rng.normal(0, 0.5, n), rng.normal(0, 0.5, n)]
    attrs = [rng.normal(0, 1, n)]
    part(db, axes, attrs, (300, 200), (-1, -1), (1, 1), ops=ops)


def test_count_only_and_1d(db):
    rng = np.random.default_rng(6)
    n = 500_000
    part(db, [rng.uniform(0, 1, n)], [], (100_000,), (0,), (1,))
    part(db, [rng.uniform(0, 1, n), rng.uniform(0, 1, n)], [], (1000, 1000), (0, 0), (1, 1))


def test_attrs_mixed_ops_and_wide_exponents(db):
    """Per-attribute op sets; values spanning 2^-40..2^40 (fixed-point range and
    the f64 L2 fallback), signed zeros, exactly representable sums (bit-exact)."""
    rng = np.random.default_rng(7)
    n = 400_003
    axes = [rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)]
    wide = rng.choice([-1.0, 1.0], n) * np.exp2(rng.integers(-40, 40, n).astype(np.float64))
    zeros = rng.choice([-0.0, 0.0], n)
    dyadic = rng.integers(-2 ** 20, 2 ** 20, n) * 2.0 ** -20
    ops = [("sum", "avg"), ("min", "max"), ("sum", "min", "max", "avg")]
    ref = oracle.databin(axes, [wide, zeros, dyadic], (400, 300), (-1, -1), (1, 1))
    out = run_gpu(db, axes, [wide, zeros, dyadic], (400, 300), (-1, -1), (1, 1), ops=ops, route="partition")
    assert out["profile"].variant & 15 == 4
    compare(out, ref, ops)
    assert np.array_equal(out["sum"][2], ref["sum"][2])          # dyadic: exact in any order


def test_hot_bin_contention_exact(db):
    """WE4-style: every row in one bin (one tile, max shared-memory contention)."""
    n = 1_000_000
    m = (np.arange(n) % 1000 + 1).astype(np.float64)
    part(db, [np.full(n, 0.3), np.full(n, 0.3)], [m], (512, 512), (0, 0), (1, 1), exact=True)


def test_auto_bounds_and_nonfinite_axes(db):
    rng = np.random.default_rng(8)
    n = 200_000
    x, y = rng.uniform(-3, 7, n), rng.uniform(2, 4, n)
    x[::97] = np.nan          # NaN rows: ignored by the bounds (R4), outside the mesh
    y[1::89] = np.nan
    part(db, [x, y], [rng.uniform(0, 1, n)], (256, 256), bounds_auto=True)


def test_deterministic_ignores_route(db):
    rng = np.random.default_rng(9)
    n = 100_000
    axes = [rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)]
    attrs = [rng.uniform(0, 1, n)]
    ref = oracle.databin(axes, attrs, (64, 64), (-1, -1), (1, 1))
    out = run_gpu(db, axes, attrs, (64, 64), (-1, -1), (1, 1), deterministic=True, route="partition")
    assert out["profile"].variant & 15 == 3
    compare(out, ref, exact=True)


def test_auto_route_choice(db):
    """Auto: uniform data on a mesh much larger than a window -> partition;
    the Plummer core (C3 mesh) -> window (k_bin_fast); results agree either way."""
    rng = np.random.default_rng(10)
    n = 1_000_000
    axes = [rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)]
    attrs = [rng.uniform(0.5, 1.5, n)]
    ref = oracle.databin(axes, attrs, (512, 512), (-1, -1), (1, 1))
    out = run_gpu(db, axes, attrs, (512, 512), (-1, -1), (1, 1))
    assert out["profile"].variant & 15 == 4
    compare(out, ref)
    w = synth.CONFIGS["c3"]
    axes, attrs = workload_inputs(w, n=1_000_000)
    ref = oracle.databin(axes, attrs, w.res, w.lo, w.hi)
    out = run_gpu(db, axes, attrs, w.res, w.lo, w.hi)
    assert out["profile"].variant & 15 in (1, 2) and out["profile"].variant & 16
    compare(out, ref)


def test_window_route_forced_on_uniform(db):
    rng = np.random.default_rng(11)
    n = 500_000
    axes = [rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)]
    attrs = [rng.uniform(0.5, 1.5, n)]
    ref = oracle.databin(axes, attrs, (512, 512), (-1, -1), (1, 1))
    out = run_gpu(db, axes, attrs, (512, 512), (-1, -1), (1, 1), route="window")
    assert out["profile"].variant & 15 == 1
    compare(out, ref)


# ---------------------------------------------------------------- full size (BASELINE.json configs[3])
@pytest.mark.slow
def test_c4_full_1B_256cube(db):
    """C4 at its full 1B rows on one B200 in the bench's launch configuration
    (auto route -> partition route, two-level grouping into thousands of
    tiles, 64-bit row offsets), every one of the 16.7M bins compared with the
    oracle.  The oracle streams the seeded rows chunk by chunk in partition
    mode P (``oracle.databin_blocks`` is bit-identical to
    ``oracle.databin(..., P)``), P worker threads on the host cores:
    counts/min/max bit-exact, sums within reading R8."""
    import os

    import torch
    w = synth.CONFIGS["c4"]
    dev = torch.device("cuda:0")
    names = list(w.axes) + list(w.attrs)
    cols = [torch.empty(w.n, dtype=torch.float64, device=dev) for _ in names]
    st = torch.cuda.current_stream(dev).cuda_stream
    for t, c in zip(cols, names):
        synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, w.n, t.data_ptr(), st)
    torch.cuda.synchronize(dev)
    hs = [db.wrap_tensor(t) for t in cols]
    spec = db.make_spec(w.res, w.lo, w.hi, nattr=len(w.attrs))
    h = db.bin_init(spec, db.make_placement(device_id=0))
    try:
        db.bin_profile_enable(h, True)
        t = db.bin_execute(h, hs[:3], hs[3:])
        out = db.result_to_numpy(h, t, spec)
        variant = db.bin_profile_read(h).variant
    finally:
        db.bin_finalize(h)
        for a in hs:
            db.bin_array_release(a)
        del cols
        torch.cuda.empty_cache()
    assert variant & 15 == 4, variant                      # the partition route, as bench.py --workload c4 runs it

    def rows(s, c):
        return ([synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c, 1) for x in w.axes],
                [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c, 1) for x in w.attrs])

    P = max(1, min(os.cpu_count() or 1, 24))
    ref = oracle.databin_blocks(rows, w.n, w.res, w.lo, w.hi, len(w.attrs), P=P)
    assert ref["n_in"] == w.n and ref["n_out"] == 0
    compare(out, ref)
