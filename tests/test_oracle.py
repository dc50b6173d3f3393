"""Pins for the CPU oracle (run with -m "not gpu").

Each test pins the oracle to something other than itself: worked examples
with hand-derived values (WE1-WE8), library
routines on inputs where they must agree (numpy histogramdd / bincount /
ufunc.at), integer closed forms, math.fsum error bounds (Higham gamma_{n-1}),
and invariants of the method.
"""
import math
import struct

import numpy as np
import pytest

import oracle

INF = math.inf


def f2b(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def empty_bin_ok(r, b, a=0):
    """Reading R5: identities of every reduction for an empty bin."""
    assert r["count"][b] == 0
    assert f2b(r["sum"][a, b]) == f2b(0.0)
    assert r["min"][a, b] == INF and r["max"][a, b] == -INF
    assert math.isnan(r["avg"][a, b])


# ---------------------------------------------------------------- worked examples
def test_we1_single_particle():
    # m = 2 at (0.1, 0.1), 2x2 over [-1,1]^2 -> bin (1,1) = idx 3
    r = oracle.databin([[0.1], [0.1]], [[2.0]], [2, 2], [-1, -1], [1, 1])
    assert r["count"].tolist() == [0, 0, 0, 1]
    assert r["sum"][0, 3] == 2.0 and r["min"][0, 3] == 2.0
    assert r["max"][0, 3] == 2.0 and r["avg"][0, 3] == 2.0
    for b in range(3):
        empty_bin_ok(r, b)
    assert (r["n_in"], r["n_out"]) == (1, 0)


def test_we2_edges_dyadic():
    # 4x4 over [0,1]^2, y = 0.5 -> iy = 2; x on edges; hi belongs to the last bin;
    # one ulp outside either bound is out (readings R1/R2).
    xs = [0.0, 0.25, 0.5, 0.75, 1.0, -2.0 ** -52, 1.0 + 2.0 ** -52]
    r = oracle.databin([xs, [0.5] * 7], [[1.0] * 7], [4, 4], [0, 0], [1, 1])
    assert (r["n_in"], r["n_out"]) == (5, 2)
    expect = np.zeros(16, np.uint64)
    expect[[8, 9, 10]] = 1
    expect[11] = 2
    assert r["count"].tolist() == expect.tolist()


def test_we3_massive_body_interior_edge():
    # 32x32 over [-1,1]^2, scale = 16 exactly: (0,0) -> (16,16) -> 16 + 32*16 = 528
    r = oracle.databin([[0.0], [0.0]], [[1000.0]], [32, 32], [-1, -1], [1, 1])
    assert np.flatnonzero(r["count"]).tolist() == [528]


def test_we4_integer_masses_exact_and_contention():
    m = np.arange(1, 1001, dtype=np.float64)
    r = oracle.databin([np.full(1000, 0.3), np.full(1000, 0.3)], [m], [8, 8], [0, 0], [1, 1])
    b = 2 + 8 * 2
    assert r["count"][b] == 1000
    assert r["sum"][0, b] == 500500.0 and r["avg"][0, b] == 500.5
    assert r["min"][0, b] == 1.0 and r["max"][0, b] == 1000.0


def test_we5_sum_is_in_row_order():
    e = 2.0 ** -53
    r = oracle.databin([[0.5] * 3], [[1.0, e, e]], [1], [0], [1])
    assert r["sum"][0, 0] == 1.0                     # (1 + e) + e = 1 (ties to even)
    r = oracle.databin([[0.5] * 3], [[e, e, 1.0]], [1], [0], [1])
    assert r["sum"][0, 0] == 1.0 + 2.0 ** -52         # (e + e) + 1 = 1 + 2^-52


def test_we6_average_rounding():
    r = oracle.databin([[0.5] * 3], [[0.1] * 3], [1], [0], [1])
    assert r["sum"][0, 0] == 0.30000000000000004
    assert r["avg"][0, 0] == 0.10000000000000002     # = max + 1 ulp (reading R9)
    assert r["avg"][0, 0] > r["max"][0, 0]


def test_we7_signed_zero_total_order():
    for vals in ([-0.0, 0.0], [0.0, -0.0]):
        r = oracle.databin([[0.5] * 2], [vals], [1], [0], [1])
        assert f2b(r["min"][0, 0]) == f2b(-0.0)
        assert f2b(r["max"][0, 0]) == f2b(0.0)


@pytest.mark.parametrize("lo,hi,k_e", [(0.0, 8.0, 3), (-4.0, 4.0, 3), (0.0, 0.5, -1)])
def test_we8_dyadic_closed_form(lo, hi, k_e):
    # lo..hi spans 2^e; res = 64 = 2^6; x = lo + j*2^(e-40) exactly, so
    # k = floor(j * 2^(6-40)) = j >> 34, clamped to 63 (integer arithmetic only).
    rng = np.random.default_rng(8)
    j = rng.integers(0, 2 ** 40 + 1, size=20000, dtype=np.int64)
    j[:3] = [0, 2 ** 40, 2 ** 40 - 1]
    x = lo + j.astype(np.float64) * 2.0 ** (k_e - 40)
    assert np.all(x - lo == j.astype(np.float64) * 2.0 ** (k_e - 40))  # exact inputs
    r = oracle.databin([x], [np.ones_like(x)], [64], [lo], [hi])
    k = np.minimum(j >> 34, 63)
    assert r["count"].tolist() == np.bincount(k, minlength=64).astype(np.uint64).tolist()


def test_upper_clamp_for_every_inside_x():
    # Reading R2: any x <= hi whose index rounds to res goes to res-1.
    rng = np.random.default_rng(2)
    found = 0
    for _ in range(4000):
        lo, hi = np.sort(rng.uniform(-10, 10, 2))
        res = int(rng.integers(2, 5000))
        x = np.nextafter(hi, -np.inf)
        if math.floor((x - lo) * (res / (hi - lo))) >= res:
            r = oracle.databin([[x, hi]], [[1.0, 1.0]], [res], [lo], [hi])
            assert r["count"][res - 1] == 2 and r["n_out"] == 0
            found += 1
    assert found > 10


def test_nan_and_inf_are_outside():
    r = oracle.databin([[np.nan, np.inf, -np.inf, 0.5]], [[1.0] * 4], [2], [0], [1])
    assert (r["n_in"], r["n_out"]) == (1, 3)


def test_empty_input_manual_and_auto():
    r = oracle.databin([np.zeros(0), np.zeros(0)], [np.zeros(0)], [3, 2], [0, 0], [1, 1])
    assert r["count"].sum() == 0 and (r["n_in"], r["n_out"]) == (0, 0)
    for b in range(6):
        empty_bin_ok(r, b)
    with pytest.raises(ValueError):
        oracle.databin([np.zeros(0)], [], [4], bounds_auto=True)


# ---------------------------------------------------------------- auto bounds
def test_auto_bounds_examples():
    # SPEC.md:353-355
    lo, hi = oracle.bounds([np.array([-1.0, 0.0, 2.0])])
    assert (lo[0], hi[0]) == (-1.0, 2.0)
    r = oracle.databin([[5.0, 5.0, 5.0]], [[1.0, 2.0, 3.0]], [4], bounds_auto=True)
    assert (r["lo"][0], r["hi"][0]) == (4.5, 5.5)     # reading R4
    assert r["count"].tolist() == [0, 0, 3, 0]


def test_auto_bounds_ignore_nan_rows():
    # reading R4: NaN rows do not define bounds (and then fall outside the mesh);
    # numpy's nanmin/nanmax are the independent reference; -0.0 < +0.0 (R6)
    rng = np.random.default_rng(15)
    x = rng.uniform(-3, 7, 1000)
    x[[0, 17, 999]] = np.nan
    lo, hi = oracle.bounds([x])
    assert (lo[0], hi[0]) == (np.nanmin(x), np.nanmax(x))
    lo, hi = oracle.bounds([np.array([np.nan, 0.0, -0.0, np.nan])])
    assert np.signbit(lo[0]) and not np.signbit(hi[0])
    with pytest.raises(ValueError):
        oracle.bounds([np.array([np.nan, np.nan])])
    r = oracle.databin([x], [np.ones(1000)], [10], bounds_auto=True)
    assert (r["n_in"], r["n_out"]) == (997, 3)


def test_auto_bounds_nothing_outside():
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = int(rng.integers(1, 3000))
        ax = [rng.standard_normal(n) * rng.uniform(0.1, 100) for _ in range(2)]
        r = oracle.databin(ax, [rng.uniform(0.5, 1.5, n)], [17, 9], bounds_auto=True)
        assert r["n_out"] == 0 and r["n_in"] == n
        assert r["lo"].tolist() == [a.min() for a in ax]
        assert r["hi"].tolist() == [a.max() for a in ax]


# ---------------------------------------------------------------- library routines
def _centred_inputs(rng, res, lo, hi, n):
    """Rows at bin centres +- 0.3 widths: no formula can disagree on the bin."""
    ks = [rng.integers(0, r_, n) for r_ in res]
    axes = []
    for d, r_ in enumerate(res):
        w = (hi[d] - lo[d]) / r_
        axes.append(lo[d] + (ks[d] + 0.5 + rng.uniform(-0.3, 0.3, n)) * w)
    return ks, axes


@pytest.mark.parametrize("res", [[16, 16], [5, 7, 3], [33], [64, 2, 2]])
def test_counts_match_numpy_histogramdd(res):
    rng = np.random.default_rng(len(res) * 100 + res[0])
    lo = rng.uniform(-5, 0, len(res))
    hi = lo + rng.uniform(0.5, 7, len(res))
    n = 5000
    _, axes = _centred_inputs(rng, res, lo, hi, n)
    r = oracle.databin(axes, [np.ones(n)], res, lo, hi)
    h, _ = np.histogramdd(np.stack(axes, 1), bins=res, range=list(zip(lo, hi)))
    assert r["count"].tolist() == h.astype(np.uint64).ravel(order="F").tolist()  # x fastest


@pytest.mark.parametrize("res", [[16, 16], [4, 5, 6]])
def test_sum_min_max_match_bincount_and_ufunc_at(res):
    rng = np.random.default_rng(11)
    lo = np.full(len(res), -1.0)
    hi = np.full(len(res), 1.0)
    n = 20000
    ks, axes = _centred_inputs(rng, res, lo, hi, n)
    lin = np.ravel_multi_index(ks, res, order="F")
    B = int(np.prod(res))
    vals = [rng.uniform(0.5, 1.5, n), rng.uniform(-1, 1, n)]
    r = oracle.databin(axes, vals, res, lo, hi)
    for a, v in enumerate(vals):
        # np.bincount accumulates in row order: bit-identical to the sequential fold
        s = np.bincount(lin, weights=v, minlength=B)
        occupied = np.bincount(lin, minlength=B) > 0
        assert np.array_equal(r["sum"][a][occupied].view(np.uint64), s[occupied].view(np.uint64))
        mn = np.full(B, np.inf)
        mx = np.full(B, -np.inf)
        np.minimum.at(mn, lin, v)
        np.maximum.at(mx, lin, v)
        assert np.array_equal(r["min"][a], mn) and np.array_equal(r["max"][a], mx)
        with np.errstate(invalid="ignore", divide="ignore"):
            avg = s / np.bincount(lin, minlength=B)
        assert np.array_equal(r["avg"][a][occupied], avg[occupied])


def test_sum_within_fsum_error_bound():
    rng = np.random.default_rng(3)
    n = 3000
    x = rng.uniform(0, 1, n)
    v = rng.standard_normal(n) * 10.0 ** rng.uniform(-3, 3, n)
    r = oracle.databin([x], [v], [4], [0], [1])
    k = np.minimum(np.floor(x * 4).astype(int), 3)
    u = 2.0 ** -53
    for b in range(4):
        vb = v[k == b]
        m = len(vb)
        gamma = (m - 1) * u / (1 - (m - 1) * u)
        exact = math.fsum(vb)
        assert abs(r["sum"][0, b] - exact) <= gamma * np.abs(vb).sum()
        assert r["sumabs"][0, b] == pytest.approx(np.abs(vb).sum(), rel=1e-12)


# ---------------------------------------------------------------- brute force
def test_brute_force_per_bin_scan():
    """A differently structured reference: for each bin, scan every row."""
    rng = np.random.default_rng(4)
    n_edge = 0
    for trial in range(30):
        ndim = int(rng.integers(1, 4))
        res = [int(rng.integers(1, 5)) for _ in range(ndim)]
        n = int(rng.integers(0, 60))
        lo = rng.uniform(-1, 0, ndim)
        hi = lo + rng.uniform(0.5, 2, ndim)
        axes = [rng.uniform(lo[d] - 0.2, hi[d] + 0.2, n) for d in range(ndim)]
        v = rng.integers(-50, 50, n).astype(np.float64)   # integer: order-free sums
        r = oracle.databin(axes, [v], res, lo, hi)
        B = int(np.prod(res))
        for b in range(B):
            cell = []
            rem = b
            for d in range(ndim):
                cell.append(rem % res[d])
                rem //= res[d]
            members, edge = [], []
            for i in range(n):
                ok = True
                for d in range(ndim):
                    x = axes[d][i]
                    if not (lo[d] <= x <= hi[d]):
                        ok = False
                        break
                    w = (hi[d] - lo[d]) / res[d]
                    # the cell's closed interval [lo + c*w, lo + (c+1)*w], upper edge to
                    # the next cell except the last; rows within 1e-9 of an interior edge
                    # may fall on either side of it (WE2/WE8 pin those exactly)
                    t = (x - lo[d]) / w
                    if abs(t - round(t)) < 1e-9 and 0 < round(t) < res[d]:
                        if round(t) - 1 <= cell[d] <= round(t):
                            ok = None
                        else:
                            ok = False
                            break
                        continue
                    c = min(int(math.floor(t)), res[d] - 1)
                    if c != cell[d]:
                        ok = False
                        break
                if ok is None:
                    edge.append(v[i])
                elif ok:
                    members.append(v[i])
            assert len(members) <= r["count"][b] <= len(members) + len(edge)
            if not edge:
                assert r["count"][b] == len(members)
                if members:
                    assert r["sum"][0, b] == sum(members)
                    assert r["min"][0, b] == min(members) and r["max"][0, b] == max(members)
                else:
                    empty_bin_ok(r, b)
            n_edge += len(edge)
        assert r["count"].sum() == r["n_in"]
    assert n_edge < 10  # the edge exclusion stays rare (random uniform coordinates)


# ---------------------------------------------------------------- invariants
def test_invariants_conservation_and_ordering():
    rng = np.random.default_rng(6)
    n = 50000
    axes = [rng.uniform(-1.2, 1.2, n), rng.uniform(-1.2, 1.2, n)]
    m = rng.uniform(0.5, 1.5, n)
    r = oracle.databin(axes, [m], [32, 32], [-1, -1], [1, 1])
    assert r["count"].sum() == r["n_in"] and r["n_in"] + r["n_out"] == n
    inside = (np.abs(axes[0]) <= 1) & (np.abs(axes[1]) <= 1)
    assert r["n_in"] == inside.sum()
    assert math.isclose(r["sum"].sum() + m[~inside].sum(), m.sum(), rel_tol=1e-12)
    occ = r["count"] > 0
    slack = 1e-12 * np.abs(r["max"][0][occ])
    assert np.all(r["min"][0][occ] <= r["avg"][0][occ] + slack)
    assert np.all(r["avg"][0][occ] <= r["max"][0][occ] + slack)


def test_partition_mode_laws():
    rng = np.random.default_rng(7)
    n = 10007
    axes = [rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)]
    m = rng.uniform(0.5, 1.5, n)
    mi = rng.integers(1, 1000, n).astype(np.float64)
    base = oracle.databin(axes, [m, mi], [16, 8], [-1, -1], [1, 1], P=1)
    for P in (2, 3, 8, 20000):
        r = oracle.databin(axes, [m, mi], [16, 8], [-1, -1], [1, 1], P=P)
        assert np.array_equal(r["count"], base["count"])
        assert np.array_equal(r["min"], base["min"]) and np.array_equal(r["max"], base["max"])
        assert (r["n_in"], r["n_out"]) == (base["n_in"], base["n_out"])
        assert np.all(np.abs(r["sum"] - base["sum"]) <= 1e-12 * base["sumabs"])
        assert np.array_equal(r["sum"][1], base["sum"][1])  # integer sums: order-free
    # P-partition equals folding per-block grids in rank order
    P = 3
    cuts = [(k * n) // P for k in range(P + 1)]
    parts = [oracle.databin([a[cuts[k]:cuts[k + 1]] for a in axes], [m[cuts[k]:cuts[k + 1]]],
                            [16, 8], [-1, -1], [1, 1]) for k in range(P)]
    s = np.zeros_like(parts[0]["sum"])
    for p in parts:
        s = s + p["sum"]
    r = oracle.databin(axes, [m], [16, 8], [-1, -1], [1, 1], P=P)
    assert np.array_equal(r["sum"].view(np.uint64), s.view(np.uint64))


# ---------------------------------------------------------------- Eq. (1)
def test_eq1_examples():
    # SPEC.md:238-247 hand evaluations of PAPER.md:418
    assert oracle.eq1_device(0, 4, 1, 0, 4) == 0
    assert oracle.eq1_device(5, 4, 1, 0, 4) == 1
    assert oracle.eq1_device(2, 3, 1, 1, 4) == 3
    assert [oracle.eq1_device(r, 4, 1, 0, 4) for r in range(8)] == [0, 1, 2, 3, 0, 1, 2, 3]
    assert [oracle.eq1_device(r, 1, 1, 3, 4) for r in range(4)] == [3, 3, 3, 3]


def test_eq1_properties():
    for n_a in (1, 2, 4, 8):
        for n_u in range(1, n_a + 1):
            for s in (1, 2, 3):
                for d0 in range(n_a):
                    ds = [oracle.eq1_device(r, n_u, s, d0, n_a) for r in range(64)]
                    assert all(0 <= d < n_a for d in ds)
                    assert all(ds[r] == ds[r + n_u] for r in range(64 - n_u))  # period n_u
    assert [oracle.eq1_device(r, 8, 1, 0, 8) for r in range(8)] == list(range(8))


# ---------------------------------------------------------------- unusable bounds (reading R4)
def test_auto_bounds_infinite_or_overflowing_are_degenerate():
    # R4: realised bounds must be finite with a finite width and scale; the
    # plain definition has no bin for (x - lo) * scale = NaN, so such inputs
    # are BIN_EDEGENERATE (auto) -- never an index computed from NaN
    for col in ([0.0, 1.0, np.inf], [-np.inf, 0.0, 1.0], [np.inf, np.inf], [-np.inf]):
        with pytest.raises(oracle.Degenerate):
            oracle.databin([col], [np.ones(len(col))], [4], bounds_auto=True)
    big = np.finfo(np.float64).max
    with pytest.raises(oracle.Degenerate):      # width hi - lo overflows to +inf
        oracle.databin([[-big, big]], [[1.0, 1.0]], [4], bounds_auto=True)
    with pytest.raises(oracle.Degenerate):      # scale res / width overflows (subnormal width)
        oracle.databin([[0.0, 5e-324]], [[1.0, 1.0]], [4], bounds_auto=True)
    with pytest.raises(oracle.Degenerate):      # lo == hi and +-0.5 rounds away (R4 widening fails)
        oracle.databin([[1e300, 1e300]], [[1.0, 1.0]], [4], bounds_auto=True)
    # NaN rows are still skipped: finite rows alone define usable bounds
    r = oracle.databin([[0.0, np.nan, 1.0]], [[1.0, 2.0, 3.0]], [2], bounds_auto=True)
    assert (r["lo"][0], r["hi"][0], r["count"].tolist(), r["n_out"]) == (0.0, 1.0, [1, 1], 1)
    # 2D: one bad axis is enough
    with pytest.raises(oracle.Degenerate):
        oracle.databin([[0.0, 1.0], [0.0, np.inf]], [], [2, 2], bounds_auto=True)


def test_manual_bounds_must_be_usable():
    big = np.finfo(np.float64).max
    for lo, hi in ((0.0, np.inf), (-np.inf, 0.0), (np.nan, 1.0), (0.0, np.nan), (1.0, 1.0), (2.0, 1.0),
                   (-big, big), (0.0, 5e-324)):
        with pytest.raises(oracle.InvalidArgument):
            oracle.databin([[0.5]], [[1.0]], [4], [lo], [hi])
    # the largest usable widths still bin (scale finite, every in-bounds index finite)
    r = oracle.databin([[-big / 2, big / 4, big / 2]], [[1.0, 2.0, 3.0]], [2], [-big / 2], [big / 2])
    assert r["count"].tolist() == [1, 2]
    r = oracle.databin([[0.0, 1e-300]], [[1.0, 2.0]], [2], [0.0], [1e-300])
    assert r["count"].tolist() == [1, 1]


# ---------------------------------------------------------------- streamed partition mode
@pytest.mark.parametrize("P", [1, 2, 5])
def test_databin_blocks_is_partition_mode(P):
    """oracle.databin_blocks (the streamed form used for the 1B-row C4 check)
    is the partition mode of oracle_databin step for step: bit-identical in
    every output for any chunking, including chunks that split blocks."""
    import synth
    w = synth.CONFIGS["c4"]
    n = 300_007

    def rows(s, c):
        return ([synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c) for x in w.axes],
                [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[x], s, c) for x in ("mass", "vx")])

    axes, attrs = rows(0, n)
    ref = oracle.databin(axes, attrs, [16, 8, 4], [-1, -1, -1], [1, 1, 0.5], P=P)
    got = oracle.databin_blocks(rows, n, [16, 8, 4], [-1, -1, -1], [1, 1, 0.5], 2, P=P, chunk=65_537)
    for k in ("count", "sum", "sumabs", "min", "max", "avg"):
        assert np.array_equal(np.asarray(ref[k]).view(np.uint64), np.asarray(got[k]).view(np.uint64)), k
    assert (ref["n_in"], ref["n_out"]) == (got["n_in"], got["n_out"])
    assert got["n_out"] > 0
