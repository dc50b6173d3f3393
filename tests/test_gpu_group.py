"""Cross-rank combine (SURVEY §8 row a6 + a7) on ONE B200.

A one-device rank group (``bin_init_group``) bins P contiguous row blocks
into P ranks' accumulators and combines them with the fused peer combine +
finalize kernel -- the same device code (barrier words, rank-order sum fold,
exact-digit add, min/max, finalize, all-gather into every rank) that one
process per GPU runs over NVLink.  The result is checked against the
oracle's partition mode P (rows split as [floor(rN/P), floor((r+1)N/P))):
bit-exact for deterministic mode and exact sums, reading R8 for fast sums,
and every rank must hold the identical result.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from tests.gpu_util import bits, compare

pytestmark = pytest.mark.gpu


def _blocks(n, P):
    return [(r * n // P, (r + 1) * n // P) for r in range(P)]


def run_group(db, P, mode, n=20_001, res=(64, 64), nattr=1, ops=("sum", "min", "max", "avg"), route="auto",
              seed=0, executes=1, lo=None, hi=None, cols=None, check=True, exec_mode=None):
    """Bins n rows as P ranks of a one-device group; checks every rank's result
    against the oracle in partition mode P.  Returns rank 0's output."""
    import torch
    dev = torch.device("cuda:0")
    D = len(res)
    if cols is None:
        rng = np.random.default_rng(seed)
        axes = [rng.standard_normal(n) * 0.45 for _ in range(D)]
        attrs = [rng.uniform(0.5, 1.5, n) if a == 0 else rng.standard_normal(n) * 10 ** (a - 1) for a in range(nattr)]
    else:
        axes, attrs = cols
        n = len(axes[0])
    lo = [-1.0] * D if lo is None else lo
    hi = [1.0] * D if hi is None else hi
    spec = db.make_spec(res, lo, hi, nattr=nattr, ops=ops, deterministic=(mode == "det"), route=route,
                        exact=(mode == "exact"))
    pl = db.make_placement(device_id=0) if exec_mode is None else db.make_placement(device_id=0, exec=exec_mode)
    hs = db.bin_init_group(spec, P, pl)
    keep, arrays = [], []
    try:
        # each rank's columns live on its own stream (lockstep per rank)
        streams = [torch.cuda.Stream(dev) for _ in range(P)]
        shards = []
        for r, (b0, b1) in enumerate(_blocks(n, P)):
            ts = [torch.from_numpy(np.ascontiguousarray(c[b0:b1])).to(dev) for c in axes + attrs]
            keep += ts
            torch.cuda.synchronize(dev)
            hnd = [db.wrap_tensor(t, stream=streams[r].cuda_stream) for t in ts]
            arrays += hnd
            shards.append((hnd[:D], hnd[D:]))
        outs = None
        for _ in range(executes):
            t = db.bin_execute_group(hs, shards)
            outs = [db.result_to_numpy(h, t, spec) for h in hs]
        if check:
            ref = oracle.databin(axes, attrs, list(res), lo, hi, P=P, exact=(mode == "exact"))
            for r, out in enumerate(outs):
                if mode == "exact":
                    refx = dict(ref)
                    refx["sum"] = ref["sum_exact"]
                    refx["avg"] = ref["avg_exact"]
                    compare(out, refx, ops=ops, exact=True)
                else:
                    compare(out, ref, ops=ops, exact=(mode == "det"))
                if r:  # the all-gather: every rank holds the same final arrays
                    o0 = outs[0]
                    assert np.array_equal(out["count"], o0["count"])
                    for k in ("sum", "min", "max", "avg"):
                        for a in range(nattr):
                            if o0[k][a] is not None:
                                assert np.array_equal(bits(out[k][a]), bits(o0[k][a])), (r, k, a)
        return outs[0]
    finally:
        for h in hs:
            db.bin_finalize(h)
        for a in arrays:
            db.bin_array_release(a)


@pytest.mark.parametrize("P", [2, 3, 4, 8])
@pytest.mark.parametrize("mode", ["fast", "det", "exact"])
def test_group_combine_vs_partition_oracle(db, P, mode):
    """P ranks, one summed + one min/max attribute: the TMA bulk slice for
    P in {2, 4, 8}, the generic per-bin slice for P = 3 and exact sums."""
    run_group(db, P, mode, n=50_003, res=(64, 64), seed=P)


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("mode", ["fast", "det", "exact"])
def test_group_several_attributes(db, P, mode):
    """Four attributes (generic slice: several sums and min/max rows per bin)."""
    run_group(db, P, mode, n=30_001, res=(32, 48), nattr=4, seed=10 + P)


@pytest.mark.parametrize("route", ["window", "partition"])
@pytest.mark.parametrize("P", [2, 4])
def test_group_routes(db, route, P):
    run_group(db, P, "fast", n=200_001, res=(256, 256), route=route, seed=20 + P)


def test_group_3d_and_1d(db):
    run_group(db, 4, "fast", n=100_000, res=(16, 16, 16), seed=31)
    run_group(db, 2, "det", n=10_001, res=(100,), seed=32)


def test_group_op_subsets(db):
    run_group(db, 2, "fast", n=20_000, nattr=2, ops=[("sum",), ("min", "max")], seed=41)
    run_group(db, 4, "det", n=20_000, nattr=1, ops=("avg",), seed=42)
    run_group(db, 2, "fast", n=20_000, nattr=0, ops=(), seed=43)


def test_group_ranks_without_rows(db):
    """n < P: some ranks hold no rows (their partials are identities)."""
    run_group(db, 8, "fast", n=5, seed=51)
    run_group(db, 4, "det", n=3, seed=52)
    run_group(db, 4, "exact", n=0 + 2, seed=53)


def test_group_repeated_executes(db):
    """Executes alternate between the two result slots (barrier epochs 1..5)."""
    run_group(db, 4, "fast", n=40_000, executes=5, seed=61)
    run_group(db, 2, "exact", n=40_000, executes=3, seed=62)


def test_group_async_side_streams(db):
    run_group(db, 4, "fast", n=40_000, exec_mode=db.BIN_EXEC_ASYNC, seed=71)


def test_group_plummer_contention(db):
    """C3-shaped (Plummer, 512^2) slice of the bench workload, 4 ranks."""
    import synth
    from tests.gpu_util import workload_inputs
    w = synth.CONFIGS["c3"]
    axes, attrs = workload_inputs(w, n=2_000_000)
    run_group(db, 4, "fast", res=tuple(w.res), lo=list(w.lo), hi=list(w.hi), cols=(axes, attrs))
    run_group(db, 2, "det", res=tuple(w.res), lo=list(w.lo), hi=list(w.hi), cols=(axes, attrs))


def test_group_errors(db):
    spec = db.make_spec((8, 8), [0, 0], [1, 1], nattr=1)
    with pytest.raises(db.BinError) as e:
        db.bin_init_group(spec, 0, db.make_placement(device_id=0))
    assert e.value.code == 1
    auto = db.make_spec((8, 8), nattr=1, bounds_auto=True)
    with pytest.raises(db.BinError) as e:
        db.bin_init_group(auto, 2, db.make_placement(device_id=0))
    assert e.value.code == 7
    hs = db.bin_init_group(spec, 2, db.make_placement(device_id=0))
    try:
        import torch
        t = torch.zeros(4, dtype=torch.float64, device="cuda:0")
        a = db.wrap_tensor(t)
        with pytest.raises(db.BinError) as e:  # a member is not a stand-alone handle
            db.bin_execute(hs[0], [a, a], [a])
        assert e.value.code == 10
        with pytest.raises(db.BinError) as e:  # ranks in the wrong order
            db.bin_execute_group([hs[1], hs[0]], [([a, a], [a]), ([a, a], [a])])
        assert e.value.code == 10
        db.bin_array_release(a)
    finally:
        for h in hs:
            db.bin_finalize(h)


@pytest.mark.slow
def test_group_c3_full_size_4_ranks(db):
    """The bench's multi-GPU configuration at full size on one B200: C3 (100M
    Plummer rows, 512^2) as 4 ranks of 25M rows each, the same fused combine
    body as `bench.py --gpus 4`, against the oracle's partition mode P = 4."""
    import synth
    from tests.gpu_util import workload_inputs
    w = synth.CONFIGS["c3"]
    axes, attrs = workload_inputs(w)
    out = run_group(db, 4, "fast", res=tuple(w.res), lo=list(w.lo), hi=list(w.hi), cols=(axes, attrs))
    assert out["n_in"] + out["n_out"] == w.n
