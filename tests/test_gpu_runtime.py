"""GPU tests of the runtime state that carries across executes of one handle
(handle.cpp): the per-CTA window cache of k_bin_fast (reused for 16
executes, re-sampled when the row count changes), the accumulator identities
written on the prep stream while the previous execute still runs, the auto
route's asynchronous re-probe, the two result slots, and zero-row executes
between ordinary ones.  Every result is compared with the oracle."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_util import compare, workload_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_available):
    if not cuda_available:
        pytest.fail("GPU tests need a CUDA device")


def _dev(cols):
    import torch
    ts = [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols]
    torch.cuda.synchronize()
    return ts


def test_window_cache_follows_changing_inputs(db):
    """One handle, inputs whose size and distribution change between executes:
    the cached windows are only a speed hint, results always match."""
    w = synth.CONFIGS["c3"]
    spec = db.make_spec(w.res, w.lo, w.hi, nattr=1, route="window")
    h = db.bin_init(spec, db.make_placement(device_id=0))
    rng = np.random.default_rng(21)
    cases = []
    ax, at = workload_inputs(w, n=600_001)
    cases.append((ax, at))
    cases.append(([rng.uniform(-16, 16, 400_000), rng.uniform(-16, 16, 400_000)], [rng.uniform(0, 1, 400_000)]))
    cases.append(([rng.normal(5, 0.5, 600_001), rng.normal(-3, 0.5, 600_001)], [rng.uniform(-1, 1, 600_001)]))
    for rep in range(3):                      # same row count: cached windows of a different distribution
        for axes, attrs in cases:
            ts = _dev(axes + attrs)
            hs = [db.wrap_tensor(t) for t in ts]
            t = db.bin_execute(h, hs[:2], hs[2:])
            compare(db.result_to_numpy(h, t, spec), oracle.databin(axes, attrs, w.res, w.lo, w.hi))
            for a in hs:
                db.bin_array_release(a)
    db.bin_finalize(h)


def test_back_to_back_executes_both_slots(db):
    """Many executes enqueued without waiting (the prep stream zeroes a slot
    while the other slot's execute runs): each of the last two tickets holds
    its own inputs' result."""
    import torch
    rng = np.random.default_rng(22)
    n = 300_000
    sets = [([rng.normal(0, s, n), rng.normal(0, s, n)], [rng.uniform(0.5, 1.5, n)]) for s in (0.3, 0.6, 1.0, 2.0)]
    devs = [_dev(ax + at) for ax, at in sets]
    spec = db.make_spec((256, 256), (-2, -2), (2, 2), nattr=1)
    h = db.bin_init(spec, db.make_placement(device_id=0))
    handles = [[db.wrap_tensor(x) for x in d] for d in devs]
    tickets = []
    for k in range(12):
        hs = handles[k % 4]
        tickets.append((k % 4, db.bin_execute(h, hs[:2], hs[2:])))
    for which, t in tickets[-2:]:
        ax, at = sets[which]
        compare(db.result_to_numpy(h, t, spec), oracle.databin(ax, at, (256, 256), (-2, -2), (2, 2)))
    db.bin_finalize(h)
    for hs in handles:
        for a in hs:
            db.bin_array_release(a)
    torch.cuda.synchronize()


def test_zero_rows_between_executes(db):
    rng = np.random.default_rng(23)
    n = 200_000
    axes, attrs = [rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)], [rng.uniform(0, 1, n)]
    full = _dev(axes + attrs)
    empty = _dev([np.zeros(0)] * 3)
    spec = db.make_spec((128, 128), (-1, -1), (1, 1), nattr=1)
    h = db.bin_init(spec, db.make_placement(device_id=0))
    ref = oracle.databin(axes, attrs, (128, 128), (-1, -1), (1, 1))
    ref0 = oracle.databin([np.zeros(0)] * 2, [np.zeros(0)], (128, 128), (-1, -1), (1, 1))
    for src, r in ((full, ref), (empty, ref0), (full, ref), (empty, ref0), (full, ref)):
        hs = [db.wrap_tensor(x) for x in src]
        t = db.bin_execute(h, hs[:2], hs[2:])
        compare(db.result_to_numpy(h, t, spec), r, exact=r is ref0)
        for a in hs:
            db.bin_array_release(a)
    db.bin_finalize(h)


def test_auto_route_recheck_switches_route(db):
    """Auto route: the first execute probes synchronously; later probes run in
    the background every 64 executes and switch the route when the data's
    spread changes.  Results match the oracle on both routes."""
    rng = np.random.default_rng(24)
    n = 200_000
    clustered = ([rng.normal(0, 0.02, n), rng.normal(0, 0.02, n)], [rng.uniform(0.5, 1.5, n)])
    spread = ([rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)], [rng.uniform(0.5, 1.5, n)])
    dc, ds = _dev(clustered[0] + clustered[1]), _dev(spread[0] + spread[1])
    spec = db.make_spec((512, 512), (-1, -1), (1, 1), nattr=1)
    h = db.bin_init(spec, db.make_placement(device_id=0))
    db.bin_profile_enable(h, True)
    hc = [db.wrap_tensor(x) for x in dc]
    hsp = [db.wrap_tensor(x) for x in ds]
    t = db.bin_execute(h, hc[:2], hc[2:])
    compare(db.result_to_numpy(h, t, spec), oracle.databin(*clustered, (512, 512), (-1, -1), (1, 1)))
    assert db.bin_profile_read(h).variant & 15 in (1, 2)           # window route for the clustered data
    variants = set()
    for k in range(140):                                            # two re-probe periods on spread-out data
        t = db.bin_execute(h, hsp[:2], hsp[2:])
        if k % 20 == 19:
            db.bin_wait(h, t)
            variants.add(db.bin_profile_read(h).variant & 15)
    compare(db.result_to_numpy(h, t, spec), oracle.databin(*spread, (512, 512), (-1, -1), (1, 1)))
    assert 4 in variants                                            # switched to the partition route
    db.bin_finalize(h)
    for a in hc + hsp:
        db.bin_array_release(a)
