"""Fan-in execute (bin_execute_shards; the paper's dedicated-device placement,
PAPER.md:496-497): several row blocks -- from this GPU, host memory or other
GPUs -- binned as one batch must equal the oracle on the concatenated rows
(deterministic mode: bit-exact in shard order; exact sums: bit-exact)."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import bits, compare

pytestmark = pytest.mark.gpu


def shard_handles(db, cols_per_shard, where):
    import torch
    keep, shards = [], []
    for cols, w in zip(cols_per_shard, where):
        hs = []
        for c in cols:
            if w == "host":
                t = torch.from_numpy(np.ascontiguousarray(c)).pin_memory()
            else:
                t = torch.from_numpy(np.ascontiguousarray(c)).to(torch.device(w))
            keep.append(t)
            hs.append(db.wrap_tensor(t))
        shards.append(hs)
    import torch
    torch.cuda.synchronize()
    return keep, shards


def run_shards(db, cols_per_shard, where, nax, res, lo, hi, **kw):
    keep, shards = shard_handles(db, cols_per_shard, where)
    spec = db.make_spec(res, lo, hi, nattr=len(cols_per_shard[0]) - nax, **kw)
    h = db.bin_init(spec, db.make_placement(device_id=0, exec=db.BIN_EXEC_PEER))
    try:
        t = db.bin_execute_shards(h, [(s[:nax], s[nax:]) for s in shards])
        out = db.result_to_numpy(h, t, spec)
    finally:
        db.bin_finalize(h)
        for s in shards:
            for a in s:
                db.bin_array_release(a)
    del keep
    return out


def gen(rng, n, nattr=1):
    return [rng.normal(0, 0.7, n), rng.normal(0, 0.7, n)] + [rng.uniform(0.5, 1.5, n) for _ in range(nattr)]


@pytest.mark.parametrize("mode", ["atomic", "deterministic", "exact"])
def test_shards_local_and_host(db, mode):
    rng = np.random.default_rng(41)
    sizes = [300_001, 0, 17, 1_000_000, 5]
    parts = [gen(rng, n) for n in sizes]
    where = ["cuda:0", "host", "cuda:0", "host", "cuda:0"]
    kw = dict(deterministic=mode == "deterministic", exact=mode == "exact")
    out = run_shards(db, parts, where, 2, (128, 96), (-2, -2), (2, 2), **kw)
    cat = [np.concatenate([p[i] for p in parts]) for i in range(3)]
    ref = oracle.databin(cat[:2], cat[2:], (128, 96), (-2, -2), (2, 2), exact=mode == "exact")
    compare(out, ref, exact=mode == "deterministic")
    if mode == "exact":
        assert np.array_equal(bits(out["sum"][0]), bits(ref["sum_exact"][0]))


def test_shards_auto_bounds_3d(db):
    rng = np.random.default_rng(42)
    parts = [[rng.normal(0, 1, n) for _ in range(3)] + [rng.normal(0, 1, n)] for n in (50_000, 70_001, 3)]
    out = run_shards(db, parts, ["cuda:0"] * 3, 3, (16, 16, 16), None, None, bounds_auto=True)
    cat = [np.concatenate([p[i] for p in parts]) for i in range(4)]
    ref = oracle.databin(cat[:3], cat[3:], (16, 16, 16), bounds_auto=True)
    compare(out, ref)
    assert np.array_equal(out["lo"], ref["lo"]) and np.array_equal(out["hi"], ref["hi"])


def test_shards_from_other_gpus(db):
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    G = torch.cuda.device_count()
    rng = np.random.default_rng(43)
    parts = [gen(rng, 400_000 + k) for k in range(G - 1)]
    where = [f"cuda:{k + 1}" for k in range(G - 1)]
    out = run_shards(db, parts, where, 2, (256, 256), (-2, -2), (2, 2), deterministic=True)
    cat = [np.concatenate([p[i] for p in parts]) for i in range(3)]
    compare(out, oracle.databin(cat[:2], cat[2:], (256, 256), (-2, -2), (2, 2)), exact=True)


def test_shards_errors(db):
    import torch
    spec = db.make_spec((4,), (0,), (1,), nattr=1)
    h = db.bin_init(spec, db.make_placement(device_id=0))
    a = torch.zeros(10, dtype=torch.float64, device="cuda:0")
    b = torch.zeros(11, dtype=torch.float64, device="cuda:0")
    ha, hb = db.wrap_tensor(a), db.wrap_tensor(b)
    try:
        with pytest.raises(db.BinError) as e:
            db.bin_execute_shards(h, [([ha], [hb])])                 # lengths differ within a shard
        assert e.value.code == 2
        t = db.bin_execute_shards(h, [([ha], [ha]), ([hb], [hb])])  # lengths may differ across shards
        assert db.result_to_numpy(h, t, spec)["n_in"] == 21
    finally:
        db.bin_finalize(h)
        db.bin_array_release(ha)
        db.bin_array_release(hb)
