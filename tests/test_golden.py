"""Golden fixtures (tests/golden/*.json): hand-derived worked examples, each
citing the passage it follows (see tests/golden/README.md).

The oracle is pinned to them with -m "not gpu"; the CUDA path (through the C
ABI) is checked against the same expected values with -m gpu, in atomic mode
(bit-exact where the fixture's partial sums are exact in any order) and in
deterministic mode (always bit-exact).
"""
import glob
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.json")) if not p.endswith("eq1_placement.json"))


def _num(v):
    return float(v) if isinstance(v, str) else float(v)


def _column(c):
    if isinstance(c, dict):
        if "fill" in c:
            v, n = c["fill"]
            return np.full(int(n), _num(v), np.float64)
        a, b = c["range"]
        return np.arange(a, b, dtype=np.float64)
    return np.array([_num(v) for v in c], np.float64)


def load(path):
    with open(path) as f:
        case = json.load(f)
    assert case.get("cite"), f"{path}: every fixture cites its passage"
    case["axes_np"] = [_column(c) for c in case["axes"]]
    case["attrs_np"] = [_column(c) for c in case["attrs"]]
    return case


def _bits(x):
    return int(np.float64(x).view(np.uint64))


def check(out, case, exact_sum=True):
    """out: dict with count/sum/min/max/avg arrays (attribute 0), n_in, n_out."""
    e = case["expect"]
    assert (int(out["n_in"]), int(out["n_out"])) == (e["n_in"], e["n_out"])
    if "lo" in e:
        assert [_bits(v) for v in out["lo"]] == [_bits(_num(v)) for v in e["lo"]]
        assert [_bits(v) for v in out["hi"]] == [_bits(_num(v)) for v in e["hi"]]
    bins = {int(k): v for k, v in e["bins"].items()}
    B = len(out["count"])
    for b in range(B):
        if b not in bins:
            assert out["count"][b] == 0
            assert _bits(out["sum"][0][b]) == _bits(0.0)
            assert out["min"][0][b] == math.inf and out["max"][0][b] == -math.inf
            assert math.isnan(out["avg"][0][b])
            continue
        x = bins[b]
        assert int(out["count"][b]) == x["count"], b
        for k in ("min", "max"):
            assert _bits(out[k][0][b]) == _bits(_num(x[k])), (b, k, out[k][0][b], x[k])
        for k in ("sum", "avg"):
            if exact_sum:
                assert _bits(out[k][0][b]) == _bits(_num(x[k])), (b, k, out[k][0][b], x[k])
            else:   # reading R8: any order within 1e-12 * sum|v|
                sabs = float(np.sum(np.abs(case["attrs_np"][0])))
                assert abs(out[k][0][b] - _num(x[k])) <= 1e-12 * sabs, (b, k)


@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[:-5])
def test_oracle_golden(path):
    case = load(path)
    sp = case["spec"]
    r = oracle.databin(case["axes_np"], case["attrs_np"], sp["res"], sp.get("lo"), sp.get("hi"),
                       bounds_auto=sp.get("bounds_auto", False))
    check(r, case, exact_sum=True)
    # partition mode agrees exactly whenever the sums are order-free
    if case["exact_any_order"] and len(case["axes_np"][0]) >= 2:
        r2 = oracle.databin(case["axes_np"], case["attrs_np"], sp["res"], sp.get("lo"), sp.get("hi"),
                            bounds_auto=sp.get("bounds_auto", False), P=2)
        check(r2, case, exact_sum=True)


def test_oracle_eq1_golden():
    with open(os.path.join(GOLDEN, "eq1_placement.json")) as f:
        case = json.load(f)
    for c in case["cases"]:
        assert oracle.eq1_device(c["r"], c["n_u"], c["s"], c["d0"], c["n_a"]) == c["device"], c


@pytest.mark.gpu
@pytest.mark.parametrize("det", [False, True], ids=["atomic", "deterministic"])
@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[:-5])
def test_gpu_golden(path, det):
    import paper_2310_02926_b200 as db
    from tests.gpu_util import run_gpu
    case = load(path)
    sp = case["spec"]
    out = run_gpu(db, case["axes_np"], case["attrs_np"], sp["res"], sp.get("lo"), sp.get("hi"),
                  bounds_auto=sp.get("bounds_auto", False), deterministic=det)
    check(out, case, exact_sum=det or case["exact_any_order"])


@pytest.mark.gpu
@pytest.mark.parametrize("route", ["window", "partition"])
@pytest.mark.parametrize("path", CASES, ids=lambda p: os.path.basename(p)[:-5])
def test_gpu_golden_routes(path, route):
    import paper_2310_02926_b200 as db
    from tests.gpu_util import run_gpu
    case = load(path)
    sp = case["spec"]
    out = run_gpu(db, case["axes_np"], case["attrs_np"], sp["res"], sp.get("lo"), sp.get("hi"),
                  bounds_auto=sp.get("bounds_auto", False), route=route)
    check(out, case, exact_sum=case["exact_any_order"])


def test_gpu_resolve_device_golden():
    """bin_resolve_device (host logic of the C ABI, no GPU compute) on Eq. (1)'s examples."""
    import paper_2310_02926_b200 as db
    with open(os.path.join(GOLDEN, "eq1_placement.json")) as f:
        case = json.load(f)
    for c in case["cases"]:
        pl = db.make_placement(device_start=c["d0"], device_stride=c["s"], devices_to_use=c["n_u"])
        assert db.bin_resolve_device(pl, c["r"], c["n_a"]) == c["device"], c
