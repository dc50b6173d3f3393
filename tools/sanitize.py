"""Small-input driver for memory-safety runs: every kernel family of
libdatabin once, on C1 and a few small random and route-forcing cases, each
checked against the oracle.  Run it under compute-sanitizer where that is
available, or (as on this GPU pool, where compute-sanitizer is closed) against
the checked build, whose kernels bounds-check every computed window index,
bin index and scatter position and trap on a failure:

  python tools/build_variants.py checked=DATABIN_CHECKED
  DATABIN_LIB=paper_2310_02926_b200/variants/checked.so python tools/sanitize.py
  compute-sanitizer --tool racecheck python tools/sanitize.py [--quick]

Kernels covered: k_prep, k_bounds, k_probe, k_bin_fast (full-grid and hot
window + queue), k_bin (general), k_window, the partition route (keys, scans,
scatter, refine, reduce), the deterministic sort path, exact sums, k_finalize,
the fused multi-instance kernels, and the one-GPU rank group's peer combine
(when the library exports it).
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402  (test infrastructure: checks the sanitized runs)
import synth  # noqa: E402
import paper_2310_02926_b200 as db  # noqa: E402
from tests.gpu_util import compare, run_gpu, workload_inputs  # noqa: E402


def case(name, axes, attrs, res, lo=None, hi=None, bounds_auto=False, **kw):
    ref = oracle.databin(axes, attrs, res, lo, hi, bounds_auto=bounds_auto)
    out = run_gpu(db, axes, attrs, res, lo, hi, bounds_auto=bounds_auto, **kw)
    compare(out, ref, exact=kw.get("deterministic", False))
    if kw.get("exact"):
        refx = oracle.databin(axes, attrs, res, lo, hi, bounds_auto=bounds_auto, exact=True)
        assert np.array_equal(out["sum"][0].view(np.uint64), refx["sum_exact"][0].view(np.uint64))
    print(f"ok {name}", flush=True)


def main():
    quick = "--quick" in sys.argv
    w = synth.CONFIGS["c1"]
    axes, attrs = workload_inputs(w)
    case("c1 manual (full-grid k_bin_fast)", axes, attrs, w.res, w.lo, w.hi)
    case("c1 auto bounds", axes, attrs, w.res, bounds_auto=True)
    case("c1 deterministic", axes, attrs, w.res, w.lo, w.hi, deterministic=True)
    case("c1 exact", axes, attrs, w.res, w.lo, w.hi, exact=True)
    rng = np.random.default_rng(7)
    n = 20_001 if quick else 100_001
    ax = [rng.standard_normal(n) * 0.4, rng.standard_normal(n) * 0.4]
    at = [rng.uniform(0.5, 1.5, n)]
    case("512^2 window + queue", ax, at, [512, 512], [-1, -1], [1, 1], route="window")
    case("512^2 partition", ax, at, [512, 512], [-1, -1], [1, 1], route="partition")
    case("512^2 exact window", ax, at, [512, 512], [-1, -1], [1, 1], route="window", exact=True)
    at4 = [rng.standard_normal(n) for _ in range(4)]
    case("256^2 4 attrs general kernel", ax, at4, [256, 256], [-1, -1], [1, 1], route="window")
    case("256^2 4 attrs partition", ax, at4, [256, 256], [-1, -1], [1, 1], route="partition")
    ax3 = [rng.uniform(-1, 1, n) for _ in range(3)]
    case("3D 128^3 partition (two-level)", ax3, at, [128, 128, 128], [-1] * 3, [1] * 3, route="partition")
    case("3D 64^3 deterministic", ax3, at, [64, 64, 64], [-1] * 3, [1] * 3, deterministic=True)
    case("auto route + auto bounds", ax, at, [512, 512], bounds_auto=True)
    # fused instance sets
    from tests.test_multi import oracle_of, paper_step_instances, run_multi, synth_cols
    cols = synth_cols(5_001 if quick else 30_001)
    insts = paper_step_instances(32)
    outs, _ = run_multi(db, cols, insts)
    for d, out in zip(insts, outs):
        compare(out, oracle_of(cols, d))
    print("ok multi paper step", flush=True)
    if hasattr(db, "bin_init_group"):
        from tests.test_gpu_group import run_group
        for P in (2, 4):
            for mode in ("fast", "det", "exact"):
                run_group(db, P, mode, n=8_001, res=(64, 64))
                print(f"ok group P={P} {mode}", flush=True)
    print("SANITIZE DONE", flush=True)


if __name__ == "__main__":
    main()
