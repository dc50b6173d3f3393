"""Helpers for the GPU parity tests: run the CUDA path through the C ABI on
seeded inputs, and compare element by element with the oracle.

Tolerances:
  count, n_in, n_out, min, max : bit-exact
  sum  : |s_gpu - s_oracle| <= 1e-12 * sum_bin |v|   (reading R8; atomic order varies)
  avg  : |a_gpu - a_oracle| <= 1e-12 * sum_bin |v| / count + 2 ulp(a_oracle)
  deterministic mode, or exactly representable partial sums: everything bit-exact
"""
from __future__ import annotations

import numpy as np

ALL_OPS = ("sum", "min", "max", "avg")


def bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def run_gpu(db, axes, attrs, res, lo=None, hi=None, ops=ALL_OPS, bounds_auto=False, deterministic=False,
            placement=None, offset=0, host_inputs=False, device=0, return_handle=False, route="auto",
            exact=False):
    import torch
    dev = torch.device(f"cuda:{device}")
    cols = list(axes) + list(attrs)
    keep = []
    handles = []
    for c in cols:
        c = np.ascontiguousarray(c, dtype=np.float64)
        if host_inputs:
            t = torch.empty(len(c) + offset, dtype=torch.float64).pin_memory()
            t[offset:] = torch.from_numpy(c)
        else:
            t = torch.empty(len(c) + offset, dtype=torch.float64, device=dev)
            t[offset:] = torch.from_numpy(c).to(dev)
        t = t[offset:]
        keep.append(t)
        handles.append(db.wrap_tensor(t))
    torch.cuda.synchronize(dev)
    spec = db.make_spec(res, lo, hi, nattr=len(attrs), ops=ops, bounds_auto=bounds_auto,
                        deterministic=deterministic, route=route, exact=exact)
    pl = placement if placement is not None else db.make_placement(device_id=device)
    h = db.bin_init(spec, pl)
    db.bin_profile_enable(h, True)
    try:
        t = db.bin_execute(h, handles[:len(axes)], handles[len(axes):])
        out = db.result_to_numpy(h, t, spec)
        out["profile"] = db.bin_profile_read(h)
    finally:
        db.bin_finalize(h)
        for a in handles:
            db.bin_array_release(a)
    return out


def _per_attr_ops(ops, nattr):
    if nattr and isinstance(ops, list) and len(ops) == nattr and not isinstance(ops[0], str):
        return ops
    return [ops] * nattr


def compare(out, ref, ops=ALL_OPS, exact=False, nattr=None):
    """Asserts GPU output `out` matches oracle `ref` under the parity bar."""
    nattr = len(ref["sum"]) if nattr is None else nattr
    assert out["n_in"] == ref["n_in"], (out["n_in"], ref["n_in"])
    assert out["n_out"] == ref["n_out"], (out["n_out"], ref["n_out"])
    assert np.array_equal(out["count"], ref["count"]), f"count mismatch at {np.flatnonzero(out['count'] != ref['count'])[:10]}"
    cnt = ref["count"]
    occ = cnt > 0
    for a, aops in enumerate(_per_attr_ops(ops, nattr)):
        for k in ("min", "max"):
            if k in aops:
                assert np.array_equal(bits(out[k][a]), bits(ref[k][a])), \
                    f"{k}[{a}] mismatch at {np.flatnonzero(bits(out[k][a]) != bits(ref[k][a]))[:10]}"
            else:
                assert out[k][a] is None
        if "sum" in aops:
            s, r = out["sum"][a], ref["sum"][a]
            if exact:
                assert np.array_equal(bits(s), bits(r)), f"sum[{a}] not bit-exact at {np.flatnonzero(bits(s) != bits(r))[:10]}"
            else:
                assert np.array_equal(bits(s[~occ]), bits(r[~occ]))          # empty bins: +0.0
                err = np.abs(s - r)
                lim = 1e-12 * ref["sumabs"][a]
                bad = np.flatnonzero(err > lim)
                assert bad.size == 0, f"sum[{a}] off at bins {bad[:10]}: {err[bad[:3]]} > {lim[bad[:3]]}"
        else:
            assert out["sum"][a] is None
        if "avg" in aops:
            g, r = out["avg"][a], ref["avg"][a]
            assert np.all(np.isnan(g[~occ])) and np.all(np.isnan(r[~occ]))
            if exact:
                assert np.array_equal(bits(g[occ]), bits(r[occ]))
            else:
                lim = 1e-12 * ref["sumabs"][a][occ] / cnt[occ] + 2 * np.spacing(np.abs(r[occ]))
                assert np.all(np.abs(g[occ] - r[occ]) <= lim)
        else:
            assert out["avg"][a] is None


def workload_inputs(w, n=None, start=0):
    """Host-generated columns of a synth workload (independent of the CUDA path)."""
    import synth
    n = w.n if n is None else n
    axes = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], start, n) for c in w.axes]
    attrs = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], start, n) for c in w.attrs]
    return axes, attrs
