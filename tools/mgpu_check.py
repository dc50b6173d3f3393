#!/usr/bin/env python
"""Multi-GPU parity check (launch with torchrun, one process per GPU).

Each rank generates its contiguous row shard of a seeded workload on its own
GPU, bins it through the C ABI with the NCCL cross-rank combine,
and rank 0 compares the combined result with the CPU oracle:
  atomic mode        -> oracle P=1 under the parity bar (counts/min/max exact)
  deterministic mode -> oracle partition mode P=world, bit-exact
Prints one JSON line per case on rank 0; exits non-zero on any mismatch.

  torchrun --standalone --nproc-per-node 2 tools/mgpu_check.py [--rows N]
"""
import argparse
import json
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=3_000_001)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2310_02926_b200 as db
    import synth
    from tests.gpu_util import compare

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    ok = True
    cases = [
        ("plummer_2d_512", synth.CONFIGS["c3"], args.rows, False),
        ("uniform_2d_256_4attr", synth.CONFIGS["c2"], args.rows // 2, False),
        ("uniform_3d_64", synth.CONFIGS["c4"], args.rows // 2, False),
        ("plummer_2d_auto_bounds", synth.CONFIGS["c3"], args.rows // 3, True),
    ]
    for name, w, n, auto in cases:
        res = w.res if name != "uniform_3d_64" else (64, 64, 64)
        r0, r1 = (rank * n) // world, ((rank + 1) * n) // world
        cols = []
        for c in list(w.axes) + list(w.attrs):
            t = torch.empty(r1 - r0, dtype=torch.float64, device=dev)
            synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], r0, r1 - r0, t.data_ptr(),
                              torch.cuda.current_stream(dev).cuda_stream)
            cols.append(t)
        torch.cuda.synchronize(dev)
        hs = [db.wrap_tensor(t) for t in cols]
        D = len(w.axes)
        for det, route, exact in ((False, "auto", False), (False, "window", False), (False, "partition", False),
                                  (True, "auto", False), (False, "auto", True), (False, "partition", True)):
            obj = [db.bin_nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            spec = db.make_spec(res, None if auto else w.lo, None if auto else w.hi, nattr=len(w.attrs),
                                ops=w.ops, bounds_auto=auto, deterministic=det, route=route, exact=exact)
            h = db.bin_init(spec, db.make_placement(), rank=rank, nranks=world, nccl_id=obj[0])
            db.bin_profile_enable(h, True)
            t = db.bin_execute(h, hs[:D], hs[D:])
            out = db.result_to_numpy(h, t, spec)
            variant = db.bin_profile_read(h).variant
            db.bin_finalize(h)
            if rank == 0:
                import oracle
                axes = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, n) for c in w.axes]
                attrs = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, n) for c in w.attrs]
                ref = oracle.databin(axes, attrs, res, None if auto else w.lo, None if auto else w.hi,
                                     bounds_auto=auto, P=world if det else 1, exact=exact)
                status = "ok"
                try:
                    compare(out, ref, w.ops, exact=det)
                    if exact:  # exact sums: bit-identical to the once-rounded exact sum for any rank count
                        for a in range(len(w.attrs)):
                            assert np.array_equal(out["sum"][a].view(np.uint64), ref["sum_exact"][a].view(np.uint64))
                            occ = ref["count"] > 0
                            assert np.array_equal(out["avg"][a][occ].view(np.uint64),
                                                  ref["avg_exact"][a][occ].view(np.uint64))
                    if auto:
                        assert np.array_equal(out["lo"], ref["lo"]) and np.array_equal(out["hi"], ref["hi"])
                except AssertionError as e:  # noqa: PERF203
                    status = "FAIL: " + str(e)[:300]
                    ok = False
                print(json.dumps({"case": name, "deterministic": det, "exact": exact, "route": route, "variant": variant,
                                  "world": world, "rows": n,
                                  "res": list(res), "status": status, "n_in": out["n_in"],
                                  "n_out": out["n_out"]}), flush=True)
            dist.barrier()
        for a in hs:
            db.bin_array_release(a)
    # fused multi-instance set (bin_multi_*): the paper-step shape (R19) plus an
    # auto-bounded instance, combined across ranks by the grouped NCCL allreduces
    n = args.rows // 3
    r0, r1 = (rank * n) // world, ((rank + 1) * n) // world
    cols = []
    for c in range(7):
        t = torch.empty(r1 - r0, dtype=torch.float64, device=dev)
        synth.fill_device(synth.UNIFORM, 1, 6, c, r0, r1 - r0, t.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
        cols.append(t)
    torch.cuda.synchronize(dev)
    hs = [db.wrap_tensor(t) for t in cols]
    systems = [(0, 1), (0, 2), (1, 2), (4, 5), (4, 6), (5, 6), (0, 4), (1, 5), (2, 6)]
    insts = [dict(res=(64, 64), lo=(-1.0, -1.0), hi=(1.0, 1.0), axes=sy, attrs=tuple(range(7)), auto=False)
             for sy in systems] + [dict(res=(50,), axes=(3,), attrs=(4, 5), auto=True)]
    specs = [db.make_spec(d["res"], None if d["auto"] else d["lo"], None if d["auto"] else d["hi"],
                          nattr=len(d["attrs"]), bounds_auto=d["auto"], exact=d["auto"]) for d in insts]
    obj = [db.bin_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    m = db.bin_multi_init([db.make_multi_op(sp, d["axes"], d["attrs"]) for sp, d in zip(specs, insts)], 7,
                          db.make_placement(), rank=rank, nranks=world, nccl_id=obj[0])
    t = db.bin_multi_execute(m, hs)
    outs = [db.result_to_numpy(m, t, sp, op=k) for k, sp in enumerate(specs)]
    db.bin_multi_finalize(m)
    if rank == 0:
        import oracle
        host = [synth.fill_host(synth.UNIFORM, 1, 6, c, 0, n) for c in range(7)]
        for k, (d, out) in enumerate(zip(insts, outs)):
            ref = oracle.databin([host[i] for i in d["axes"]], [host[i] for i in d["attrs"]], d["res"],
                                 None if d["auto"] else d["lo"], None if d["auto"] else d["hi"], bounds_auto=d["auto"],
                                 exact=True)
            status = "ok"
            try:
                compare(out, ref)
                if d["auto"]:  # the exact instance: once-rounded exact sums across ranks
                    for a in range(len(d["attrs"])):
                        assert np.array_equal(out["sum"][a].view(np.uint64), ref["sum_exact"][a].view(np.uint64))
                if d["auto"]:
                    assert np.array_equal(out["lo"], ref["lo"]) and np.array_equal(out["hi"], ref["hi"])
            except AssertionError as e:  # noqa: PERF203
                status = "FAIL: " + str(e)[:300]
                ok = False
            print(json.dumps({"case": f"multi_instance_{k}", "axes": list(d["axes"]), "world": world, "rows": n,
                              "res": list(d["res"]), "status": status, "n_in": out["n_in"],
                              "n_out": out["n_out"]}), flush=True)
    dist.barrier()
    for a in hs:
        db.bin_array_release(a)
    flag = torch.tensor([0 if ok else 1], device=dev)
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    try:
        main()
    except Exception:
        traceback.print_exc()
        sys.exit(2)
