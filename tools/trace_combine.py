#!/usr/bin/env python
"""Per-execute phase trace of the NVLink peer combine (DATABIN_TRACE) on C3
shards -- torchrun, diagnosis only.  ITERS executes, every other one waited."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["DATABIN_TRACE"] = "1"


def main():
    import torch
    import torch.distributed as dist

    import paper_2310_02926_b200 as db
    import synth
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    w = synth.CONFIGS[os.environ.get("WL", "c3")]
    n = w.n // world
    cols = []
    for c in list(w.axes) + list(w.attrs):
        t = torch.empty(n, dtype=torch.float64, device=dev)
        synth.fill_device(w.dist, w.central, w.seed, synth.COLUMNS[c], rank * n, n, t.data_ptr(), 0)
        cols.append(t)
    torch.cuda.synchronize()
    obj = [db.bin_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    spec = db.make_spec(w.res, w.lo, w.hi, nattr=len(w.attrs))
    h = db.bin_init(spec, db.make_placement(), rank=rank, nranks=world, nccl_id=obj[0])
    hs = [db.wrap_tensor(t) for t in cols]
    D = len(w.axes)
    for it in range(int(os.environ.get("ITERS", "8"))):
        t = db.bin_execute(h, hs[:D], hs[D:])
        if it % 2 == 1:
            db.bin_wait(h, t)
    db.bin_wait(h, t)
    db.bin_finalize(h)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
