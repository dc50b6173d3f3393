"""Multi-rank host logic on CPU (gloo, world_size 2): the row sharding used by
bench.py / tools/mgpu_check.py and the cross-rank combine semantics of
PAPER.md:479 -- counts add, min/max fold, sums either all-reduced (atomic
mode, within tolerance) or gathered and folded in rank order (deterministic
mode, bit-identical to the oracle's partition mode P = world)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [0, 1, 7, 1000, 100_000_001])
def test_shards_partition_the_rows(world, n):
    cuts = [bench.shard(n, r, world) for r in range(world)]
    assert cuts[0][0] == 0 and cuts[-1][1] == n
    for (a0, a1), (b0, b1) in zip(cuts, cuts[1:]):
        assert a1 == b0 and a0 <= a1
    sizes = [b - a for a, b in cuts]
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        w = synth.CONFIGS["c3"]
        n = 200_001
        r0, r1 = bench.shard(n, rank, world)
        axes = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], r0, r1 - r0) for c in w.axes]
        attrs = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], r0, r1 - r0) for c in w.attrs]
        part = oracle.databin(axes, attrs, (64, 64), (-4, -4), (4, 4))
        cnt = torch.from_numpy(part["count"].astype(np.int64))
        mn = torch.from_numpy(part["min"][0].copy())
        mx = torch.from_numpy(part["max"][0].copy())
        sm = torch.from_numpy(part["sum"][0].copy())
        dist.all_reduce(cnt)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        gathered = [torch.zeros_like(sm) for _ in range(world)]
        dist.all_gather(gathered, sm)
        folded = torch.zeros_like(sm)
        for g in gathered:          # rank order, from +0.0
            folded = folded + g
        s_all = sm.clone()
        dist.all_reduce(s_all)
        # the unique-id broadcast bench.py uses for the library's NCCL communicator
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        if rank == 0:
            full_axes = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, n) for c in w.axes]
            full_attrs = [synth.fill_host(w.dist, w.central, w.seed, synth.COLUMNS[c], 0, n) for c in w.attrs]
            refP = oracle.databin(full_axes, full_attrs, (64, 64), (-4, -4), (4, 4), P=world)
            ref1 = oracle.databin(full_axes, full_attrs, (64, 64), (-4, -4), (4, 4), P=1)
            assert np.array_equal(cnt.numpy().astype(np.uint64), ref1["count"])
            assert np.array_equal(mn.numpy(), ref1["min"][0]) and np.array_equal(mx.numpy(), ref1["max"][0])
            assert np.array_equal(folded.numpy().view(np.uint64), refP["sum"][0].view(np.uint64))
            assert np.all(np.abs(s_all.numpy() - ref1["sum"][0]) <= 1e-12 * ref1["sumabs"][0])
            assert obj[0] == bytes(range(128))
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))


@pytest.mark.parametrize("world", [2])
def test_gloo_combine_matches_oracle_partition_mode(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(results) == [(r, "ok") for r in range(world)], results
