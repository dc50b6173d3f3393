"""GPU tests of view resolution and placement (§8 row a1; PAPER.md:346-389,
:406-435, :490-505): lockstep on the producer's stream, asynchronous side
stream with snapshot (the paper's deep copy) and with in-place reads guarded
by the inputs-released event, host (pageable / pinned) and managed inputs,
analysis on another GPU fed over NVLink, and the zero-copy discipline.  Every
result is compared with the oracle."""
import ctypes
import glob
import os

import numpy as np
import pytest

import oracle
from tests.gpu_util import compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu(cuda_available):
    if not cuda_available:
        pytest.fail("GPU tests need a CUDA device")


def _cudart():
    import nvidia.cuda_runtime as cr
    libs = glob.glob(os.path.join(list(cr.__path__)[0], "lib", "libcudart.so*"))
    lib = ctypes.CDLL(sorted(libs)[0])
    lib.cudaStreamWaitEvent.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint]
    return lib


def _data(n=400_003, seed=7):
    rng = np.random.default_rng(seed)
    return [rng.standard_normal(n) * 4, rng.standard_normal(n) * 4], [rng.uniform(0.5, 1.5, n)]


RES, LO, HI = (128, 128), (-16.0, -16.0), (16.0, 16.0)


def _execute(db, handles, placement, nattr=1):
    spec = db.make_spec(RES, LO, HI, nattr=nattr)
    h = db.bin_init(spec, placement)
    t = db.bin_execute(h, handles[:2], handles[2:])
    return h, t, spec


def test_lockstep_runs_on_the_producer_stream(db):
    import torch
    axes, attrs = _data()
    ref = oracle.databin(axes, attrs, RES, LO, HI)
    s = torch.cuda.Stream()
    ts = [torch.from_numpy(c).cuda() for c in axes + attrs]
    torch.cuda.synchronize()
    hs = [db.wrap_tensor(t, stream=s.cuda_stream) for t in ts]
    h, t, spec = _execute(db, hs, db.make_placement(device_id=0, exec=db.BIN_EXEC_SYNC))
    assert db.bin_stream(h) == s.cuda_stream                       # ordered with the producer's work
    compare(db.result_to_numpy(h, t, spec), ref)
    db.bin_finalize(h)
    for a in hs:
        db.bin_array_release(a)


@pytest.mark.parametrize("snapshot", [1, 0])
def test_async_side_stream_inputs_released(db, snapshot):
    """The producer overwrites its arrays as soon as bin_inputs_released fires;
    with the snapshot that is right after the copy, in place it
    is after the binning kernel -- either way the result is the original data's."""
    import torch
    cudart = _cudart()
    axes, attrs = _data(seed=11)
    ref = oracle.databin(axes, attrs, RES, LO, HI)
    prod = torch.cuda.Stream()
    ts = [torch.from_numpy(c).cuda() for c in axes + attrs]
    torch.cuda.synchronize()
    hs = [db.wrap_tensor(t, stream=prod.cuda_stream) for t in ts]
    h, t, spec = _execute(db, hs, db.make_placement(device_id=0, exec=db.BIN_EXEC_ASYNC, async_snapshot=snapshot))
    assert db.bin_stream(h) != prod.cuda_stream                    # a side stream
    ev = db.bin_inputs_released(h, t)
    assert cudart.cudaStreamWaitEvent(ctypes.c_void_p(prod.cuda_stream), ctypes.c_void_p(ev), 0) == 0
    with torch.cuda.stream(prod):                                  # the "solver" moves on
        for x in ts:
            x.fill_(1e300)
    compare(db.result_to_numpy(h, t, spec), ref)
    db.bin_finalize(h)
    for a in hs:
        db.bin_array_release(a)


@pytest.mark.parametrize("pinned", [False, True])
def test_host_inputs_are_staged(db, pinned):
    import torch
    axes, attrs = _data(seed=13)
    ref = oracle.databin(axes, attrs, RES, LO, HI)
    ts = [torch.from_numpy(c) for c in axes + attrs]
    if pinned:
        ts = [t.pin_memory() for t in ts]
    hs = [db.wrap_tensor(t, mode=db.BIN_SYNC) for t in ts]
    h, t, spec = _execute(db, hs, db.make_placement(device_id=0))
    compare(db.result_to_numpy(h, t, spec), ref)
    db.bin_finalize(h)
    for a in hs:
        db.bin_array_release(a)


def test_managed_inputs_read_in_place(db):
    axes, attrs = _data(seed=17)
    ref = oracle.databin(axes, attrs, RES, LO, HI)
    hs = []
    for c in axes + attrs:
        a = db.bin_array_alloc(len(c), 0, db.BIN_ALLOC_CUDA_UVA)
        db.bin_copy(db.bin_array_data(a), c.ctypes.data, c.nbytes)
        hs.append(a)
    before = db.bin_alloc_stats()
    h, t, spec = _execute(db, hs, db.make_placement(device_id=0))
    compare(db.result_to_numpy(h, t, spec), ref)
    db.bin_finalize(h)
    assert db.bin_alloc_stats()["live"] == before["live"]          # nothing staged
    for a in hs:
        db.bin_array_release(a)


def test_zero_copy_device_inputs_allocate_nothing_per_execute(db):
    """zero-copy wrap + same-device access performs no allocation."""
    import torch
    axes, attrs = _data(seed=19)
    ref = oracle.databin(axes, attrs, RES, LO, HI)
    ts = [torch.from_numpy(c).cuda() for c in axes + attrs]
    torch.cuda.synchronize()
    before = db.bin_alloc_stats()
    hs = [db.wrap_tensor(t) for t in ts]
    assert db.bin_alloc_stats() == before                          # wrap: no allocation
    spec = db.make_spec(RES, LO, HI, nattr=1)
    h = db.bin_init(spec, db.make_placement(device_id=0))
    after_init = db.bin_alloc_stats()
    for _ in range(3):
        t = db.bin_execute(h, hs[:2], hs[2:])
    assert db.bin_alloc_stats() == after_init                      # executes: no allocation
    compare(db.result_to_numpy(h, t, spec), ref)
    db.bin_finalize(h)
    for a in hs:
        db.bin_array_release(a)
    assert db.bin_alloc_stats()["live"] == before["live"]


def test_device_array_host_view_and_release_callback(db):
    """get_accessible D->H temporary is freed with the view; the wrap's release
    callback fires once, after in-flight library work (Listing 1 contract)."""
    import torch
    x = torch.arange(1000, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    fired = []
    cb = db.RELEASE_FN(lambda ctx, ptr: fired.append(ptr))
    a = db.bin_array_wrap(x.data_ptr(), 1000, 0, db.BIN_ALLOC_EXTERNAL, 0, db.BIN_SYNC, cb, 0)
    before = db.bin_alloc_stats()
    p, v = db.bin_array_get_accessible(a, -1)
    assert p != x.data_ptr() and db.bin_alloc_stats()["live"] == before["live"] + 1
    host = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(1000,))
    assert host.tolist() == list(range(1000))
    db.bin_array_release(v)
    assert db.bin_alloc_stats()["live"] == before["live"] and fired == []
    db.bin_array_release(a)
    assert fired == [x.data_ptr()]


def test_peer_placement_over_nvlink(db):
    """the analysis runs on another GPU; inputs move by peer copy."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs (gpurun --gpus 2)")
    axes, attrs = _data(seed=23)
    ref = oracle.databin(axes, attrs, RES, LO, HI)
    ts = [torch.from_numpy(c).to("cuda:0") for c in axes + attrs]
    torch.cuda.synchronize()
    hs = [db.wrap_tensor(t) for t in ts]
    h, t, spec = _execute(db, hs, db.make_placement(device_id=1, exec=db.BIN_EXEC_PEER))
    out = db.result_to_numpy(h, t, spec)
    assert out["device"] == 1
    compare(out, ref)
    p, v = db.bin_array_get_accessible(hs[0], 1)                   # peer view: temporary on GPU 1
    assert p != ts[0].data_ptr()
    db.bin_array_synchronize(v)
    back = torch.empty(len(axes[0]), dtype=torch.float64)
    db.bin_copy(back.data_ptr(), p, back.numel() * 8)
    assert np.array_equal(back.numpy(), axes[0])
    db.bin_array_release(v)
    db.bin_finalize(h)
    for a in hs:
        db.bin_array_release(a)
