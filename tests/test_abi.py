"""C-ABI checks that need no GPU (-m "not gpu"): the library builds/loads,
exports every symbol include/databin.h declares, and its host-only logic
(Eq. (1) placement, argument validation, the array handle's host paths and
release-once contract) behaves as documented."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "databin.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bin_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported(db):
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(db._lib, n), n
    assert set(names) == set(db.EXPORTED)


def test_library_is_in_tree_and_sm100a(db):
    path = db.capi._build.LIB
    assert os.path.dirname(path).endswith("paper_2310_02926_b200")
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version(db):
    assert "sm_100a" in db.bin_version()


def test_eq1_matches_oracle_exhaustive(db):
    # SPEC.md:523 acceptance 1, against the independent oracle implementation
    for n_a in (1, 2, 4, 8):
        for n_u in range(1, n_a + 1):
            for s in (1, 2, 3):
                for d0 in range(n_a):
                    p = db.make_placement(device_id=db.BIN_DEVICE_AUTO, device_start=d0, device_stride=s,
                                          devices_to_use=n_u)
                    for r in range(64):
                        assert db.bin_resolve_device(p, r, n_a) == oracle.eq1_device(r, n_u, s, d0, n_a)


def test_eq1_defaults_and_overrides(db):
    p = db.bin_placement_default()
    assert (p.device_id, p.device_start, p.device_stride, p.devices_to_use) == (-2, 0, 1, 0)
    assert [db.bin_resolve_device(p, r, 4) for r in range(8)] == [0, 1, 2, 3, 0, 1, 2, 3]
    p.device_id = 2
    assert db.bin_resolve_device(p, 7, 4) == 2
    p.device_id = 5                                       # explicit ids wrap modulo n_a (R14b)
    assert [db.bin_resolve_device(p, r, 4) for r in range(3)] == [1, 1, 1]
    assert db.bin_resolve_device(p, 0, 5) == 0 and db.bin_resolve_device(p, 0, 6) == 5
    p.device_id = -3
    with pytest.raises(db.BinError) as e:
        db.bin_resolve_device(p, 0, 4)
    assert e.value.code == db.capi.BIN_EDEVICE
    p.device_id = db.BIN_DEVICE_HOST
    with pytest.raises(db.BinError) as e:
        db.bin_resolve_device(p, 0, 4)
    assert e.value.code == db.capi.BIN_ENOTSUP          # no CPU fallback, by design


def test_spec_validation_without_gpu(db, cuda_available):
    if cuda_available:
        pytest.skip("validation-order check is for the CPU box")
    bad = [db.make_spec([0, 4], [0, 0], [1, 1]),            # res < 1
           db.make_spec([4, 4], [0, 1], [1, 1]),            # lo >= hi
           db.make_spec([70000, 70000], [0, 0], [1, 1])]    # prod(res) >= 2^32
    for s in bad:
        with pytest.raises(db.BinError) as e:
            db.bin_init(s)
        assert e.value.code == db.capi.BIN_EINVAL
    s = db.make_spec([4, 4, 4], [0, 0, 0], [1, 1, 1])
    s.ndim = 4
    with pytest.raises(db.BinError) as e:
        db.bin_init(s)
    assert e.value.code == db.capi.BIN_ENOTSUP
    with pytest.raises(db.BinError) as e:   # valid spec, but no device here
        db.bin_init(db.make_spec([4], [0], [1]))
    assert e.value.code == db.capi.BIN_EDEVICE


def test_host_array_wrap_is_zero_copy_and_release_once(db):
    x = np.arange(10, dtype=np.float64)
    fired = []
    cb = db.RELEASE_FN(lambda ctx, ptr: fired.append((ctx, ptr)))
    before = db.bin_alloc_stats()
    a = db.bin_array_wrap(x.ctypes.data, 10, -1, db.BIN_ALLOC_HOST, 0, db.BIN_SYNC, cb, 1234)
    assert db.bin_alloc_stats() == before                       # wrap allocates nothing
    assert db.bin_array_data(a) == x.ctypes.data
    info = db.bin_array_info(a)
    assert (info["n"], info["device"], info["alloc"]) == (10, -1, db.BIN_ALLOC_HOST)
    p, v = db.bin_array_get_accessible(a, -1)                   # host view of host data: direct
    assert p == x.ctypes.data and db.bin_alloc_stats() == before
    db.bin_array_release(a)
    assert fired == []                                          # the view still holds it
    db.bin_array_release(v)
    assert fired == [(1234, x.ctypes.data)]
    assert db.bin_alloc_stats()["live"] == before["live"]


def test_release_once_random_interleavings(db):
    # release fires exactly once over random release orders
    rng = np.random.default_rng(0)
    x = np.zeros(4)
    for _ in range(1000):
        fired = []
        cb = db.RELEASE_FN(lambda ctx, ptr: fired.append(1))
        a = db.bin_array_wrap(x.ctypes.data, 4, -1, db.BIN_ALLOC_HOST, 0, db.BIN_SYNC, cb, 0)
        hs = [a] + [db.bin_array_get_accessible(a, -1)[1] for _ in range(int(rng.integers(0, 4)))]
        for i in rng.permutation(len(hs)):
            assert fired == []
            db.bin_array_release(hs[i])
        assert fired == [1]


def test_host_allocating_constructor(db):
    before = db.bin_alloc_stats()
    a = db.bin_array_alloc(5, -1, db.BIN_ALLOC_HOST, fill=1.0)
    assert db.bin_alloc_stats()["live"] == before["live"] + 1
    p = db.bin_array_data(a)
    vals = np.ctypeslib.as_array(ctypes.cast(p, ctypes.POINTER(ctypes.c_double)), shape=(5,))
    assert vals.tolist() == [1.0] * 5                           # Listing 2, "initialized to 1"
    db.bin_array_release(a)
    assert db.bin_alloc_stats()["live"] == before["live"]


def test_wrap_argument_errors(db):
    with pytest.raises(db.BinError) as e:
        db.bin_array_wrap(0, 5, -1, db.BIN_ALLOC_HOST)
    assert e.value.code == db.capi.BIN_EINVAL
    x = np.zeros(3)
    with pytest.raises(db.BinError) as e:
        db.bin_array_wrap(x.ctypes.data, 3, -1, db.BIN_ALLOC_HOST, dtype=7)
    assert e.value.code == db.capi.BIN_EDTYPE
