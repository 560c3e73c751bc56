"""CPU-side checks of the boundary: libddks.so builds, loads, and exports every symbol include/ddks.h declares;
host-only helpers behave; no compute calls (no GPU here)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "ddks.h")).read()
    return sorted(set(re.findall(r"DDKS_API\s+[\w\s\*]+?\b(ddks_\w+)\s*\(", hdr)))


@pytest.fixture(scope="module")
def lib():
    from paper_2106_13706_b200 import build
    build.build()
    from paper_2106_13706_b200 import ddks
    return ddks


def test_header_declares_the_north_star_calls():
    syms = _declared_symbols()
    for s in ("ddks_create", "ddks_stat", "ddks_stat_batch", "ddks_permutation_null", "ddks_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    so = lib.LIB_PATH
    out = subprocess.check_output(["nm", "-D", "--defined-only", so]).decode()
    exported = set(re.findall(r"\bT (ddks_\w+)", out))
    declared = set(_declared_symbols())
    assert declared <= exported, declared - exported
    assert declared == set(lib.EXPORTED)
    cdll = ctypes.CDLL(so)
    for s in declared:
        assert hasattr(cdll, s)


def test_library_is_sm100a_and_uses_bulk_copy(lib):
    sass = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "-sass", lib.LIB_PATH]).decode()
    assert "arch = sm_100a" in sass
    assert "UBLKCP" in sass            # cp.async.bulk (TMA bulk engine) staging of point tiles
    assert "FSET.BF.GE" in sass        # the FP32 compare of the orthant classification
    assert "ATOMS" in sass             # SMEM orthant counters


def test_shard_range_partitions(lib):
    for total in (0, 1, 7, 100, 2_000_000):
        for world in (1, 2, 3, 8):
            prev = 0
            sizes = []
            for r in range(world):
                b, e = lib.ddks_shard_range(total, world, r)
                assert b == prev and e >= b
                prev = e
                sizes.append(e - b)
            assert prev == total and max(sizes) - min(sizes) <= 1
    with pytest.raises(lib.DDKSError):
        lib.ddks_shard_range(10, 2, 2)


def test_version_and_create_without_gpu(lib):
    assert lib.ddks_version().endswith("sm100a")
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    with pytest.raises(lib.DDKSError) as e:
        lib.ddks_create()
    assert e.value.status == 6  # DDKS_ERR_CUDA: fails loudly, no CPU fallback
    with pytest.raises(lib.DDKSError) as e:
        lib.ddks_create(world=2, rank=0, nccl_id=None)
    assert e.value.status == 1


def test_null_context_is_an_argument_error_not_a_crash(lib):
    # every compute entry point rejects a NULL context with DDKS_ERR_INVALID_ARGUMENT before touching the device
    L, NULL = lib.LIB, None
    assert L.ddks_stat(NULL, NULL, 1, NULL, 1, 2, NULL, NULL) == 1
    assert L.ddks_stat_batch(NULL, NULL, NULL, 1, 1, 1, 2, NULL, NULL) == 1
    assert L.ddks_permutation_null(NULL, NULL, 1, 1, 2, NULL, 0, NULL, NULL, NULL, NULL) == 1
    assert L.ddks_stat_per_origin(NULL, NULL, 1, NULL, 1, 2, 0, 1, NULL, NULL) == 1
    assert L.ddks_significance(NULL, NULL, 1, NULL, 1, 2, 0, NULL, NULL, NULL, NULL) == 1
    assert L.ddks_significance_batch(NULL, NULL, NULL, 1, 1, 1, 2, 0, NULL, NULL) == 1
    assert L.ddks_vdks(NULL, NULL, 1, NULL, 1, 2, 4, NULL, NULL) == 1
    assert L.ddks_rdks(NULL, NULL, 1, NULL, 1, 2, NULL, NULL) == 1
    assert L.ddks_profile_read(NULL, NULL, NULL, NULL) == 1
    assert L.ddks_destroy(NULL) == 0 and L.ddks_launch_count(NULL) == 0


def test_binding_argument_checks(lib):
    # every wrapper checks shapes before the C call (a Q with fewer columns than P would be over-read), and a
    # float64 input is cast to the library's float32 with a warning (the cast can merge distinct values into ties)
    import numpy as np
    import warnings
    P = np.zeros((5, 3), np.float32)
    Q = np.zeros((4, 2), np.float32)
    for fn in (lambda: lib.ddks_stat_shard(None, P, Q, 2, 0), lambda: lib.ddks_stat_per_origin(None, P, Q, 0, 1),
               lambda: lib.ddks_stat(None, P, Q), lambda: lib.ddks_vdks(None, P, Q, 4)):
        with pytest.raises(ValueError):
            fn()
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        a = lib._Arg(np.zeros((3, 2), np.float64), np.float32)
        assert a.keep.dtype == np.float32 and any("float64" in str(x.message) for x in w)


def test_host_combine_helpers(lib):
    # the host steps after the single all-gather (include/ddks.h): max num, smallest argmax among the ranks attaining
    # it (records without origins carry -1), OR of the flags; padded per-rank item records unpadded in rank order
    assert lib.ddks_combine_records([(5, 10, 0), (7, 3, 1), (7, 2, 0), (0, -1, 0)]) == (7, 2, 1)
    assert lib.ddks_combine_records([(0, -1, 0), (0, 4, 2)]) == (0, 4, 2)
    import numpy as np
    total, world = 5, 3  # shards 2, 2, 1; chunk 2; stride 2 * 2 + 1
    g = np.array([1, 2, 11, 12, 0,   3, 4, 13, 14, 4,   5, 99, 15, 99, 1], np.uint64)
    out, flags = lib.ddks_unpad_items(g, total, world, 2)
    assert out[0].tolist() == [1, 2, 3, 4, 5] and out[1].tolist() == [11, 12, 13, 14, 15] and flags == 5
    assert lib.gather_stride(total, world, 2) == 5
