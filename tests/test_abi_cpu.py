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
