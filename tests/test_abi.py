"""CPU-side checks of the C-ABI boundary: the library loads without a GPU,
exports every symbol include/knng.h declares, and rejects bad arguments on
the host before touching CUDA (no compute calls here)."""
import os
import re

import pytest

import paper_2103_15386_b200.knng as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "knng.h")).read()
    hdr = re.sub(r"/\*.*?\*/", "", hdr, flags=re.S)
    return sorted(set(re.findall(r"\b(knng_[a-z_0-9]+)\s*\(", hdr)))


def test_library_loads_and_exports_every_declared_symbol():
    L = K.lib()
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    bound = {n for n, _, _ in K.SIGNATURES}
    assert set(declared) == bound, set(declared) ^ bound


def test_abi_version_and_status_strings():
    assert K.knng_abi_version() == 2
    L = K.lib()
    assert L.knng_status_string(0) == b"KNNG_OK"
    assert L.knng_status_string(1) == b"KNNG_E_USAGE"


@pytest.mark.parametrize("n,d,k,p,iters,msg", [
    (100, 8, 1, 1, 4, "k must be"),
    (100, 8, 33, 4, 4, "k must be"),
    (100, 8, 10, 10, 4, "sample_size"),
    (100, 8, 10, 0, 4, "sample_size"),
    (100, 8, 32, 17, 4, "<= 16"),
    (10, 8, 10, 4, 4, "n must exceed k"),
    (100, 0, 10, 4, 4, "d must be"),
    (100, 8, 10, 4, 0, "iters"),
    (100, 8, 10, 4, 300, "iters"),
])
def test_build_usage_errors_before_any_cuda_call(n, d, k, p, iters, msg):
    L = K.lib()
    st = L.knng_build(None, K.KNNG_F32, n, d, k, K.KNNG_L2SQ, iters, p, 0, None, None, None, 0, None)
    assert st == K.KNNG_E_USAGE
    assert msg in K.knng_last_error()


def test_cosine_requires_f32_and_unknown_enums():
    L = K.lib()
    assert L.knng_build(None, K.KNNG_U8, 100, 8, 10, K.KNNG_COSINE, 4, 4, 0, None, None, None, 0, None) == 1
    assert "cosine" in K.knng_last_error()
    assert L.knng_build(None, 7, 100, 8, 10, 0, 4, 4, 0, None, None, None, 0, None) == 1
    assert L.knng_build(None, 0, 100, 8, 10, 9, 4, 4, 0, None, None, None, 0, None) == 1


def test_host_pointers_rejected_as_device_arguments():
    import numpy as np
    x = np.zeros((100, 8), np.float32)
    ids = np.zeros((100, 10), np.uint32)
    L = K.lib()
    st = L.knng_build(x.ctypes.data, 0, 100, 8, 10, 0, 4, 4, 0, ids.ctypes.data, ids.ctypes.data, None, 0, None)
    assert st == K.KNNG_E_USAGE


def test_workspace_size_query():
    assert K.knng_build_workspace_bytes(0, 100, 8, 1, 1) == 0  # invalid -> 0
    small = K.knng_build_workspace_bytes(0, 10_000, 16, 10, 8)
    big = K.knng_build_workspace_bytes(0, 1_000_000, 128, 32, 16)
    assert 0 < small < big
    # C2 (SIFT1M shape) fits easily in 180 GB: ~2.2 GB of graph state
    assert big < 3 << 30
    cos = K.knng_build_workspace_bytes(0, 1_000_000, 128, 32, 16, "cosine")
    # cosine: +normalised f32 copy of the rows; L2 f32: +exact u8 copy
    assert cos - big >= 1_000_000 * 128 * 3
    L = K.lib()
    assert L.knng_merge_workspace_bytes(0, 5000, 5000, 16, 10, 8, 0) > K.knng_build_workspace_bytes(0, 10_000, 16, 10, 8)


def test_merge_and_bruteforce_usage_errors():
    L = K.lib()
    # nB < floor(k/2)
    st = L.knng_merge(None, 100, None, None, None, 3, None, None, 0, 8, 10, 0, 4, 4, 0, 0, None, None, None, 0, None)
    assert st == K.KNNG_E_USAGE
    st = L.knng_bruteforce(None, 0, 100, 8, 0, None, 10, 40, None, None, None)
    assert st == K.KNNG_E_USAGE


def test_launch_counter_and_timing_api_without_gpu():
    assert K.knng_launch_count() >= 0
    K.knng_set_timing(True)
    K.knng_reset_timing()
    assert K.knng_kernel_time("k_join") == (0.0, 0)
    K.knng_set_timing(False)


def test_iter_stats_struct_matches_header():
    hdr = open(os.path.join(ROOT, "include", "knng.h")).read()
    body = hdr[hdr.index("typedef struct {"):hdr.index("} knng_iter_stats;")]
    body = re.sub(r"/\*.*?\*/", "", body, flags=re.S)
    fields = re.findall(r"int64_t\s+(\w+);", body)
    assert fields == [f for f, _ in K.IterStats._fields_]
