"""The C-ABI library loads, exports every symbol include/quick.h declares, and its host-side
argument validation returns the documented status codes (no compute calls without a GPU)."""
import ctypes
import os
import re

import pytest

from _helpers import ROOT

quick = pytest.importorskip("paper_2402_10076_b200.quick")


def declared_functions():
    src = open(os.path.join(ROOT, "include", "quick.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(quick_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for required in ("quick_pack_weights", "quick_w4a16_gemm", "quick_unpack_weights", "quick_packed_bytes"):
        assert required in names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(quick.LIB_PATH)
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_layout_version_and_sizes():
    assert quick.quick_layout_version() == 1
    assert quick.quick_packed_bytes(4096, 4096, 128) == 4096 * 4096 // 2 + 32 * 4096 * 5 // 2
    assert quick.quick_packed_bytes(8192, 28672, 128) == 8192 * 28672 // 2 + 64 * 28672 * 5 // 2
    assert quick.quick_packed_bytes(512, 100, 128) == 0     # N % 8
    assert quick.quick_packed_bytes(100, 128, 4) == 0       # K % 64 / G % 32
    assert quick.quick_packed_bytes(0, 128, 128) == 0


def test_status_strings():
    for s, name in enumerate(["QUICK_OK", "QUICK_ERR_INVALID_ARG", "QUICK_ERR_UNSUPPORTED", "QUICK_ERR_CUDA"]):
        assert quick.quick_status_string(s) == name


def test_gemm_argument_validation_before_any_cuda_call():
    lib = quick.raw_library()
    null = ctypes.c_void_p(0)
    dummy = ctypes.c_void_p(1 << 20)
    # M == 0 is a no-op, even with null pointers (BLAS convention, reading R15)
    assert lib.quick_w4a16_gemm(null, null, 0, 256, 512, 128, null, null) == quick.QUICK_OK
    assert lib.quick_w4a16_gemm(dummy, dummy, -1, 256, 512, 128, dummy, null) == quick.QUICK_ERR_INVALID_ARG
    assert lib.quick_w4a16_gemm(dummy, dummy, 8, 256, 500, 128, dummy, null) == quick.QUICK_ERR_INVALID_ARG
    assert lib.quick_w4a16_gemm(dummy, dummy, 8, 200, 512, 128, dummy, null) == quick.QUICK_ERR_UNSUPPORTED
    assert lib.quick_w4a16_gemm(dummy, dummy, 8, 256, 512, 16, dummy, null) == quick.QUICK_ERR_UNSUPPORTED
    assert lib.quick_w4a16_gemm(null, dummy, 8, 256, 512, 128, dummy, null) == quick.QUICK_ERR_INVALID_ARG
    # misaligned X (16 B required)
    assert lib.quick_w4a16_gemm(ctypes.c_void_p((1 << 20) + 2), dummy, 8, 256, 512, 128, dummy, null) == \
        quick.QUICK_ERR_UNSUPPORTED
    # _ex overrides
    ex = lib.quick_w4a16_gemm_ex
    z = ctypes.c_size_t(0)
    assert ex(dummy, dummy, 8, 256, 512, 128, dummy, 100, 0, 0, 0, null, z, null) == quick.QUICK_ERR_INVALID_ARG  # ldy<N
    assert ex(dummy, dummy, 8, 256, 512, 128, dummy, 260, 0, 0, 0, null, z, null) == quick.QUICK_ERR_UNSUPPORTED  # ldy%8
    assert ex(dummy, dummy, 8, 256, 512, 128, dummy, 256, 0, 48, 0, null, z, null) == quick.QUICK_ERR_UNSUPPORTED  # tile
    assert ex(dummy, dummy, 8, 256, 512, 128, dummy, 256, 0, 16, 9, null, z, null) == quick.QUICK_ERR_UNSUPPORTED  # S>8
    assert ex(dummy, dummy, 8, 256, 128, 128, dummy, 256, 0, 16, 3, null, z, null) == quick.QUICK_ERR_UNSUPPORTED  # S>KT
    # a workspace size without a (256-byte aligned) workspace pointer
    assert ex(dummy, dummy, 8, 256, 512, 128, dummy, 256, 0, 0, 0, null, ctypes.c_size_t(4096), null) == \
        quick.QUICK_ERR_INVALID_ARG
    assert ex(dummy, dummy, 8, 256, 512, 128, dummy, 256, 0, 0, 0, ctypes.c_void_p((1 << 20) + 64),
              ctypes.c_size_t(4096), null) == quick.QUICK_ERR_INVALID_ARG
    # unknown flag bits
    assert ex(dummy, dummy, 8, 256, 512, 128, dummy, 256, 1 << 8, 0, 0, null, z, null) == quick.QUICK_ERR_UNSUPPORTED


def test_plan_validation():
    with pytest.raises(quick.QuickError):
        quick.quick_gemm_plan(8, 200, 512, 128)
    with pytest.raises(quick.QuickError):
        quick.quick_gemm_plan(8, 256, 512, 128, flags=1 << 8)


def test_workspace_bytes_is_zero_for_invalid_or_workspace_free_calls():
    assert quick.quick_workspace_bytes(0, 4096, 4096, 128) == 0            # M == 0: no launch
    assert quick.quick_workspace_bytes(8, 200, 512, 128) == 0              # unsupported shape
    assert quick.quick_workspace_bytes(8, 256, 512, 128, tile_n=48) == 0   # bad tile
    # forced cluster split-K and the large-M plans never use the workspace
    assert quick.quick_workspace_bytes(8, 4096, 4096, 128, split_k=4) == 0
    assert quick.quick_workspace_bytes(1024, 4096, 4096, 128) == 0
    assert quick.quick_workspace_bytes(8, 4096, 4096, 128, flags=quick.QUICK_FLAG_NO_STREAMK) == 0


def test_pack_rejects_mismatched_metadata():
    import numpy as np
    K, N, G = 256, 128, 64
    qw = np.zeros((K, N // 8), np.uint32)
    sc = np.ones((K // G, N), np.float16)
    zr = np.zeros((K // G, N // 8), np.uint32)
    quick.quick_pack_weights(qw, sc, zr, G)                       # consistent: fine
    with pytest.raises(ValueError):
        quick.quick_pack_weights(qw, sc, zr, 128)                 # scales rows != K / G
    with pytest.raises(ValueError):
        quick.quick_pack_weights(qw, sc.astype(np.float32), zr, G)   # not fp16
    with pytest.raises(ValueError):
        quick.quick_pack_weights(qw, sc, zr[:, :4], G)            # zeros columns != N / 8
    with pytest.raises(ValueError):
        quick.quick_pack_weights(qw, sc, zr, 96)                  # G does not divide K


def test_epilogue_validation():
    lib = quick.raw_library()
    null = ctypes.c_void_p(0)
    assert lib.quick_f32_to_f16(null, null, 0, null) == quick.QUICK_OK
    assert lib.quick_f32_to_f16(null, null, 8, null) == quick.QUICK_ERR_INVALID_ARG
    assert lib.quick_gather_columns(null, null, 0, 4, 8, null) == quick.QUICK_ERR_INVALID_ARG
    d = ctypes.c_void_p(1 << 20)
    assert lib.quick_gather_columns(d, d, 2, 4, 12, null) == quick.QUICK_ERR_UNSUPPORTED
    assert lib.quick_dequant_weights(null, 512, 256, 128, null, null) == quick.QUICK_ERR_INVALID_ARG


def test_bias_entry_point_validation():
    """quick_w4a16_gemm_bias: a null bias is INVALID_ARG; bias with the SiLU epilogue or a misaligned
    bias is UNSUPPORTED -- all decided on the host before any CUDA call."""
    lib = quick.raw_library()
    null = ctypes.c_void_p(0)
    d = ctypes.c_void_p(1 << 20)
    args = (8, 256, 512, 128, d, 256)
    assert lib.quick_w4a16_gemm_bias(d, d, null, *args, 0, 0, 0, null, 0, null) == quick.QUICK_ERR_INVALID_ARG
    assert lib.quick_w4a16_gemm_bias(d, d, d, *args, quick.QUICK_FLAG_SILU_MUL, 0, 0, null, 0, null) == \
        quick.QUICK_ERR_UNSUPPORTED
    assert lib.quick_w4a16_gemm_bias(d, d, ctypes.c_void_p((1 << 20) + 2), *args, 0, 0, 0, null, 0, null) == \
        quick.QUICK_ERR_UNSUPPORTED
    assert lib.quick_w4a16_gemm_bias(null, null, d, 0, 256, 512, 128, null, 256, 0, 0, 0, null, 0, null) == \
        quick.QUICK_OK   # M == 0
