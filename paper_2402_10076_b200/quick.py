"""Thin ctypes binding of libquick.so (include/quick.h): argument marshalling only.

Every step of the path runs inside libquick.so (host repack in C++, GEMM and epilogues in
sm_100a kernels).  torch is used for device memory and streams only.  There is no fallback:
if the library is missing this module raises at import time.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libquick.so")

QUICK_OK, QUICK_ERR_INVALID_ARG, QUICK_ERR_UNSUPPORTED, QUICK_ERR_CUDA = 0, 1, 2, 3
QUICK_FLAG_OUT_F32, QUICK_FLAG_PDL, QUICK_FLAG_NO_STREAMK = 1, 2, 4


class QuickError(RuntimeError):
    def __init__(self, fn, status, cuda_err=0):
        self.status = status
        self.cuda_error = cuda_err
        super().__init__(f"{fn} failed: {_status_string(status)} (cudaError {cuda_err})")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libquick.so not built at {LIB_PATH}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    c_int, c_void_p, c_size_t, c_uint32 = ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32
    sigs = {
        "quick_layout_version": (c_uint32, []),
        "quick_packed_bytes": (c_size_t, [c_int, c_int, c_int]),
        "quick_pack_weights": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]),
        "quick_unpack_weights": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
        "quick_w4a16_gemm": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
        "quick_w4a16_gemm_ex": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int,
                                        c_int, c_int, c_int, c_void_p]),
        "quick_gemm_plan": (c_int, [c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
        "quick_dequant_weights": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
        "quick_f32_to_f16": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
        "quick_gather_columns": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]),
        "quick_status_string": (ctypes.c_char_p, [c_int]),
        "quick_last_cuda_error": (c_int, []),
    }
    for name, (res, args) in sigs.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


_lib = _load()


def _status_string(s):
    return _lib.quick_status_string(int(s)).decode()


def _check(fn, status):
    if status != QUICK_OK:
        raise QuickError(fn, status, _lib.quick_last_cuda_error() if status == QUICK_ERR_CUDA else 0)


def _np_ptr(a):
    return ctypes.c_void_p(a.ctypes.data)


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# ----------------------------------------------------------------------------- host side
def quick_layout_version() -> int:
    return int(_lib.quick_layout_version())


def quick_packed_bytes(K: int, N: int, group_size: int) -> int:
    return int(_lib.quick_packed_bytes(K, N, group_size))


def quick_pack_weights(qweight, scales, zeros, group_size: int) -> np.ndarray:
    """AWQ (qweight uint32 [K][N/8], scales fp16 [K/G][N], zeros uint32 [K/G][N/8]) -> v1 blob (uint8)."""
    qweight = np.ascontiguousarray(qweight, dtype=np.uint32)
    zeros = np.ascontiguousarray(zeros, dtype=np.uint32)
    scales = np.ascontiguousarray(np.asarray(scales).view(np.uint16) if np.asarray(scales).dtype == np.float16
                                  else np.asarray(scales, dtype=np.uint16))
    K, N = qweight.shape[0], qweight.shape[1] * 8
    nbytes = quick_packed_bytes(K, N, group_size)
    out = np.empty(max(nbytes, 1), dtype=np.uint8)
    _check("quick_pack_weights", _lib.quick_pack_weights(_np_ptr(qweight), _np_ptr(scales), _np_ptr(zeros),
                                                         group_size, K, N, _np_ptr(out)))
    return out[:nbytes]


def quick_unpack_weights(packed, group_size: int, K: int, N: int):
    """Exact inverse of quick_pack_weights -> (qweight uint32, scales fp16, zeros uint32)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    qweight = np.empty((K, N // 8), dtype=np.uint32)
    scales = np.empty((K // group_size, N), dtype=np.uint16)
    zeros = np.empty((K // group_size, N // 8), dtype=np.uint32)
    _check("quick_unpack_weights", _lib.quick_unpack_weights(_np_ptr(packed), group_size, K, N, _np_ptr(qweight),
                                                             _np_ptr(scales), _np_ptr(zeros)))
    return qweight, scales.view(np.float16), zeros


def quick_gemm_plan(M: int, N: int, K: int, group_size: int):
    tn, sk, nc = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check("quick_gemm_plan", _lib.quick_gemm_plan(M, N, K, group_size, ctypes.byref(tn), ctypes.byref(sk),
                                                   ctypes.byref(nc)))
    pair = _lib.quick_debug_plan_pair(M, N, K, group_size) == 1   # CTA pairs (cta_group::2)
    return {"tile_n": tn.value, "split_k": sk.value, "num_ctas": nc.value, "pair": pair}


# ----------------------------------------------------------------------------- device side
def quick_w4a16_gemm(x, packed, N: int, K: int, group_size: int, out=None, *, ldy=None, out_fp32=False,
                     pdl=False, no_streamk=False, tile_n: int = 0, split_k: int = 0, stream=None):
    """Y = X . dequant(Wq) on the GPU.  x: cuda fp16 [M][K]; packed: cuda uint8 blob.
    Returns `out` (allocated if None): fp16 [M][N] (fp32 if out_fp32)."""
    import torch
    assert x.is_cuda and x.dtype == torch.float16 and x.is_contiguous() and x.dim() == 2 and x.shape[1] == K
    assert packed.is_cuda and packed.dtype == torch.uint8
    M = x.shape[0]
    if out is None:
        out = torch.empty((M, N), device=x.device, dtype=torch.float32 if out_fp32 else torch.float16)
    ld = out.stride(0) if ldy is None else ldy
    _check("quick_w4a16_gemm_ex", _lib.quick_w4a16_gemm_ex(
        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(packed.data_ptr()), M, N, K, group_size,
        ctypes.c_void_p(out.data_ptr()), ld, (QUICK_FLAG_OUT_F32 if out_fp32 else 0) | (QUICK_FLAG_PDL if pdl else 0)
        | (QUICK_FLAG_NO_STREAMK if no_streamk else 0),
        tile_n, split_k, _stream_handle(stream)))
    return out


def quick_w4a16_gemm_raw(x_ptr: int, packed_ptr: int, M: int, N: int, K: int, group_size: int, y_ptr: int,
                         stream_handle: int, flags: int = 0, tile_n: int = 0, split_k: int = 0, ldy: int = 0):
    """Plain C-ABI call on raw device pointers (`quick_w4a16_gemm`, or `_ex` when any option is set)."""
    if flags or tile_n or split_k or ldy:
        _check("quick_w4a16_gemm_ex", _lib.quick_w4a16_gemm_ex(
            ctypes.c_void_p(x_ptr), ctypes.c_void_p(packed_ptr), M, N, K, group_size, ctypes.c_void_p(y_ptr),
            ldy or N, flags, tile_n, split_k, ctypes.c_void_p(stream_handle)))
        return
    _check("quick_w4a16_gemm", _lib.quick_w4a16_gemm(ctypes.c_void_p(x_ptr), ctypes.c_void_p(packed_ptr), M, N, K,
                                                     group_size, ctypes.c_void_p(y_ptr),
                                                     ctypes.c_void_p(stream_handle)))


def quick_dequant_weights(packed, K: int, N: int, group_size: int, out=None, stream=None):
    import torch
    if out is None:
        out = torch.empty((K, N), device=packed.device, dtype=torch.float16)
    _check("quick_dequant_weights", _lib.quick_dequant_weights(ctypes.c_void_p(packed.data_ptr()), K, N, group_size,
                                                               ctypes.c_void_p(out.data_ptr()),
                                                               _stream_handle(stream)))
    return out


def quick_f32_to_f16(src, dst=None, stream=None):
    import torch
    if dst is None:
        dst = torch.empty(src.shape, device=src.device, dtype=torch.float16)
    _check("quick_f32_to_f16", _lib.quick_f32_to_f16(ctypes.c_void_p(src.data_ptr()), ctypes.c_void_p(dst.data_ptr()),
                                                     src.numel(), _stream_handle(stream)))
    return dst


def quick_gather_columns(src, P: int, M: int, Nr: int, dst=None, stream=None):
    import torch
    if dst is None:
        dst = torch.empty((M, P * Nr), device=src.device, dtype=torch.float16)
    _check("quick_gather_columns", _lib.quick_gather_columns(ctypes.c_void_p(src.data_ptr()),
                                                             ctypes.c_void_p(dst.data_ptr()), P, M, Nr,
                                                             _stream_handle(stream)))
    return dst


def quick_status_string(status: int) -> str:
    return _status_string(status)


def quick_last_cuda_error() -> int:
    return int(_lib.quick_last_cuda_error())


def raw_library():
    """The ctypes handle (tests check symbol exports and raw status codes)."""
    return _lib
