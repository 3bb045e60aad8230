"""Thin ctypes binding of libquick.so (include/quick.h): argument marshalling only.

Every step of the path runs inside libquick.so (host repack in C++, GEMM and epilogues in
sm_100a kernels).  torch is used for device memory and streams only.  There is no fallback:
if the library is missing this module raises at import time.
"""
import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# QUICK_LIB: an alternative in-tree build of the same library (A/B timing of build variants, tools/)
LIB_PATH = os.environ.get("QUICK_LIB") or os.path.join(_PKG, "libquick.so")

QUICK_OK, QUICK_ERR_INVALID_ARG, QUICK_ERR_UNSUPPORTED, QUICK_ERR_CUDA = 0, 1, 2, 3
QUICK_FLAG_OUT_F32, QUICK_FLAG_PDL, QUICK_FLAG_NO_STREAMK, QUICK_FLAG_SILU_MUL, QUICK_FLAG_BF16 = 1, 2, 4, 8, 16


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
        "quick_import_gptq": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p,
                                      c_void_p, c_void_p, c_void_p]),
        "quick_pack_weights_device": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_void_p,
                                              c_void_p]),
        "quick_gather_k": (c_int, [c_void_p, c_void_p, c_int, c_int, c_void_p, c_void_p]),
        "quick_pack_gate_up": (c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int,
                                       c_int, c_void_p]),
        "quick_w4a16_gemm": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
        "quick_w4a16_gemm_ex": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int,
                                        c_int, c_int, c_int, c_void_p, c_size_t, c_void_p]),
        "quick_w4a16_gemm_bias": (c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int,
                                          c_int, c_int, c_int, c_void_p, c_size_t, c_void_p]),
        "quick_workspace_bytes": (c_size_t, [c_int, c_int, c_int, c_int, c_int, c_int, c_int]),
        "quick_gemm_plan": (c_int, [c_int, c_int, c_int, c_int, c_int, c_size_t, c_void_p, c_void_p, c_void_p,
                                    c_void_p]),
        "quick_dequant_weights": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_void_p]),
        "quick_dequant_weights_ex": (c_int, [c_void_p, c_int, c_int, c_int, c_void_p, c_int, c_void_p]),
        "quick_f32_to_f16": (c_int, [c_void_p, c_void_p, c_size_t, c_void_p]),
        "quick_gather_columns": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_void_p]),
        "quick_peer_alloc": (c_int, [c_size_t, c_void_p]),
        "quick_peer_free": (c_int, [c_void_p]),
        "quick_peer_export": (c_int, [c_void_p, c_void_p]),
        "quick_peer_import": (c_int, [c_void_p, c_void_p]),
        "quick_peer_close": (c_int, [c_void_p]),
        "quick_tp_barrier": (c_int, [c_void_p, c_int, c_int, c_void_p]),
        "quick_tp_column_gemm": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_int, c_void_p,
                                         c_int, c_int, c_int, c_void_p, c_size_t, c_void_p]),
        "quick_tp_row_gemm": (c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_void_p, c_void_p, c_int,
                                      c_void_p, c_int, c_int, c_int, c_void_p, c_size_t, c_void_p]),
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
    """AWQ (qweight uint32 [K][N/8], scales fp16 [K/G][N], zeros uint32 [K/G][N/8]) -> v1 blob (uint8).
    Shapes and dtypes are checked here: the C packer trusts them."""
    qweight, scales, zeros = np.asarray(qweight), np.asarray(scales), np.asarray(zeros)
    if qweight.ndim != 2 or qweight.dtype not in (np.uint32, np.int32):
        raise ValueError(f"qweight must be a 2-D uint32/int32 array [K][N/8], got {qweight.dtype} {qweight.shape}")
    K, N = qweight.shape[0], qweight.shape[1] * 8
    if group_size <= 0 or K % group_size:
        raise ValueError(f"group_size {group_size} must divide K={K}")
    if scales.dtype not in (np.float16, np.uint16):
        raise ValueError(f"scales must be float16 (or their uint16 bits), got {scales.dtype}")
    if scales.shape != (K // group_size, N):
        raise ValueError(f"scales shape {scales.shape} != (K/G, N) = {(K // group_size, N)}")
    if zeros.dtype not in (np.uint32, np.int32) or zeros.shape != (K // group_size, N // 8):
        raise ValueError(f"zeros must be uint32/int32 (K/G, N/8) = {(K // group_size, N // 8)}, "
                         f"got {zeros.dtype} {zeros.shape}")
    qweight = np.ascontiguousarray(qweight).view(np.uint32)
    zeros = np.ascontiguousarray(zeros).view(np.uint32)
    scales = np.ascontiguousarray(scales).view(np.uint16)
    nbytes = quick_packed_bytes(K, N, group_size)
    out = np.empty(max(nbytes, 1), dtype=np.uint8)
    _check("quick_pack_weights", _lib.quick_pack_weights(_np_ptr(qweight), _np_ptr(scales), _np_ptr(zeros),
                                                         group_size, K, N, _np_ptr(out)))
    return out[:nbytes]


def _awq_checked(qweight, scales, zeros, group_size):
    qweight, scales, zeros = np.asarray(qweight), np.asarray(scales), np.asarray(zeros)
    if qweight.ndim != 2 or qweight.dtype not in (np.uint32, np.int32):
        raise ValueError(f"qweight must be a 2-D uint32/int32 array [K][N/8], got {qweight.dtype} {qweight.shape}")
    K, N = qweight.shape[0], qweight.shape[1] * 8
    if group_size <= 0 or K % group_size:
        raise ValueError(f"group_size {group_size} must divide K={K}")
    if scales.dtype not in (np.float16, np.uint16) or scales.shape != (K // group_size, N):
        raise ValueError(f"scales must be float16 (K/G, N) = {(K // group_size, N)}, got {scales.dtype} {scales.shape}")
    if zeros.dtype not in (np.uint32, np.int32) or zeros.shape != (K // group_size, N // 8):
        raise ValueError(f"zeros must be uint32/int32 (K/G, N/8) = {(K // group_size, N // 8)}, "
                         f"got {zeros.dtype} {zeros.shape}")
    return (np.ascontiguousarray(qweight).view(np.uint32), np.ascontiguousarray(scales).view(np.uint16),
            np.ascontiguousarray(zeros).view(np.uint32), K, N)


def quick_pack_gate_up(gate, up, group_size: int) -> np.ndarray:
    """Fused gate||up blob (quick.h): gate / up = (qweight, scales, zeros) AWQ tuples with I columns each;
    the GEMM with QUICK_FLAG_SILU_MUL on it returns SiLU(X.gate) * (X.up) [M][I]."""
    qg, sg, zg, K, I = _awq_checked(*gate, group_size)
    qu, su, zu, K2, I2 = _awq_checked(*up, group_size)
    if (K2, I2) != (K, I):
        raise ValueError(f"gate {K}x{I} and up {K2}x{I2} shapes differ")
    nbytes = quick_packed_bytes(K, 2 * I, group_size)
    out = np.empty(max(nbytes, 1), dtype=np.uint8)
    _check("quick_pack_gate_up", _lib.quick_pack_gate_up(_np_ptr(qg), _np_ptr(sg), _np_ptr(zg), _np_ptr(qu),
                                                         _np_ptr(su), _np_ptr(zu), group_size, K, I, _np_ptr(out)))
    return out[:nbytes]


def quick_import_gptq(qweight, qzeros, scales, group_size: int, g_idx=None, zero_plus_one: bool = True):
    """AutoGPTQ tensors (qweight [K/8][N], qzeros [K/G][N/8] storing zero - zero_plus_one, scales fp16
    [K/G][N], optional g_idx [K]) -> (qweight_awq, scales, zeros_awq, perm) in the AWQ format with the
    rows sorted by group (quick.h quick_import_gptq).  Pack the result with quick_pack_weights and feed
    the GEMM X[:, perm] (quick_gather_k) when perm is not the identity."""
    qweight = np.ascontiguousarray(qweight).view(np.uint32)
    qzeros = np.ascontiguousarray(qzeros).view(np.uint32)
    scales = np.ascontiguousarray(scales)
    K, N = qweight.shape[0] * 8, qweight.shape[1]
    if group_size <= 0 or K % group_size:
        raise ValueError(f"group_size {group_size} must divide K={K}")
    if scales.dtype not in (np.float16, np.uint16) or scales.shape != (K // group_size, N):
        raise ValueError(f"scales must be float16 (K/G, N) = {(K // group_size, N)}")
    if qzeros.shape != (K // group_size, N // 8):
        raise ValueError(f"qzeros must be (K/G, N/8) = {(K // group_size, N // 8)}")
    scales = scales.view(np.uint16)
    gi = None
    if g_idx is not None:
        gi = np.ascontiguousarray(g_idx, dtype=np.int32)
        if gi.shape != (K,):
            raise ValueError(f"g_idx must have K={K} entries")
    qa = np.empty((K, N // 8), np.uint32)
    sa = np.empty((K // group_size, N), np.uint16)
    za = np.empty((K // group_size, N // 8), np.uint32)
    perm = np.empty(K, np.int32)
    _check("quick_import_gptq", _lib.quick_import_gptq(
        _np_ptr(qweight), _np_ptr(qzeros), _np_ptr(scales), _np_ptr(gi) if gi is not None else None,
        1 if zero_plus_one else 0, group_size, K, N, _np_ptr(qa), _np_ptr(sa), _np_ptr(za), _np_ptr(perm)))
    return qa, sa.view(np.float16), za, perm


def quick_pack_weights_device(qweight, scales, zeros, group_size: int, out=None, stream=None):
    """quick_pack_weights on the GPU: torch cuda tensors qweight int32/uint32 [K][N/8], scales fp16 [K/G][N],
    zeros int32 [K/G][N/8] -> the v1 blob (cuda uint8), bit-identical to the host packer."""
    import torch
    K, N = qweight.shape[0], qweight.shape[1] * 8
    for t, shape in ((qweight, (K, N // 8)), (scales, (K // group_size, N)), (zeros, (K // group_size, N // 8))):
        if not (t.is_cuda and t.is_contiguous() and tuple(t.shape) == shape and t.element_size() in (2, 4)):
            raise ValueError(f"device AWQ tensors must be contiguous cuda tensors of shape {shape}")
    if scales.dtype not in (torch.float16, torch.int16) or qweight.element_size() != 4 or zeros.element_size() != 4:
        raise ValueError("qweight / zeros must be 32-bit, scales fp16")
    nbytes = quick_packed_bytes(K, N, group_size)
    if out is None:
        out = torch.empty(nbytes, dtype=torch.uint8, device=qweight.device)
    _check("quick_pack_weights_device", _lib.quick_pack_weights_device(
        ctypes.c_void_p(qweight.data_ptr()), ctypes.c_void_p(scales.data_ptr()), ctypes.c_void_p(zeros.data_ptr()),
        group_size, K, N, ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)))
    return out


def quick_gather_k(x, perm, out=None, stream=None):
    """Xp[m][k'] = X[m][perm[k']] on the GPU (x cuda fp16 [M][K], perm cuda int32 [K])."""
    import torch
    M, K = x.shape
    if out is None:
        out = torch.empty_like(x)
    _check("quick_gather_k", _lib.quick_gather_k(ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(perm.data_ptr()), M, K,
                                                 ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)))
    return out


def quick_unpack_weights(packed, group_size: int, K: int, N: int):
    """Exact inverse of quick_pack_weights -> (qweight uint32, scales fp16, zeros uint32)."""
    packed = np.ascontiguousarray(packed, dtype=np.uint8)
    qweight = np.empty((K, N // 8), dtype=np.uint32)
    scales = np.empty((K // group_size, N), dtype=np.uint16)
    zeros = np.empty((K // group_size, N // 8), dtype=np.uint32)
    _check("quick_unpack_weights", _lib.quick_unpack_weights(_np_ptr(packed), group_size, K, N, _np_ptr(qweight),
                                                             _np_ptr(scales), _np_ptr(zeros)))
    return qweight, scales.view(np.float16), zeros


def quick_gemm_plan(M: int, N: int, K: int, group_size: int, *, flags: int = 0, workspace_bytes: int = 0):
    """The plan quick_w4a16_gemm_ex would launch for this shape with a workspace of that size."""
    tn, sk, nc, pr = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _check("quick_gemm_plan", _lib.quick_gemm_plan(M, N, K, group_size, flags, workspace_bytes, ctypes.byref(tn),
                                                   ctypes.byref(sk), ctypes.byref(nc), ctypes.byref(pr)))
    return {"tile_n": tn.value, "split_k": sk.value, "num_ctas": nc.value, "pair": pr.value == 1}


def quick_workspace_bytes(M: int, N: int, K: int, group_size: int, *, flags: int = 0, tile_n: int = 0,
                          split_k: int = 0) -> int:
    return int(_lib.quick_workspace_bytes(M, N, K, group_size, flags, tile_n, split_k))


def workspace_for(shapes, group_size: int, device, *, flags: int = 0):
    """A zeroed caller-owned workspace (torch uint8 tensor) large enough for every (M, N, K) in
    `shapes` (memory plumbing only; the library never allocates)."""
    import torch
    nb = max([quick_workspace_bytes(M, N, K, group_size, flags=flags) for (M, N, K) in shapes] + [256])
    return torch.zeros(nb, dtype=torch.uint8, device=device)


# ----------------------------------------------------------------------------- device side
def quick_w4a16_gemm(x, packed, N: int, K: int, group_size: int, out=None, *, ldy=None, out_fp32=False,
                     pdl=False, no_streamk=False, tile_n: int = 0, split_k: int = 0, workspace=None,
                     flags: int = 0, stream=None, bias=None):
    """Y = X . dequant(Wq) (+ bias) on the GPU.  x: cuda fp16 [M][K]; packed: cuda uint8 blob;
    workspace: optional zeroed cuda uint8 tensor (quick_workspace_bytes) enabling stream-K plans;
    bias: optional cuda [N] tensor of x's dtype (quick_w4a16_gemm_bias).
    Returns `out` (allocated if None): fp16 [M][N] (fp32 if out_fp32)."""
    import torch
    if x.dtype == torch.bfloat16:          # the bf16 variant: bf16 X, scales (in the blob) and Y
        flags |= QUICK_FLAG_BF16
    if not (x.is_cuda and x.dtype in (torch.float16, torch.bfloat16) and x.is_contiguous() and x.dim() == 2
            and x.shape[1] == K):
        raise ValueError(f"x must be a contiguous cuda float16 / bfloat16 [M][{K}] tensor")
    if not (packed.is_cuda and packed.dtype == torch.uint8 and packed.is_contiguous()):
        raise ValueError("packed must be a contiguous cuda uint8 tensor")
    if packed.numel() != quick_packed_bytes(K, N, group_size):
        raise ValueError(f"packed has {packed.numel()} bytes, expected {quick_packed_bytes(K, N, group_size)}")
    M = x.shape[0]
    want = torch.float32 if out_fp32 else x.dtype
    n_out = N // 2 if (flags & QUICK_FLAG_SILU_MUL) else N
    if out is None:
        out = torch.empty((M, n_out), device=x.device, dtype=want)
    elif not (out.is_cuda and out.dtype == want and out.dim() == 2 and out.shape[0] >= M and out.shape[1] >= n_out
              and out.stride(1) == 1 and out.device == x.device):
        raise ValueError(f"out must be a cuda {want} [>= {M}][>= {n_out}] tensor with unit column stride")
    ld = out.stride(0) if ldy is None else ldy
    ws_ptr, ws_bytes = None, 0
    if workspace is not None:
        if not (workspace.is_cuda and workspace.dtype == torch.uint8 and workspace.is_contiguous()):
            raise ValueError("workspace must be a contiguous cuda uint8 tensor")
        ws_ptr, ws_bytes = workspace.data_ptr(), workspace.numel()
    fl = flags | (QUICK_FLAG_OUT_F32 if out_fp32 else 0) | (QUICK_FLAG_PDL if pdl else 0) \
        | (QUICK_FLAG_NO_STREAMK if no_streamk else 0)
    if bias is not None:
        if not (bias.is_cuda and bias.dtype == x.dtype and bias.is_contiguous() and bias.dim() == 1
                and bias.numel() == N and bias.device == x.device):
            raise ValueError(f"bias must be a contiguous cuda {x.dtype} [{N}] tensor")
        _check("quick_w4a16_gemm_bias", _lib.quick_w4a16_gemm_bias(
            ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(packed.data_ptr()), ctypes.c_void_p(bias.data_ptr()),
            M, N, K, group_size, ctypes.c_void_p(out.data_ptr()), ld, fl, tile_n, split_k, ctypes.c_void_p(ws_ptr),
            ws_bytes, _stream_handle(stream)))
        return out
    _check("quick_w4a16_gemm_ex", _lib.quick_w4a16_gemm_ex(
        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(packed.data_ptr()), M, N, K, group_size,
        ctypes.c_void_p(out.data_ptr()), ld, fl, tile_n, split_k, ctypes.c_void_p(ws_ptr), ws_bytes,
        _stream_handle(stream)))
    return out


def quick_w4a16_gemm_raw(x_ptr: int, packed_ptr: int, M: int, N: int, K: int, group_size: int, y_ptr: int,
                         stream_handle: int, flags: int = 0, tile_n: int = 0, split_k: int = 0, ldy: int = 0,
                         ws_ptr: int = 0, ws_bytes: int = 0):
    """Plain C-ABI call on raw device pointers (`quick_w4a16_gemm`, or `_ex` when any option is set)."""
    if flags or tile_n or split_k or ldy or ws_bytes:
        _check("quick_w4a16_gemm_ex", _lib.quick_w4a16_gemm_ex(
            ctypes.c_void_p(x_ptr), ctypes.c_void_p(packed_ptr), M, N, K, group_size, ctypes.c_void_p(y_ptr),
            ldy or N, flags, tile_n, split_k, ctypes.c_void_p(ws_ptr or None), ws_bytes,
            ctypes.c_void_p(stream_handle)))
        return
    _check("quick_w4a16_gemm", _lib.quick_w4a16_gemm(ctypes.c_void_p(x_ptr), ctypes.c_void_p(packed_ptr), M, N, K,
                                                     group_size, ctypes.c_void_p(y_ptr),
                                                     ctypes.c_void_p(stream_handle)))


def quick_dequant_weights(packed, K: int, N: int, group_size: int, out=None, stream=None, bf16: bool = False):
    import torch
    if out is None:
        out = torch.empty((K, N), device=packed.device, dtype=torch.bfloat16 if bf16 else torch.float16)
    _check("quick_dequant_weights_ex", _lib.quick_dequant_weights_ex(
        ctypes.c_void_p(packed.data_ptr()), K, N, group_size, ctypes.c_void_p(out.data_ptr()),
        QUICK_FLAG_BF16 if bf16 else 0, _stream_handle(stream)))
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


# ----------------------------------------------------------------------------- peer memory / fused TP
QUICK_IPC_HANDLE_BYTES = 64


def _ptr_array(ptrs):
    arr = (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(int(p)) for p in ptrs])
    return arr


def quick_peer_alloc(nbytes: int) -> int:
    p = ctypes.c_void_p()
    _check("quick_peer_alloc", _lib.quick_peer_alloc(nbytes, ctypes.byref(p)))
    return int(p.value)


def quick_peer_free(ptr: int):
    _check("quick_peer_free", _lib.quick_peer_free(ctypes.c_void_p(ptr)))


def quick_peer_export(ptr: int) -> bytes:
    buf = ctypes.create_string_buffer(QUICK_IPC_HANDLE_BYTES)
    _check("quick_peer_export", _lib.quick_peer_export(ctypes.c_void_p(ptr), buf))
    return buf.raw


def quick_peer_import(handle: bytes) -> int:
    p = ctypes.c_void_p()
    _check("quick_peer_import", _lib.quick_peer_import(ctypes.create_string_buffer(handle, len(handle)),
                                                       ctypes.byref(p)))
    return int(p.value)


def quick_peer_close(ptr: int):
    _check("quick_peer_close", _lib.quick_peer_close(ctypes.c_void_p(ptr)))


def quick_tp_barrier(flag_ptrs, rank: int, stream=None):
    _check("quick_tp_barrier", _lib.quick_tp_barrier(_ptr_array(flag_ptrs), len(flag_ptrs), rank,
                                                     _stream_handle(stream)))


def quick_tp_column_gemm(x, packed, N_local: int, K: int, group_size: int, y_ptrs, ldy: int, flag_ptrs, rank: int,
                         *, flags: int = 0, workspace=None, stream=None):
    """Column-parallel GEMM, all-gather fused into the epilogue (quick.h): y_ptrs / flag_ptrs = every rank's
    buffer as mapped in this process."""
    ws_ptr, ws_bytes = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    _check("quick_tp_column_gemm", _lib.quick_tp_column_gemm(
        ctypes.c_void_p(x.data_ptr()), ctypes.c_void_p(packed.data_ptr()), x.shape[0], N_local, K, group_size,
        _ptr_array(y_ptrs), ldy, _ptr_array(flag_ptrs), len(y_ptrs), rank, flags, ctypes.c_void_p(ws_ptr),
        ws_bytes, _stream_handle(stream)))


def quick_tp_row_gemm(x_local, packed, N: int, K_local: int, group_size: int, part_ptrs, y_ptrs, ldy: int, flag_ptrs,
                      rank: int, *, flags: int = 0, workspace=None, stream=None):
    """Row-parallel GEMM + peer-memory fp32 all-reduce (quick.h)."""
    ws_ptr, ws_bytes = (workspace.data_ptr(), workspace.numel()) if workspace is not None else (None, 0)
    _check("quick_tp_row_gemm", _lib.quick_tp_row_gemm(
        ctypes.c_void_p(x_local.data_ptr()), ctypes.c_void_p(packed.data_ptr()), x_local.shape[0], N, K_local,
        group_size, _ptr_array(part_ptrs), _ptr_array(y_ptrs), ldy, _ptr_array(flag_ptrs), len(y_ptrs), rank,
        flags, ctypes.c_void_p(ws_ptr), ws_bytes, _stream_handle(stream)))


def quick_status_string(status: int) -> str:
    return _status_string(status)


def quick_last_cuda_error() -> int:
    return int(_lib.quick_last_cuda_error())


def raw_library():
    """The ctypes handle (tests check symbol exports and raw status codes)."""
    return _lib
