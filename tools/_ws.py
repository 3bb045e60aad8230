"""Tools helper: one caller-owned stream-K workspace per process (the library never allocates).
Tools launch serially on one stream, so sharing it is safe (quick.h: no concurrent launches)."""
import torch

from paper_2402_10076_b200 import quick

WS_BYTES = 16 << 20
_ws = None


def ws():
    global _ws
    if _ws is None:
        _ws = torch.zeros(WS_BYTES, dtype=torch.uint8, device="cuda")
    return _ws


def gemm_raw(*a, **k):
    w = ws()
    return quick.quick_w4a16_gemm_raw(*a, ws_ptr=w.data_ptr(), ws_bytes=w.numel(), **k)


def gemm(*a, **k):
    return quick.quick_w4a16_gemm(*a, workspace=ws(), **k)


def plan(M, N, K, G, flags=0):
    return quick.quick_gemm_plan(M, N, K, G, flags=flags, workspace_bytes=WS_BYTES)
