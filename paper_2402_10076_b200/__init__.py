"""QUICK (arXiv 2402.10076) W4A16 GEMM, B200-native (sm_100a).

    from paper_2402_10076_b200 import quick
    blob = quick.quick_pack_weights(qweight, scales, zeros, 128)        # offline, host
    y = quick.quick_w4a16_gemm(x, torch.from_numpy(blob).cuda(), N, K, 128)

The package holds only what the hot path needs: csrc/ (CUDA kernels + C-ABI, built into
libquick.so), the ctypes binding (quick.py) and tensor-parallel plumbing (tp.py).
"""
__all__ = ["quick", "tp", "build"]
