"""Load-path ceiling: the kernel with dequant + MMA skipped (debug flag 1<<30) vs the full kernel,
per plan, on cold weights (graph of L launches over rotating copies)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

DBG = 1 << 30
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
L = 16


def timeit(launch):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(L):
            launch(i)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / L)
    return best


SHAPES = [(16, 28672, 8192), (16, 4096, 4096), (16, 13824, 5120)]
for (M, N, K) in SHAPES:
    p = synth.make_problem(0, M, N, K, 128)
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, 128)).cuda()
    R = max(2, int(np.ceil(300e6 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
    y = torch.empty((M, N), device="cuda", dtype=torch.float16)
    wb = blob.numel()
    # warm the stream-K workspace outside capture
    _ws.gemm_raw(x.data_ptr(), blob.data_ptr(), M, N, K, 128, y.data_ptr(), stream.cuda_stream)
    for name, flags, tn, sk, hot in [("full sk", 0, 0, 0, 0), ("nocompute sk", DBG, 0, 0, 0),
                                     ("full cluster", 4, 0, 0, 0), ("nocompute cluster", DBG | 4, 0, 0, 0),
                                     ("nomma sk", 1 << 27, 0, 0, 0), ("nosttm sk", 1 << 25, 0, 0, 0),
                                     ("full sk L2-hot", 0, 0, 0, 1), ("nomma sk L2-hot", 1 << 27, 0, 0, 1),
                                     ("nosttm sk L2-hot", 1 << 25, 0, 0, 1), ("nocompute sk L2-hot", DBG, 0, 0, 1)]:
        if hot and wb > 60e6:
            continue   # does not stay in L2
        us = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[0 if hot else i % R].data_ptr(), M, N,
                                                          K, 128, y.data_ptr(), stream.cuda_stream, flags, tn, sk))
        print(f"{M}x{N}x{K} {name:18s} {us:8.2f} us  {wb / us / 1e3:7.1f} GB/s ({wb / us / 1e3 / 6547:.3f} of HBM)",
              flush=True)
    del copies
    torch.cuda.empty_cache()
