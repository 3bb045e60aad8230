"""Decompose the small-problem latency: per-launch time (CUDA-graph replay of L launches, rotating
cold weights) of (a) the full kernel, (b) the load path only (debug flag, no dequant/MMA),
(c) tiny problems where the fixed costs dominate, (d) an empty kernel for the launch gap.
usage: python tools/latency_probe.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

DBG_NOCOMPUTE = 1 << 30
DBG_EXIT_TOP = 1 << 29
DBG_EXIT_PROLOGUE = 1 << 28
DBG_NO_MMA = 1 << 27
DBG_ONE_CTA = 1 << 26
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
L = 32


def timeit(fn_launch, reps=5):
    fn_launch(0)   # eager first: the stream-K workspace is allocated outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(L):
            fn_launch(i)
    g.replay()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1e3 / L)
    return best


z = torch.zeros(1, device=dev)
print(f"empty torch kernel (fill 1 elem): {timeit(lambda i: z.fill_(1.0)):.2f} us")
G = 128
import sys as _s
shapes = [(16, 128, 128), (16, 128, 1024), (16, 1024, 1024), (1, 4096, 4096), (16, 4096, 4096), (16, 28672, 8192)]
if len(_s.argv) > 1:
    shapes = [tuple(int(v) for v in a.split("x")) for a in _s.argv[1:]]
for (M, N, K) in shapes:
    p = synth.make_problem(0, M, N, K, G)
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).to(dev)
    R = max(2, int(np.ceil(2.5 * l2 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).to(dev)
    y = torch.empty((M, N), device=dev, dtype=torch.float16)
    xp, yp = x.data_ptr(), y.data_ptr()
    h = stream.cuda_stream
    wb = K * N // 2 + (K // G) * N * 5 // 2
    res = []
    for name, tn, sk, fl in [("exit-top", 0, 0, DBG_EXIT_TOP), ("exit-prologue", 0, 0, DBG_EXIT_PROLOGUE),
                             ("exit-top+pdl", 0, 0, DBG_EXIT_TOP | quick.QUICK_FLAG_PDL), ("auto", 0, 0, 0), ("auto+pdl", 0, 0, quick.QUICK_FLAG_PDL), ("nocompute", 0, 0, DBG_NOCOMPUTE),
                             ("cluster", 16, 4 if K >= 512 else 1, 0), ("cluster-nocomp", 16, 4 if K >= 512 else 1, DBG_NOCOMPUTE),
                             ("nosplit", 16, 1, 0), ("nomma", 0, 0, DBG_NO_MMA), ("onecta", 0, 0, DBG_ONE_CTA),
                             ("onecta-nocomp", 0, 0, DBG_ONE_CTA | DBG_NOCOMPUTE), ("onecta-nomma", 0, 0, DBG_ONE_CTA | DBG_NO_MMA)]:
        try:
            t = timeit(lambda i: _ws.gemm_raw(xp, copies[i % R].data_ptr(), M, N, K, G, yp, h,
                                                            flags=fl, tile_n=tn, split_k=sk))
            res.append(f"{name} {t:.2f}")
        except Exception as e:  # noqa: BLE001
            res.append(f"{name} err {str(e)[:40]}")
    print(f"M={M} N={N} K={K} plan={_ws.plan(M, N, K, G)} hbm-floor {wb / 6.65e3 / 1e3 * 1e3:.2f} us :: " + " | ".join(res))
