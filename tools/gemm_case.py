"""One (M, N, K, flags[, tile, split]) GEMM case timed as graph replays in a fresh process (a
failing case cannot poison the next one).  usage: python tools/gemm_case.py M N K flags [tile split]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

M, N, K = (int(v) for v in sys.argv[1:4])
flags = int(sys.argv[4], 0)
tn = int(sys.argv[5]) if len(sys.argv) > 5 else 0
sk = int(sys.argv[6]) if len(sys.argv) > 6 else 0
p = synth.make_problem(0, M, N, K, 128)
blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, 128)).cuda()
R = max(2, int(np.ceil(300e6 / blob.numel())))
copies = [blob] + [blob.clone() for _ in range(R - 1)]
x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
y = torch.empty((M, N), device="cuda", dtype=torch.float16)
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
h = stream.cuda_stream
try:
    _ws.gemm_raw(x.data_ptr(), blob.data_ptr(), M, N, K, 128, y.data_ptr(), h, flags, tn, sk)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(16):
            _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, 128, y.data_ptr(), h, flags,
                                       tn, sk)
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    g.replay()
    b.record(stream)
    torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / 16
    print(f"{M}x{N}x{K} flags {flags:#x} tile {tn} split {sk}: {us:.2f} us, tensor frac "
          f"{2 * M * N * K / us / 1e6 / 1671.5:.3f}, hbm frac {(K * N // 2 + K * N // 128 * 5 // 2) / us / 1e3 / 6445:.3f}")
except Exception as e:  # noqa: BLE001
    print(f"{M}x{N}x{K} flags {flags:#x} tile {tn} split {sk}: ERROR {str(e).splitlines()[0]}")
