"""Single-shape GEMM driver for ncu captures: `reps` launches of quick_w4a16_gemm at (M, N, K),
each on a different weight copy (cold L2 under ncu's --cache-control all anyway)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

ap = argparse.ArgumentParser()
ap.add_argument("--M", type=int, default=1)
ap.add_argument("--N", type=int, default=4096)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--G", type=int, default=128)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--tile_n", type=int, default=0)
ap.add_argument("--split_k", type=int, default=0)
ap.add_argument("--flags", type=lambda v: int(v, 0), default=0)
a = ap.parse_args()
p = synth.make_problem(0, a.M, a.N, a.K, a.G)
blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, a.G)).cuda()
copies = [blob] + [blob.clone() for _ in range(a.reps - 1)]
x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
y = torch.empty((a.M, a.N), device="cuda", dtype=torch.float16)
for r in range(a.reps):
    if a.flags:
        _ws.gemm_raw(x.data_ptr(), copies[r].data_ptr(), a.M, a.N, a.K, a.G, y.data_ptr(),
                                   torch.cuda.current_stream().cuda_stream, flags=a.flags, tile_n=a.tile_n,
                                   split_k=a.split_k)
    else:
        _ws.gemm(x, copies[r], a.N, a.K, a.G, out=y, tile_n=a.tile_n, split_k=a.split_k)
torch.cuda.synchronize()
print("plan", _ws.plan(a.M, a.N, a.K, a.G))
