"""Accumulation-precision diagnostic at the largest K (8192 x 28672, M = 256): error of the GPU
path vs the fp64 oracle for several split-K factors, next to an emulated exact-fp32 accumulation
(16-k chunk sums rounded to fp32, ascending k)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

M, N, K, G = 256, 8192, 28672, 128
p = synth.make_problem(M + N, M=M, N=N, K=K, G=G)
cols = np.arange(0, N, N // 128)[:128]
q = oracle.unpack_awq(p.qweight)[:, cols]
z = oracle.unpack_awq(p.zeros)[:, cols]
w = oracle.dequant(oracle.pack_awq(q), p.scales[:, cols], oracle.pack_awq(z), G)
ref = oracle.gemm(p.x, w)
x64, w64 = p.x.astype(np.float64), w.astype(np.float64)
acc = np.zeros((M, len(cols)), dtype=np.float32)
for k0 in range(0, K, 16):
    acc = (acc.astype(np.float64) + x64[:, k0:k0 + 16] @ w64[k0:k0 + 16]).astype(np.float32)
emu = acc.astype(np.float16).astype(np.float64)


def stats(y, name):
    err = np.abs(y - ref)
    big = np.abs(ref) >= 1e-2
    rel = err[big] / np.abs(ref[big])
    res = oracle.tol_check(y, ref)
    print(f"{name:28s} max_abs={err.max():.3e} mean_abs={err.mean():.3e} max_rel(|ref|>=1e-2)={rel.max():.3e} "
          f"fails={res['n_fail']} |y|~{np.abs(ref).mean():.2f}", flush=True)


stats(emu, "emulated fp32 (16-k chunks)")
blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).cuda()
x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
for tn, sk in ((256, 1), (256, 2), (256, 4), (256, 8), (64, 1), (16, 1), (16, 8)):
    y = _ws.gemm(x, blob, N, K, G, tile_n=tn, split_k=sk, out_fp32=True)
    torch.cuda.synchronize()
    stats(y.cpu().numpy()[:, cols].astype(np.float64), f"gpu tile={tn} split={sk} fp32out")
