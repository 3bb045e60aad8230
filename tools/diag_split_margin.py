"""Tolerance margin of the long-K accumulation (reading R15) per split-K factor: the worst ratio
|y - ref| / bound of the BJ tolerance (bound = 1e-3 where |ref| < 1e-2, else 1e-2 |ref|) over sampled
columns of 8192 x 28672 (K = 28672, the largest BJ K), several seeds and the unit-scale stress set, for
forced plans (tile, split, pair).  ratio < 1 passes; the plan cap needs headroom for unseen inputs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (tools: accuracy diagnostics)
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402

N, K, G = 8192, 28672, 128
PAIR = 1 << 20
cases = [(int(s.split(":")[0]), int(s.split(":")[1].rstrip("p")), s.endswith("p")) for s in
         (sys.argv[1].split(",") if len(sys.argv) > 1 else ["128:1p", "128:2p", "128:3p", "128:4p", "16:1", "16:2", "16:4"])]
M = int(sys.argv[2]) if len(sys.argv) > 2 else 256
sets = [("rand", s) for s in range(4)] + [("unit", 7)]
worst = {c: 0.0 for c in cases}
for kind, seed in sets:
    p = synth.make_problem(seed * 31 + M, M=M, N=N, K=K, G=G) if kind == "rand" else \
        synth.make_structured("unit", seed, M=M, N=N, K=K, G=G)
    cols = np.random.default_rng(seed).choice(N, 384, replace=False)
    q = oracle.unpack_awq(p.qweight)[:, cols]
    z = oracle.unpack_awq(p.zeros)[:, cols]
    w = oracle.dequant(oracle.pack_awq(q), p.scales[:, cols], oracle.pack_awq(z), G)
    ref = oracle.gemm(p.x, w)
    bound = np.where(np.abs(ref) < 1e-2, 1e-3, 1e-2 * np.abs(ref))
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).cuda()
    x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
    for (tn, sk, pr) in cases:
        y = torch.empty((M, N), device="cuda", dtype=torch.float16)
        _ws.gemm_raw(x.data_ptr(), blob.data_ptr(), M, N, K, G, y.data_ptr(), torch.cuda.current_stream().cuda_stream,
                     quick.QUICK_FLAG_NO_STREAMK | (PAIR if pr else 0), tn, sk)
        torch.cuda.synchronize()
        r = float(np.max(np.abs(y.float().cpu().numpy()[:, cols] - ref) / bound))
        worst[(tn, sk, pr)] = max(worst[(tn, sk, pr)], r)
        print(f"{kind} seed {seed} tile {tn} split {sk} pair {pr}: worst err/bound {r:.3f}", flush=True)
print("WORST over sets:", {f"t{k[0]}s{k[1]}{'p' if k[2] else ''}": round(v, 3) for k, v in worst.items()})
