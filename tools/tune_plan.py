"""Measure every (tile_n, split_k) launch plan for the BASELINE shapes and M points on the B200.
Each timing = CUDA-graph replay of L launches, weights rotating over copies > 2.5 x L2 (cold HBM).
Writes JSON lines to gpurun_out/tune.jsonl (input to the plan heuristic)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

OUT = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "tune.jsonl")
shapes = [(4096, 4096), (13824, 5120), (5120, 13824), (28672, 8192), (8192, 28672)]
Ms = [1, 4, 16, 32, 64, 128, 256, 512, 1024]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    shapes = [(4096, 4096), (28672, 8192)]
    Ms = [1, 16, 64, 128, 256, 1024]
G = 128
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
f = open(OUT, "a")
L = 24


def timeit(fn_launch, reps=3):
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


for (N, K) in shapes:
    p = synth.make_problem(0, 1, N, K, G)
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).to(dev)
    R = max(2, int(np.ceil(2.5 * l2 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    wb = K * N // 2 + (K // G) * N * 5 // 2
    for M in Ms:
        x = torch.from_numpy(synth.make_x(M, M, K).view(np.int16)).view(torch.float16).to(dev)
        y = torch.empty((M, N), device=dev, dtype=torch.float16)
        auto = _ws.plan(M, N, K, G)
        cover = 16 if M <= 16 else 32 if M <= 32 else 64 if M <= 64 else 128 if M <= 128 else 256
        results = []
        for tn in (16, 32, 64, 128, 256):
            if tn > cover or tn * 8 < cover:
                continue
            for sk in (1, 2, 3, 4, 5, 6, 8):
                if sk > K // 64:
                    continue
                try:
                    us = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                                                      y.data_ptr(), stream.cuda_stream, 0, tn, sk))
                except Exception as e:  # noqa
                    us = None
                results.append((tn, sk, us))
        us_auto = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                                               y.data_ptr(), stream.cuda_stream))
        us_pdl = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                                              y.data_ptr(), stream.cuda_stream, quick.QUICK_FLAG_PDL))
        ok = [r for r in results if r[2] is not None]
        best = min(ok, key=lambda r: r[2])
        rec = {"N": N, "K": K, "M": M, "auto": auto, "us_auto": round(us_auto, 3), "us_auto_pdl": round(us_pdl, 3),
               "best": {"tile_n": best[0], "split_k": best[1], "us": round(best[2], 3)},
               "hbm_frac_best": round((wb + 2 * M * K + 2 * M * N) / (best[2] * 1e-6) / 6547.2e9, 4),
               "tc_frac_best": round(2 * M * N * K / (best[2] * 1e-6) / 1674.4e12, 4),
               "all": [(a, b, None if c is None else round(c, 3)) for a, b, c in results]}
        f.write(json.dumps(rec) + "\n")
        f.flush()
        print(N, K, M, "auto", auto, round(us_auto, 2), "pdl", round(us_pdl, 2), "best", best[:2], round(best[2], 2),
              "hbm%", rec["hbm_frac_best"], "tc%", rec["tc_frac_best"], flush=True)
    del copies, blob
    torch.cuda.empty_cache()
