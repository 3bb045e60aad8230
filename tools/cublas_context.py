"""Context only (not a target): the W4A16 GEMM (automatic plan, ordinary launches) against cuBLAS fp16
dense GEMM (torch.matmul) on the pre-dequantized weights (4x the weight bytes), both as CUDA-graph
replays over rotating weight copies larger than L2.  One line per point; JSON to gpurun_out/."""
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

G = 128
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
out = open(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "cublas_context.jsonl"), "a")
TC = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                 "MEASURED_PEAKS.json")))["bf16_tflops"]
HBM = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                  "MEASURED_PEAKS.json")))["hbm_gbs"]


def timeit(launch, L=16, reps=5):
    launch(0)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for i in range(L):
            launch(i)
    g.replay()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        g.replay()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3 / L)
    return float(np.median(ts))


# argv: shapes "NxK,NxK" and M points "1,16,..." (default: the round-1 context set)
SHAPES = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")] if len(sys.argv) > 1 else \
    [(4096, 4096), (13824, 5120), (28672, 8192)]
MS = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [16, 128, 256, 512, 1024]
for (N, K) in SHAPES:
    p = synth.make_problem(0, 1, N, K, G)
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).cuda()
    R = max(2, int(np.ceil(300e6 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    wd = quick.quick_dequant_weights(blob, K, N, G)
    nW = max(2, int(np.ceil(300e6 / (wd.numel() * 2))))
    wds = [wd] + [wd.clone() for _ in range(nW - 1)]
    for M in MS:
        x = torch.from_numpy(synth.make_x(M, M, K).view(np.int16)).view(torch.float16).cuda()
        y = torch.empty((M, N), device="cuda", dtype=torch.float16)
        h = stream.cuda_stream
        t_q = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                                           y.data_ptr(), h))
        t_p = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                             y.data_ptr(), h, flags=quick.QUICK_FLAG_PDL))
        t_c = timeit(lambda i: torch.matmul(x, wds[i % nW], out=y))
        F = 2 * M * N * K
        B = K * N // 2 + (K // G) * N * 5 // 2 + 2 * M * K + 2 * M * N
        rec = {"N": N, "K": K, "M": M, "us_quick": round(t_q, 3), "us_quick_pdl": round(t_p, 3),
               "us_cublas_fp16_dense": round(t_c, 3),
               "quick_tensor_frac": round(F / t_q / 1e6 / TC, 4), "cublas_tensor_frac": round(F / t_c / 1e6 / TC, 4),
               "quick_hbm_frac": round(B / t_q / 1e3 / HBM, 4), "speedup_vs_cublas": round(t_c / t_q, 3),
               "plan": _ws.plan(M, N, K, G)}
        out.write(json.dumps(rec) + "\n")
        print(rec, flush=True)
    del copies, wds, wd
    torch.cuda.empty_cache()
