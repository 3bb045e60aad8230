"""Ablation (the paper's Fig. 2 question on B200): the dequantized A stage in TMEM
(tcgen05.st + TS MMA, the design) against the same stage written back to shared memory (STS.128,
SWIZZLE_128B K-major, conflict-free) + SS MMA.  Same plan, same weights; checks bit-identity and
times both as CUDA-graph replays on cold weights.  Appends JSON lines to gpurun_out/ablation.jsonl."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (tools: parity of the ablation variant)
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

ABL = 1 << 21
G = 128
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
out = open(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "ablation.jsonl"), "a")


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


# argv: cases "MxNxKxTILExSPLIT,..." (default: the round-1 set)
cases = [tuple(int(v) for v in c.split("x")) for c in sys.argv[1].split(",")] if len(sys.argv) > 1 else \
    [(16, 4096, 4096, 16, 4), (16, 28672, 8192, 16, 1), (128, 4096, 4096, 128, 4), (512, 4096, 4096, 128, 1),
     (1024, 28672, 8192, 128, 1)]
for (M, N, K, tn, sk) in cases:
    p = synth.make_problem(0, M, N, K, G)
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).cuda()
    R = max(2, int(np.ceil(300e6 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
    y0 = torch.empty((M, N), device="cuda", dtype=torch.float16)
    y1 = torch.empty_like(y0)
    h = stream.cuda_stream
    _ws.gemm_raw(x.data_ptr(), blob.data_ptr(), M, N, K, G, y0.data_ptr(), h,
                               quick.QUICK_FLAG_NO_STREAMK, tn, sk)
    _ws.gemm_raw(x.data_ptr(), blob.data_ptr(), M, N, K, G, y1.data_ptr(), h, ABL, tn, sk)
    torch.cuda.synchronize()
    same = bool(torch.equal(y0.view(torch.int16), y1.view(torch.int16)))
    cols = np.arange(0, N, max(1, N // 256))[:256]
    cols = cols[: len(cols) // 8 * 8]
    q = oracle.unpack_awq(p.qweight)[:, cols]
    z = oracle.unpack_awq(p.zeros)[:, cols]
    w = oracle.dequant(oracle.pack_awq(q), p.scales[:, cols], oracle.pack_awq(z), G)
    ref = oracle.gemm(p.x, w)
    tol_tmem = oracle.tol_check(y0.float().cpu().numpy()[:, cols], ref)
    tol_smem = oracle.tol_check(y1.float().cpu().numpy()[:, cols], ref)
    diff = (y0.float() - y1.float()).abs().max().item()
    t_tmem = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                                          y0.data_ptr(), h, quick.QUICK_FLAG_NO_STREAMK, tn, sk))
    t_smem = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                                          y1.data_ptr(), h, ABL, tn, sk))
    # context only: cuBLAS fp16 GEMM on the dequantized weights (4x the weight bytes), rotating copies
    wd = quick.quick_dequant_weights(blob, K, N, G)
    nW = max(2, int(np.ceil(300e6 / (wd.numel() * 2))))
    wds = [wd] + [wd.clone() for _ in range(nW - 1)]
    yc = torch.empty((M, N), device="cuda", dtype=torch.float16)
    t_cublas = timeit(lambda i: torch.matmul(x, wds[i % nW], out=yc))
    del wds, wd
    rec = {"M": M, "N": N, "K": K, "tile_n": tn, "split_k": sk, "bit_identical": same, "max_abs_diff": diff,
           "us_cublas_fp16_dense": round(t_cublas, 3),
           "tmem_tol_ok": tol_tmem["ok"], "smem_tol_ok": tol_smem["ok"],
           "us_tmem_a": round(t_tmem, 3), "us_smem_a": round(t_smem, 3), "smem_over_tmem": round(t_smem / t_tmem, 3)}
    out.write(json.dumps(rec) + "\n")
    print(rec, flush=True)
    del copies
    torch.cuda.empty_cache()
