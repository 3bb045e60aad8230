"""Mistral-7B linear stack as a real 32-layer chain (BASELINE.json configs[4]): per layer QKV, O, the fused
gate||up GEMM with its SiLU*mul epilogue, and down, each layer with its own weight copies (3.6 GB in
all: every launch streams from HBM), chained through their activations (O -> gate_up -> down -> next
layer's QKV / O input; attention and norms are not on the path).  The whole 32-layer step is one CUDA
graph of PDL launches.  (An L2-prefetch variant was measured harmful and removed:
profiles/r02_l2_prefetch_negative.txt.)  JSON to gpurun_out/layer_chain.jsonl.

    python tools/layer_chain.py [Ms=1,16,64,256]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402

Ms = [int(v) for v in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 16, 64, 256]
L, G, H, I = 32, 128, 4096, 14336
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
out = open(os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "layer_chain.jsonl"), "a")


def blob_of(N, K, seed):
    return torch.from_numpy(quick.quick_pack_weights(synth.make_qweight(seed, K, N), synth.make_scales(seed, K, N, G),
                                                     synth.make_zeros(seed, K, N, G), G)).to(dev)


gate = (synth.make_qweight(3, H, I), synth.make_scales(3, H, I, G), synth.make_zeros(3, H, I, G))
up = (synth.make_qweight(4, H, I), synth.make_scales(4, H, I, G), synth.make_zeros(4, H, I, G))
base = {"qkv": blob_of(6144, H, 1), "o": blob_of(H, H, 2),
        "gu": torch.from_numpy(quick.quick_pack_gate_up(gate, up, G)).to(dev), "down": blob_of(H, I, 5)}
layers = [{k: (v if l == 0 else v.clone()) for k, v in base.items()} for l in range(L)]
ws = _ws.ws()
h = stream.cuda_stream
for M in Ms:
    x = torch.from_numpy(synth.make_x(M, M, H).view(np.int16)).view(torch.float16).to(dev)
    attn = torch.from_numpy(synth.make_x(M + 1, M, H).view(np.int16)).view(torch.float16).to(dev)
    qkv = torch.empty((M, 6144), device=dev, dtype=torch.float16)
    yo = torch.empty((M, H), device=dev, dtype=torch.float16)
    hh = torch.empty((M, I), device=dev, dtype=torch.float16)
    xs = [x, torch.empty_like(x)]

    def step():
        seq = []
        for l in range(L):
            xin, xout = xs[l % 2], xs[(l + 1) % 2]
            seq += [(layers[l]["qkv"], xin, qkv, 6144, H, 0), (layers[l]["o"], attn, yo, H, H, 0),
                    (layers[l]["gu"], yo, hh, 2 * I, H, quick.QUICK_FLAG_SILU_MUL), (layers[l]["down"], hh, xout, H, I, 0)]
        for i, (w, xi, yi, N, K, fl) in enumerate(seq):
            quick.quick_w4a16_gemm_raw(xi.data_ptr(), w.data_ptr(), M, N, K, G, yi.data_ptr(), h,
                                       flags=quick.QUICK_FLAG_PDL | fl, ldy=yi.shape[1], ws_ptr=ws.data_ptr(),
                                       ws_bytes=ws.numel())

    res = {"M": M}
    for variant in ("plain",):
        step()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            step()
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        res[variant] = {"ms_per_step": round(ms, 4), "tokens_per_s": round(M / (ms * 1e-3), 1),
                                              "us_per_layer": round(1e3 * ms / L, 3)}
        del g
    out.write(json.dumps(res) + "\n")
    out.flush()
    print(res, flush=True)
