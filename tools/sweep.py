"""Auto-plan timing sweep on the B200: for each (N, K) shape and M, the automatic plan timed as
CUDA-graph replays of L launches (weights rotating over > 2.5 x L2 of copies, so every launch
reads HBM), with and without PDL, and with the stream-K schedule disabled.  One JSON line per
point to gpurun_out/sweep.jsonl and a table on stdout.

    python tools/sweep.py [shapes=all|small|big] [Ms=1,16,64,...]
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
import _ws  # noqa: E402  (caller-owned stream-K workspace)

SHAPES = {"small": [(4096, 4096)],
          "mistral": [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)],
          "fig7": [(8192, 8192)],
          "big": [(28672, 8192), (8192, 28672)],
          "all": [(4096, 4096), (13824, 5120), (5120, 13824), (28672, 8192), (8192, 28672)]}
which = sys.argv[1] if len(sys.argv) > 1 else "all"
Ms = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 4, 16, 32, 64, 128, 256, 512, 1024]
modes = sys.argv[3].split(",") if len(sys.argv) > 3 else ["auto", "pdl", "nosk"]
G = 128
OUT = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "sweep.jsonl")
os.makedirs(os.path.dirname(OUT), exist_ok=True)
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "MEASURED_PEAKS.json")))
HBM, TC = peaks["hbm_gbs"] * 1e9, peaks["bf16_tflops"] * 1e12
dev = torch.device("cuda:0")
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
l2 = torch.cuda.get_device_properties(0).L2_cache_size
L = 16
FLAGS = {"auto": 0, "pdl": quick.QUICK_FLAG_PDL, "nosk": quick.QUICK_FLAG_NO_STREAMK,
         "sk": quick.QUICK_FLAG_PDL | (1 << 17),   # debug: stream-K whenever the tile allows it
         "pdlearly": quick.QUICK_FLAG_PDL | (1 << 24),
         "onecta": quick.QUICK_FLAG_PDL | (1 << 26),   # debug: stream-K with one CTA per SM
         "exittop": quick.QUICK_FLAG_PDL | (1 << 29),  # debug: return at kernel entry (launch cost)
         "exitpro": quick.QUICK_FLAG_PDL | (1 << 28),  # debug: return after the prologue
         "nocomp": quick.QUICK_FLAG_PDL | (1 << 30),   # debug: loads only
         "nomma": quick.QUICK_FLAG_PDL | (1 << 27),    # debug: dequant + TMEM stores, no MMA
         "mmasync": quick.QUICK_FLAG_PDL | (1 << 18)}  # ablation: register-fragment mma.sync decode kernel


def timeit(launch, reps=5):
    for i in range(2):
        launch(i)   # eager first: allocates the stream-K workspace outside capture
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


f = open(OUT, "a")
for (N, K) in SHAPES[which]:
    p = synth.make_problem(0, 1, N, K, G)
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).to(dev)
    R = max(2, int(np.ceil(2.5 * l2 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    for M in Ms:
        x = torch.from_numpy(synth.make_x(M, M, K).view(np.int16)).view(torch.float16).to(dev)
        y = torch.empty((M, N), device=dev, dtype=torch.float16)
        B = K * N // 2 + (K // G) * N * 5 // 2 + 2 * M * K + 2 * M * N
        F = 2 * M * N * K
        rec = {"N": N, "K": K, "M": M, "plan": _ws.plan(M, N, K, G)}
        for mode in modes:
            # "auto" / "pdl" / "nosk", or a forced plan "t<tile>s<split>[p]" (e.g. t256s2, t256s2p)
            fl, tn, sk = FLAGS.get(mode, 0), 0, 0
            if mode.startswith("t"):   # "t<tile>s<split>[p][e]": p = CTA pair (cta_group::2), e = early PDL trigger
                fl = quick.QUICK_FLAG_PDL   # forced plans are timed with PDL, like the bench
                if mode.endswith("k"):   # k = force the stream-K schedule (split must be 0)
                    fl |= 1 << 17
                mm = mode.rstrip("k")
                if mm.endswith("e"):
                    fl |= 1 << 24
                if mm.rstrip("e").endswith("p"):
                    fl |= 1 << 20
                tn, sk = (int(v) for v in mm[1:].rstrip("e").rstrip("p").split("s"))
                if tn > 2 * M and tn > 16:
                    continue
            us = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G,
                                                              y.data_ptr(), stream.cuda_stream, fl, tn, sk))
            rec[mode] = {"us": round(us, 3), "hbm": round(B / (us * 1e-6) / HBM, 4),
                         "tc": round(F / (us * 1e-6) / TC, 4)}
        f.write(json.dumps(rec) + "\n")
        f.flush()
        print(N, K, M, rec["plan"], " ".join("%s %.2fus hbm %.3f tc %.3f" % (m, rec[m]["us"], rec[m]["hbm"],
                                                                            rec[m]["tc"]) for m in modes if m in rec),
              flush=True)
    del copies, blob
    torch.cuda.empty_cache()
