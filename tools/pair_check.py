"""CTA-pair (cta_group::2) plan check on the B200: one (M, N, K, tile, split) case per process
(a failing case cannot poison the next).  Compares the pair plan with the ordinary plan of the
same tile/split (expected bit-identical: same MMA K order per output) and with an fp32
reference through the library's dequant, then times both as CUDA-graph replays.

    python tools/pair_check.py M N K tile split [pdl]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

M, N, K, tn, sk = (int(v) for v in sys.argv[1:6])
pdl = quick.QUICK_FLAG_PDL if len(sys.argv) > 6 and sys.argv[6] == "pdl" else 0
PAIR = 1 << 20
G = 128
p = synth.make_problem(0, M, N, K, G)
blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).cuda()
x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
h = stream.cuda_stream


def run(flags, y):
    _ws.gemm_raw(x.data_ptr(), blob.data_ptr(), M, N, K, G, y.data_ptr(), h, flags, tn, sk)


tag = f"{M}x{N}x{K} tile {tn} split {sk}{' pdl' if pdl else ''}"
try:
    y0 = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float16)
    y1 = torch.full((M, N), float("nan"), device="cuda", dtype=torch.float16)
    run(pdl, y0)
    run(pdl | PAIR, y1)
    torch.cuda.synchronize()
    w = quick.quick_dequant_weights(blob, K, N, G).float()   # [K, N] or [N, K]
    if w.shape[0] != K:
        w = w.t()
    ref = x.float() @ w
    err1 = ((y1.float() - ref).abs() / ref.abs().clamp_min(1e-2)).max().item()
    ident = torch.equal(y0.view(torch.int16), y1.view(torch.int16))
    nbad = int((y0.view(torch.int16) != y1.view(torch.int16)).sum().item())
    R = max(2, int(np.ceil(300e6 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    ts = {}
    for name, fl in (("base", pdl), ("pair", pdl | PAIR)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            for i in range(16):
                _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, G, y1.data_ptr(), h, fl,
                                           tn, sk)
        g.replay()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b) * 1e3 / 16)
        ts[name] = best
    F = 2 * M * N * K
    print(f"{tag}: identical {ident} (diff {nbad}) max rel err pair {err1:.2e} | base {ts['base']:.2f} us "
          f"({F / ts['base'] / 1e6 / 1671.5:.3f}) pair {ts['pair']:.2f} us ({F / ts['pair'] / 1e6 / 1671.5:.3f})",
          flush=True)
except Exception as e:  # noqa: BLE001
    print(f"{tag}: ERROR {str(e).splitlines()[0]}", flush=True)
