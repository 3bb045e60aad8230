"""Bring-up diagnostics: run small structured problems through the C-ABI and save Y next to the
oracle's reference under gpurun_out/diag/ for offline inspection."""
import os
import sys
import traceback

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", "diag")
os.makedirs(out, exist_ok=True)
dev = torch.device("cuda:0")
cases = [("onehot", 16, 256, 512, 128, 16, 1), ("onehot", 16, 128, 64, 64, 16, 1),
         ("intexact", 16, 128, 128, 128, 16, 1), ("random", 8, 256, 512, 128, 16, 1),
         ("random", 8, 256, 512, 128, 16, 4), ("random", 200, 256, 512, 128, 256, 1),
         ("random", 64, 256, 512, 128, 64, 2)]
for kind, M, N, K, G, tn, sk in cases:
    tag = f"{kind}_M{M}_N{N}_K{K}_G{G}_t{tn}_s{sk}"
    try:
        p = synth.make_problem(1, M, N, K, G) if kind == "random" else synth.make_structured(kind, 1, M, N, K, G)
        blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).to(dev)
        x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).to(dev)
        y = _ws.gemm(x, blob, N, K, G, tile_n=tn, split_k=sk)
        torch.cuda.synchronize()
        ref = oracle.w4a16_reference(p.x, p.qweight, p.scales, p.zeros, G)
        yn = y.float().cpu().numpy()
        res = oracle.tol_check(yn, ref)
        np.savez(os.path.join(out, tag + ".npz"), y=yn, ref=ref, x=p.x, qweight=p.qweight, scales=p.scales,
                 zeros=p.zeros)
        print(tag, "OK" if res["ok"] else "FAIL", res, flush=True)
    except Exception:
        print(tag, "EXC", traceback.format_exc(), flush=True)
        break
