"""Back-to-back PDL launches of one GEMM (eager, same stream) from a fresh process, weights
rotating over cloned copies (as tools/sweep.py does), then a check of the CUDA error state and
of the result against a non-PDL launch.
usage: python tools/pdl_repro.py M N K [reps] [flags] [copies] [ref_first]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)

M, N, K = (int(v) for v in sys.argv[1:4])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 20
flags = int(sys.argv[5], 0) if len(sys.argv) > 5 else quick.QUICK_FLAG_PDL
ncopies = int(sys.argv[6]) if len(sys.argv) > 6 else 3
ref_first = int(sys.argv[7]) if len(sys.argv) > 7 else 0
p = synth.make_problem(0, M, N, K, 128)
blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, 128)).cuda()
copies = [blob] + [blob.clone() for _ in range(ncopies - 1)]
x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
y = torch.empty((M, N), device="cuda", dtype=torch.float16)
if ref_first:
    _ws.gemm(x, blob, N, K, 128, out=y)
    torch.cuda.synchronize()
print("plan", _ws.plan(M, N, K, 128), "flags", hex(flags), flush=True)
s = torch.cuda.current_stream().cuda_stream
for r in range(reps):
    _ws.gemm_raw(x.data_ptr(), copies[r % ncopies].data_ptr(), M, N, K, 128, y.data_ptr(), s, flags)
torch.cuda.synchronize()
y_ref = _ws.gemm(x, blob, N, K, 128)
torch.cuda.synchronize()
print("ok, bit-equal to a non-PDL launch:", bool(torch.equal(y, y_ref)), flush=True)
