"""Timeline of a PDL chain of the same GEMM (tracing build of the kernel, debug hook quick_debug_set_trace):
L launches back to back with QUICK_FLAG_PDL on one stream, each recording per CTA (smid, start, end,
griddep release) in globaltimer ns into its own buffer.  Prints, per launch, the first/median/last CTA
start, griddep release and end relative to the previous launch's last CTA end -- where the time of one
GEMM in a chain goes.  usage: python tools/trace_chain.py M N K [L]"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2402_10076_b200 import quick  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402

M, N, K = (int(v) for v in sys.argv[1:4])
L = int(sys.argv[4]) if len(sys.argv) > 4 else 6
XF = int(sys.argv[5], 0) if len(sys.argv) > 5 else 0   # extra flags (e.g. 0x1000000: early PDL trigger)
TN = int(sys.argv[6]) if len(sys.argv) > 6 else 0      # forced tile / split (0 = automatic)
SK = int(sys.argv[7]) if len(sys.argv) > 7 else 0
G, STRIDE = 128, 8 + 7 * 256
lib = quick.raw_library()
lib.quick_debug_set_trace.argtypes = [ctypes.c_void_p]
p = synth.make_problem(0, M, N, K, G)
blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).cuda()
copies = [blob.clone() for _ in range(max(L + 4, int(4e8 // blob.numel())))]
x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
y = torch.empty((M, N), device="cuda", dtype=torch.float16)
plan = _ws.plan(M, N, K, G, flags=quick.QUICK_FLAG_PDL | XF)
NCTA = max(plan["num_ctas"], 1024)
bufs = [torch.zeros(16 * STRIDE + 4 * max(NCTA, 4096), dtype=torch.int64, device="cuda") for _ in range(L)]
s = torch.cuda.current_stream().cuda_stream
for w in range(3):   # warm-up (untraced)
    _ws.gemm_raw(x.data_ptr(), copies[w].data_ptr(), M, N, K, G, y.data_ptr(), s, quick.QUICK_FLAG_PDL | XF, TN, SK)
torch.cuda.synchronize()
# the traced launches are captured in one CUDA graph (eager launches of short kernels are host-bound:
# the GPU would idle between them), each with its own trace buffer
stream = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    for i in range(L):
        lib.quick_debug_set_trace(ctypes.c_void_p(bufs[i].data_ptr()))
        _ws.gemm_raw(x.data_ptr(), copies[3 + i].data_ptr(), M, N, K, G, y.data_ptr(), stream.cuda_stream,
                     quick.QUICK_FLAG_PDL | XF, TN, SK)
lib.quick_debug_set_trace(ctypes.c_void_p(0))
g.replay()
torch.cuda.synchronize()
print("plan", plan, "launches", L)
prev_end = None
for i in range(L):
    r = bufs[i].cpu().numpy()[16 * STRIDE:].reshape(-1, 4)[:NCTA]
    r = r[r[:, 1] > 0]
    st, en, gd = r[:, 1].astype(np.int64), r[:, 2].astype(np.int64), r[:, 3].astype(np.int64)
    base = prev_end if prev_end is not None else st.min()
    q = lambda a: "%7.2f/%7.2f/%7.2f" % ((a.min() - base) / 1e3, (np.median(a) - base) / 1e3, (a.max() - base) / 1e3)
    gdv = gd[gd > 0]
    print(f"launch {i}: CTAs {len(r)}  start {q(st)}  griddep {q(gdv) if len(gdv) else '-'}  end {q(en)}  us "
          f"(rel. to the previous launch's last CTA end)")
    prev_end = en.max()
