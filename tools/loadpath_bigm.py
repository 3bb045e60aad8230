import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = ["x"]
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "loadpath_bench.py")).read().split("SHAPES = ")[0])
import numpy as np, torch, synth
from paper_2402_10076_b200 import quick
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import _ws  # noqa: E402  (caller-owned stream-K workspace)
for (M, N, K) in [(1024, 28672, 8192), (512, 4096, 4096), (1024, 4096, 4096)]:
    p = synth.make_problem(0, M, N, K, 128)
    blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, 128)).cuda()
    R = max(2, int(np.ceil(300e6 / blob.numel())))
    copies = [blob] + [blob.clone() for _ in range(R - 1)]
    x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
    y = torch.empty((M, N), device="cuda", dtype=torch.float16)
    _ws.gemm_raw(x.data_ptr(), blob.data_ptr(), M, N, K, 128, y.data_ptr(), stream.cuda_stream)
    for name, flags in [("full", 0), ("nocompute (loads only)", 1 << 30), ("nomma (loads+dequant+STTM)", 1 << 27)]:
        us = timeit(lambda i: _ws.gemm_raw(x.data_ptr(), copies[i % R].data_ptr(), M, N, K, 128,
                                                          y.data_ptr(), stream.cuda_stream, flags))
        print(f"{M}x{N}x{K} plan {_ws.plan(M, N, K, 128)} {name:28s} {us:8.2f} us  tensor frac {2*M*N*K/us/1e6/1671.5:.3f}", flush=True)
    del copies
    torch.cuda.empty_cache()
