"""Per-stage clock64 trace of the W4A16 kernel pipeline (debug hook quick_debug_set_trace).
usage: python tools/trace_gemm.py M N K [tile_n split_k]"""
import ctypes
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
tn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
sk = int(sys.argv[5]) if len(sys.argv) > 5 else 0
FLAGS = int(os.environ.get("TRACE_FLAGS", "0"), 0)   # extra launch flags (e.g. 0x100000: CTA pair)
G, TS, STRIDE = 128, 256, 8 + 7 * 256
lib = quick.raw_library()
lib.quick_debug_set_trace.argtypes = [ctypes.c_void_p]
p = synth.make_problem(0, M, N, K, G)
blob = torch.from_numpy(quick.quick_pack_weights(p.qweight, p.scales, p.zeros, G)).cuda()
copies = [blob.clone() for _ in range(max(4, int(3e8 // blob.numel())))]
x = torch.from_numpy(p.x.view(np.int16)).view(torch.float16).cuda()
y = torch.empty((M, N), device="cuda", dtype=torch.float16)
NCTA = _ws.plan(M, N, K, G)["num_ctas"] if not (tn or sk) else 4096
tr = torch.zeros(16 * STRIDE + 4 * max(NCTA, 4096), dtype=torch.int64, device="cuda")


def run(w):
    _ws.gemm_raw(x.data_ptr(), w.data_ptr(), M, N, K, G, y.data_ptr(), 0, FLAGS, tn, sk)


for i in range(3):
    run(copies[i])
torch.cuda.synchronize()
lib.quick_debug_set_trace(ctypes.c_void_p(tr.data_ptr()))
run(copies[-1])
torch.cuda.synchronize()
lib.quick_debug_set_trace(ctypes.c_void_p(0))
tt = tr.cpu().numpy()
t = tt[:16 * STRIDE].reshape(16, STRIDE)
rec = tt[16 * STRIDE:].reshape(-1, 4)[:, :3]
rec = rec[rec[:, 1] > 0]
if len(rec):
    t0 = rec[:, 1].min()
    span = (rec[:, 2].max() - t0) / 1e3
    per_sm = {}
    for smid, a, b in rec:
        per_sm.setdefault(int(smid), []).append(((a - t0) / 1e3, (b - t0) / 1e3))
    cnt = np.bincount([len(v) for v in per_sm.values()])
    busy = np.array([max(b for _, b in v) for v in per_sm.values()])
    dur = (rec[:, 2] - rec[:, 1]) / 1e3
    print(f"ALL CTAs: {len(rec)} on {len(per_sm)} SMs, CTAs/SM histogram {cnt.tolist()}, kernel span {span:.2f} us, "
          f"CTA duration min/med/max {dur.min():.2f}/{np.median(dur):.2f}/{dur.max():.2f} us, SM finish min/med/max "
          f"{busy.min():.2f}/{np.median(busy):.2f}/{busy.max():.2f} us, start skew max {(rec[:,1].max()-t0)/1e3:.2f} us")
    full = tt[16 * STRIDE:].reshape(-1, 4)
    idx = np.nonzero(full[:, 1] > 0)[0]
    # per SM: the CTAs sharing it, by launch index (is the same one always the fast one?)
    by_sm = {}
    for i in idx:
        by_sm.setdefault(int(full[i, 0]), []).append((int(i), (full[i, 2] - full[i, 1]) / 1e3))
    pairs = [sorted(v) for v in by_sm.values() if len(v) == 2]
    if pairs:
        lo = np.array([p[0][1] for p in pairs])
        hi = np.array([p[1][1] for p in pairs])
        print(f"SMs with 2 CTAs: {len(pairs)}; lower-index CTA duration mean {lo.mean():.2f} us, higher-index "
              f"{hi.mean():.2f} us; lower-index faster on {int((lo < hi).sum())} SMs; index gap "
              f"{np.mean([p[1][0] - p[0][0] for p in pairs]):.1f}")
    d_all = (full[idx, 2] - full[idx, 1]) / 1e3
    slow = idx[d_all > 2 * np.median(d_all)]
    print("slow CTAs (lin idx, smid, start us, dur us):",
          [(int(i), int(full[i, 0]), round((full[i, 1] - t0) / 1e3, 2), round((full[i, 2] - full[i, 1]) / 1e3, 2)) for i in slow[:20]])
print("plan", _ws.plan(M, N, K, G), "tile", tn, "split", sk)
names = ["P_before_empty", "P_issued", "D_full", "D_aempty_ok", "D_afull_arrived", "M_afull_ok", "M_committed"]
for c in range(16):
    row = t[c]
    if row[0] == 0:
        continue
    nst = int(row[3])
    n = min(nst, TS)
    ev = row[8:].reshape(7, TS)[:, :n].astype(np.int64) - int(row[0])
    print(f"CTA {c} sm {row[4]} nst {nst}: setup->end {int(row[2]) - int(row[0])} cyc, dfull at {int(row[1]) - int(row[0])}"
          + (f", split-K: partials stored {int(row[5]) - int(row[0])}, cluster sync 1 {int(row[6]) - int(row[0])},"
             f" reduced {int(row[7]) - int(row[0])}" if row[5] else ""))
    if c < 2:
        for i in list(range(min(n, 6))) + list(range(max(6, n - 3), n)):
            print("  it", i, " ".join(f"{nm}={ev[j, i]}" for j, nm in enumerate(names)))
    if n > 8:
        mid = slice(4, n - 2)
        d = lambda a: float(np.mean(np.diff(a[mid])))
        print("   per-stage interval: " + " ".join(f"{nm}={d(ev[j]):.0f}" for j, nm in enumerate(names)))
        print("   latencies: issue->full %.0f  full->aempty %.0f  aempty->afull %.0f  afull->mma %.0f  mma issue %.0f" % (
            np.mean(ev[2, mid] - ev[1, mid]), np.mean(ev[3, mid] - ev[2, mid]), np.mean(ev[4, mid] - ev[3, mid]),
            np.mean(ev[5, mid] - ev[4, mid]), np.mean(ev[6, mid] - ev[5, mid])))
        # MMA commit (stage i) -> dequant sees aempty for stage i + 4
        if n > 12:
            print("   commit(i)->aempty(i+4) %.0f" % np.mean(ev[3, 8:n - 2] - ev[6, 4:n - 6]))
