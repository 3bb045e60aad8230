"""Print the resident CTAs / clusters the plan sees for every kernel variant (debug)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401  (initialises the CUDA context)
from paper_2402_10076_b200 import quick  # noqa: E402

lib = quick.raw_library()
f = lib.quick_debug_resident
f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
torch.cuda.init()
for bn in (16, 32, 64, 128, 256):
    for sk in (0, 1):
        if sk and bn > 64:
            continue
        sm, rg = ctypes.c_int(), ctypes.c_int()
        res = [f(bn, sk, S, ctypes.byref(sm), ctypes.byref(rg)) for S in (1, 2, 4, 8)]
        print(f"tile {bn:3d} sk {sk}: smem {sm.value} B regs {rg.value}  resident S=1,2,4,8: {res}")
res = {}
for bn in (128, 256):
    res[f"t{bn}"] = [f(bn, 0, S, None, None) for S in range(1, 9)]
    res[f"t{bn}p"] = [f(bn, 2, S, None, None) for S in range(1, 5)]
print("resident (S = 1..):", res)
