"""Build libquick.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels with the repo)."""
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libquick.so")
SOURCES = [os.path.join(CSRC, "quick_gemm.cu"), os.path.join(CSRC, "quick_repack.cu"), os.path.join(CSRC, "quick_tp.cu"), os.path.join(CSRC, "quick_pack.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "quick_ptx.cuh"), os.path.join(ROOT, "include", "quick.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",   # not -arch=sm_100a: tcgen05 needs the 'a' target only
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3",
    "-shared",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build libquick.so")


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False, out: str = None, defines=()) -> str:
    """Compile libquick.so next to this file (or `out` with extra -D defines: A/B build variants);
    returns its path."""
    target = out or LIB
    if not force and out is None and up_to_date():
        return LIB
    tmp = target + ".tmp"
    cmd = [nvcc_path(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"), "-o", tmp,
           *SOURCES, "-lpthread"]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    print(build(force=True, verbose=True))
