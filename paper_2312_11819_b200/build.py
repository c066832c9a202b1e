"""In-tree build of the engine library (no JIT cache, travels with gpurun snapshots).

    python -m paper_2312_11819_b200.build          # -> paper_2312_11819_b200/lib/librlhf_b200.so

Every .cu is compiled for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``:
plain ``-arch=sm_100a`` would also embed compute_100 PTX, which rejects tcgen05).
Host C++ is compiled by nvcc's host compiler into the same shared object.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(PKG, "lib", "librlhf_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
INCLUDES = ["-I" + os.path.join(ROOT, "include"), "-I" + CSRC, "-I" + os.path.join(CSRC, "kernels")]
COMMON = ["-O3", "-std=c++17", "-Xcompiler", "-fPIC", "-ccbin", "g++"] + INCLUDES


def sources():
    out = []
    for sub in ("kernels", "host"):
        d = os.path.join(CSRC, sub)
        for f in sorted(os.listdir(d)):
            if f.endswith((".cu", ".cpp")):
                out.append(os.path.join(d, f))
    return out


def headers():
    hs = []
    for base in (os.path.join(ROOT, "include"), CSRC):
        for dp, _, fs in os.walk(base):
            hs += [os.path.join(dp, f) for f in fs if f.endswith((".h", ".hpp", ".cuh"))]
    return hs


def _compile(src: str, hdr_mtime: float, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj
    if src.endswith(".cu"):
        cmd = [NVCC] + ARCH + COMMON + ["-lineinfo", "-Xptxas", "-v" if verbose else "-O3", "-c", src, "-o", obj]
    else:
        cmd = [NVCC] + COMMON + ["-x", "c++", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        print(r.stderr, file=sys.stderr)
    return obj


def build(verbose: bool = False) -> str:
    """Compile every CUDA/C++ source for sm_100a and link librlhf_b200.so."""
    os.makedirs(OBJ, exist_ok=True)
    hm = max(os.path.getmtime(h) for h in headers())
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, hm, verbose), srcs))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [NVCC] + ARCH + ["-shared", "-ccbin", "g++", "-o", LIB] + objs + \
            ["-lcudart_static", "-lpthread", "-ldl", "-lrt"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
