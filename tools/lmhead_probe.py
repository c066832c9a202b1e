"""Decode LM head at the c2 shape from HBM (distinct weight copies per launch, nothing in L2):
the persistent GEMM with the top-2 epilogue (current path) vs the cluster decode GEMM
(rlhf_gemm_decode, fp32 logits out, no top-2) at several K-split counts, PDL graph.

    python tools/lmhead_probe.py [--V 50272] [--B 32] [--d 768]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200 import ops  # noqa: E402
from paper_2312_11819_b200.capi import lib  # noqa: E402
from paper_2312_11819_b200.ops import GemmParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--V", type=int, default=50272)
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--d", type=int, default=768)
a = ap.parse_args()
L = lib()
L.rlhf_gemm.argtypes = [C.POINTER(GemmParams), C.c_void_p]
Ws = [(torch.randn(a.V, a.d, device="cuda") * 0.05).bfloat16() for _ in range(20)]
hf = torch.randn(a.B, a.d, device="cuda").bfloat16()
tiles = (a.V + 127) // 128
top2 = torch.empty(tiles * a.B * 4, device="cuda")
logits = torch.empty(a.B, a.V, device="cuda")


def top2_gemm(W, st):
    p = GemmParams()
    p.M, p.N, p.K, p.batch, p.batch_h = a.V, a.B, a.d, 1, 1
    p.A, p.lda, p.B, p.ldb = W.data_ptr(), a.d, hf.data_ptr(), a.d
    p.C, p.c_f32, p.c_rs, p.c_cs, p.alpha = logits.data_ptr(), 1, 1, a.V, 1.0
    p.top2 = top2.data_ptr()
    assert L.rlhf_gemm(C.byref(p), C.c_void_p(st)) == 0


def timed(fn):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for W in Ws[:2]:
            fn(W, s.cuda_stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            L.rlhf_set_pdl(1)
            for W in Ws:
                fn(W, s.cuda_stream)
            L.rlhf_set_pdl(0)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (3 * len(Ws))


us = timed(top2_gemm)
print(f"persistent GEMM + top-2: {us:7.2f} us/launch  {a.V * a.d * 2 / us / 1e3:7.0f} GB/s")
for splits in (1, 2, 3, 4, 6):
    try:
        us = timed(lambda W, st, sp=splits: ops.gemm_decode(W, hf, out=logits, splits=sp))
        print(f"decode GEMM splits={splits}: {us:7.2f} us/launch  {a.V * a.d * 2 / us / 1e3:7.0f} GB/s")
    except Exception as ex:  # noqa: BLE001
        print(f"decode GEMM splits={splits}: {ex}")
