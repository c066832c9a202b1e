"""Time the decode LM head alone at the c2 shape: the tied-embedding GEMM with the top-2
epilogue (rlhf_gemm, column-major out, logits never stored) and the tile merge
(rlhf_argmax_tiles), each as a CUDA graph of 20 launches.

    python tools/lmhead_bench.py [--V 50272] [--B 32] [--d 768]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200.capi import lib  # noqa: E402
from paper_2312_11819_b200.ops import GemmParams  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--V", type=int, default=50272)
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--d", type=int, default=768)
a = ap.parse_args()
L = lib()
L.rlhf_gemm.argtypes = [C.POINTER(GemmParams), C.c_void_p]
L.rlhf_argmax_tiles.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_int,
                                C.c_void_p]
W = (torch.randn(a.V, a.d, device="cuda") * 0.05).bfloat16()
hf = torch.randn(a.B, a.d, device="cuda").bfloat16()
tiles = (a.V + 127) // 128
top2 = torch.empty(tiles * a.B * 4, device="cuda")
logits = torch.empty(a.B * a.V, device="cuda")
tok = torch.zeros(a.B, 600, device="cuda", dtype=torch.int32)
pos = torch.zeros(2, device="cuda", dtype=torch.int32)
margin = torch.zeros(a.B, 600, device="cuda")
p = GemmParams()
p.M, p.N, p.K, p.batch, p.batch_h = a.V, a.B, a.d, 1, 1
p.A, p.lda, p.B, p.ldb = W.data_ptr(), a.d, hf.data_ptr(), a.d
p.C, p.c_f32, p.c_rs, p.c_cs, p.alpha = logits.data_ptr(), 1, 1, a.V, 1.0
p.top2 = top2.data_ptr()


def gemm(st):
    assert L.rlhf_gemm(C.byref(p), C.c_void_p(st)) == 0


def merge(st):
    assert L.rlhf_argmax_tiles(top2.data_ptr(), tiles, a.B, tok.data_ptr(), 600, pos.data_ptr(), margin.data_ptr(), 0,
                               C.c_void_p(st)) == 0


s = torch.cuda.Stream()
for name, fn in (("lm-head GEMM + top-2", gemm), ("argmax_tiles", merge)):
    with torch.cuda.stream(s):
        fn(s.cuda_stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                fn(s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 100 * 1e3
    print(f"{name}: {t:7.2f} us/launch" + (f"  {a.V * a.d * 2 / t / 1e3:7.1f} GB/s (weights)" if fn is gemm else ""))
