"""Achieved HBM bandwidth of the decode GEMM on large weights (graph of back-to-back
launches over distinct weight copies, so nothing stays in L2).

    python tools/decode_gemm_bw.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200 import ops  # noqa: E402
from paper_2312_11819_b200.capi import lib  # noqa: E402

for name, M, K, N, splits in [("c3 W1", 8192, 2048, 16, 4), ("c3 W2", 2048, 8192, 16, 16), ("c3 W2", 2048, 8192, 16, 8), ("c3 qkv", 6144, 2048, 16, 4), ("c3 qkv", 6144, 2048, 16, 8), ("c3 W1", 8192, 2048, 16, 8),
                              ("c3 O", 2048, 2048, 16, 8), ("c3 O", 2048, 2048, 16, 16), ("c3 O", 2048, 2048, 16, 4),
                              ("c2 W1", 3072, 768, 32, 8), ("c2 qkv", 2304, 768, 32, 8)]:
    copies = max(2, int(2e9 // (M * K * 2)))
    Ws = [torch.randn(M, K, device="cuda").bfloat16() for _ in range(min(copies, 24))]
    X = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(N, M, device="cuda")
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for W in Ws:
            ops.gemm_decode(W, X, out=out, splits=splits)
        with torch.cuda.graph(g, stream=s):
            lib().rlhf_set_pdl(1)
            for W in Ws:
                ops.gemm_decode(W, X, out=out, splits=splits)
            lib().rlhf_set_pdl(0)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / len(Ws)
    print(f"{name:7s} M={M:5d} K={K:5d} N={N} splits={splits}: {us:7.2f} us/launch  {M * K * 2 / us / 1e3:7.0f} GB/s")
