"""Decode-GEMM bandwidth at LLaMA-7B shapes (c4): the cluster split-K decode kernel at
several slice counts vs the persistent GEMM the engine uses for >= 148 tiles.

    python tools/decode_gemm_bw_7b.py [batch]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200 import ops  # noqa: E402
from paper_2312_11819_b200.capi import lib  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8


def timed(fn, copies):
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for i in range(copies):
            fn(i)
        with torch.cuda.graph(g, stream=s):
            lib().rlhf_set_pdl(1)
            for i in range(copies):
                fn(i)
            lib().rlhf_set_pdl(0)
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / copies


for name, M, K, splits_list in [("qkv", 12288, 4096, [1, 2, 4]), ("wo", 4096, 4096, [2, 4, 8, 16]),
                                ("w1 gate|up", 22016, 4096, [1, 2]), ("w2", 4096, 11008, [4, 8, 16]),
                                ("lm head", 32000, 4096, [1])]:
    copies = max(2, min(16, int(3e9 // (M * K * 2))))
    Ws = [torch.randn(M, K, device="cuda").bfloat16() for _ in range(copies)]
    X = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
    for sp in splits_list:
        try:
            us = timed(lambda i: ops.gemm_decode(Ws[i], X, out=out, splits=sp, out_f32=False), copies)
            print(f"{name:10s} M={M:5d} K={K:5d} N={N} decode splits={sp:2d}: {us:8.2f} us  {M * K * 2 / us / 1e3:6.0f} GB/s",
                  flush=True)
        except Exception as e:
            print(name, sp, "failed", e)
    outc = torch.empty(N, M, device="cuda", dtype=torch.bfloat16)
    us = timed(lambda i: ops.gemm(Ws[i], X, out=outc, out_f32=False, swap_out=True), copies)
    print(f"{name:10s} M={M:5d} K={K:5d} N={N} persistent GEMM : {us:8.2f} us  {M * K * 2 / us / 1e3:6.0f} GB/s", flush=True)
    del Ws
    torch.cuda.empty_cache()
