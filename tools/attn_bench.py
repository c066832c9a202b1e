"""Time rlhf_attn_decode alone (CUDA graph of 20 launches) at the c2 decode shape.

    python tools/attn_bench.py [--ctx 384] [--B 32] [--H 12] [--hd 64] [--smax 512]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2312_11819_b200 import ops
from paper_2312_11819_b200.capi import lib

ap = argparse.ArgumentParser()
ap.add_argument("--ctx", type=int, nargs="+", default=[257, 384, 512])
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--H", type=int, default=12)
ap.add_argument("--hd", type=int, default=64)
ap.add_argument("--smax", type=int, default=512)
ap.add_argument("--pdl", action="store_true", help="programmatic dependent launches inside the graph")
ap.add_argument("--layers", type=int, default=12, help="distinct KV caches cycled (defeats L2 reuse)")
a = ap.parse_args()
d = a.H * a.hd
qkv = torch.randn(a.B, 3 * d, device="cuda").bfloat16()
caches = [(torch.randn(a.B, a.H, a.smax, a.hd, device="cuda").bfloat16(),
           torch.randn(a.B, a.H, a.smax, a.hd, device="cuda").bfloat16()) for _ in range(a.layers)]
for ctx in a.ctx:
    pos = torch.tensor([ctx - 1], device="cuda", dtype=torch.int32)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for kc, vc in caches:
            ops.attn_decode(qkv, kc, vc, pos)
        with torch.cuda.graph(g, stream=s):
            if a.pdl:
                lib().rlhf_set_pdl(1)
            for _ in range(2):
                for kc, vc in caches:
                    ops.attn_decode(qkv, kc, vc, pos)
            lib().rlhf_set_pdl(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    n = 2 * a.layers
    us = e0.elapsed_time(e1) / n * 1e3
    byts = a.B * a.H * ctx * a.hd * 2 * 2
    print(f"ctx {ctx:5d}: {us:7.2f} us/launch  {byts / us / 1e3:7.0f} GB/s  ({byts / 1e6:.1f} MB)")
