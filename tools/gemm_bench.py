"""Time the tcgen05 GEMM on the PPO step's shapes (CUDA events, warm, through the C-ABI).

    python tools/gemm_bench.py [--shape M,N,K[,a_mn,b_mn]] [--iters 20] [--only-first]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200 import ops  # noqa: E402

SHAPES = [  # c2 (OPT-125m, B=32, S=512): forward, dgrad, wgrad, LM head; decode (swap-AB, Bg=32)
    ("fwd W1", 16384, 3072, 768, 0, 0, 1),
    ("fwd W2", 16384, 768, 3072, 0, 0, 1),
    ("fwd qkv", 16384, 2304, 768, 0, 0, 1),
    ("dgrad W1", 16384, 768, 3072, 0, 1, 1),
    ("wgrad W1", 3072, 768, 16384, 1, 1, 2),
    ("fwd Wo", 16384, 768, 768, 0, 0, 1),
    ("dgrad qkv", 16384, 768, 2304, 0, 1, 1),
    ("wgrad qkv", 2304, 768, 16384, 1, 1, 2),
    ("wgrad W2", 768, 3072, 16384, 1, 1, 2),
    ("wgrad Wo", 768, 768, 16384, 1, 1, 8),
    ("lm head", 8192, 50272, 768, 0, 0, 1),
    ("dec qkv", 2304, 32, 768, 0, 0, 6),
    ("dec W2", 768, 32, 3072, 0, 0, 8),
    ("dec lmhead", 50272, 32, 768, 0, 0, 1),
]

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--only-first", action="store_true")
a = ap.parse_args()
for name, M, N, K, amn, bmn, split in (SHAPES[:1] if a.only_first else SHAPES):
    A = torch.randn((K, M) if amn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if bmn else (N, K), device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.float32 if split > 1 or name.startswith("wgrad") else torch.bfloat16)
    f = lambda: ops.gemm(A, B, a_mn=bool(amn), b_mn=bool(bmn), out=C, out_f32=C.dtype == torch.float32, split_k=split)
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / a.iters * 1e-3
    fl = 2.0 * M * N * K
    by = 2.0 * (M * K + N * K) + C.element_size() * M * N
    print(f"{name:12s} M={M:6d} N={N:6d} K={K:6d} split={split}  {t*1e6:9.1f} us  {fl/t/1e12:7.1f} TFLOP/s  {by/t/1e9:7.1f} GB/s")
