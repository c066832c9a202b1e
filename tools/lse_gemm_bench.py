"""Time the LM-head pair GEMM with the log-sum-exp epilogue (logits never stored) at the c2
Forward shape (rows = B*R = 8192, V = 50272, d = 768) against the same GEMM storing bf16
logits, to see what the epilogue costs on top of the tensor-core work.

    python tools/lse_gemm_bench.py [--rows 8192] [--V 50272] [--d 768]
"""
import argparse
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200.capi import lib  # noqa: E402
from paper_2312_11819_b200.ops import GemmParams, _stream  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=8192)
ap.add_argument("--V", type=int, default=50272)
ap.add_argument("--d", type=int, default=768)
a = ap.parse_args()
R, P = 256, 256
Bq = a.rows // R
x = (torch.randn(a.rows, a.d, device="cuda") * 0.5).bfloat16()
w = (torch.randn(a.V, a.d, device="cuda") * 0.1).bfloat16()
tokens = torch.randint(0, a.V, (Bq, P + R), device="cuda", dtype=torch.int32)
tiles = (a.V + 255) // 256
part = torch.empty(a.rows * tiles * 2 * 2, device="cuda")
tgt = torch.empty(a.rows, device="cuda")
out = torch.empty(a.rows, a.V, device="cuda", dtype=torch.bfloat16)
L = lib()
L.rlhf_gemm.argtypes = [C.POINTER(GemmParams), C.c_void_p]


def params(lse):
    p = GemmParams()
    p.M, p.N, p.K, p.batch, p.batch_h = a.rows, a.V, a.d, 1, 1
    p.A, p.lda, p.B, p.ldb = x.data_ptr(), a.d, w.data_ptr(), a.d
    p.C, p.c_f32, p.c_rs, p.c_cs, p.alpha = out.data_ptr(), 0, a.V, 1, 1.0
    if lse:
        p.lse_part, p.lse_tgt, p.lse_tokens = part.data_ptr(), tgt.data_ptr(), tokens.data_ptr()
        p.lse_S, p.lse_P, p.lse_R = P + R, P, R
    return p


for lse in (True, False):
    p = params(lse)
    for _ in range(3):
        assert L.rlhf_gemm(C.byref(p), _stream()) == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        L.rlhf_gemm(C.byref(p), _stream())
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / n * 1e3
    print(f"{'lse epilogue' if lse else 'bf16 logits '}: {t:8.1f} us  {2 * a.rows * a.V * a.d / t / 1e6:7.1f} TFLOP/s")
