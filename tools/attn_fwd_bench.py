"""Time rlhf_attn_fwd_fused (the fused causal attention forward) alone at the c2 shape,
v2 (default) against v1 (RLHF_ATTN_FWD_V1=1 in a second process).

    python tools/attn_fwd_bench.py [--B 32] [--H 12] [--S 512] [--want-p]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ctypes as C  # noqa: E402

from paper_2312_11819_b200.capi import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=32)
ap.add_argument("--H", type=int, default=12)
ap.add_argument("--S", type=int, nargs="+", default=[256, 512])
a = ap.parse_args()
for S in a.S:
    d = a.H * 64
    L = lib()
    L.rlhf_attn_fwd_fused.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p,
                                      C.c_void_p, C.c_void_p]
    qkv = torch.randn(a.B * S, 3 * d, device="cuda").bfloat16()
    P = torch.empty(a.B, a.H, S, S, device="cuda", dtype=torch.bfloat16)
    O = torch.empty(a.B * S, d, device="cuda", dtype=torch.bfloat16)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def run(want_p):
        assert L.rlhf_attn_fwd_fused(qkv.data_ptr(), a.B, a.H, 64, S, 0.125, P.data_ptr() if want_p else None,
                                     O.data_ptr(), st) == 0

    for want_p in (False, True):
        for _ in range(3):
            run(want_p)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            run(want_p)
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / n * 1e3
        fl = 2 * 2 * a.B * a.H * (S * (S + 128) / 2) * 64  # causal tiles QK^T + PV
        print(f"{'v1' if os.environ.get('RLHF_ATTN_FWD_V1') else 'v2'} S={S} want_p={int(want_p)}: {t:8.1f} us "
              f"{fl / t / 1e6:7.1f} TFLOP/s")
