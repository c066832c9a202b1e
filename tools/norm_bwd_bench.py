"""Time rlhf_layernorm_bwd / rlhf_rmsnorm_bwd at training shapes (CUDA events, 20 reps).

    python tools/norm_bwd_bench.py
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200.capi import lib  # noqa: E402

L = lib()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
P = lambda t: C.c_void_p(t.data_ptr())
L.rlhf_rmsnorm_bwd.argtypes = [C.c_void_p] * 6 + [C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
L.rlhf_layernorm_bwd.argtypes = [C.c_void_p] * 8 + [C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
for kind, M, d in [("ln", 16384, 768), ("ln", 8192, 2048), ("rms", 8192, 2048), ("rms", 4096, 4096),
                   ("rms", 1024, 4096), ("rms", 2048, 4096), ("ln", 2048, 2048), ("ln", 4096, 2048), ("rms", 8192, 4096)]:
    x, dy, dx = (torch.randn(M, d, device="cuda") for _ in range(3))
    mean, rstd = torch.randn(M, device="cuda"), torch.rand(M, device="cuda") + 0.5
    g = torch.randn(d, device="cuda").bfloat16()
    dg, db = torch.zeros(d, device="cuda"), torch.zeros(d, device="cuda")
    ws = torch.empty((M // 8 + 1) * 2 * d + 64, device="cuda")  # room for any rows-per-block

    def run():
        if kind == "rms":
            return L.rlhf_rmsnorm_bwd(P(dy), P(x), P(rstd), P(g), P(dx), P(dg), M, d, P(ws), ws.numel(), s)
        return L.rlhf_layernorm_bwd(P(dy), P(x), P(mean), P(rstd), P(g), P(dx), P(dg), P(db), M, d, P(ws), ws.numel(), s)
    for _ in range(3):
        assert run() == 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        run()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 20
    byts = 4.0 * M * d * 4  # dy, x read; dx read + write
    print(f"{kind:3s} M={M:6d} d={d:5d}: {us:8.1f} us  {byts / us / 1e3:6.0f} GB/s", flush=True)
