"""Per-CTA phase timing of one tcgen05 GEMM launch (clock64 probes in gemm_sm100_kernel).

Phases: 0 entry | 1 after barrier init + TMEM alloc | 2 producer got first free slot |
3 MMA saw first stage land (TMA latency) | 4 MMA issued the unit | 5 epilogue saw the
accumulator | 6 epilogue done (partials written) | 7 unit complete (split-K fixup done).
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2312_11819_b200 import ops  # noqa: E402

CASES = [("dec Wo", 768, 32, 768, 6), ("dec W2", 768, 32, 3072, 8), ("dec qkv", 2304, 32, 768, 6),
         ("fwd W1", 16384, 3072, 768, 1)]
L = ops._declare_gemm()
for name, M, N, K, split in CASES:
    W = torch.randn(M, K, device="cuda").bfloat16()
    X = torch.randn(N, K, device="cuda").bfloat16()
    out = torch.zeros(N, M, device="cuda")
    probe = torch.zeros(4096 * 16, device="cuda", dtype=torch.int64)
    ws = torch.zeros(64 << 20, device="cuda", dtype=torch.uint8)
    cnt = torch.zeros(65536, device="cuda", dtype=torch.int32)
    p = ops.GemmParams()
    p.M, p.N, p.K, p.batch, p.batch_h = M, N, K, 1, 1
    p.A, p.lda, p.B, p.ldb = W.data_ptr(), K, X.data_ptr(), K
    if N <= 64:
        p.C, p.c_f32, p.c_rs, p.c_cs = out.data_ptr(), 1, 1, M
    else:
        out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        p.C, p.c_f32, p.c_rs, p.c_cs = out.data_ptr(), 0, N, 1
    p.alpha, p.split_k = 1.0, split
    p.workspace, p.workspace_bytes, p.counters, p.counters_len = ws.data_ptr(), ws.numel(), cnt.data_ptr(), 65536
    for it in range(3):
        probe.zero_()
        p.probe = probe.data_ptr() if it == 2 else None
        torch.cuda.synchronize()
        assert L.rlhf_gemm(C.byref(p), C.c_void_p(torch.cuda.current_stream().cuda_stream)) == 0
        torch.cuda.synchronize()
    pr = probe.view(-1, 16).cpu().numpy().astype(np.int64)
    pr = pr[pr[:, 0] > 0]
    d = (pr - pr[:, :1]).astype(np.float64) / 1.9e3  # cycles -> us at ~1.9 GHz
    med = np.median(d, axis=0)
    mx = np.max(d, axis=0)
    print(f"{name:8s} ctas={len(pr):4d}  median us per phase: " + " ".join(f"{v:7.2f}" for v in med[:12]))
    print(f"{'':8s} {'':9s}  max    us per phase: " + " ".join(f"{v:7.2f}" for v in mx[:12]))
