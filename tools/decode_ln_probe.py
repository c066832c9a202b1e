"""Decode GEMM with and without the fused LayerNorm prologue (clock64 probes + graph timing).
Phases as tools/decode_probe.py (3 = operand ready: after the wait, or after the LN prologue)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_11819_b200 import ops
for name, M, K, N, splits in [("c2 qkv", 2304, 768, 32, 4), ("c2 W1", 3072, 768, 32, 4), ("c3 qkv", 6144, 2048, 16, 4)]:
    W = torch.randn(M, K, device="cuda").bfloat16(); X = torch.randn(N, K, device="cuda").bfloat16()
    x = torch.randn(N, K, device="cuda"); g = torch.randn(K, device="cuda").bfloat16(); b = torch.randn(K, device="cuda").bfloat16()
    for ln in (None, (x, g, b)):
        probe = torch.zeros(4096 * 16, device="cuda", dtype=torch.int64)
        for it in range(3):
            probe.zero_(); torch.cuda.synchronize()
            ops.gemm_decode(W, X, splits=splits, probe=probe if it == 2 else None, ln=ln); torch.cuda.synchronize()
        pr = probe.view(-1, 16).cpu().numpy()[:, :9].astype(np.int64)
        pr = pr[pr[:, 0] > 0]
        d = (pr - pr[:, :1]) / 1.9e3
        tag = f"{name} {'ln' if ln else '--'}"
        print(f"{tag:10s} ctas={len(pr):3d} median:", " ".join(f"{v:6.2f}" for v in np.median(d, 0)))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gr = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ops.gemm_decode(W, X, splits=splits, ln=ln)
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    ops.gemm_decode(W, X, splits=splits, ln=ln)
        torch.cuda.synchronize()
        e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
        print(f"{'':10s} graph-replayed avg {e0.elapsed_time(e1) / 20 * 1e3:.2f} us per launch")
