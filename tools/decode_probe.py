"""Phase timing of the cluster split-K decode GEMM (clock64 probes, us at ~1.9 GHz).
0 entry | 1 init+TMEM | 2 weight TMA issued | 3 after griddepcontrol.wait | 4 accumulator ready |
5 partial in smem | 6 cluster barrier 1 | 7 reduction+stores done | 8 cluster barrier 2"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2312_11819_b200 import ops
for name, M, K, splits in [("Wo", 768, 768, 4), ("W2", 768, 3072, 8), ("qkv", 2304, 768, 4), ("W1", 3072, 768, 4)]:
    W = torch.randn(M, K, device="cuda").bfloat16(); X = torch.randn(32, K, device="cuda").bfloat16()
    probe = torch.zeros(4096 * 16, device="cuda", dtype=torch.int64)
    for it in range(3):
        probe.zero_(); torch.cuda.synchronize()
        ops.gemm_decode(W, X, splits=splits, probe=probe if it == 2 else None); torch.cuda.synchronize()
    pr = probe.view(-1, 16).cpu().numpy()[:, :13].astype(np.int64)
    pr = pr[pr[:, 0] > 0]
    d = (pr - pr[:, :1]) / 1.9e3
    print(f"{name:4s} ctas={len(pr):3d} median:", " ".join(f"{v:6.2f}" for v in np.median(d, 0)))
    print(f"{'':4s} {'':8s} max   :", " ".join(f"{v:6.2f}" for v in d.max(0)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ops.gemm_decode(W, X, splits=splits)
        with torch.cuda.graph(g, stream=s):
            for _ in range(20):
                ops.gemm_decode(W, X, splits=splits)
    torch.cuda.synchronize()
    e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
    print(f"     graph-replayed avg {e0.elapsed_time(e1) / 20 * 1e3:.2f} us per launch")
