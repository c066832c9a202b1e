"""One c3 FFN-down decode GEMM (M=2048, K=8192, N=16, 16 K-slices) a few times; used
under `ncu --set full` (launch 3 is profiled)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200 import ops  # noqa: E402

M, K, N, splits = int(os.environ.get("M", 2048)), int(os.environ.get("K", 8192)), 16, int(os.environ.get("SPLITS", 16))
W = torch.randn(M, K, device="cuda").bfloat16()
X = torch.randn(N, K, device="cuda").bfloat16()
out = torch.empty(N, M, device="cuda")
for _ in range(4):
    ops.gemm_decode(W, X, out=out, splits=splits)
torch.cuda.synchronize()
print("ok")
