"""Run the c2 FFN up-projection GEMM (M=16384, N=3072, K=768, bf16 out) a few times
through the C-ABI; used under `ncu --set full` for profiles/ (launch 4 is profiled)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200 import ops  # noqa: E402

M, N, K = 16384, 3072, 768
x = torch.randn(M, K, device="cuda").bfloat16()
w = torch.randn(N, K, device="cuda").bfloat16()
y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(5):
    ops.gemm(x, w, out=y, out_f32=False)
torch.cuda.synchronize()
print("ok")
