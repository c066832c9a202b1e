"""Time the batched attention GEMMs of the c2 training step (B=32, H=12, S=512, hd=64)
through the C-ABI (CUDA events, warm): S = QK^T (causal tile skip), O = P V (causal
k-range), dV = P^T dO, dQ = dS K, dK = dS^T Q, dP = dO V^T."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2312_11819_b200.ops import GemmParams, gemm_batched  # noqa: E402

B, S, H, hd = 32, 512, 12, 64
d = H * hd
qkv = torch.randn(B * S, 3 * d, device="cuda").bfloat16()
P = torch.randn(B, H, S, S, device="cuda").bfloat16()
dO = torch.randn(B * S, d, device="cuda").bfloat16()
out_s = torch.empty(B, H, S, S, device="cuda")
out_o = torch.empty(B * S, d, device="cuda").bfloat16()


def params(M, N, K, A, a_mn, lda, ash, asb, Bp, b_mn, ldb, bsh, bsb, C, c_f32, crs, ccs, csh, csb, causal):
    p = GemmParams()
    p.M, p.N, p.K, p.batch, p.batch_h = M, N, K, B * H, H
    p.A, p.a_mn_major, p.lda, p.a_stride_h, p.a_stride_b = A, a_mn, lda, ash, asb
    p.B, p.b_mn_major, p.ldb, p.b_stride_h, p.b_stride_b = Bp, b_mn, ldb, bsh, bsb
    p.C, p.c_f32, p.c_rs, p.c_cs, p.c_stride_h, p.c_stride_b = C, c_f32, crs, ccs, csh, csb
    p.alpha, p.causal = 1.0, causal
    return p


q, k, v = qkv.data_ptr(), qkv.data_ptr() + 2 * d, qkv.data_ptr() + 4 * d
cases = {
    "QK^T (S fp32)": params(S, S, hd, q, 0, 3 * d, hd, S * 3 * d, k, 0, 3 * d, hd, S * 3 * d,
                            out_s.data_ptr(), 1, S, 1, S * S, H * S * S, 1),
    "P V (O bf16)": params(S, hd, S, P.data_ptr(), 0, S, S * S, H * S * S, v, 1, 3 * d, hd, S * 3 * d,
                           out_o.data_ptr(), 0, d, 1, hd, S * d, 2),
    "P^T dO (dV)": params(S, hd, S, P.data_ptr(), 1, S, S * S, H * S * S, dO.data_ptr(), 1, d, hd, S * d,
                          out_o.data_ptr(), 0, d, 1, hd, S * d, 3),
}
for name, p in cases.items():
    for _ in range(3):
        gemm_batched(p)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gemm_batched(p)
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 10 * 1e-3
    fl = 2.0 * B * H * S * S * hd / 2
    print(f"{name:16s} {t*1e6:8.1f} us   {fl/t/1e12:7.1f} TFLOP/s (causal half)")

# fused scores + softmax vs QK^T GEMM (fp32 scores) + softmax kernel
from paper_2312_11819_b200 import ops  # noqa: E402
from paper_2312_11819_b200.capi import lib  # noqa: E402
import ctypes as C  # noqa: E402

Pf = torch.zeros(B, H, S, S, device="cuda", dtype=torch.bfloat16)
L = lib()
L.rlhf_attn_fwd_fused.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p,
                                  C.c_void_p]
L.rlhf_attn_softmax.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
for name, f in [("fused -> P", lambda: L.rlhf_attn_fwd_fused(qkv.data_ptr(), B, H, hd, S, 0.125, Pf.data_ptr(), None, st)),
                ("fused -> O", lambda: L.rlhf_attn_fwd_fused(qkv.data_ptr(), B, H, hd, S, 0.125, None, out_o.data_ptr(), st)),
                ("fused -> P, O", lambda: L.rlhf_attn_fwd_fused(qkv.data_ptr(), B, H, hd, S, 0.125, Pf.data_ptr(),
                                                                out_o.data_ptr(), st)),
                ("softmax only", lambda: L.rlhf_attn_softmax(out_s.data_ptr(), Pf.data_ptr(), B * H, S, st))]:
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:16s} {e0.elapsed_time(e1) / 10 * 1e3:8.1f} us")
