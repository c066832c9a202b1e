"""Decode attention (rlhf_attn_decode) vs a plain PyTorch fp32 reference.

Contract: scores in fp32, probabilities normalised then rounded
to bf16, P.V accumulated in fp32, output rounded to bf16.  Contexts cover one
staged chunk, exact chunk boundaries and several chunks (C = 256 positions for
hd 64, 128 for hd 128).
"""
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("hd,H", [(64, 12), (128, 4)])
@pytest.mark.parametrize("ctx", [1, 17, 128, 129, 256, 257, 700, 1280])
def test_attn_decode_matches_torch(hd, H, ctx):
    import torch
    from paper_2312_11819_b200 import ops
    torch.manual_seed(ctx * 7 + hd)
    B, Smax = 5, 1280
    d = H * hd
    qkv = torch.randn(B, 3 * d, device="cuda").bfloat16()
    kc = torch.randn(B, H, Smax, hd, device="cuda").bfloat16()
    vc = torch.randn(B, H, Smax, hd, device="cuda").bfloat16()
    pos = torch.tensor([ctx - 1], device="cuda", dtype=torch.int32)
    got = ops.attn_decode(qkv, kc, vc, pos).float()
    q = qkv[:, :d].float().view(B, H, 1, hd)
    s = (q @ kc[:, :, :ctx].float().transpose(-1, -2)) / hd ** 0.5
    p = torch.softmax(s, -1).bfloat16().float()
    ref = (p @ vc[:, :, :ctx].float()).view(B, d)
    torch.testing.assert_close(got, ref, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("ctx", [1, 190, 193, 384, 511])
def test_attn_decode_large_grid_matches_torch(ctx):
    """B*H > 3 CTAs per SM (OPT-1.3B decode: 16 x 32): the 3-slot ring variant."""
    import torch
    from paper_2312_11819_b200 import ops
    torch.manual_seed(ctx)
    B, H, hd, Smax = 16, 32, 64, 512
    d = H * hd
    qkv = torch.randn(B, 3 * d, device="cuda").bfloat16()
    kc = torch.randn(B, H, Smax, hd, device="cuda").bfloat16()
    vc = torch.randn(B, H, Smax, hd, device="cuda").bfloat16()
    pos = torch.tensor([ctx - 1], device="cuda", dtype=torch.int32)
    got = ops.attn_decode(qkv, kc, vc, pos).float()
    q = qkv[:, :d].float().view(B, H, 1, hd)
    s = (q @ kc[:, :, :ctx].float().transpose(-1, -2)) / hd ** 0.5
    p = torch.softmax(s, -1).bfloat16().float()
    ref = (p @ vc[:, :, :ctx].float()).view(B, d)
    torch.testing.assert_close(got, ref, atol=2e-2, rtol=2e-2)


@pytest.mark.parametrize("B,H,S", [(2, 3, 128), (2, 12, 512), (3, 4, 256)])
def test_attn_fwd_fused_matches_torch(B, H, S):
    """Fused attention forward (tcgen05 scores in TMEM, online softmax, P tiles in smem,
    P.V accumulated in TMEM) vs fp32 torch: P within bf16 rounding with exact zeros above
    the diagonal, O = bf16(P_bf16 V) within bf16 rounding; P-only and O-only modes agree."""
    import torch
    from paper_2312_11819_b200 import ops
    torch.manual_seed(S + H)
    hd = 64
    d = H * hd
    qkv = (torch.randn(B * S, 3 * d, device="cuda") * 1.5).bfloat16()
    P, O = ops.attn_fwd_fused(qkv, B, H, S, 0.125)
    q = qkv[:, :d].float().view(B, S, H, hd).transpose(1, 2)
    k = qkv[:, d:2 * d].float().view(B, S, H, hd).transpose(1, 2)
    v = qkv[:, 2 * d:].float().view(B, S, H, hd).transpose(1, 2)
    s = (q @ k.transpose(-1, -2)) * 0.125
    mask = torch.ones(S, S, device="cuda", dtype=torch.bool).tril()
    ref = torch.softmax(s.masked_fill(~mask, float("-inf")), -1)
    torch.cuda.synchronize()
    Pf = P.float()
    assert (Pf - ref).abs().max().item() <= 4e-3 * ref.abs().max().item() + 1e-6
    assert (Pf[..., ~mask] == 0).all()
    # O from the kernel's own bf16 probabilities (the rounding contract), fp32 accumulation
    o_ref = (Pf @ v).transpose(1, 2).reshape(B * S, d)
    assert (O.float() - o_ref).abs().max().item() <= 1e-2 * o_ref.abs().max().item() + 1e-3
    P2, _ = ops.attn_fwd_fused(qkv, B, H, S, 0.125, want_o=False)
    _, O2 = ops.attn_fwd_fused(qkv, B, H, S, 0.125, want_p=False)
    torch.cuda.synchronize()
    assert torch.equal(P2, P) and torch.equal(O2, O)


@pytest.mark.gpu
@pytest.mark.parametrize("B,H,S", [(2, 3, 128), (2, 4, 256), (1, 2, 384), (3, 2, 512)])
def test_attn_bwd_ds_fused_matches_torch(B, H, S):
    """Fused score gradient (dO V^T in TMEM, D = rowsum(P dP), dS = bf16(P (dP - D) scale)) against
    fp32 torch on the kernel's own bf16 P, and against the unfused GEMM + softmax-backward pair."""
    import ctypes as C
    import torch
    from paper_2312_11819_b200 import ops
    from paper_2312_11819_b200.capi import lib
    torch.manual_seed(B * S + H)
    hd, d, scale = 64, H * 64, 0.125
    qkv = (torch.randn(B * S, 3 * d, device="cuda") * 1.5).bfloat16()
    dO = torch.randn(B * S, d, device="cuda").bfloat16()
    P, _ = ops.attn_fwd_fused(qkv, B, H, S, scale)
    dS = ops.attn_bwd_ds_fused(dO, qkv, P, B, H, S, scale)
    v = qkv[:, 2 * d:].float().view(B, S, H, hd).transpose(1, 2)
    g = dO.float().view(B, S, H, hd).transpose(1, 2)
    dP = g @ v.transpose(-1, -2)
    Pf = P.float()
    D = (Pf * dP).sum(-1, keepdim=True)
    ref = Pf * (dP - D) * scale
    mask = torch.ones(S, S, device="cuda", dtype=torch.bool).tril()
    torch.cuda.synchronize()
    got = dS.float()
    assert (got[..., ~mask] == 0).all()
    err = (got - ref).abs().max().item()
    assert err <= 1e-2 * ref.abs().max().item() + 1e-4, err
    # the unfused pair: fp32 dP from the batched GEMM path, then rlhf_attn_softmax_bwd
    L = lib()
    L.rlhf_attn_softmax_bwd.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_float, C.c_void_p]
    dPc = dP.contiguous()
    dS2 = torch.zeros_like(dS)
    assert L.rlhf_attn_softmax_bwd(P.data_ptr(), dPc.data_ptr(), dS2.data_ptr(), B * H, S, scale, ops._stream()) == 0
    torch.cuda.synchronize()
    # same inputs up to the fp32 summation order of dP and D: bf16 results within one rounding step
    diff = (got - dS2.float()).abs()
    assert diff.max().item() <= 2e-2 * ref.abs().max().item() + 1e-4
    assert (diff > 0).float().mean().item() < 0.05
