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
