"""LLaMA-family element kernels (csrc/kernels/llama.cu, rowwise.cu RMS path) against
plain torch fp32 references of the same ops, through the C-ABI.

Tolerances: outputs are bf16-rounded, so |mine - ref| <= 1 bf16 ulp of the value
(rel 2^-8) plus fp32 reassociation noise; reductions (dgamma) rel 1e-4.
"""
import ctypes as C
import math

import pytest
import torch

from paper_2312_11819_b200.capi import lib

pytestmark = pytest.mark.gpu
dev = "cuda"


def _s():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def rope_table(S, hd):
    i = torch.arange(hd // 2, dtype=torch.float64)
    ang = torch.arange(S, dtype=torch.float64)[:, None] * torch.pow(torch.tensor(10000.0, dtype=torch.float64),
                                                                     -2.0 * i / hd)[None]
    return torch.stack([torch.cos(ang).float(), torch.sin(ang).float()], -1).contiguous()  # [S, hd/2, 2]


def bf(x):
    return x.to(torch.bfloat16).float()


@pytest.mark.parametrize("M,d", [(37, 128), (256, 2048), (64, 4096), (2048, 4096), (1000, 1536), (100, 1100)])
def test_rmsnorm_fwd_bwd(M, d):
    L = lib()
    torch.manual_seed(0)
    x = torch.randn(M, d, device=dev) * 3
    g = (1 + 0.1 * torch.randn(d, device=dev)).to(torch.bfloat16)
    y = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
    rstd = torch.empty(M, device=dev)
    assert L.rlhf_rmsnorm(_p(x), _p(g), _p(y), _p(rstd), M, d, _s()) == 0
    rs = 1.0 / torch.sqrt((x * x).mean(-1) + 1e-6)
    ref = x * rs[:, None] * g.float()
    torch.testing.assert_close(y.float(), bf(ref), atol=1e-2, rtol=1e-2)
    torch.testing.assert_close(rstd, rs, rtol=1e-5, atol=0)
    # backward: dx += rs (dy g - xhat mean(dy g xhat)), dg += sum dy xhat
    dy = torch.randn(M, d, device=dev)
    dx = torch.full((M, d), 0.5, device=dev)
    dg = torch.full((d,), 0.25, device=dev)
    ws = torch.empty(((M + 15) // 16) * d + 64, device=dev)  # room for 16-row pair blocks
    L.rlhf_rmsnorm_bwd.argtypes = [C.c_void_p] * 6 + [C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
    assert L.rlhf_rmsnorm_bwd(_p(dy), _p(x), _p(rstd), _p(g), _p(dx), _p(dg), M, d, _p(ws), ws.numel(), _s()) == 0
    xr = x.clone().requires_grad_(True)
    gr = g.float().clone().requires_grad_(True)
    out = xr / torch.sqrt((xr * xr).mean(-1, keepdim=True) + 1e-6) * gr
    out.backward(dy)
    torch.testing.assert_close(dx, 0.5 + xr.grad, rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(dg, 0.25 + gr.grad, rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("M,d,ws_rows", [(50, 768, 64), (300, 2048, 16), (300, 2048, 64), (70, 1040, 64),
                                          (8192, 2048, 16)])
def test_layernorm_bwd(M, d, ws_rows):
    """LayerNorm backward (d = 2048 takes the two-warps-per-row pair kernel) vs torch autograd."""
    L = lib()
    torch.manual_seed(2)
    x = torch.randn(M, d, device=dev) * 2 + 0.3
    g = (1 + 0.1 * torch.randn(d, device=dev)).to(torch.bfloat16)
    b = (0.1 * torch.randn(d, device=dev)).to(torch.bfloat16)
    y = torch.empty(M, d, device=dev, dtype=torch.bfloat16)
    mean, rstd = torch.empty(M, device=dev), torch.empty(M, device=dev)
    assert L.rlhf_layernorm(_p(x), _p(g), _p(b), _p(y), _p(mean), _p(rstd), M, d, _s()) == 0
    dy = torch.randn(M, d, device=dev)
    dx = torch.full((M, d), 0.5, device=dev)
    dg = torch.full((d,), 0.25, device=dev)
    db = torch.full((d,), -0.25, device=dev)
    ws = torch.empty(((M + ws_rows - 1) // ws_rows) * 2 * d + 64, device=dev)
    L.rlhf_layernorm_bwd.argtypes = [C.c_void_p] * 8 + [C.c_int, C.c_int, C.c_void_p, C.c_size_t, C.c_void_p]
    assert L.rlhf_layernorm_bwd(_p(dy), _p(x), _p(mean), _p(rstd), _p(g), _p(dx), _p(dg), _p(db), M, d, _p(ws),
                                ws.numel(), _s()) == 0
    xr = x.clone().requires_grad_(True)
    gr = g.float().clone().requires_grad_(True)
    br = b.float().clone().requires_grad_(True)
    torch.nn.functional.layer_norm(xr, (d,), gr, br, 1e-5).backward(dy)
    torch.testing.assert_close(dx, 0.5 + xr.grad, rtol=1e-4, atol=1e-4)
    torch.testing.assert_close(dg, 0.25 + gr.grad, rtol=1e-4, atol=2e-3)
    torch.testing.assert_close(db, -0.25 + br.grad, rtol=1e-4, atol=2e-3)


@pytest.mark.parametrize("B,T,H,hd", [(3, 40, 4, 64), (2, 16, 2, 128)])
def test_rope_qkv_forward_inverse_and_cache(B, T, H, hd):
    L = lib()
    torch.manual_seed(1)
    d = H * hd
    S = 96
    tab = rope_table(S, hd).to(dev)
    qkv = torch.randn(B * T, 3 * d, device=dev).to(torch.bfloat16)
    orig = qkv.clone()
    p0 = 5
    Smax = 64
    kc = torch.zeros(B, H, Smax, hd, device=dev, dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    L.rlhf_rope_qkv.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    assert L.rlhf_rope_qkv(_p(qkv), B, T, p0, None, H, hd, _p(tab), 0, _p(kc), _p(vc), Smax, _s()) == 0
    pos = torch.arange(T, device=dev) + p0
    c, s = tab[pos, :, 0], tab[pos, :, 1]  # [T, hd/2]

    def rot(x):  # x [B, T, H, hd]
        x0, x1 = x[..., : hd // 2], x[..., hd // 2:]
        cc, ss = c[None, :, None], s[None, :, None]
        return torch.cat([x0 * cc - x1 * ss, x1 * cc + x0 * ss], -1)

    o = orig.float().view(B, T, 3, H, hd)
    exp_q, exp_k = bf(rot(o[:, :, 0])), bf(rot(o[:, :, 1]))
    got = qkv.float().view(B, T, 3, H, hd)
    torch.testing.assert_close(got[:, :, 0], exp_q, atol=2e-2, rtol=1e-2)
    torch.testing.assert_close(got[:, :, 1], exp_k, atol=2e-2, rtol=1e-2)
    torch.testing.assert_close(got[:, :, 2], o[:, :, 2], atol=0, rtol=0)  # v untouched
    torch.testing.assert_close(kc[:, :, p0:p0 + T].float(), got[:, :, 1].transpose(1, 2), atol=0, rtol=0)
    torch.testing.assert_close(vc[:, :, p0:p0 + T].float(), o[:, :, 2].transpose(1, 2), atol=0, rtol=0)
    assert kc[:, :, :p0].abs().sum() == 0 and kc[:, :, p0 + T:].abs().sum() == 0
    # inverse rotation brings q, k back (up to the two bf16 roundings)
    assert L.rlhf_rope_qkv(_p(qkv), B, T, p0, None, H, hd, _p(tab), 1, None, None, 0, _s()) == 0
    torch.testing.assert_close(qkv.float(), orig.float(), atol=5e-2, rtol=2e-2)


def test_rope_decode_position_from_device():
    L = lib()
    B, H, hd, Smax = 4, 2, 64, 32
    d = H * hd
    tab = rope_table(Smax, hd).to(dev)
    qkv = torch.randn(B, 3 * d, device=dev).to(torch.bfloat16)
    q_ref = qkv.clone()
    kc = torch.zeros(B, H, Smax, hd, device=dev, dtype=torch.bfloat16)
    vc = torch.zeros_like(kc)
    pos = torch.tensor([17], device=dev, dtype=torch.int32)
    assert L.rlhf_rope_qkv(_p(qkv), B, 1, 0, _p(pos), H, hd, _p(tab), 0, _p(kc), _p(vc), Smax, _s()) == 0
    q2 = q_ref.clone()
    assert L.rlhf_rope_qkv(_p(q2), B, 1, 17, None, H, hd, _p(tab), 0, None, None, 0, _s()) == 0
    torch.testing.assert_close(qkv, q2, atol=0, rtol=0)
    torch.testing.assert_close(kc[:, :, 17].reshape(B, d), qkv[:, d:2 * d], atol=0, rtol=0)


@pytest.mark.parametrize("rows,ff", [(33, 384), (128, 11008)])
def test_swiglu_fwd_bwd(rows, ff):
    L = lib()
    torch.manual_seed(2)
    gu = (torch.randn(rows, 2 * ff, device=dev) * 2).to(torch.bfloat16)
    act = torch.empty(rows, ff, device=dev, dtype=torch.bfloat16)
    assert L.rlhf_swiglu(_p(gu), _p(act), rows, ff, _s()) == 0
    g, u = gu.float()[:, :ff], gu.float()[:, ff:]
    torch.testing.assert_close(act.float(), bf(g * torch.sigmoid(g) * u), atol=1e-2, rtol=1e-2)
    dact = torch.randn(rows, ff, device=dev).to(torch.bfloat16)
    dgu = torch.empty_like(gu)
    assert L.rlhf_swiglu_bwd(_p(gu), _p(dact), _p(dgu), rows, ff, _s()) == 0
    gr, ur = g.clone().requires_grad_(True), u.clone().requires_grad_(True)
    (gr * torch.sigmoid(gr) * ur).backward(dact.float())
    torch.testing.assert_close(dgu.float()[:, :ff], bf(gr.grad), atol=2e-2, rtol=1e-2)
    torch.testing.assert_close(dgu.float()[:, ff:], bf(ur.grad), atol=2e-2, rtol=1e-2)
    assert math.isfinite(dgu.float().sum().item())
