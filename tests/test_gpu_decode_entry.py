"""Decode step entry fused with the greedy sampler (rlhf_argmax_embed_ln / _rmsnorm) vs the
two launches it replaces (rlhf_argmax_tiles with the position advance, then rlhf_embed_ln /
rlhf_embed_rmsnorm): token, margin, position, residual row x and normalised row y must be
bit-identical, free-running (the merged token is embedded) and teacher-forced (predictions
to a separate buffer, the given token embedded).  GPU only.  Every tensor's dtype is explicit:
tests/golden/make_golden.py switches torch's default dtype to float64 when an earlier test
imports it."""
import ctypes as C

import pytest
import torch

pytestmark = pytest.mark.gpu


def _lib():
    from paper_2312_11819_b200.capi import lib
    L = lib()
    vp, i64 = C.c_void_p, C.c_int64
    L.rlhf_argmax_tiles.argtypes = [vp, C.c_int, C.c_int, vp, i64, vp, vp, C.c_int, vp]
    L.rlhf_embed_ln.argtypes = [vp, i64, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, vp, vp]
    L.rlhf_embed_rmsnorm.argtypes = [vp, i64, C.c_int, vp, vp, C.c_int, vp, vp, vp, vp]
    L.rlhf_argmax_embed_ln.argtypes = [vp, C.c_int, vp, vp, vp, i64, C.c_int, vp, vp, vp, C.c_int, vp, vp, vp, vp, vp]
    L.rlhf_argmax_embed_rmsnorm.argtypes = [vp, C.c_int, vp, vp, vp, i64, C.c_int, vp, vp, C.c_int, vp, vp, vp, vp]
    return L


def _top2_partials(logits):
    """[B, V] fp32 -> [tiles, B, 4] (max, row id bits, second max, 0) per 128-row tile."""
    B, V = logits.shape
    tiles = (V + 127) // 128
    pad = torch.full((B, tiles * 128), -float("inf"), device=logits.device, dtype=torch.float32)
    pad[:, :V] = logits
    v, i = pad.view(B, tiles, 128).topk(2, dim=2)
    ids = (i[..., 0] + torch.arange(tiles, device=logits.device).view(1, -1) * 128).int()
    out = torch.zeros(tiles, B, 4, device=logits.device, dtype=torch.float32)
    out[..., 0] = v[..., 0].t()
    out[..., 1] = ids.t().contiguous().view(torch.float32)
    out[..., 2] = v[..., 1].t()
    return out, tiles


@pytest.mark.parametrize("rms", [False, True])
@pytest.mark.parametrize("teacher", [False, True])
@pytest.mark.parametrize("B,d,V", [(32, 768, 50272), (13, 2048, 1000)])
def test_argmax_embed_matches_two_launches(rms, teacher, B, d, V):
    torch.manual_seed(B + d)
    L = _lib()
    S = 24
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    E = (torch.randn(V, d, device="cuda", dtype=torch.float32) * 0.1).bfloat16()
    Pm = (torch.randn(S, d, device="cuda", dtype=torch.float32) * 0.1).bfloat16()
    g = (1 + 0.1 * torch.randn(d, device="cuda", dtype=torch.float32)).bfloat16()
    b = (0.1 * torch.randn(d, device="cuda", dtype=torch.float32)).bfloat16()
    t2, tiles = _top2_partials(torch.randn(B, V, device="cuda", dtype=torch.float32))
    tok0 = torch.randint(0, V, (B, S), device="cuda", dtype=torch.int32)
    p0 = 9
    outs = []
    for fused in (False, True):
        tok = tok0.clone()
        pred = torch.full((B, S), -1, device="cuda", dtype=torch.int32)
        dst = pred if teacher else tok
        margin = torch.zeros(B, S, device="cuda", dtype=torch.float32)
        pos = torch.tensor([p0, 0], device="cuda", dtype=torch.int32)
        x = torch.zeros(B, d, device="cuda", dtype=torch.float32)
        y = torch.zeros(B, d, device="cuda", dtype=torch.bfloat16)
        if fused:
            if rms:
                r = L.rlhf_argmax_embed_rmsnorm(t2.data_ptr(), tiles, dst.data_ptr(), margin.data_ptr(), tok.data_ptr(), S,
                                                B, pos.data_ptr(), E.data_ptr(), d, x.data_ptr(), g.data_ptr(),
                                                y.data_ptr(), st)
            else:
                r = L.rlhf_argmax_embed_ln(t2.data_ptr(), tiles, dst.data_ptr(), margin.data_ptr(), tok.data_ptr(), S, B,
                                           pos.data_ptr(), E.data_ptr(), Pm.data_ptr(), d, x.data_ptr(), g.data_ptr(),
                                           b.data_ptr(), y.data_ptr(), st)
            assert r == 0
        else:
            assert L.rlhf_argmax_tiles(t2.data_ptr(), tiles, B, dst.data_ptr(), S, pos.data_ptr(), margin.data_ptr(), 1,
                                       st) == 0
            if rms:
                r = L.rlhf_embed_rmsnorm(tok.data_ptr(), S, B, pos.data_ptr(), E.data_ptr(), d, x.data_ptr(),
                                         g.data_ptr(), y.data_ptr(), st)
            else:
                r = L.rlhf_embed_ln(tok.data_ptr(), S, B, pos.data_ptr(), E.data_ptr(), Pm.data_ptr(), d, x.data_ptr(),
                                    g.data_ptr(), b.data_ptr(), y.data_ptr(), st)
            assert r == 0
        torch.cuda.synchronize()
        outs.append((tok, pred, margin, pos, x, y))
    for a, c in zip(*outs):
        assert torch.equal(a, c)
    tok, pred, margin, pos, x, y = outs[1]
    assert pos.tolist() == [p0 + 1, 0]  # advanced once, ticket reset
    # the merged token is the full-vocabulary argmax of the partials
    exp = t2[..., 1].t().contiguous().view(torch.int32).gather(1, t2[..., 0].t().argmax(dim=1, keepdim=True)).squeeze(1)
    assert torch.equal((pred if teacher else tok)[:, p0 + 1], exp)
