"""Thin torch-tensor wrappers over the per-op C-ABI (include/rlhf_kernels.h).

Used by the GPU numerics tests and for ad-hoc kernel timing.  The engine itself
(csrc/host/engine.cpp) calls the same entry points from C++.  Every call goes to
the sm_100a library; there is no fallback.
"""
from __future__ import annotations

import ctypes as C

import torch

from .capi import lib


class GemmParams(C.Structure):
    _fields_ = [("M", C.c_int), ("N", C.c_int), ("K", C.c_int), ("batch", C.c_int), ("batch_h", C.c_int),
                ("A", C.c_void_p), ("a_mn_major", C.c_int), ("lda", C.c_int64), ("a_stride_h", C.c_int64),
                ("a_stride_b", C.c_int64),
                ("B", C.c_void_p), ("b_mn_major", C.c_int), ("ldb", C.c_int64), ("b_stride_h", C.c_int64),
                ("b_stride_b", C.c_int64),
                ("C", C.c_void_p), ("c_f32", C.c_int), ("c_rs", C.c_int64), ("c_cs", C.c_int64),
                ("c_stride_h", C.c_int64), ("c_stride_b", C.c_int64),
                ("alpha", C.c_float), ("accumulate", C.c_int),
                ("bias", C.c_void_p), ("bias_f32", C.c_int), ("bias_along_m", C.c_int),
                ("relu", C.c_int),
                ("aux", C.c_void_p), ("aux_rs", C.c_int64), ("aux_cs", C.c_int64),
                ("residual", C.c_void_p), ("causal", C.c_int), ("split_k", C.c_int), ("block_n", C.c_int),
                ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
                ("counters", C.c_void_p), ("counters_len", C.c_int), ("probe", C.c_void_p), ("top2", C.c_void_p),
                ("lse_part", C.c_void_p), ("lse_tgt", C.c_void_p), ("lse_tokens", C.c_void_p), ("lse_S", C.c_int),
                ("lse_P", C.c_int), ("lse_R", C.c_int)]


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _declare_gemm():
    L = lib()
    L.rlhf_gemm.argtypes = [C.POINTER(GemmParams), C.c_void_p]
    L.rlhf_gemm_workspace_bytes.argtypes = [C.POINTER(GemmParams)]
    L.rlhf_gemm_workspace_bytes.restype = C.c_size_t
    return L


def gemm(a: torch.Tensor, b: torch.Tensor, *, a_mn: bool = False, b_mn: bool = False, out: torch.Tensor | None = None,
         out_f32: bool = True, alpha: float = 1.0, accumulate: bool = False, bias: torch.Tensor | None = None,
         bias_along_m: bool = False, relu: bool = False, aux: torch.Tensor | None = None,
         residual: torch.Tensor | None = None, split_k: int = 1,
         block_n: int = 0, swap_out: bool = False) -> torch.Tensor:
    """2-D GEMM: C[M,N] = A[M,K] . B[N,K]^T with the C-ABI's operand conventions.

    a_mn: `a` is stored [K, M] (M contiguous); b_mn: `b` is stored [K, N].
    swap_out: write C transposed (element (m,n) at n*M + m) into `out` [N, M].
    """
    L = _declare_gemm()
    M = a.shape[1] if a_mn else a.shape[0]
    K = a.shape[0] if a_mn else a.shape[1]
    N = b.shape[1] if b_mn else b.shape[0]
    if out is None:
        shape = (N, M) if swap_out else (M, N)
        out = torch.zeros(shape, device=a.device, dtype=torch.float32 if out_f32 else torch.bfloat16)
    p = GemmParams()
    p.M, p.N, p.K, p.batch, p.batch_h = M, N, K, 1, 1
    p.A, p.a_mn_major, p.lda = a.data_ptr(), int(a_mn), a.stride(0)
    p.B, p.b_mn_major, p.ldb = b.data_ptr(), int(b_mn), b.stride(0)
    p.C, p.c_f32 = out.data_ptr(), int(out.dtype == torch.float32)
    p.c_rs, p.c_cs = (1, M) if swap_out else (out.stride(0), 1)
    p.alpha, p.accumulate = alpha, int(accumulate)
    if bias is not None:
        p.bias, p.bias_f32, p.bias_along_m = bias.data_ptr(), int(bias.dtype == torch.float32), int(bias_along_m)
    p.relu = int(relu)
    if aux is not None:
        p.aux, p.aux_rs, p.aux_cs = aux.data_ptr(), p.c_rs, p.c_cs
    if residual is not None:
        p.residual = residual.data_ptr()
    p.split_k, p.block_n = split_k, block_n
    keep = []
    if split_k > 1:
        ws_bytes = L.rlhf_gemm_workspace_bytes(C.byref(p))
        ws = torch.empty(ws_bytes // 4 + 1, device=a.device, dtype=torch.float32)
        cnt = torch.zeros(65536, device=a.device, dtype=torch.int32)
        keep += [ws, cnt]
        p.workspace, p.workspace_bytes = ws.data_ptr(), ws_bytes
        p.counters, p.counters_len = cnt.data_ptr(), cnt.numel()
    st = L.rlhf_gemm(C.byref(p), _stream())
    if st != 0:
        raise RuntimeError(f"rlhf_gemm failed with status {st}")
    return out


def gemm_kernel_name(M: int, N: int, K: int) -> str:
    """Kernel rlhf_gemm dispatches a row-major bf16 Y[M,N] = X[M,K] W[N,K]^T to."""
    L = lib()
    L.rlhf_gemm_kernel_name.argtypes = [C.POINTER(GemmParams)]
    L.rlhf_gemm_kernel_name.restype = C.c_char_p
    p = GemmParams()
    p.M, p.N, p.K, p.batch, p.batch_h = M, N, K, 1, 1
    p.lda, p.ldb, p.c_rs, p.c_cs = K, K, N, 1
    return L.rlhf_gemm_kernel_name(C.byref(p)).decode()


def gemm_batched(params: GemmParams) -> None:
    L = _declare_gemm()
    st = L.rlhf_gemm(C.byref(params), _stream())
    if st != 0:
        raise RuntimeError(f"rlhf_gemm failed with status {st}")


class GemmDecodeParams(C.Structure):
    _fields_ = [("M", C.c_int), ("N", C.c_int), ("K", C.c_int), ("W", C.c_void_p), ("ldw", C.c_int64),
                ("X", C.c_void_p), ("ldx", C.c_int64), ("Y", C.c_void_p), ("y_f32", C.c_int), ("ldy", C.c_int64),
                ("bias", C.c_void_p), ("relu", C.c_int), ("residual", C.c_void_p), ("splits", C.c_int),
                ("pdl", C.c_int), ("probe", C.c_void_p), ("ln_x", C.c_void_p), ("ln_g", C.c_void_p),
                ("ln_b", C.c_void_p), ("kcache", C.c_void_p), ("vcache", C.c_void_p), ("pos", C.c_void_p),
                ("kv_d", C.c_int), ("kv_hd", C.c_int), ("kv_H", C.c_int), ("kv_Smax", C.c_int),
                ("ln_stats_out", C.c_void_p), ("ln_stats_parts_out", C.c_void_p), ("ln_stats_in", C.c_void_p),
                ("ln_stats_parts", C.c_int)]


def gemm_decode(W: torch.Tensor, X: torch.Tensor, *, out: torch.Tensor | None = None, bias=None, relu=False,
                residual=None, splits: int = 1, out_f32: bool = True, probe=None, ln=None, stats_out=None,
                stats_in=None) -> torch.Tensor:
    """Y[N, M] = X[N, K] . W[M, K]^T (+bias[M]) (relu) (+residual) via rlhf_gemm_decode."""
    L = lib()
    L.rlhf_gemm_decode.argtypes = [C.POINTER(GemmDecodeParams), C.c_void_p]
    M, K = W.shape
    N = X.shape[0] if X is not None else ln[0].shape[0]
    if out is None:
        out = torch.zeros(N, M, device=W.device, dtype=torch.float32 if out_f32 else torch.bfloat16)
    p = GemmDecodeParams(M, N, K, W.data_ptr(), W.stride(0), X.data_ptr() if X is not None else None,
                         X.stride(0) if X is not None else K, out.data_ptr(),
                         int(out.dtype == torch.float32), out.stride(0), bias.data_ptr() if bias is not None else None,
                         int(relu), residual.data_ptr() if residual is not None else None, splits, 0,
                         probe.data_ptr() if probe is not None else None)
    if ln is not None:  # (x fp32 [N, K], gamma bf16 [K], beta bf16 [K])
        p.ln_x, p.ln_g, p.ln_b = ln[0].data_ptr(), ln[1].data_ptr(), ln[2].data_ptr()
    parts = C.c_int(0)
    if stats_out is not None:  # partials fp32 [>= CTAs * N * 2]; the CTA count comes back on the host
        p.ln_stats_out, p.ln_stats_parts_out = stats_out.data_ptr(), C.cast(C.pointer(parts), C.c_void_p)
    if stats_in is not None:  # (partials, count)
        p.ln_stats_in, p.ln_stats_parts = stats_in[0].data_ptr(), int(stats_in[1])
    st = L.rlhf_gemm_decode(C.byref(p), _stream())
    if st != 0:
        raise RuntimeError(f"rlhf_gemm_decode failed with status {st}")
    return (out, parts.value) if stats_out is not None else out


def layernorm(x: torch.Tensor, g: torch.Tensor, b: torch.Tensor) -> torch.Tensor:
    """bf16(LayerNorm(x) * g + b) of fp32 rows x [N, d] via rlhf_layernorm (eps 1e-5)."""
    L = lib()
    L.rlhf_layernorm.argtypes = [C.c_void_p] * 6 + [C.c_int, C.c_int, C.c_void_p]
    N, d = x.shape
    y = torch.empty(N, d, device=x.device, dtype=torch.bfloat16)
    st = L.rlhf_layernorm(x.data_ptr(), g.data_ptr(), b.data_ptr(), y.data_ptr(), None, None, N, d, _stream())
    if st != 0:
        raise RuntimeError(f"rlhf_layernorm failed with status {st}")
    return y


def attn_decode(qkv: torch.Tensor, kcache: torch.Tensor, vcache: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
    """Decode attention of one new token per sample (rlhf_attn_decode).

    qkv [B, 3*d] bf16 (q in columns [0, d)); kcache / vcache [B, H, Smax, hd] bf16;
    pos int32[1] on the device: keys [0, pos] are attended.  Returns [B, d] bf16.
    """
    L = lib()
    L.rlhf_attn_decode.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.c_void_p, C.c_void_p]
    B, H, Smax, hd = kcache.shape
    out = torch.empty(B, H * hd, device=qkv.device, dtype=torch.bfloat16)
    rc = L.rlhf_attn_decode(qkv.data_ptr(), B, H, hd, Smax, kcache.data_ptr(), vcache.data_ptr(), pos.data_ptr(),
                            out.data_ptr(), _stream())
    if rc:
        raise RuntimeError(f"rlhf_attn_decode failed ({rc})")
    return out


def attn_bwd_ds_fused(dO: torch.Tensor, qkv: torch.Tensor, P: torch.Tensor, B: int, H: int, S: int,
                      scale: float) -> torch.Tensor:
    """Score gradient of causal attention (rlhf_attn_bwd_ds_fused): dS = bf16(P (dO V^T - D) scale),
    D = rowsum(P * dO V^T); dS bf16 [B, H, S, S], columns past the query block's diagonal tile
    left 0 (the buffer is zero-initialised here)."""
    L = lib()
    L.rlhf_attn_bwd_ds_fused.argtypes = [C.c_void_p] * 4 + [C.c_int] * 4 + [C.c_float, C.c_void_p]
    hd = qkv.shape[1] // (3 * H)
    dS = torch.zeros(B, H, S, S, device=qkv.device, dtype=torch.bfloat16)
    rc = L.rlhf_attn_bwd_ds_fused(dO.data_ptr(), qkv.data_ptr(), P.data_ptr(), dS.data_ptr(), B, H, hd, S, scale,
                                  _stream())
    if rc:
        raise RuntimeError(f"rlhf_attn_bwd_ds_fused failed ({rc})")
    return dS


def attn_fwd_fused(qkv: torch.Tensor, B: int, H: int, S: int, alpha: float, want_p: bool = True, want_o: bool = True):
    """Fused causal attention forward (rlhf_attn_fwd_fused) from packed qkv rows:
    returns (P bf16 [B, H, S, S] or None, O bf16 [B*S, H*hd] or None)."""
    L = lib()
    L.rlhf_attn_fwd_fused.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p,
                                      C.c_void_p]
    hd = qkv.shape[1] // (3 * H)
    P = torch.zeros(B, H, S, S, device=qkv.device, dtype=torch.bfloat16) if want_p else None
    O = torch.zeros(B * S, H * hd, device=qkv.device, dtype=torch.bfloat16) if want_o else None
    rc = L.rlhf_attn_fwd_fused(qkv.data_ptr(), B, H, hd, S, alpha, P.data_ptr() if want_p else None,
                               O.data_ptr() if want_o else None, _stream())
    if rc:
        raise RuntimeError(f"rlhf_attn_fwd_fused failed ({rc})")
    return P, O
