"""FlashMatch (K7): tcgen05 online-softmax attention for the MASt3R ViT blocks.

Speedy MASt3R replaces the self/cross attention of the ViT-Large encoder and
ViT-Base decoder with a FlashAttention-2 style fused kernel (
the reference ships no code for it).  This module is the
Python face of ``fnl_flashmatch_fwd`` (include/fastnn_b200.h): binary16
Q/K/V/O, fp32 scores and accumulation, head_dim 64, non-causal.

PyTorch is only the container for device memory and the stream; the attention
itself always runs in ``libfastnn_b200.so`` -- there is no fallback path.
"""
import math

from . import _fastnn

HEAD_DIM = 64


def _strides3(t):
    """[B, H, N, 64] view -> element strides (batch, head, token)."""
    if t.dim() != 4 or t.shape[-1] != HEAD_DIM or t.stride(-1) != 1:
        raise ValueError("flashmatch: tensors must be [B, H, N, 64] with a contiguous head_dim")
    return (t.stride(0), t.stride(1), t.stride(2))


def flashmatch(q, k, v, scale=None, out=None):
    """softmax(q k^T * scale) v for [B, H, N, 64] binary16 CUDA tensors.

    Any [B, H, N, 64] views are accepted as long as head_dim is contiguous and
    strides are multiples of 8 elements -- e.g. q/k/v sliced out of a fused QKV
    projection ``qkv.view(B, N, 3, H, 64).permute(2, 0, 3, 1, 4)`` without a
    copy.  ``out`` (same convention) receives the result; by default a new
    contiguous [B, H, Nq, 64] tensor.  Runs asynchronously on torch's current
    stream.
    """
    import torch

    for name, t in (("q", q), ("k", k), ("v", v)):
        if t.dtype != torch.float16 or not t.is_cuda:
            raise ValueError(f"flashmatch: {name} must be a float16 CUDA tensor")
    B, H, Nq, D = q.shape
    if k.shape[:2] != (B, H) or v.shape != k.shape or D != HEAD_DIM:
        raise ValueError(f"flashmatch: shape mismatch q{tuple(q.shape)} k{tuple(k.shape)} v{tuple(v.shape)}")
    Nkv = k.shape[2]
    if out is None:
        out = torch.empty((B, H, Nq, D), dtype=torch.float16, device=q.device)
    elif out.shape != q.shape or out.dtype != torch.float16:
        raise ValueError("flashmatch: out must match q")
    if scale is None:
        scale = 1.0 / math.sqrt(D)
    stream = torch.cuda.current_stream(q.device).cuda_stream
    _fastnn._flashmatch_fwd(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), B, H, Nq, Nkv, D,
                            float(scale), _strides3(q), _strides3(k), _strides3(v), _strides3(out), stream)
    return out
