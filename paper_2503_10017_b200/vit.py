"""Random-init MASt3R ViT blocks around FlashMatch.

MASt3R's encoder is a ViT-Large (24 blocks, width 1024, 16 heads) applied to
both images, its decoder a ViT-Base (12 blocks, width 768, 12 heads) whose
blocks run self-attention on one image's tokens and cross-attention to the
other image's tokens.  At 512x384 with 16x16 patches
each image has 768 tokens of head_dim 64.  Speedy MASt3R's FlashMatch puts a
fused attention kernel into every one of those attention calls
(PAPER.md:134-139); here that kernel is K7 (flashmatch.py).

This harness exists to measure and test K7 inside the real block structure:
LayerNorm / GEMMs / GELU are plain library ops (cuBLAS via torch, fp16), the
attention always goes through ``flashmatch``.  Weights are random (no
checkpoints offline); the local-feature head maps decoder tokens to unit-norm
24-d descriptor maps, the input of the FastNN-Lite matcher.
"""
import math

import torch
import torch.nn.functional as F

from .flashmatch import flashmatch

PATCH = 16
HEAD_DIM = 64


def _linear(g, fan_in, fan_out, device, sides=1):
    """Xavier-normal weights [sides, out, in] (sides > 1: one set per image side)."""
    w = torch.randn((sides, fan_out, fan_in), generator=g) * math.sqrt(2.0 / (fan_in + fan_out))
    return (w.to(device=device, dtype=torch.float16),
            torch.zeros((sides, 1, fan_out), device=device, dtype=torch.float16))


def _apply(x, wb):
    """x [S*, N, in] @ W^T + b with shared (S=1) or per-side weights."""
    w, b = wb
    if w.shape[0] == 1:
        return F.linear(x, w[0], b[0, 0])
    return torch.baddbmm(b, x, w.transpose(1, 2))


class Block:
    """Pre-LN transformer block: self-attn (+ cross-attn) + MLP, fp16.  The two
    image sides travel stacked as batch [2, N, C]; the decoder has one weight
    set per side (sides=2), so every attention call covers both images in ONE
    FlashMatch launch."""

    def __init__(self, g, width, heads, cross, device, sides=1):
        self.width, self.heads, self.cross = width, heads, cross
        self.qkv = _linear(g, width, 3 * width, device, sides)
        self.proj = _linear(g, width, width, device, sides)
        if cross:
            self.q_x = _linear(g, width, width, device, sides)
            self.kv_x = _linear(g, width, 2 * width, device, sides)
            self.proj_x = _linear(g, width, width, device, sides)
        self.fc1 = _linear(g, width, 4 * width, device, sides)
        self.fc2 = _linear(g, 4 * width, width, device, sides)

    def _ln(self, x):
        return F.layer_norm(x, (self.width,))

    def self_attn(self, x, attn):
        B, N, C = x.shape
        qkv = _apply(self._ln(x), self.qkv).view(B, N, 3, self.heads, HEAD_DIM).permute(2, 0, 3, 1, 4)
        o = torch.empty((B, N, C), dtype=x.dtype, device=x.device)
        attn(qkv[0], qkv[1], qkv[2], o.view(B, N, self.heads, HEAD_DIM).permute(0, 2, 1, 3))
        return x + _apply(o, self.proj)

    def cross_attn(self, x, y, attn):
        B, N, C = x.shape
        q = _apply(self._ln(x), self.q_x).view(B, N, self.heads, HEAD_DIM).permute(0, 2, 1, 3)
        kv = _apply(self._ln(y), self.kv_x).view(B, y.shape[1], 2, self.heads, HEAD_DIM).permute(2, 0, 3, 1, 4)
        o = torch.empty((B, N, C), dtype=x.dtype, device=x.device)
        attn(q, kv[0], kv[1], o.view(B, N, self.heads, HEAD_DIM).permute(0, 2, 1, 3))
        return x + _apply(o, self.proj_x)

    def mlp(self, x):
        return x + _apply(F.gelu(_apply(self._ln(x), self.fc1)), self.fc2)


def flash_attn(q, k, v, out):
    """K7 FlashMatch (the product path)."""
    flashmatch(q, k, v, out=out)


def torch_attn(q, k, v, out):
    """Library attention (torch SDPA) -- comparison arm for tests/bench only."""
    out.copy_(F.scaled_dot_product_attention(q, k, v))


class MASt3RViT:
    """ViT-L encoder (shared by both images) + ViT-B decoder (one per image
    side, self + cross attention) + local-feature descriptor head."""

    def __init__(self, height=512, width=384, desc_dim=24, enc_depth=24, dec_depth=12, seed=0,
                 device="cuda"):
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.h, self.w, self.desc_dim = height // PATCH, width // PATCH, desc_dim
        self.tokens = self.h * self.w
        self.patch = _linear(g, 3 * PATCH * PATCH, 1024, device)
        self.pos = (torch.randn((1, self.tokens, 1024), generator=g) * 0.02).to(device, torch.float16)
        self.enc = [Block(g, 1024, 16, False, device) for _ in range(enc_depth)]
        self.enc_to_dec = _linear(g, 1024, 768, device)
        self.dec = [Block(g, 768, 12, True, device, sides=2) for _ in range(dec_depth)]
        self.head = _linear(g, 768, desc_dim * PATCH * PATCH, device)

    def attention_calls(self):
        """(batch, heads, nq, nkv) of every attention launch of one pair forward
        (the two image sides are batched into each launch)."""
        enc = [(2, 16, self.tokens, self.tokens)] * len(self.enc)
        dec = [(2, 12, self.tokens, self.tokens)] * (2 * len(self.dec))  # self + cross per block
        return enc + dec

    def encode(self, imgs, attn=flash_attn):
        """imgs [B, 3, H, W] fp16 -> tokens [B, N, 1024]."""
        B = imgs.shape[0]
        x = F.unfold(imgs, PATCH, stride=PATCH).transpose(1, 2)  # [B, N, 3*16*16]
        x = _apply(x, self.patch) + self.pos
        for blk in self.enc:
            x = blk.mlp(blk.self_attn(x, attn))
        return x

    def decode(self, f, attn=flash_attn):
        """f [2, N, 1024] encoder tokens of both images -> [2, N, 768]; side s
        cross-attends to side 1-s (CroCo/DUSt3R decoder)."""
        x = _apply(f, self.enc_to_dec)
        for blk in self.dec:
            x = blk.self_attn(x, attn)
            x = blk.cross_attn(x, x.flip(0), attn)
            x = blk.mlp(x)
        return x

    def descriptors(self, x):
        """decoder tokens [B, N, 768] -> unit-norm descriptor maps [B, H, W, d] fp32."""
        B = x.shape[0]
        d = _apply(x, self.head).float()  # [B, N, d*16*16]
        d = d.view(B, self.h, self.w, self.desc_dim, PATCH, PATCH).permute(0, 1, 4, 2, 5, 3)
        d = d.reshape(B, self.h * PATCH, self.w * PATCH, self.desc_dim)
        return F.normalize(d, dim=-1)

    @torch.no_grad()
    def forward_pair(self, img1, img2, attn=flash_attn):
        """One image pair -> (D1, D2) descriptor maps, [H, W, d] fp32 each."""
        d = self.descriptors(self.decode(self.encode(torch.stack([img1, img2]), attn), attn))
        return d[0], d[1]
