"""K7 FlashMatch parity: the tcgen05 attention kernel vs the float64 oracle
(oracle/attention.py) and torch fp32 math attention on the same binary16
inputs.  Tolerance (BASELINE.json north_star: attention outputs within 1e-3
relative): ||O - ref||_F / ||ref||_F <= 1e-3 and max|O - ref| <= 2e-3 * max|ref|
(the binary16 output alone contributes ~2.8e-4 relative)."""
import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REL_F = 1e-3
REL_MAX = 2e-3


def _check(out, ref):
    out = out.astype(np.float64)
    err = out - ref
    rel_f = np.linalg.norm(err) / np.linalg.norm(ref)
    rel_max = np.abs(err).max() / np.abs(ref).max()
    assert rel_f <= REL_F and rel_max <= REL_MAX, (rel_f, rel_max)
    return rel_f, rel_max


def _rand(torch, shape, seed, scale=1.0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return (torch.randn(shape, generator=g) * scale).to(torch.float16)


@pytest.mark.parametrize("B,H,Nq,Nkv", [(2, 16, 768, 768), (1, 3, 300, 200), (1, 2, 128, 129),
                                         (1, 1, 5, 77), (3, 12, 768, 256), (1, 4, 1000, 768)])
def test_flashmatch_vs_oracle(fnl, B, H, Nq, Nkv):
    import torch
    from oracle import attention
    from paper_2503_10017_b200.flashmatch import flashmatch
    q = _rand(torch, (B, H, Nq, 64), 1)
    k = _rand(torch, (B, H, Nkv, 64), 2)
    v = _rand(torch, (B, H, Nkv, 64), 3)
    out = flashmatch(q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    ref = attention.attention(q.numpy(), k.numpy(), v.numpy())
    _check(out.cpu().numpy(), ref)


def test_flashmatch_vs_torch_fp32_and_strided_qkv(fnl):
    """q/k/v read in place from a fused QKV projection [B, N, 3, H, 64];
    output written in place into [B, N, H*64] (the layout the next GEMM wants)."""
    import torch
    from paper_2503_10017_b200.flashmatch import flashmatch
    B, N, H = 2, 768, 12
    qkv = _rand(torch, (B, N, 3 * H * 64), 7).cuda()
    v5 = qkv.view(B, N, 3, H, 64).permute(2, 0, 3, 1, 4)
    q, k, v = v5[0], v5[1], v5[2]
    o = torch.empty((B, N, H * 64), dtype=torch.float16, device="cuda")
    flashmatch(q, k, v, out=o.view(B, N, H, 64).permute(0, 2, 1, 3))
    ref = torch.softmax((q.float() @ k.float().transpose(-1, -2)) / math.sqrt(64), dim=-1) @ v.float()
    ref = ref.permute(0, 2, 1, 3).reshape(B, N, H * 64)
    torch.cuda.synchronize()
    _check(o.cpu().numpy(), ref.cpu().double().numpy())


def test_flashmatch_large_logits(fnl):
    """Peaked softmax (|logits| ~ 100): the online max keeps exp2 in range."""
    import torch
    from oracle import attention
    from paper_2503_10017_b200.flashmatch import flashmatch
    q = _rand(torch, (1, 2, 256, 64), 11, scale=4.0)
    k = _rand(torch, (1, 2, 384, 64), 12, scale=4.0)
    v = _rand(torch, (1, 2, 384, 64), 13)
    out = flashmatch(q.cuda(), k.cuda(), v.cuda())
    torch.cuda.synchronize()
    _check(out.cpu().numpy(), attention.attention(q.numpy(), k.numpy(), v.numpy()))


def test_flashmatch_rejects_bad_args(fnl):
    import torch
    from paper_2503_10017_b200.flashmatch import flashmatch
    q = torch.zeros((1, 1, 8, 32), dtype=torch.float16, device="cuda")
    with pytest.raises(ValueError):
        flashmatch(q, q, q)
    q = torch.zeros((1, 1, 8, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        flashmatch(q, q, q)
