"""FlashMatch inside the random-init MASt3R ViT blocks (config C3 harness):
the product attention (K7) against the library attention arm, and the
resulting descriptor maps fed to the FastNN-Lite matcher."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).norm() / b.norm())


def test_vit_blocks_flashmatch_vs_library_attention(fnl):
    import torch
    from paper_2503_10017_b200 import vit
    model = vit.MASt3RViT(enc_depth=2, dec_depth=2, seed=3)
    g = torch.Generator(device="cpu").manual_seed(4)
    imgs = torch.randn((2, 3, 512, 384), generator=g).to("cuda", torch.float16)
    with torch.no_grad():
        f_ours = model.encode(imgs, vit.flash_attn)
        f_lib = model.encode(imgs, vit.torch_attn)
        assert _rel(f_ours, f_lib) < 1e-3
        x_ours = model.decode(f_ours, vit.flash_attn)
        x_lib = model.decode(f_ours, vit.torch_attn)
        assert _rel(x_ours, x_lib) < 1e-3
        d_ours = model.descriptors(x_ours)
        d_lib = model.descriptors(x_lib)
    assert d_ours.shape == (2, 512, 384, 24)
    assert _rel(d_ours, d_lib) < 1e-3


def test_vit_descriptors_feed_the_matcher(fnl):
    import torch
    from paper_2503_10017_b200 import vit
    model = vit.MASt3RViT(height=128, width=96, enc_depth=1, dec_depth=1, seed=5)
    g = torch.Generator(device="cpu").manual_seed(6)
    img = torch.randn((3, 128, 96), generator=g).to("cuda", torch.float16)
    d1, d2 = model.forward_pair(img, img)
    torch.cuda.synchronize()
    D1 = np.ascontiguousarray(d1.cpu().numpy())
    D2 = np.ascontiguousarray(d2.cpu().numpy())
    assert D1.shape == (128, 96, 24) and np.isfinite(D1).all()
    matches, report = fnl.reciprocal_match(D1, D2, backend="tensor", metric="dot")
    assert matches.shape[1] == 3
