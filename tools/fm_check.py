"""FlashMatch numerics spot-check across shapes (max |err| vs torch fp32), one line per shape."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10017_b200 import flashmatch  # noqa: E402

shapes = [(1, 1, 128, 128), (1, 1, 128, 768), (1, 2, 256, 768), (2, 16, 768, 768), (2, 12, 768, 768),
          (1, 3, 300, 200), (1, 1, 5, 77), (1, 4, 1000, 768)]
for B, H, Nq, Nkv in shapes:
    g = torch.Generator().manual_seed(1)
    q = torch.randn(B, H, Nq, 64, generator=g).half().cuda()
    k = torch.randn(B, H, Nkv, 64, generator=g).half().cuda()
    v = torch.randn(B, H, Nkv, 64, generator=g).half().cuda()
    o = flashmatch(q, k, v)
    torch.cuda.synchronize()
    ref = torch.softmax((q.float() @ k.float().transpose(-1, -2)) / 8.0, -1) @ v.float()
    err = (o.float() - ref).abs().max().item()
    rel = ((o.float() - ref).norm() / ref.norm()).item()
    print(B, H, Nq, Nkv, f"max_err={err:.3e} rel={rel:.3e}", flush=True)
