"""Per-launch FlashMatch time (CUDA events, 50 back-to-back launches) at the
C3 shapes, for the kernel version in FNL_FM_VERSION, beside torch SDPA."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10017_b200 import flashmatch  # noqa: E402

for B, H, N in [(2, 16, 768), (2, 12, 768)]:
    q = torch.randn(B, H, N, 64, device="cuda").half()
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    o = torch.empty_like(q)
    for name, fn in (("flashmatch", lambda: flashmatch(q, k, v, out=o)),
                     ("sdpa", lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))):
        for _ in range(5):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"v{os.environ.get('FNL_FM_VERSION', '5')} {name} [{B},{H},{N},64]: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us",
              flush=True)
