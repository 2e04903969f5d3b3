"""FlashMatch phase trace of CTA 0 (FNL_FM_TRACE=1): clock64 stamps relative
to kernel entry.  0 entry, 34 TMEM allocated, 3+j S(j) ready (tile 0), 10+j
row max known, 20+j P(j) published, 63 exit."""
import os
import sys

import numpy as np
import torch

os.environ.setdefault("FNL_FM_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10017_b200 as fnl  # noqa: E402
from paper_2503_10017_b200 import _fastnn  # noqa: E402

for B, H in ((2, 12), (2, 16)):
    q = torch.randn((B, H, 768, 64), device="cuda").half()
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    for _ in range(3):
        fnl.flashmatch(q, k, v)
    torch.cuda.synchronize()
    st = np.array(_fastnn._flashmatch_trace(), dtype=np.int64)
    t0 = st[0]
    rel = {i: int(st[i] - t0) for i in range(64) if st[i] >= t0 and st[i] - t0 < 10**7}
    print(f"[{B},{H},768,64]:", rel, flush=True)
