"""Per-launch FlashMatch time at the C3 shapes (50 launches captured in one
CUDA graph, so host launch cost is excluded), beside torch SDPA."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_10017_b200 import flashmatch  # noqa: E402


def graph_time(fn, n=50, reps=5):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (n * reps) * 1e3


for B, H, N in [(2, 16, 768), (2, 12, 768)]:
    q = torch.randn(B, H, N, 64, device="cuda").half()
    k = torch.randn_like(q)
    v = torch.randn_like(q)
    o = torch.empty_like(q)
    for name, fn in (("flashmatch", lambda: flashmatch(q, k, v, out=o)),
                     ("sdpa", lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v))):
        print(f"{name} [{B},{H},{N},64]: {graph_time(fn):.2f} us", flush=True)
