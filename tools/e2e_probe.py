"""Time the host-buffer batch API (bench.py e2e leg) for a given sub-batch size."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10017_b200 as fnl
B, H, W, D = 128, 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(16)]
h1 = torch.empty((B, H, W, D), dtype=torch.float32, pin_memory=True)
h2 = torch.empty((B, H, W, D), dtype=torch.float32, pin_memory=True)
for i in range(B):
    h1[i].copy_(torch.from_numpy(pool[i % 16])); h2[i].copy_(torch.from_numpy(pool[(i + 5) % 16]))
n1, n2 = h1.numpy(), h2.numpy()
fnl.reciprocal_match_batch(n1, n2, backend="tensor", stride=8, metric="dot")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(2):
    fnl.reciprocal_match_batch(n1, n2, backend="tensor", stride=8, metric="dot")
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 2
print(f"sub={os.environ.get('FNL_BATCH_SUB', 16)}: {dt * 1e3:.1f} ms per {B} pairs = {B / dt:.0f} pairs/s")
