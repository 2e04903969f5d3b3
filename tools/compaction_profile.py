"""Drive the compaction / convergence kernels at the bench shape (128 C2 pairs)
for ncu: harvest (cycle check + stable compaction + convergence), gather,
confidence compaction."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10017_b200 as fnl
B, H, W, D = 128, 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(16)]
d1 = torch.stack([torch.from_numpy(pool[i % 16]) for i in range(B)]).cuda()
d2 = torch.stack([torch.from_numpy(pool[(i + 5) % 16]) for i in range(B)]).cuda()
out = torch.empty((B, 3072, 3), dtype=torch.int32, device="cuda"); cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
for _ in range(2):
    fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, out.data_ptr(), cnt.data_ptr(),
                                backend="tensor", stride=8, metric="dot", max_distance=-0.5)
torch.cuda.synchronize()
print("matches kept", int(cnt.sum()))
