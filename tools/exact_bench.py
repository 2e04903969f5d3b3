"""Reference-semantics backends (K4 exact CUDA-core path) at C2: device-resident pairs/s."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10017_b200 as fnl
B, H, W, D = 16, 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(8)]
d1 = torch.stack([torch.from_numpy(pool[i % 8]) for i in range(B)]).cuda()
d2 = torch.stack([torch.from_numpy(pool[(i + 3) % 8]) for i in range(B)]).cuda()
out = torch.empty((B, 3072, 3), dtype=torch.int32, device="cuda"); cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
for be in ("single", "hybrid", "tensor"):
    run = lambda: fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, out.data_ptr(), cnt.data_ptr(),
                                              backend=be, stride=8, metric="dot")
    run(); torch.cuda.synchronize()
    t = time.perf_counter(); st = run(); torch.cuda.synchronize(); dt = time.perf_counter() - t
    rows = sum(s["query_rows"] for s in st)
    print(f"{be}: {B / dt:.0f} pairs/s, {rows * H * W * 48 / dt / 1e12:.1f} TFLOP/s algorithmic")
