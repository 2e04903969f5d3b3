"""Where the timed C2 step goes besides kernels: per step, CUDA events on the
stream around each reciprocal_match_device call and host wall time of the
call, so GPU idle time between and inside steps shows up.  Usage (on a B200):
python tools/step_gaps.py [steps] [pairs]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10017_b200 as fnl  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
H, W, D = 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(8)]
d1 = torch.stack([torch.from_numpy(pool[i % 8]) for i in range(B)]).cuda()
d2 = torch.stack([torch.from_numpy(pool[(i + 3) % 8]) for i in range(B)]).cuda()
samples = (H // 8) * (W // 8)
out = torch.empty((B, samples, 3), dtype=torch.int32, device="cuda")
cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()


def step():
    fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, out.data_ptr(), cnt.data_ptr(),
                                backend="single", stride=8, metric="dot", stream=s.cuda_stream,
                                with_stats=False)


for _ in range(3):
    step()
torch.cuda.synchronize()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
host = []
t_all = time.perf_counter()
e_all0, e_all1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e_all0.record(s)
for i in range(steps):
    ev[i][0].record(s)
    t = time.perf_counter()
    step()
    host.append((time.perf_counter() - t) * 1e3)
    ev[i][1].record(s)
e_all1.record(s)
torch.cuda.synchronize()
gpu = [a.elapsed_time(b) for a, b in ev]
gaps = [ev[i][1].elapsed_time(ev[i + 1][0]) for i in range(steps - 1)]
tot = e_all0.elapsed_time(e_all1)
# the same steps with the GPU left idle 50 ms before each (power / clock recovery)
gpu_idle = []
for i in range(min(steps, 10)):
    torch.cuda.synchronize()
    time.sleep(0.05)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    step()
    b.record(s)
    torch.cuda.synchronize()
    gpu_idle.append(a.elapsed_time(b))
print(f"after 50 ms idle: GPU per step median {np.median(gpu_idle):.3f} ms")
print(f"steps {steps} pairs {B}: total {tot:.2f} ms = {tot / steps:.3f} ms/step; "
      f"GPU per step (events) median {np.median(gpu):.3f} min {min(gpu):.3f} max {max(gpu):.3f}; "
      f"host call median {np.median(host):.3f} ms; gaps between steps median {np.median(gaps):.3f} ms")
