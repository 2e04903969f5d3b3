"""Is a pinned H2D cudaMemcpyAsync asynchronous w.r.t. the host (torch vs our library)?"""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
x = torch.empty((1 << 28,), dtype=torch.float32, pin_memory=True)   # 1 GiB
y = torch.empty_like(x, device="cuda")
s = torch.cuda.Stream()
torch.cuda.synchronize()
with torch.cuda.stream(s):
    t = time.perf_counter(); y.copy_(x, non_blocking=True); dt = time.perf_counter() - t
torch.cuda.synchronize()
print(f"torch non_blocking H2D 1 GiB: host call {dt*1e3:.2f} ms")
