import torch, time
x = torch.empty((4831838208 // 4,), dtype=torch.float32, pin_memory=True)
y = torch.empty_like(x, device="cuda")
for _ in range(2): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 3
print(f"H2D {x.numel()*4/dt/1e9:.1f} GB/s, {dt*1e3:.1f} ms per 4.83 GB")
