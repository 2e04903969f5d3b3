"""Does an H2D copy on one stream overlap a kernel on another on this box?"""
import os, time, torch
print("CUDA_DEVICE_MAX_CONNECTIONS =", os.environ.get("CUDA_DEVICE_MAX_CONNECTIONS"))
x = torch.empty((1 << 28,), dtype=torch.float32, pin_memory=True)
y = torch.empty_like(x, device="cuda")
a = torch.randn((8192, 8192), device="cuda", dtype=torch.bfloat16)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def gemms(n):
    for _ in range(n):
        a @ a
torch.cuda.synchronize()
for label, fn in [("copy only", lambda: y.copy_(x, non_blocking=True)), ("gemm only", lambda: gemms(60))]:
    torch.cuda.synchronize(); t = time.perf_counter(); fn(); torch.cuda.synchronize()
    print(f"{label}: {(time.perf_counter() - t) * 1e3:.1f} ms")
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(s1):
    gemms(60)
with torch.cuda.stream(s2):
    y.copy_(x, non_blocking=True)
torch.cuda.synchronize()
print(f"both on two streams: {(time.perf_counter() - t) * 1e3:.1f} ms")
