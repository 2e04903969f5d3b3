"""Timeline of one host-buffer batch call (CUPTI via torch.profiler): are the
H2D sub-batch uploads overlapping the matcher kernels?"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10017_b200 as fnl
B, H, W, D = 128, 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(8)]
h1 = torch.empty((B, H, W, D), dtype=torch.float32, pin_memory=True)
h2 = torch.empty((B, H, W, D), dtype=torch.float32, pin_memory=True)
for i in range(B):
    h1[i].copy_(torch.from_numpy(pool[i % 8])); h2[i].copy_(torch.from_numpy(pool[(i + 3) % 8]))
n1, n2 = h1.numpy(), h2.numpy()
fnl.reciprocal_match_batch(n1, n2, backend="tensor", stride=8, metric="dot")
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    fnl.reciprocal_match_batch(n1, n2, backend="tensor", stride=8, metric="dot")
    torch.cuda.synchronize()
prof.export_chrome_trace("gpurun_out/e2e_trace.json")
ev = json.load(open("gpurun_out/e2e_trace.json"))["traceEvents"]
rows = [(e["ts"], e.get("dur", 0), e.get("cat"), e["name"][:40], e.get("args", {}).get("stream"))
        for e in ev if e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
rows.sort()
t0 = rows[0][0] if rows else 0
last = {}
for ts, dur, cat, name, stream in rows:
    if cat == "gpu_memcpy" or name.startswith("fnl::<unnamed>::pack") or "harvest" in name:
        print(f"{(ts - t0) / 1e3:9.2f} ms +{dur / 1e3:7.2f} ms  s={stream} {cat:10s} {name}")
