"""GPU timeline of back-to-back reciprocal_match_device calls (CUPTI through
torch.profiler): per call, kernel busy time, idle gaps between kernels, and
the largest gaps with the kernels around them.  Usage (on a B200):
python tools/call_timeline.py [pairs] [calls] [out.json]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10017_b200 as fnl  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 5
out_path = sys.argv[3] if len(sys.argv) > 3 else None
H, W, D = 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(8)]
d1 = torch.stack([torch.from_numpy(pool[i % 8]) for i in range(B)]).cuda()
d2 = torch.stack([torch.from_numpy(pool[(i + 3) % 8]) for i in range(B)]).cuda()
samples = (H // 8) * (W // 8)
out = torch.empty((B, samples, 3), dtype=torch.int32, device="cuda")
cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream()


def call():
    fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, out.data_ptr(), cnt.data_ptr(),
                                backend="single", stride=8, metric="dot", stream=s.cuda_stream,
                                with_stats=False)


for _ in range(3):
    call()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(calls):
        call()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
k = sorted(((e.time_range.start, e.time_range.end, e.name) for e in ev), key=lambda x: x[0])
# calls start at a pack kernel preceded by the previous call's last kernel
starts = [i for i, x in enumerate(k) if "pack" in x[2]][::2]
res = []
for ci in range(len(starts)):
    a = starts[ci]
    b = starts[ci + 1] if ci + 1 < len(starts) else len(k)
    seg = k[a:b]
    busy = sum(e - s0 for s0, e, _ in seg)
    wall = seg[-1][1] - seg[0][0]
    gaps = [(seg[i + 1][0] - seg[i][1], seg[i][2][:40], seg[i + 1][2][:40]) for i in range(len(seg) - 1)]
    hist = {"<3us": 0.0, "3-10us": 0.0, "10-30us": 0.0, ">30us": 0.0}
    for g, _, _ in gaps:
        hist["<3us" if g < 3 else "3-10us" if g < 10 else "10-30us" if g < 30 else ">30us"] += g
    res.append({"kernels": len(seg), "wall_us": wall, "busy_us": busy, "idle_us": wall - busy,
                "gap_hist_us": hist, "top_gaps": sorted(gaps, reverse=True)[:8]})
for r in res:
    print(f"kernels {r['kernels']} wall {r['wall_us']:.1f} us busy {r['busy_us']:.1f} idle {r['idle_us']:.1f} "
          f"gaps {', '.join(f'{k}: {v:.0f}' for k, v in r['gap_hist_us'].items())}")
r = res[len(res) // 2]
for g in r["top_gaps"]:
    print(f"  gap {g[0]:7.1f} us after {g[1]} before {g[2]}")
agg = {}
for s0, e, n in k[starts[len(starts) // 2]:(starts[len(starts) // 2 + 1] if len(starts) > len(starts) // 2 + 1 else len(k))]:
    n = n.split("(")[0][:50]
    agg[n] = agg.get(n, 0.0) + (e - s0)
for n, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"  {v:8.1f} us {n}")
if out_path:
    json.dump(res, open(out_path, "w"), indent=1)
