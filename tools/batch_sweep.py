"""Pairs per call vs latency and throughput of the device API (C2 maps,
backend single, no stats): one JSON line per batch size.  Usage (on a B200):
python tools/batch_sweep.py [out.json]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10017_b200 as fnl  # noqa: E402

H, W, D = 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(16)]
res = []
for B in (1, 2, 4, 8, 16, 32, 64, 128):
    d1 = torch.stack([torch.from_numpy(pool[i % 16]) for i in range(B)]).cuda()
    d2 = torch.stack([torch.from_numpy(pool[(i + 5) % 16]) for i in range(B)]).cuda()
    out = torch.empty((B, 3072, 3), dtype=torch.int32, device="cuda")
    cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()

    def call():
        fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, out.data_ptr(), cnt.data_ptr(),
                                    backend="single", stride=8, metric="dot", stream=s.cuda_stream,
                                    with_stats=False)
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    n = max(3, 64 // B)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(n):
        call()
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    r = {"pairs_per_call": B, "ms_per_call": round(ms, 4), "pairs_per_s": round(B / ms * 1e3, 1), "calls": n}
    print(json.dumps(r), flush=True)
    res.append(r)
    del d1, d2
if len(sys.argv) > 1:
    json.dump({"workload": "C2 512x384 d=24 stride 8, dot, backend single, device API without stats "
               "(batches <= 16 replay the loop as a CUDA graph); CUDA events over back-to-back calls",
               "rows": res}, open(sys.argv[1], "w"), indent=1)
