"""Two host threads, each matching half the batch on its own stream/context:
does the GPU fill one stream's host gaps with the other's kernels?"""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2503_10017_b200 as fnl
B, H, W, D = 128, 512, 384, 24
pool = [fnl.gen_random(H, W, D, 1000 + i) for i in range(16)]
d1 = torch.stack([torch.from_numpy(pool[i % 16]) for i in range(B)]).cuda()
d2 = torch.stack([torch.from_numpy(pool[(i + 5) % 16]) for i in range(B)]).cuda()
S = 3072
out = torch.empty((B, S, 3), dtype=torch.int32, device="cuda")
cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]

def run(lo, hi, st):
    fnl.reciprocal_match_device(d1[lo].data_ptr(), d2[lo].data_ptr(), hi - lo, H, W, D, out[lo].data_ptr(),
                                cnt[lo].data_ptr(), backend="tensor", stride=8, metric="dot", stream=st.cuda_stream)

def step(nthreads):
    per = B // nthreads
    ths = [threading.Thread(target=run, args=(i * per, (i + 1) * per, streams[i])) for i in range(nthreads)]
    for t in ths: t.start()
    for t in ths: t.join()

for n in (1, 2, 4):
    for _ in range(2): step(n)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): step(n)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 5
    print(f"{n} thread(s): {dt * 1e3:.2f} ms per {B} pairs = {B / dt:.0f} pairs/s")
