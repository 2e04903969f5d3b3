"""K7 FlashMatch throughput at config C3 (MASt3R ViT-L encoder + ViT-B decoder,
512x384 -> 768 tokens, head_dim 64): every attention launch of one pair
forward, timed with CUDA events; plus the whole random-init ViT forward with
K7 vs the library attention.  Used by bench.py (flashmatch section)."""
import math

import torch


def attention_flops(calls):
    return sum(4.0 * b * h * nq * nkv * 64 for b, h, nq, nkv in calls)


def time_calls(calls, attn, reps=20, warmup=3):
    bufs = {}
    g = torch.Generator(device="cpu").manual_seed(0)
    for shape in dict.fromkeys(calls):  # one input set per distinct (batch, heads, nq, nkv)
        b, h, nq, nkv = shape
        q = torch.randn((b, h, nq, 64), generator=g).to("cuda", torch.float16)
        k = torch.randn((b, h, nkv, 64), generator=g).to("cuda", torch.float16)
        v = torch.randn((b, h, nkv, 64), generator=g).to("cuda", torch.float16)
        bufs[shape] = (q, k, v, torch.empty_like(q))
    seq = [bufs[c] for c in calls]

    def run():
        for q, k, v, o in seq:
            attn(q, k, v, o)

    # captured once into a CUDA graph: the GPU time of the 48 launches, not
    # the Python launch cost
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(warmup):
            run()
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        run()
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def time_forward(model, attn, reps=5, warmup=2):
    """One pair forward replayed from a CUDA graph (the forward is hundreds of
    small launches; the graph removes the host launch cost)."""
    g = torch.Generator(device="cpu").manual_seed(1)
    img1 = torch.randn((3, 512, 384), generator=g).to("cuda", torch.float16)
    img2 = torch.randn((3, 512, 384), generator=g).to("cuda", torch.float16)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(warmup):
            model.forward_pair(img1, img2, attn)
    torch.cuda.current_stream().wait_stream(side)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        model.forward_pair(img1, img2, attn)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run(peak_tflops):
    from paper_2503_10017_b200 import vit
    model = vit.MASt3RViT(seed=0)
    calls = model.attention_calls()
    flops = attention_flops(calls)
    ms = time_calls(calls, vit.flash_attn)
    ms_lib = time_calls(calls, vit.torch_attn)
    fwd = time_forward(model, vit.flash_attn)
    fwd_lib = time_forward(model, vit.torch_attn)
    tf = flops / (ms / 1e3) / 1e12
    return {
        "workload": "C3: all attention launches of one MASt3R pair forward at 512x384 (768 tokens, "
                    "head_dim 64): 24 x ViT-L encoder self-attn [2 img x 16 heads] + 12 x ViT-B decoder "
                    "(self + cross) [2 sides x 12 heads]; binary16 in, fp32 accumulate",
        "attention_ms_per_pair": round(ms, 4),
        "attention_gflop_per_pair": round(flops / 1e9, 2),
        "achieved_tflops": round(tf, 1),
        "peak_tflops": peak_tflops,
        "frac": round(tf / peak_tflops, 4),
        "library_sdpa_ms_per_pair": round(ms_lib, 4),
        "vit_forward_ms_per_pair": round(fwd, 3),
        "vit_forward_ms_per_pair_library_sdpa": round(fwd_lib, 3),
        "launches_per_pair": len(calls),
    }


if __name__ == "__main__":
    import json
    import sys
    sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
    print(json.dumps(run(1635.2)))
