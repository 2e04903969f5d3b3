#!/usr/bin/env python3
"""FastNN-Lite pair-matching throughput on B200 (BASELINE.json metric).

A step = the full reciprocal matching hot path (K1 pack -> iterative K2 gather /
K3 tcgen05 score+argmax / merge / near-tie rescan / K5 harvest until
convergence) over one batch of PAIRS_PER_GPU synthetic 512x384 d=24 pairs per
GPU (config C2 shape, batched as in C4).  Pairs are independent, so ranks
shard them with no data-path collective ("scaling": "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--pairs B]
  python bench.py --impl reference ...   # the reference CPU path on the host

value : device-resident throughput (maps already in HBM), CUDA events on the
        launching stream, barrier + synchronize on both sides, max over ranks.
e2e   : the public batch API (paper_2503_10017_b200.reciprocal_match_batch) on
        pinned HOST maps: H2D of every step's inputs and D2H of its matches are
        inside the timed region.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

H, W, D, STRIDE = 512, 384, 24, 8
METRIC = "dot"                     # MASt3R descriptors are unit norm
NT = H * W
FLOP_PER_SCORE = 2 * D             # algorithmic: 2d per (query, target) score, d=24 unpadded
SPEC_DENSE_F16_TFLOPS = 2250.0    # B200 nominal dense fp16/bf16 (the doubled figure is 2:4 sparsity)
POOL = 64                          # distinct synthetic maps, seeds 1000.. (gen_random, reference generator)
METRIC_NAME = "image pairs/sec FastNN-Lite @512x384 d=24 (1/2/4/8 B200); % tensor-pipe peak"


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["bf16_tflops"]), float(p.get("bf16_tflops_sustained", 0) or 0), "measured"
    except Exception:
        return 1590.0, 1400.0, "fallback"


def gen_pool(gen_random):
    return [gen_random(H, W, D, 1000 + i) for i in range(POOL)]


def pair_maps(k):
    """Pair k of the synthetic stream: two distinct pool maps."""
    a = k % POOL
    b = (a + 1 + (k // POOL) * 7 + (k % 5)) % POOL
    if b == a:
        b = (a + 1) % POOL
    return a, b


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region.

    The sampler starts before the region (nvidia-smi needs ~0.1-0.3 s to come
    up), a reader thread timestamps every line, and summary() keeps only the
    samples taken between mark_start() and mark_end()."""

    def __init__(self, index, period_ms=25):
        self.index = index
        self.period_ms = period_ms
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def __enter__(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", str(self.period_ms)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        self.first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                self.lines.append((time.time(), line))
                self.first.set()
        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        self.first.wait(timeout=3.0)
        return self

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        parsed = []
        for ts, line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                try:
                    parsed.append((ts, (float(parts[0]), float(parts[1]), parts[3:7])))
                except ValueError:
                    pass
        rows = [r for ts, r in parsed if (self.t0 is None or ts >= self.t0) and (self.t1 is None or ts <= self.t1 + 0.05)]
        nearest = False
        if not rows and parsed and self.t0 is not None:
            # timed region shorter than the sampling period: the sample nearest to it
            mid = 0.5 * (self.t0 + (self.t1 or self.t0))
            rows = [min(parsed, key=lambda x: abs(x[0] - mid))[1]]
            nearest = True
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        out = {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
               "reasons": reasons, "samples": len(rows)}
        if nearest:
            out["nearest_sample"] = True
        return out


def dist_setup():
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
    # FNL_BENCH_DIST_BACKEND=gloo (with more ranks than GPUs) is only for
    # exercising the N>1 code path on a 1-GPU box; timings are then meaningless
    forced = os.environ.get("FNL_BENCH_DIST_BACKEND")
    if ngpu:
        local = local % ngpu
    if world > 1 and not dist.is_initialized():
        backend = forced or ("nccl" if ngpu else "gloo")
        if ngpu:
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


def allreduce(vals, op):
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return vals
    dev = "cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return t.tolist()


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ---------------------------------------------------------------- reference arm
def ref_threads():
    return max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))


def run_reference_pairs(ref, pool, first, count):
    """The unmodified reference FastNN path (oracle/_ref, compiled from
    /root/reference): reciprocal_match backend=single, dot, all host threads,
    block_size = ceil(samples / threads) so every thread gets a query block."""
    threads = ref_threads()
    samples = math.ceil(H / STRIDE) * math.ceil(W / STRIDE)
    bs = math.ceil(samples / threads)
    t0 = time.perf_counter()
    for k in range(first, first + count):
        a, b = pair_maps(k)
        ref.reciprocal_match(pool[a], pool[b], backend="single", metric=METRIC, stride=STRIDE,
                             block_size=bs, threads=threads)
    return time.perf_counter() - t0, threads


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def main_reference(args):
    world, rank, _ = dist_setup()
    if rank != 0:
        return
    from oracle import oracle
    ref = oracle.reference()
    pool = gen_pool(ref.gen_random)
    per_step = 1
    for i in range(args.warmup):
        run_reference_pairs(ref, pool, i, per_step)
    total, threads = 0.0, ref_threads()
    for i in range(args.steps):
        dt, threads = run_reference_pairs(ref, pool, args.warmup + i, per_step)
        total += dt
    pairs = args.steps * per_step
    value = pairs / total
    line = {
        "impl": "reference", "metric": METRIC_NAME, "value": value, "unit": "pairs/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * total / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (reference gen_random, 64-map pool)",
        "config": {"workload": "C2: FastNN reciprocal match, 512x384 d=24, stride 8, dot; reference "
                               "CPU path (backend single), 1 pair per step", "pairs_per_step": per_step,
                   "threads": threads, "cpu": cpu_model()},
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "reference",
                         "sample": f"{pairs} C2 pairs, reference reciprocal_match single/dot, "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- B200 arm
def main_b200(args):
    import torch
    world, rank, local = dist_setup()
    torch.cuda.set_device(local)
    import paper_2503_10017_b200 as fnl
    fnl.set_device(local)
    B = args.pairs
    first_pair = rank * B
    pool = gen_pool(fnl.gen_random)
    samples = math.ceil(H / STRIDE) * math.ceil(W / STRIDE)

    # device-resident inputs (value) and pinned host copies (e2e)
    h1 = torch.empty((B, H, W, D), dtype=torch.float32, pin_memory=True)
    h2 = torch.empty((B, H, W, D), dtype=torch.float32, pin_memory=True)
    for i in range(B):
        a, b = pair_maps(first_pair + i)
        h1[i].copy_(torch.from_numpy(pool[a]))
        h2[i].copy_(torch.from_numpy(pool[b]))
    d1 = h1.to("cuda", non_blocking=False)
    d2 = h2.to("cuda", non_blocking=False)
    out_pairs = torch.empty((B, samples, 3), dtype=torch.int32, device="cuda")
    out_counts = torch.empty((B,), dtype=torch.int32, device="cuda")
    stream = torch.cuda.current_stream()

    def step_device(with_stats=False):
        return fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, out_pairs.data_ptr(),
                                           out_counts.data_ptr(), backend=args.backend, stride=STRIDE,
                                           metric=METRIC, stream=stream.cuda_stream, with_stats=with_stats)

    for _ in range(args.warmup):
        step_device()
    # every step matches the same pairs: the per-step work (query rows, near
    # ties) comes from one untimed step with the diagnostic stats switched on
    stats = step_device(with_stats=True)
    rows_per_step = sum(s["query_rows"] for s in stats)
    ties_per_step = sum(s["near_tie_rows"] for s in stats)
    torch.cuda.synchronize()
    fnl.kernel_timing(reset=True)
    query_rows, near_ties = 0, 0
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.mark_start()
        ev0.record(stream)
        for _ in range(args.steps):
            step_device()
            query_rows += rows_per_step
            near_ties += ties_per_step
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    timing = fnl.kernel_timing(reset=True)
    matches_last = int(out_counts.sum().item())

    # ---- per-kernel-class breakdown: one extra step with events around every
    # launch (outside the timed region; events add small gaps)
    fnl.kernel_profile(enable=1, reset=True)
    t_prof0 = torch.cuda.Event(enable_timing=True)
    t_prof1 = torch.cuda.Event(enable_timing=True)
    t_prof0.record(stream)
    step_device()
    t_prof1.record(stream)
    torch.cuda.synchronize()
    prof = fnl.kernel_profile(enable=0, reset=True)
    fnl.kernel_timing(reset=True)
    prof_step_ms = t_prof0.elapsed_time(t_prof1)
    # algorithmic HBM bytes of K1: fp32 rows in, binary16 UMMA rows out, both maps
    pack_bytes = 2 * B * NT * (D * 4 + 64)
    breakdown = {k: {"ms": round(v["ms"], 4), "launches": int(v["launches"])}
                 for k, v in prof.items() if v["launches"]}
    breakdown["step_ms"] = round(prof_step_ms, 4)
    breakdown["unattributed_ms"] = round(prof_step_ms - sum(v["ms"] for v in prof.values()), 4)
    if prof["pack"]["ms"] > 0:
        breakdown["pack"]["hbm_gbs"] = round(pack_bytes / (prof["pack"]["ms"] / 1e3) / 1e9, 1)

    # ---- e2e through the public host-buffer batch API
    n1, n2 = h1.numpy(), h2.numpy()
    for _ in range(max(1, args.warmup // 2)):
        fnl.reciprocal_match_batch(n1, n2, backend=args.backend, stride=STRIDE, metric=METRIC)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        pairs_h, counts_h, _ = fnl.reciprocal_match_batch(n1, n2, backend=args.backend, stride=STRIDE,
                                                          metric=METRIC)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    barrier()

    # ---- C5: one oversized 1536x1152 pair, target columns sharded over the ranks
    c5 = None
    if not args.no_c5:
        c5 = bench_c5(fnl, world, rank, local)

    # ---- C3: FlashMatch attention at the MASt3R ViT shapes (rank 0)
    c3 = None
    if rank == 0 and not args.no_c3:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_flashmatch
        c3 = bench_flashmatch.run(peaks()[0])

    # ---- max over ranks
    max_ms, max_e2e = allreduce([elapsed_ms, e2e_s], op=__import__("torch").distributed.ReduceOp.MAX) \
        if world > 1 else (elapsed_ms, e2e_s)
    tot_rows, tot_score_ms, tot_launch = allreduce([query_rows, timing["score_ms"], timing["score_launches"]],
                                                   op=__import__("torch").distributed.ReduceOp.SUM) \
        if world > 1 else (query_rows, timing["score_ms"], timing["score_launches"])

    # ---- CPU baseline (rank 0, N=1 only): the reference on a bounded sample
    cpu = None
    parity = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle
        ref = oracle.reference()
        done, spent, threads = 0, 0.0, ref_threads()
        while done < 1 or (spent < args.cpu_seconds and done < 64):
            dt, threads = run_reference_pairs(ref, pool, done, 1)
            spent += dt
            done += 1
        cpu = {"value": done / spent, "unit": "pairs/s", "cores": threads, "kind": "reference",
               "sample": f"{done} C2 pairs (512x384 d=24 stride 8, dot), reference reciprocal_match "
                         f"backend=single, {threads} threads, {spent:.1f} s; host CPU {cpu_model()}"}
        # the same reference as the checker (untimed): the tensor backend must
        # equal reference backend=single on binary16-rounded maps, bit for bit,
        # for the first pairs of the last timed step's batch
        got_pairs = out_pairs[:args.parity_pairs].cpu().numpy()
        got_counts = out_counts[:args.parity_pairs].cpu().numpy()
        same = 0
        for i in range(min(args.parity_pairs, B)):
            a, b = pair_maps(i)
            want, _ = ref.reciprocal_match(oracle.half_round_array(pool[a]), oracle.half_round_array(pool[b]),
                                           backend="single", metric=METRIC, stride=STRIDE,
                                           block_size=math.ceil(samples / threads), threads=threads)
            n = int(got_counts[i])
            same += int(n == len(want) and np.array_equal(got_pairs[i, :n].astype(np.uint32), want))
        parity = {"pairs_checked": min(args.parity_pairs, B), "identical": same,
                  "checker": "oracle/_ref reciprocal_match backend=single on binary16-rounded maps "
                             "(the tensor backend's contract), (i, j, iter) triples of the last timed step"}

    if rank != 0:
        return
    pairs_total = B * world * args.steps
    value = pairs_total / (max_ms / 1000.0)
    e2e_value = B * world * args.e2e_steps / max_e2e
    peak_burst, peak_sust, peak_kind = peaks()
    flops = FLOP_PER_SCORE * NT * tot_rows
    achieved = flops / (tot_score_ms / 1000.0) / 1e12 if tot_score_ms > 0 else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "tc_scan_ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                pj = json.load(f)
            # ncu figure of one captured launch, scaled per pair to this run's launches
            traffic = pj["dram_bytes_per_launch"] / pj.get("pairs_in_launch", 1) * B
        except Exception:
            traffic = None
    line = {
        "metric": METRIC_NAME, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16", "data": "synthetic",
        "config": {"workload": "C2/C4: FastNN-Lite reciprocal matching of 512x384 d=24 pairs, stride 8 "
                               "(3072 samples), T=10, convergence 0.99, dot metric, tensor backend "
                               "(binary16 in / fp32 accumulate, exact near-tie re-decision)",
                   "pairs_per_gpu_per_step": B, "global_batch": B * world, "height": H, "width": W,
                   "dim": D, "stride": STRIDE, "backend": args.backend, "parallelism": f"pairs dp{world}",
                   "inputs": f"pool of {POOL} gen_random maps (seeds 1000..{1000 + POOL - 1}), pair k = "
                             f"(map k%64, distinct partner); {B * 2 * H * W * D * 4 / 1e9:.2f} GB fp32 "
                             "per GPU per step > 126 MB L2 (no L2 flush needed)",
                   "query_rows_per_step": tot_rows / args.steps,
                   "near_tie_rows_per_step": near_ties / args.steps if world == 1 else None,
                   "matches_per_step_rank0": matches_last,
                   "kernel_breakdown_rank0": breakdown},
        "e2e": {"value": e2e_value, "unit": "pairs/s",
                "h2d_bytes_per_step": int(2 * B * H * W * D * 4),
                "d2h_bytes_per_step": int(B * samples * 3 * 4 + B * 4)},
        "gpu_launches": int(timing["total_launches"]),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s",
                     "frac": (achieved / peak_burst) if achieved else None, "traffic": traffic,
                     "kernel": "tc_scan_kernel (tcgen05 score + running argmax)",
                     "flop_per_score": FLOP_PER_SCORE, "peak_kind": f"{peak_kind} bf16 dense burst",
                     "frac_of_sustained": (achieved / peak_sust) if (achieved and peak_sust) else None,
                     "frac_of_spec": (achieved / SPEC_DENSE_F16_TFLOPS) if achieved else None,
                     "kernel_share_of_step": (tot_score_ms / world) / max_ms / 1.0,
                     "avg_launch_ms": tot_score_ms / max(1, tot_launch)},
        "cpu_baseline": cpu,
        "parity_sample": parity,
        "clocks": clk.summary(),
        "c5_sharded_pair": c5,
        "c3_flashmatch": c3,
    }
    print(json.dumps(line), flush=True)


C5_H, C5_W = 1536, 1152


def bench_c5(fnl, world, rank, local, reps=3):
    """Config C5: one 1536x1152 d=24 pair (1,769,472 px/image, 27,648 samples),
    every NN pass scanning 1/world of the target columns per rank with one
    int64 MIN all-reduce of the per-query (dist, index) keys (NCCL).  Device
    time per pair, max over ranks."""
    import torch
    from paper_2503_10017_b200.shard import match_sharded
    D1 = torch.from_numpy(fnl.gen_random(C5_H, C5_W, D, 2606)).cuda()
    D2 = torch.from_numpy(fnl.gen_random(C5_H, C5_W, D, 2607)).cuda()
    stream = torch.cuda.current_stream()
    match_sharded(D1, D2, stride=STRIDE, metric=METRIC)  # warm-up (workspace, packing)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        pairs, counts, stats = match_sharded(D1, D2, stride=STRIDE, metric=METRIC)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ms = allreduce([ms], op=__import__("torch").distributed.ReduceOp.MAX)[0] if world > 1 else ms
    rows = stats[0]["query_rows"]
    flops = FLOP_PER_SCORE * C5_H * C5_W * rows
    peer = None
    if world > 1:
        # the same pair with the peer-memory transport (keys pushed by the merge
        # epilogues into every rank's IPC-mapped buffer, peer-memory barrier)
        from paper_2503_10017_b200.shard import PeerTransport
        try:
            peers = PeerTransport(((C5_H + 7) // 8) * ((C5_W + 7) // 8), None)
            try:
                match_sharded(D1, D2, stride=STRIDE, metric=METRIC, transport="p2p", peers=peers)
                barrier()
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(reps):
                    pp, pc, _ = match_sharded(D1, D2, stride=STRIDE, metric=METRIC, transport="p2p", peers=peers)
                e1.record(stream)
                torch.cuda.synchronize()
                pms = e0.elapsed_time(e1) / reps
                pms = allreduce([pms], op=__import__("torch").distributed.ReduceOp.MAX)[0]
                same = bool(torch.equal(pp[0, : int(pc[0])], pairs[0, : int(counts[0])]))
                peer = {"transport": "CUDA IPC peer memory, atomicMin pushes fused into the merge epilogues",
                        "ms_per_pair": round(pms, 3), "pairs_per_s": round(1000.0 / pms, 2),
                        "matches_equal_nccl": same}
            finally:
                torch.cuda.synchronize()
                barrier()
                peers.close()
        except Exception as e:  # reported, not fatal: the NCCL number above stands
            peer = {"error": str(e)[:200]}
    return {"workload": f"C5: one {C5_H}x{C5_W} d=24 pair (gen_random 2606/2607), stride 8 "
                        f"({((C5_H + 7) // 8) * ((C5_W + 7) // 8)} samples), dot, tensor backend, target columns "
                        f"sharded over {world} rank(s), int64 MIN all-reduce of (dist, index) keys per NN pass",
            "shards": world, "ms_per_pair": round(ms, 3), "pairs_per_s": round(1000.0 / ms, 2),
            "query_rows": int(rows), "iterations": int(stats[0]["iterations"]),
            "matches": int(counts[0].item()),
            "aggregate_tflops": round(flops / (ms / 1e3) / 1e12, 1), "peer_memory": peer}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--pairs", type=int, default=128, help="pairs per GPU per step")
    ap.add_argument("--backend", default="tensor")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--parity-pairs", type=int, default=2, help="pairs of the timed batch re-checked against the reference")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the sharded 1536x1152 pair (config C5)")
    ap.add_argument("--no-c3", action="store_true", help="skip the FlashMatch attention section (config C3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        main_reference(args)
    else:
        main_b200(args)


if __name__ == "__main__":
    main()
