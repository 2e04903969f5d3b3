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


def node_pool(gen_random, local_rank, local_world):
    """The 64-map pool (1.21 GB fp32), generated ONCE per node: local rank 0
    writes it to /dev/shm and the other ranks of the node map the same pages
    read-only after a barrier, so 8 ranks hold one copy instead of eight."""
    if local_world <= 1:
        return gen_pool(gen_random)
    path = f"/dev/shm/fnl_bench_pool_{H}x{W}x{D}_{POOL}_{os.getppid()}.npy"
    if local_rank == 0:
        arr = np.lib.format.open_memmap(path + ".tmp", mode="w+", dtype=np.float32, shape=(POOL, H, W, D))
        for i in range(POOL):
            arr[i] = gen_random(H, W, D, 1000 + i)
        arr.flush()
        del arr
        os.replace(path + ".tmp", path)
    barrier()
    pool = np.load(path, mmap_mode="r")
    barrier()
    if local_rank == 0:
        os.unlink(path)  # the mappings stay valid
    return [pool[i] for i in range(POOL)]


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
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", str(world)))
    pool = node_pool(fnl.gen_random, int(os.environ.get("LOCAL_RANK", "0")), local_world)
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

    # the timed step stays host-driven whatever the batch size: its K3
    # launches are bracketed by CUDA events (roofline.achieved), which a
    # replayed loop graph would not carry
    graph_max = fnl.loop_graph_max_pairs(0)
    for _ in range(args.warmup):
        step_device()
    # every step matches the same pairs: the per-step work (query rows, near
    # ties) comes from one untimed step with the diagnostic stats switched on
    stats = step_device(with_stats=True)
    rows_per_step = sum(s["query_rows"] for s in stats)
    # rows K3 actually scores (reverse queries answered by the memo excluded):
    # the roofline of the kernel is taken on these, the step-level figure on
    # the reference's own query rows
    computed_per_step = sum(s["computed_query_rows"] for s in stats)
    ties_per_step = sum(s["near_tie_rows"] for s in stats)
    rescans_per_step = sum(s["rescan_rows"] for s in stats)
    torch.cuda.synchronize()
    fnl.kernel_timing(reset=True)
    query_rows, near_ties, computed_rows = 0, 0, 0
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        clk.mark_start()
        ev0.record(stream)
        for _ in range(args.steps):
            step_device()
            query_rows += rows_per_step
            computed_rows += computed_per_step
            near_ties += ties_per_step
        ev1.record(stream)
        torch.cuda.synchronize()
        clk.mark_end()
    barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    timing = fnl.kernel_timing(reset=True)
    matches_last = int(out_counts.sum().item())
    # which pairs each rank matched and how many matches it found (the shards
    # are disjoint contiguous pair ranges; no data-path collective)
    by_rank = [(first_pair, first_pair + B, matches_last)]
    if world > 1:
        import torch.distributed as dist
        by_rank = [None] * world
        dist.all_gather_object(by_rank, (first_pair, first_pair + B, matches_last))

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
    pack_bytes = 2 * B * NT * (D * 4 + 16 * ((D + 7) // 8))  # fp32 in, the stored binary16 chunks out (dot)
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

    # ---- the other backends on the same batch (same stream, CUDA events):
    # the paper's Alg. 3 as the `tensor` backend and the reference's hybrid;
    # their last outputs feed the parity section
    other = {}
    other_outputs = {}
    for bk in [x for x in ("single", "hybrid", "tensor") if x != args.backend]:
        if args.no_other_backends:
            break
        op = torch.empty_like(out_pairs)
        oc = torch.empty_like(out_counts)

        def run_bk():
            fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), B, H, W, D, op.data_ptr(), oc.data_ptr(),
                                        backend=bk, stride=STRIDE, metric=METRIC, stream=stream.cuda_stream,
                                        with_stats=False)
        for _ in range(2):
            run_bk()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrep = max(3, args.steps // 2)
        e0.record(stream)
        for _ in range(nrep):
            run_bk()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / nrep
        ms = allreduce([ms], op=torch.distributed.ReduceOp.MAX)[0] if world > 1 else ms
        other[bk] = {"pairs_per_s": round(B * world / (ms / 1e3), 1), "ms_per_step": round(ms, 3),
                     "steps": nrep}
        other_outputs[bk] = (op, oc)
    fnl.kernel_timing(reset=True)

    # ---- configs[1]: ONE 512x384 pair per call (latency; device-resident, same
    # backend), the batch-1 view of the metric next to the batched value
    single = None
    fnl.loop_graph_max_pairs(graph_max)  # a single pair per call replays its loop as a CUDA graph
    if not args.no_other_backends:
        op1 = torch.empty_like(out_pairs[:1])
        oc1 = torch.empty_like(out_counts[:1])

        def run_one():
            fnl.reciprocal_match_device(d1.data_ptr(), d2.data_ptr(), 1, H, W, D, op1.data_ptr(), oc1.data_ptr(),
                                        backend=args.backend, stride=STRIDE, metric=METRIC,
                                        stream=stream.cuda_stream, with_stats=False)
        for _ in range(3):
            run_one()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        nrep = 20
        e0.record(stream)
        for _ in range(nrep):
            run_one()
        e1.record(stream)
        torch.cuda.synchronize()
        ms1 = e0.elapsed_time(e1) / nrep
        single = {"workload": "configs[1]: one C2 pair per call (pair 0 of the batch), device-resident, backend "
                              + args.backend + ", CUDA events over 20 back-to-back calls",
                  "ms_per_pair": round(ms1, 3), "pairs_per_s": round(1e3 / ms1, 1),
                  "identical_to_batched": bool(torch.equal(oc1[0], out_counts[0]) and
                                               torch.equal(op1[0, :int(oc1[0])], out_pairs[0, :int(oc1[0])]))}
    fnl.loop_graph_max_pairs(0)
    fnl.kernel_timing(reset=True)

    # ---- C5: one oversized 1536x1152 pair, target columns sharded over the ranks
    c5 = None
    if not args.no_c5:
        c5 = bench_c5(fnl, world, rank, local, args.backend)

    # ---- C3: FlashMatch attention at the MASt3R ViT shapes (rank 0)
    c3 = None
    if rank == 0 and not args.no_c3:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import bench_flashmatch
        c3 = bench_flashmatch.run(peaks()[0])

    # ---- max over ranks
    max_ms, max_e2e = allreduce([elapsed_ms, e2e_s], op=__import__("torch").distributed.ReduceOp.MAX) \
        if world > 1 else (elapsed_ms, e2e_s)
    tot_rows, tot_computed, tot_score_ms, tot_launch = allreduce(
        [query_rows, computed_rows, timing["score_ms"], timing["score_launches"]],
        op=__import__("torch").distributed.ReduceOp.SUM) \
        if world > 1 else (query_rows, computed_rows, timing["score_ms"], timing["score_launches"])

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
        parity = parity_checks(fnl, ref, oracle, pool, B, args, samples, threads, out_pairs, out_counts,
                               other_outputs)

    if rank != 0:
        return
    pairs_total = B * world * args.steps
    value = pairs_total / (max_ms / 1000.0)
    e2e_value = B * world * args.e2e_steps / max_e2e
    peak_burst, peak_sust, peak_kind = peaks()
    flops = FLOP_PER_SCORE * NT * tot_computed
    achieved = flops / (tot_score_ms / 1000.0) / 1e12 if tot_score_ms > 0 else None
    # the whole step against the same peak, on the reference's query rows
    step_tflops = FLOP_PER_SCORE * NT * tot_rows / (max_ms / 1000.0) / 1e12 / world
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
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f16 in / f16 accumulate (tensor-core candidate scores, certified margin); fp32 reference chain for the decision",
        "data": "synthetic",
        "config": {"workload": "C2/C4: FastNN-Lite reciprocal matching of 512x384 d=24 pairs, stride 8 "
                               f"(3072 samples), T=10, convergence 0.99, dot metric, backend {args.backend} "
                               "on the tcgen05 route (HybridCast: binary16-in tensor-core scores, accumulated "
                               "in binary16 when the norms allow it, nominate candidate sub-tiles; the winner "
                               "is decided by the reference chain in the backend's own arithmetic, so results "
                               "are identical to the reference's)",
                   "pairs_per_gpu_per_step": B, "global_batch": B * world, "height": H, "width": W,
                   "dim": D, "stride": STRIDE, "backend": args.backend, "parallelism": f"pairs dp{world}",
                   "inputs": f"pool of {POOL} gen_random maps (seeds 1000..{1000 + POOL - 1}), pair k = "
                             f"(map k%64, distinct partner); {B * 2 * H * W * D * 4 / 1e9:.2f} GB fp32 "
                             "per GPU per step > 126 MB L2 (no L2 flush needed)",
                   "query_rows_per_step": tot_rows / args.steps,
                   "computed_query_rows_per_step": tot_computed / args.steps,
                   "near_tie_rows_per_step": near_ties / args.steps if world == 1 else None,
                   "rescan_rows_per_step": rescans_per_step if world == 1 else None,
                   "matches_per_step_rank0": matches_last,
                   "pairs_by_rank": [[int(a), int(b)] for a, b, _ in by_rank],
                   "matches_by_rank": [int(m) for _, _, m in by_rank],
                   "host_staging_per_rank_gb": round(2 * B * H * W * D * 4 / 1e9, 2),
                   "pool": f"{POOL} maps, {POOL * H * W * D * 4 / 1e9:.2f} GB, one copy per node (/dev/shm)",
                   "kernel_breakdown_rank0": breakdown},
        "e2e": {"value": e2e_value, "unit": "pairs/s",
                "h2d_bytes_per_step": int(2 * B * H * W * D * 4),
                "d2h_bytes_per_step": int(B * samples * 3 * 4 + B * 4)},
        "gpu_launches": int(timing["total_launches"]),
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_burst, "unit": "TFLOP/s",
                     "frac": (achieved / peak_burst) if achieved else None, "traffic": traffic,
                     "kernel": "tc_scan_kernel (tcgen05 scores + running top-6 sub-tile maxima)",
                     "flop_per_score": FLOP_PER_SCORE, "peak_kind": f"{peak_kind} bf16 dense burst",
                     "frac_of_sustained": (achieved / peak_sust) if (achieved and peak_sust) else None,
                     "frac_of_spec": (achieved / SPEC_DENSE_F16_TFLOPS) if achieved else None,
                     "kernel_share_of_step": (tot_score_ms / world) / max_ms / 1.0,
                     "step_tflops_per_gpu": step_tflops,
                     "step_frac": step_tflops / peak_burst,
                     "rows_basis": "achieved: K3 TFLOP/s on the rows it scores (reverse queries answered by the "
                                   "reverse-NN memo excluded); step_*: the reference's query rows over the "
                                   "whole timed step",
                     "avg_launch_ms": tot_score_ms / max(1, tot_launch)},
        "cpu_baseline": cpu,
        "parity_sample": parity,
        "other_backends": other,
        "c2_single_pair": single,
        "clocks": clk.summary(),
        "c5_sharded_pair": c5,
        "c3_flashmatch": c3,
    }
    print(json.dumps(line), flush=True)


def parity_checks(fnl, ref, oracle, pool, B, args, samples, threads, out_pairs, out_counts, other_outputs):
    """Re-check outputs of the timed batch against the reference run on the
    SAME fp32 maps (untimed, rank 0):
      * the headline backend: ordered (i, j, iter) MatchSets identical to the
        reference's same backend, for parity_pairs pairs spread over the batch;
      * hybrid vs the reference's hybrid (2 pairs);
      * the paper's Alg. 3 (`tensor`: binary16 in, fp32 compare) vs the
        reference `single` on the unrounded maps: MatchSets, and per grid query
        the forward NN, where a disagreement is only allowed when the fp32
        top-2 distance gap is below eps_q, the bound on what binary16 input
        rounding can move a distance by (both candidates)."""
    bs = math.ceil(samples / threads)
    idx = sorted({int(round(x)) for x in np.linspace(0, B - 1, min(args.parity_pairs, B))})

    def ref_match(i, backend):
        a, b = pair_maps(i)
        m, _ = ref.reciprocal_match(pool[a], pool[b], backend=backend, metric=METRIC, stride=STRIDE,
                                    block_size=bs, threads=threads)
        return m

    def same(op, oc, i, want):
        n = int(oc[i].item())
        return n == len(want) and np.array_equal(op[i, :n].cpu().numpy().astype(np.uint32), want)

    ref_single = {}
    head = 0
    for i in idx:
        want = ref_match(i, "single" if args.backend in ("single", "tensor") else args.backend)
        ref_single[i] = want
        head += int(same(out_pairs, out_counts, i, want))
    out = {"pairs_checked": len(idx), "pair_indices": idx, "identical": head,
           "checker": f"oracle/_ref (the unmodified reference compiled from /root/reference) reciprocal_match "
                      f"backend={'single' if args.backend == 'tensor' else args.backend} on the same fp32 maps, "
                      f"ordered (i, j, iter) triples of the last timed step"}
    if args.backend == "tensor":
        out["note"] = "headline is Alg. 3: identical only where no near tie flips (see same_input_alg3)"
    if "hybrid" in other_outputs or args.backend == "hybrid":
        op, oc = other_outputs.get("hybrid", (out_pairs, out_counts))
        hi = idx[:2]
        out["hybrid_vs_reference_hybrid"] = {
            "pairs_checked": len(hi), "identical": sum(int(same(op, oc, i, ref_match(i, "hybrid"))) for i in hi)}
    if "tensor" in other_outputs or args.backend == "tensor":
        op, oc = other_outputs.get("tensor", (out_pairs, out_counts))
        ti = idx[:2]
        msets = sum(int(same(op, oc, i, ref_single[i])) for i in ti)
        grid = np.asarray(fnl.grid_subsample(H, W, 0, STRIDE), dtype=np.int64)
        nq = mism = above = near = 0
        eps_max = 0.0
        for i in ti:
            a, b = pair_maps(i)
            Q = pool[a].reshape(-1, D)[grid]
            T = pool[b].reshape(-1, D)
            ours = fnl.nn_tensor(Q[None], pool[b], metric=METRIC)["nearest"]
            theirs = ref.nn_single_loop(Q[None], pool[b], block_size=math.ceil(len(Q) / threads), metric=METRIC,
                                        precision="full", threads=threads)["nearest"]
            qn = np.linalg.norm(Q.astype(np.float64), axis=1)
            tn = float(np.linalg.norm(T.astype(np.float64), axis=1).max())
            # distance units (dot: -q.t); binary16 rounding u = 2^-11 per input,
            # subnormal step 2^-24, plus both fp32 chains' rounding
            eps = 2.0 * (2.0**-10 * qn * tn + 2.0**-24 * math.sqrt(D) * (qn + tn)) + 4.0 * (D + 2) * 2.0**-24 * qn * tn
            T64 = T.astype(np.float64)
            gaps = np.empty(len(Q))
            for c0 in range(0, len(Q), 256):
                s = -(Q[c0:c0 + 256].astype(np.float64) @ T64.T)
                p2 = np.partition(s, 1, axis=1)[:, :2]
                gaps[c0:c0 + 256] = p2[:, 1] - p2[:, 0]
            bad = ours != theirs
            nq += len(Q)
            mism += int(bad.sum())
            above += int((bad & (gaps > eps)).sum())
            near += int((gaps <= eps).sum())
            eps_max = max(eps_max, float(eps.max()))
        out["same_input_alg3"] = {
            "backend": "tensor (PAPER.md Alg. 3: binary16 in, fp32 accumulate and compare)",
            "vs": "reference single on the same unrounded fp32 maps",
            "matchsets_identical": f"{msets}/{len(ti)}",
            "grid_queries_checked": nq, "mismatched_queries": mism,
            "mismatches_with_gap_above_eps": above, "queries_with_gap_below_eps": near,
            "eps": "per query, distance units: 2(2^-10 |q| t_max + 2^-24 sqrt(d)(|q| + t_max)) + "
                   "4(d+2) 2^-24 |q| t_max (binary16 rounding of both inputs moves each candidate's distance "
                   f"by at most half of it); max over the sample {eps_max:.3g}"}
    return out


C5_H, C5_W = 1536, 1152


def c5_golden(backend):
    """The reference's own C5 MatchSet (tests/golden/recip_c5.npz, made from
    oracle/_ref by tests/golden/make_golden_c5.py), or None."""
    path = os.path.join(ROOT, "tests", "golden", "recip_c5.npz")
    key = f"matches_{backend}"
    if not os.path.exists(path):
        return None
    z = np.load(path)
    return z[key] if key in z else None


def bench_c5(fnl, world, rank, local, backend, reps=3):
    """Config C5: one 1536x1152 d=24 pair (1,769,472 px/image, 27,648 samples),
    every NN pass scanning 1/world of the target columns per rank with one
    int64 MIN all-reduce of the per-query (dist, index) keys (NCCL).  Device
    time per pair, max over ranks."""
    import torch
    from paper_2503_10017_b200.shard import match_sharded
    D1 = torch.from_numpy(fnl.gen_random(C5_H, C5_W, D, 2606)).cuda()
    D2 = torch.from_numpy(fnl.gen_random(C5_H, C5_W, D, 2607)).cuda()
    stream = torch.cuda.current_stream()
    match_sharded(D1, D2, stride=STRIDE, metric=METRIC, backend=backend)  # warm-up (workspace, packing)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        pairs, counts, stats = match_sharded(D1, D2, stride=STRIDE, metric=METRIC, backend=backend)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    ms = allreduce([ms], op=__import__("torch").distributed.ReduceOp.MAX)[0] if world > 1 else ms
    rows = stats[0]["query_rows"]
    computed = stats[0]["computed_query_rows"]  # reverse queries answered by the memo excluded
    flops = FLOP_PER_SCORE * C5_H * C5_W * computed
    peer = None
    if world > 1:
        # the same pair with the peer-memory transport (keys pushed by the merge
        # epilogues into every rank's IPC-mapped buffer, peer-memory barrier)
        from paper_2503_10017_b200.shard import PeerTransport
        try:
            peers = PeerTransport(((C5_H + 7) // 8) * ((C5_W + 7) // 8), None)
            try:
                match_sharded(D1, D2, stride=STRIDE, metric=METRIC, backend=backend, transport="p2p", peers=peers)
                barrier()
                torch.cuda.synchronize()
                e0.record(stream)
                for _ in range(reps):
                    pp, pc, _ = match_sharded(D1, D2, stride=STRIDE, metric=METRIC, backend=backend,
                                              transport="p2p", peers=peers)
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
    gold = c5_golden(backend)
    n = int(counts[0].item())
    parity = None
    if gold is not None:
        parity = {"identical": bool(n == len(gold) and np.array_equal(pairs[0, :n].cpu().numpy().astype(np.uint32),
                                                                         gold)),
                  "checker": f"tests/golden/recip_c5.npz: the reference's own reciprocal_match backend={backend} "
                             "on the same maps (generated from oracle/_ref)"}
    return {"workload": f"C5: one {C5_H}x{C5_W} d=24 pair (gen_random 2606/2607), stride 8 "
                        f"({((C5_H + 7) // 8) * ((C5_W + 7) // 8)} samples), dot, backend {backend}, target columns "
                        f"sharded over {world} rank(s), int64 MIN all-reduce of (dist, index) keys per NN pass",
            "shards": world, "ms_per_pair": round(ms, 3), "pairs_per_s": round(1000.0 / ms, 2),
            "query_rows": int(rows), "computed_query_rows": int(computed), "iterations": int(stats[0]["iterations"]),
            "matches": int(counts[0].item()),
            "aggregate_tflops": round(flops / (ms / 1e3) / 1e12, 1), "peer_memory": peer, "parity": parity}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--pairs", type=int, default=128, help="pairs per GPU per step")
    ap.add_argument("--backend", default="single",
                    help="headline backend: the reference's default `single` (full precision, bit-identical "
                         "to the reference on the same inputs) on the tcgen05 route")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--parity-pairs", type=int, default=8,
                    help="pairs of the timed batch (first .. last) re-checked against the reference")
    ap.add_argument("--no-other-backends", action="store_true", help="skip timing the non-headline backends")
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
