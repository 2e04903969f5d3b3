"""Command line front end of the B200 matcher: ``python -m paper_2503_10017_b200.cli``.

Mirrors the reference ``fastnn`` CLI (tools/fastnn_cli.cpp:1-452, formats in
docs/formats.md) subcommand for subcommand -- ``gen``, ``match``, ``verify``,
``bench`` -- with the same flags, defaults, output files, report / CSV schemas
and exit codes (0 ok, 1 verification failure or runtime/data error, 2 flag
validation or guard violation).  Differences, all additive:

* every backend runs on the GPU, and ``tensor`` (the tcgen05 FastNN-Lite path)
  is accepted wherever a backend is named;
* ``verify`` uses the GPU exact mutual-NN oracle, so its quadratic-oracle cap
  defaults to 1,048,576 pixels per map instead of 16,384 (``--cap`` still
  applies);
* ``bench`` times the GPU backends (wall clock around each synchronous call,
  host buffers in and out, like the reference's single-threaded timings).
"""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

EXIT_OK, EXIT_FAILURE, EXIT_USAGE = 0, 1, 2
BACKENDS = ("bruteforce", "double", "single", "hybrid", "tensor")
BENCH_HEADER = ("height,width,dim,pixels,block_size,backend,precision,metric,repeats,median_us,min_us,"
                "max_us,a_block_fetches,b_block_fetches,argmin_agreement_vs_full,half_saturated")


class GuardError(Exception):
    """Flag validation / guard violation (exit code 2)."""


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # argparse would exit(2) itself; keep the reference's code and stream
        sys.stderr.write(f"error: {message}\n")
        raise SystemExit(EXIT_USAGE)


def _fnl():
    import paper_2503_10017_b200 as fnl
    return fnl


def _resolve_manifest(path):
    """(fmap1, fmap2, truth or None) with paths relative to the manifest (fastnn_cli.cpp:86-94)."""
    with open(path) as f:
        m = json.load(f)
    base = os.path.dirname(path)
    truth = m.get("ground_truth")
    return (os.path.join(base, m["fmap1"]), os.path.join(base, m["fmap2"]),
            os.path.join(base, truth) if truth else None)


def run_gen(a):
    fnl = _fnl()
    p = fnl.gen_matched_pair(a.height, a.width, a.dim, a.seed, a.noise, a.permute)
    os.makedirs(a.out, exist_ok=True)
    d1, d2 = os.path.join(a.out, "d1.fmap"), os.path.join(a.out, "d2.fmap")
    truth, manifest = os.path.join(a.out, "truth.json"), os.path.join(a.out, "manifest.json")
    fnl.write_fmap(p["d1"], d1)
    fnl.write_fmap(p["d2"], d2)
    with open(truth, "w") as f:
        json.dump({"height": a.height, "width": a.width, "dim": a.dim, "noise_sigma": float(a.noise),
                   "permute": a.permute, "map": [int(x) for x in p["truth"]]}, f)
        f.write("\n")
    with open(manifest, "w") as f:
        json.dump({"fmap1": "d1.fmap", "fmap2": "d2.fmap", "ground_truth": "truth.json"}, f)
        f.write("\n")
    print(f"wrote {d1}, {d2}, {truth}, {manifest}")
    return EXIT_OK


def run_match(a):
    fnl = _fnl()
    if not a.manifest and (not a.in1 or not a.in2):
        raise GuardError("match needs two fmap files or --manifest")
    # flag combinations are rejected before any file is touched (fastnn_cli.cpp:96-111)
    if a.max_iters < 1 or a.block_size < 1 or a.threads < 1:
        raise GuardError("--max-iters, --block-size and --threads must be positive")
    if not (0.0 < a.convergence <= 1.0):
        raise GuardError("convergence_fraction must be in (0, 1]")
    in1, in2 = (a.in1, a.in2) if not a.manifest else _resolve_manifest(a.manifest)[:2]
    d1, d2 = fnl.read_fmap(in1), fnl.read_fmap(in2)
    stride = 0 if a.k > 0 else a.stride  # an explicit k overrides the grid stride
    matches, report = fnl.reciprocal_match(d1, d2, backend=a.backend, k=a.k, stride=stride,
                                           max_iters=a.max_iters, convergence=a.convergence,
                                           metric=a.metric, precision=a.precision,
                                           block_size=a.block_size, threads=a.threads)
    rep = json.loads(report)
    rep["seed"] = a.seed
    with open(a.out, "w") as f:
        for i, j, it in matches.tolist():
            f.write(json.dumps({"i": i, "j": j, "iter": it}, separators=(",", ":")) + "\n")
    rendered = fnl._render_report(rep, a.report_format)
    if a.report:
        with open(a.report, "w") as f:
            f.write(rendered)
    else:
        sys.stdout.write(rendered)
    sys.stderr.write(f"matches: {matches.shape[0]} (of {rep['samples']} samples, {rep['iterations']} iterations)\n")
    return EXIT_OK


def run_verify(a):
    fnl = _fnl()
    if not a.manifest and (not a.in1 or not a.in2):
        raise GuardError("verify needs two fmap files or --manifest")
    in1, in2 = (a.in1, a.in2) if not a.manifest else _resolve_manifest(a.manifest)[:2]
    d1, d2 = fnl.read_fmap(in1), fnl.read_fmap(in2)
    p1, p2 = d1.shape[0] * d1.shape[1], d2.shape[0] * d2.shape[1]
    if p1 > a.cap or p2 > a.cap:
        raise GuardError(f"map exceeds the quadratic-oracle cap ({a.cap} pixels); shrink the instance or raise --cap")
    pairs = []
    with open(a.matches) as f:
        for line in f:
            if line.strip():
                j = json.loads(line)
                pairs.append((int(j["i"]), int(j["j"])))
    oracle = fnl.mutual_nn_exact(d1, d2, metric=a.metric)  # exact, on the GPU
    forward = np.full(p1, -1, dtype=np.int64)
    forward[oracle[:, 0].astype(np.int64)] = oracle[:, 1]
    violations = 0
    for i, j in pairs:
        if not (0 <= i < p1 and forward[i] == j):
            violations += 1
            print(f"violation: pair ({i}, {j}) is not a mutual nearest neighbor")
    print(f"matched: {len(pairs)} oracle_total: {oracle.shape[0]} violations: {violations}")
    return EXIT_OK if violations == 0 else EXIT_FAILURE


def _split(s):
    return [x for x in s.split(",") if x]


def run_bench(a):
    fnl = _fnl()
    sizes = []
    for s in _split(a.sizes):
        if "x" not in s:
            raise GuardError(f"bad --sizes entry '{s}' (expected HEIGHTxWIDTH)")
        h, w = s.split("x", 1)
        sizes.append((int(h), int(w)))
    block_sizes = [int(x) for x in _split(a.block_sizes)]
    backends = _split(a.backends)
    for b in backends:
        if b not in BACKENDS:
            raise GuardError(f"unknown backend '{b}'")
    if not sizes or not block_sizes or not backends or a.repeats == 0:
        raise GuardError("bench sweep must name at least one size, block size and backend")
    rows = []
    for h, w in sizes:
        A = fnl.gen_random(h, w, a.dim, a.seed, True)
        B = fnl.gen_random(h, w, a.dim, a.seed + 1, True)
        for bs in block_sizes:
            want_ref = any(b in ("hybrid", "tensor") for b in backends)
            full_ref = fnl.nn_single_loop(A, B, block_size=bs, metric=a.metric)["nearest"] if want_ref else None
            for b in backends:
                times, res = [], None
                for _ in range(a.repeats):
                    t0 = time.perf_counter()
                    if b == "bruteforce":
                        res = fnl.nn_bruteforce(A, B, metric=a.metric)
                    elif b == "double":
                        res = fnl.nn_double_loop(A, B, block_size=bs, metric=a.metric)
                    elif b == "single":
                        res = fnl.nn_single_loop(A, B, block_size=bs, metric=a.metric)
                    elif b == "hybrid":
                        res = fnl.nn_hybridcast(A, B, block_size=bs, metric=a.metric)
                    else:
                        res = fnl.nn_tensor(A, B, metric=a.metric)
                    times.append((time.perf_counter() - t0) * 1e6)
                agree = None
                if b in ("hybrid", "tensor") and full_ref is not None:
                    agree = float(np.mean(np.asarray(res["nearest"]) == np.asarray(full_ref)))
                rows.append({
                    "height": h, "width": w, "dim": a.dim, "pixels": h * w, "block_size": bs, "backend": b,
                    "precision": "hybrid" if b in ("hybrid", "tensor") else "full", "metric": a.metric,
                    "repeats": a.repeats, "median_us": statistics.median(times), "min_us": min(times),
                    "max_us": max(times), "a_block_fetches": int(res.get("a_block_fetches", 0)),
                    "b_block_fetches": int(res.get("b_block_fetches", 0)),
                    "argmin_agreement_vs_full": agree,
                    "half_saturated": int(res.get("half_saturation_events", 0)) > 0})
    if a.format == "csv":
        lines = [BENCH_HEADER]
        for r in rows:
            ag = "" if r["argmin_agreement_vs_full"] is None else f"{r['argmin_agreement_vs_full']:.6f}"
            lines.append(",".join(str(x) for x in (
                r["height"], r["width"], r["dim"], r["pixels"], r["block_size"], r["backend"], r["precision"],
                r["metric"], r["repeats"], f"{r['median_us']:.3f}", f"{r['min_us']:.3f}", f"{r['max_us']:.3f}",
                r["a_block_fetches"], r["b_block_fetches"], ag, 1 if r["half_saturated"] else 0)))
        text = "\n".join(lines) + "\n"
    else:
        text = json.dumps(rows, indent=2) + "\n"
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        sys.stdout.write(text)
    return EXIT_OK


def _positive(v):
    x = int(v)
    if x <= 0:
        raise argparse.ArgumentTypeError(f"{v} is not a positive number")
    return x


def _nonneg(v):
    x = float(v)
    if x < 0:
        raise argparse.ArgumentTypeError(f"{v} is negative")
    return x


def build_parser():
    p = _Parser(prog="fastnn_b200", description="fast reciprocal nearest-neighbor matching over dense feature maps")
    sub = p.add_subparsers(dest="cmd", required=True, parser_class=_Parser)
    g = sub.add_parser("gen", help="generate a synthetic matched pair with ground truth")
    g.add_argument("--height", type=_positive, default=64)
    g.add_argument("--width", type=_positive, default=48)
    g.add_argument("--dim", type=_positive, default=24)
    g.add_argument("--seed", type=int, default=1)
    g.add_argument("--noise", type=_nonneg, default=0.0)
    g.add_argument("--permute", choices=("identity", "random"), default="random")
    g.add_argument("-o", "--out", required=True, help="output directory")
    m = sub.add_parser("match", help="run reciprocal matching on two fmap files")
    m.add_argument("in1", nargs="?", default="")
    m.add_argument("in2", nargs="?", default="")
    m.add_argument("--manifest", default="")
    m.add_argument("--backend", choices=BACKENDS, default="single")
    m.add_argument("--stride", type=int, default=8)
    m.add_argument("--k", type=int, default=0)
    m.add_argument("--max-iters", dest="max_iters", type=_positive, default=10)
    m.add_argument("--convergence", type=float, default=0.99)
    m.add_argument("--metric", choices=("l2", "dot"), default="l2")
    m.add_argument("--precision", choices=("full", "hybrid"), default="full")
    m.add_argument("--block-size", dest="block_size", type=_positive, default=4096)
    m.add_argument("--threads", type=_positive, default=1)
    m.add_argument("--seed", type=int, default=0)
    m.add_argument("-o", "--out", required=True)
    m.add_argument("--report", default="")
    m.add_argument("--report-format", dest="report_format", choices=("json", "csv"), default="json")
    v = sub.add_parser("verify", help="check a match file against the exhaustive mutual-NN oracle")
    v.add_argument("--matches", required=True)
    v.add_argument("in1", nargs="?", default="")
    v.add_argument("in2", nargs="?", default="")
    v.add_argument("--manifest", default="")
    v.add_argument("--metric", choices=("l2", "dot"), default="l2")
    v.add_argument("--cap", type=int, default=1 << 20)
    b = sub.add_parser("bench", help="sweep backends and report timings and fetches")
    b.add_argument("--sizes", default="512x384")
    b.add_argument("--block-sizes", dest="block_sizes", default="4096")
    b.add_argument("--backends", default="double,single,hybrid")
    b.add_argument("--metric", choices=("l2", "dot"), default="l2")
    b.add_argument("--dim", type=_positive, default=24)
    b.add_argument("--repeats", type=_positive, default=5)
    b.add_argument("--seed", type=int, default=1)
    b.add_argument("-o", "--out", default="")
    b.add_argument("--format", choices=("csv", "json"), default="csv")
    return p


def main(argv=None):
    a = build_parser().parse_args(argv)
    try:
        return {"gen": run_gen, "match": run_match, "verify": run_verify, "bench": run_bench}[a.cmd](a)
    except GuardError as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_USAGE
    except (ValueError, RuntimeError, OSError, KeyError) as e:
        sys.stderr.write(f"error: {e}\n")
        return EXIT_FAILURE


if __name__ == "__main__":
    sys.exit(main())
