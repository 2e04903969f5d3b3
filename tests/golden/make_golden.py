"""Generates tests/golden/* from the UNMODIFIED reference (oracle/_ref/_fastnn_ref,
compiled from /root/reference/proj by oracle/Makefile).  Run in the dev
container (the reference sources are not on the GPU box):

    python tests/golden/make_golden.py

Fixtures are small: maps are identified by generator arguments plus a sha256 of
the reference generator's output (the product's gen_random must reproduce the
digest), outputs are stored in full.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402

R = oracle.reference()
TIMING = ("subsample_us", "forward_nn_us", "reverse_nn_us", "harvest_us")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def report(js):
    r = json.loads(js)
    for k in TIMING:
        r.pop(k)
    return r


def main():
    out = {}
    # ---- generators: digests of the reference's libstdc++-based generators
    gens = []
    for (h, w, d, seed, norm) in [(64, 48, 24, 21, True), (64, 48, 24, 121, True), (6, 5, 8, 7, True),
                                   (5, 4, 3, 9, False), (512, 384, 24, 606, True), (512, 384, 24, 607, True),
                                   (12, 9, 8, 2111, True), (8, 8, 6, 1, True)]:
        gens.append({"args": [h, w, d, seed, norm], "sha256": sha(R.gen_random(h, w, d, seed, normalize=norm))})
    pairs = []
    for (h, w, d, seed, sigma, perm) in [(64, 48, 24, 7, 0.05, "random"), (10, 10, 8, 5, 0.0, "random"),
                                          (16, 12, 8, 901, 0.0, "identity")]:
        p = R.gen_matched_pair(h, w, d, seed, sigma, perm)
        pairs.append({"args": [h, w, d, seed, sigma, perm], "d1": sha(p["d1"]), "d2": sha(p["d2"]),
                      "truth": sha(p["truth"])})
    out["gen_random"] = gens
    out["gen_matched_pair"] = pairs

    # ---- binary16 (reference tests/test_half.cpp probes + random + midpoints)
    rng = np.random.default_rng(11)
    probes = [2048.0, 2049.0, 2051.0, 2050.5, 1.0, -2049.0, 0.0, -0.0, 65504.0, 65519.0, 65520.0, -1e9,
              2.0**-24, 2.0**-25, np.nextafter(np.float32(2.0**-25), np.float32(1)), 2.0**-14, 3e-6, 1e-8]
    mags = np.ldexp(rng.uniform(1, 2, 4000), rng.integers(-26, 17, 4000)) * rng.choice([-1, 1], 4000)
    probes = np.concatenate([np.array(probes, np.float32), mags.astype(np.float32)])
    half = np.array([R.to_half_round(float(x)) for x in probes], np.float32)
    np.savez_compressed(os.path.join(HERE, "half.npz"), probes=probes, rounded=half)

    # ---- NN and reciprocal matching at C1 (64x48 d=24)
    D1 = R.gen_random(64, 48, 24, 21)
    D2 = R.gen_random(64, 48, 24, 121)
    nn = {}
    for metric in ("l2", "dot"):
        for prec in ("full", "hybrid"):
            r = R.nn_single_loop(D1, D2, block_size=500, metric=metric, precision=prec)
            nn[f"{metric}_{prec}_nearest"] = r["nearest"]
            nn[f"{metric}_{prec}_min_dist"] = r["min_dist"]
            nn[f"{metric}_{prec}_counters"] = np.array([r["a_block_fetches"], r["b_block_fetches"],
                                                        r["half_saturation_events"]], np.uint64)
    np.savez_compressed(os.path.join(HERE, "nn_c1.npz"), **nn)

    mp = R.gen_matched_pair(64, 48, 24, 7, 0.05, "random")
    recip = []
    for name, (A, B) in (("random", (D1, D2)), ("matched", (mp["d1"], mp["d2"]))):
        for backend in ("single", "hybrid", "double", "bruteforce"):
            for metric in ("l2", "dot"):
                for prec in ("full", "hybrid"):
                    for kw in (dict(stride=8, block_size=100), dict(stride=3, convergence=1.0, block_size=77)):
                        m, rep = R.reciprocal_match(A, B, backend=backend, metric=metric, precision=prec, **kw)
                        recip.append({"pair": name, "backend": backend, "metric": metric, "precision": prec,
                                      "kwargs": kw, "matches": m.tolist(), "report": report(rep)})
    out["reciprocal_c1"] = recip

    # ---- tensor-backend reference semantics at C1: reference single on binary16-rounded maps
    h1, h2 = oracle.half_round_array(D1), oracle.half_round_array(D2)
    tens = []
    for metric in ("l2", "dot"):
        m, rep = R.reciprocal_match(h1, h2, backend="single", metric=metric)
        tens.append({"metric": metric, "matches": m.tolist(), "report": report(rep)})
    out["tensor_semantics_c1"] = tens

    # ---- grid subsample pins
    out["grid"] = [{"args": [h, w, k, s], "ids": R.grid_subsample(h, w, k=k, stride=s).tolist()}
                   for (h, w, k, s) in [(8, 8, 0, 4), (1, 1, 0, 5), (5, 7, 0, 100), (64, 64, 256, 0),
                                        (64, 48, 0, 8), (12, 9, 0, 2), (480, 640, 0, 8)] if h * w <= 4096 or s == 8]

    # ---- C2 (512x384, seeds 606/607, stride 8): match sets of the reference
    C1_ = R.gen_random(512, 384, 24, 606)
    C2_ = R.gen_random(512, 384, 24, 607)
    threads = os.cpu_count() or 1
    c2 = {}
    for metric in ("dot", "l2"):
        m, rep = R.reciprocal_match(C1_, C2_, backend="single", metric=metric, block_size=384, threads=threads)
        c2[f"single_{metric}"] = m
        c2[f"single_{metric}_history"] = np.array(report(rep)["active_history"], np.uint32)
        m, rep = R.reciprocal_match(oracle.half_round_array(C1_), oracle.half_round_array(C2_), backend="single",
                                    metric=metric, block_size=384, threads=threads)
        c2[f"tensor_{metric}"] = m
    np.savez_compressed(os.path.join(HERE, "recip_c2.npz"), **c2)

    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(out, f)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
