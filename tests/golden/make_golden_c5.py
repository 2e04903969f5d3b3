"""Generates tests/golden/recip_c5.npz: the reference MatchSet of BASELINE
config C5 (one 1536x1152 d=24 pair, gen_random seeds 2606/2607, dot, stride 8
-> 27,648 samples), from the UNMODIFIED reference (oracle/_ref/_fastnn_ref,
compiled from /root/reference/proj by oracle/Makefile), backend single and
backend hybrid.  Run in the dev container (minutes of CPU):

    python tests/golden/make_golden_c5.py

The maps are identified by the generator arguments plus the sha256 of the
reference generator's output (the product's gen_random must reproduce it).
"""
import hashlib
import json
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402

R = oracle.reference()
H, W, D, S1, S2, STRIDE = 1536, 1152, 24, 2606, 2607, 8
TIMING = ("subsample_us", "forward_nn_us", "reverse_nn_us", "harvest_us")


def main():
    threads = os.cpu_count() or 1
    D1 = R.gen_random(H, W, D, S1)
    D2 = R.gen_random(H, W, D, S2)
    samples = math.ceil(H / STRIDE) * math.ceil(W / STRIDE)
    bs = math.ceil(samples / threads)
    out = {"sha_d1": np.frombuffer(hashlib.sha256(D1.tobytes()).digest(), np.uint8),
           "sha_d2": np.frombuffer(hashlib.sha256(D2.tobytes()).digest(), np.uint8)}
    meta = {"args": [H, W, D, S1, S2, STRIDE], "metric": "dot", "threads": threads}
    for backend in ("single", "hybrid"):
        t0 = time.time()
        m, rep = R.reciprocal_match(D1, D2, backend=backend, metric="dot", stride=STRIDE, block_size=bs,
                                    threads=threads)
        r = json.loads(rep)
        for k in TIMING:
            r.pop(k)
        out[f"matches_{backend}"] = np.asarray(m, np.uint32)
        meta[f"report_{backend}"] = r
        print(backend, len(m), f"{time.time() - t0:.0f}s", flush=True)
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "recip_c5.npz"), **out)


if __name__ == "__main__":
    main()
