"""K4 exact scan at several descriptor dims: device time of one dense NN query
(backend single / hybrid, dot) -- used to check the per-dim queries-per-thread
choice (QB) against register spills."""
import os
import sys
import time

sys.path.insert(0, os.environ.get("FNL_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import paper_2503_10017_b200 as fnl

for d in (24, 48, 64):
    A = fnl.gen_random(64, 128, d, 5)
    B = fnl.gen_random(256, 256, d, 6)
    for be in ("single", "hybrid"):
        f = fnl.nn_single_loop if be == "single" else fnl.nn_hybridcast
        kw = dict(metric="dot") if be == "hybrid" else dict(metric="dot", precision="full")
        f(A, B, **kw)
        t = time.perf_counter()
        for _ in range(5):
            r = f(A, B, **kw)
        dt = (time.perf_counter() - t) / 5
        print(f"d={d} {be}: {dt * 1e3:.2f} ms, {A.shape[0] * A.shape[1] * B.shape[0] * B.shape[1] / dt / 1e9:.1f} G scores/s,"
              f" checksum {int(np.asarray(r['nearest']).astype(np.int64).sum())}")
