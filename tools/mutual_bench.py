"""Dense mutual NN at 512x384 (2 x 3.87e10 scores): tensor path vs the exact CUDA-core path."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10017_b200 as fnl
D1 = fnl.gen_random(512, 384, 24, 606); D2 = fnl.gen_random(512, 384, 24, 607)
for name, f in (("tensor", fnl.mutual_nn_tensor), ("exact", fnl.mutual_nn_exact)):
    f(D1, D2, metric="dot")
    t = time.perf_counter(); m = f(D1, D2, metric="dot"); dt = time.perf_counter() - t
    print(f"{name}: {dt * 1e3:.1f} ms, {m.shape[0]} mutual pairs, {2 * 196608 ** 2 * 48 / dt / 1e12:.0f} TFLOP/s algorithmic")
