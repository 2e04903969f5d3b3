"""Times the K3 tensor kernel on a dense 12288 x 196608 NN (d=24, dot) -- a
profiling probe, not a test.  FNL_TC_DEBUG=1/2 strips the epilogue."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2503_10017_b200 as f
A = f.gen_random(96, 128, 24, 1)
B = f.gen_random(512, 384, 24, 2)
for _ in range(2):
    f.nn_tensor(A, B, "dot")
f.kernel_timing(reset=True)
for _ in range(5):
    f.nn_tensor(A, B, "dot")
t = f.kernel_timing(reset=True)
ms = t["score_ms"] / t["score_launches"]
scores = A.shape[0] * A.shape[1] * B.shape[0] * B.shape[1]
print(f"debug={os.environ.get('FNL_TC_DEBUG','0')} tc_scan {ms:.3f} ms  {scores/ms/1e9:.2f} Tscore/s  "
      f"{48*scores/ms/1e9:.1f} TFLOP/s algorithmic  {scores/ms*1e3/148/1.965e9:.1f} scores/clk/SM")
