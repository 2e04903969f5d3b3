"""Run a dense tensor NN pass (12,288 queries x 196,608 targets) with the K3
clock trace on: FNL_TC_DEBUG=16 python tools/tc_trace_run.py; then
python tools/tc_trace.py /tmp/fnl_tc_trace.bin"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10017_b200 as fnl  # noqa: E402
D1 = fnl.gen_random(512, 384, 24, 606)
D2 = fnl.gen_random(512, 384, 24, 607)
q = D1[:32]  # 32 x 384 = 12,288 query rows
for _ in range(2):
    fnl.nn_tensor(q, D2, metric="dot")
print("ok")
