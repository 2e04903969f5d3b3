"""Time every FlashMatch kernel version at the C3 shapes (one process per
version: FNL_FM_VERSION is read once per process).
Usage: python tools/fm_versions.py [versions...]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = """
import sys, json
sys.path.insert(0, %r)
sys.path.insert(0, %r)
import bench_flashmatch as bf
from paper_2503_10017_b200 import vit
m = vit.MASt3RViT(seed=0)
calls = m.attention_calls()
print(json.dumps({"ms": bf.time_calls(calls, vit.flash_attn), "lib_ms": bf.time_calls(calls, vit.torch_attn)}))
""" % (ROOT, os.path.join(ROOT, "tools"))
for v in (sys.argv[1:] or ["2", "3"]):
    env = dict(os.environ, FNL_FM_VERSION=v)
    out = subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    print(f"v{v}: {line}")
