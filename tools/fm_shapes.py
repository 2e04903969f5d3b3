"""Per-shape FlashMatch timing (encoder [2,16,768,64] and decoder [2,12,768,64]
launches separately) for the current FNL_FM_* environment."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import bench_flashmatch as bf  # noqa: E402
from paper_2503_10017_b200 import vit  # noqa: E402
out = {}
for name, call in (("enc", (2, 16, 768, 768)), ("dec", (2, 12, 768, 768))):
    calls = [call] * 24
    out[name] = {"ms_per_launch": bf.time_calls(calls, vit.flash_attn) / 24,
                 "lib_ms_per_launch": bf.time_calls(calls, vit.torch_attn) / 24}
print(json.dumps(out))
