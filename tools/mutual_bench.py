"""Dense mutual NN at 512x384 d=24 (2 x 3.87e10 scores): the tensor route
(each map packed once, both directions back to back on the device, certified
resolution) for mutual_nn_exact (full precision) and mutual_nn_tensor
(binary16-rounded maps), vs the CUDA-core exact scan (FNL_EXACT_KERNEL=cuda_core).
Prints wall ms per call (host maps in, pairs out: includes 2 x 18.9 MB H2D) and
the device ms of the kernels (kernel_profile classes)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_10017_b200 as fnl  # noqa: E402

D1 = fnl.gen_random(512, 384, 24, 606)
D2 = fnl.gen_random(512, 384, 24, 607)
out = {}
for name, f, env in (("exact_tensor_route", fnl.mutual_nn_exact, None),
                     ("tensor_rounded", fnl.mutual_nn_tensor, None),
                     ("exact_cuda_core", fnl.mutual_nn_exact, "cuda_core")):
    if env:
        os.environ["FNL_EXACT_KERNEL"] = env
    else:
        os.environ.pop("FNL_EXACT_KERNEL", None)
    for metric in ("dot", "l2"):
        f(D1, D2, metric=metric)
        fnl.kernel_profile(enable=1, reset=True)
        reps = 3
        t = time.perf_counter()
        for _ in range(reps):
            m = f(D1, D2, metric=metric)
        dt = (time.perf_counter() - t) / reps
        prof = fnl.kernel_profile(enable=0, reset=True)
        dev_ms = sum(v["ms"] for v in prof.values()) / reps
        out[f"{name}/{metric}"] = {
            "wall_ms": round(dt * 1e3, 2), "device_ms": round(dev_ms, 2), "mutual_pairs": int(m.shape[0]),
            "classes_ms": {k: round(v["ms"] / reps, 3) for k, v in prof.items() if v["launches"]},
            "algorithmic_tflops_device": round(2 * 196608 ** 2 * 48 / (dev_ms / 1e3) / 1e12, 1)}
        print(name, metric, out[f"{name}/{metric}"], flush=True)
print(json.dumps(out))
