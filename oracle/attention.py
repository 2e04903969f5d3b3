"""FlashMatch oracle (TEST INFRASTRUCTURE ONLY).

FlashMatch has no code in the reference: PAPER.md:134-139 describes it as
FlashAttention-2 inside the ViT encoder/decoder self- and cross-attention, and
SPEC.md:15,190 excludes it from proj/.  So "parity unpinned" in the sense of
tests/golden: there are no reference golden vectors.  The checker is the
definition itself, restated in float64 numpy:

    O = softmax(Q K^T * scale) V        (per batch and head, non-causal)

evaluated on the SAME binary16 inputs the kernel consumes, with the
max-subtracted softmax.  Only tests/ and bench.py may import this module.
"""
import numpy as np


def attention(q, k, v, scale=None):
    """q [..., Nq, D], k/v [..., Nkv, D] (any float dtype) -> float64 [..., Nq, D]."""
    q = np.asarray(q, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    if scale is None:
        scale = 1.0 / np.sqrt(q.shape[-1])
    s = np.einsum("...qd,...kd->...qk", q, k) * scale
    s -= s.max(axis=-1, keepdims=True)
    p = np.exp(s)
    p /= p.sum(axis=-1, keepdims=True)
    return np.einsum("...qk,...kd->...qd", p, v)


def attention_loop(q, k, v, scale=None):
    """Pure-Python two-pass restatement for tiny cases (pins attention())."""
    nq, d = len(q), len(q[0])
    if scale is None:
        scale = 1.0 / d ** 0.5
    out = []
    for i in range(nq):
        s = [sum(float(q[i][c]) * float(k[j][c]) for c in range(d)) * scale for j in range(len(k))]
        m = max(s)
        e = [np.exp(x - m) for x in s]
        z = sum(e)
        out.append([sum(e[j] * float(v[j][c]) for j in range(len(k))) / z for c in range(d)])
    return np.array(out)
