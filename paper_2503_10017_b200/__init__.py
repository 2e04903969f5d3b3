"""B200-native FastNN-Lite / HybridCast matching path (arXiv 2503.10017, Speedy MASt3R).

Drop-in for the reference ``fastnn`` Python package (``python/fastnn/__init__.py``):
the same 14 functions with the same signatures, defaults and return types,
backed by hand-written sm_100a kernels through ``libfastnn_b200.so``.  Extra
entry points: ``nn_tensor``, ``reciprocal_match_batch``,
``reciprocal_match_device``, ``kernel_timing``.

There is no CPU fallback: importing works anywhere (host-only helpers such as
``gen_random`` and ``grid_subsample`` run on the CPU), but every matching / NN
call raises RuntimeError when no B200 is present, and the import itself fails
loudly if the compiled extension is missing.
"""
import os as _os

_here = _os.path.dirname(_os.path.abspath(__file__))
try:
    from ._fastnn import (  # noqa: F401
        _parse_report,
        _render_report,
        _tensor_selftest,
        abi_version,
        block_distances,
        device_count,
        dist_scalar,
        gen_matched_pair,
        gen_random,
        grid_subsample,
        kernel_profile,
        kernel_timing,
        loop_graph_max_pairs,
        mutual_nn_exact,
        mutual_nn_tensor,
        nn_bruteforce,
        nn_double_loop,
        nn_hybridcast,
        nn_single_loop,
        nn_tensor,
        read_fmap,
        reciprocal_match,
        reciprocal_match_batch,
        reciprocal_match_device,
        set_device,
        to_half_round,
        write_fmap,
    )
except ImportError as e:  # fail loudly: the product has no Python fallback
    raise ImportError(
        f"paper_2503_10017_b200: compiled extension missing or broken ({e}); "
        "run `python -c 'import __graft_entry__ as g; g.build()'` (or `make`) first") from e

from .flashmatch import flashmatch  # noqa: E402,F401  (K7 attention, torch tensors)

LIBRARY_PATH = _os.path.join(_here, "libfastnn_b200.so")

__all__ = [
    "block_distances",
    "dist_scalar",
    "gen_matched_pair",
    "gen_random",
    "grid_subsample",
    "mutual_nn_exact",
    "nn_bruteforce",
    "nn_double_loop",
    "nn_hybridcast",
    "nn_single_loop",
    "read_fmap",
    "reciprocal_match",
    "to_half_round",
    "write_fmap",
    # extensions of this build
    "nn_tensor",
    "mutual_nn_tensor",
    "reciprocal_match_batch",
    "reciprocal_match_device",
    "kernel_timing",
    "kernel_profile",
    "loop_graph_max_pairs",
    "flashmatch",
    "device_count",
    "set_device",
    "abi_version",
]

__version__ = "0.1.0"
