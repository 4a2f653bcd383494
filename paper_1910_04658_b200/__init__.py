"""B200-native BinSketch hot path (arXiv 1910.04658): C-ABI library + thin binding.

The product is ``libbinsketch.so`` (CUDA kernels for sm_100a behind the C ABI
in ``include/binsketch.h``); ``binsketch`` is the ctypes binding with the same
entry-point names. PyTorch supplies device memory, streams and
``torch.distributed`` only.
"""
from . import binsketch  # noqa: F401
from .binsketch import (COS, HAM, IP, JS, MEASURES, BinSketchError, andpopc, build, build_seeded,  # noqa: F401
                        card_table, device_status, estimate, make_pi, popcount, recommended_N, topk,
                        workspace_bytes, words)

__all__ = ["binsketch", "make_pi", "build", "build_seeded", "popcount", "andpopc", "estimate", "topk",
           "card_table", "device_status", "workspace_bytes", "words", "recommended_N", "BinSketchError",
           "IP", "HAM", "JS", "COS", "MEASURES"]
