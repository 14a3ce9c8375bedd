"""B200-native SpAMM hot path (cuSpAMM, arXiv 2103.13042): tile norms -> skip map ->
masked tile multiply, behind the C ABI of libspamm.so (include/spamm.h).

``from paper_2103_13042_b200 import spamm`` loads the CUDA extension (and raises if it
is missing -- there is no CPU fallback).
"""
__all__ = ["spamm"]
