"""B200-native ULTRA-HSTU (arXiv 2602.16986) hot path: the jagged semi-local HSTU
attention layer, forward and backward, behind the C-ABI library ``libuhstu``.

Importing the package is cheap; the CUDA library is loaded on first use by
``paper_2602_16986_b200.uhstu`` and raises if it is missing (no CPU fallback).
"""
__all__ = ["synth", "uhstu"]
