"""Mixed-precision GEMM of the dequantized operands in fp64 -- TEST INFRASTRUCTURE ONLY.

PAPER.md §2.1 Eq. 2 (lines 47-51):  Y = X W ~= Q(X) Q(W) * s_X s_W, and §3.2 "GEMM
Kernel" (line 143): per output tile the three segment contractions (MXFP4, MXFP6,
MXFP8) accumulate into one result that is returned in BFloat16 (abstract line 6).

Weights are in PyTorch Linear layout W[N, K] (so Y = X W^T); both operands are
reordered with the same permutation (line 151), so

    Y_ref[m, n] = sum_g sum_{k in segment g} dqA_g[m, k] * dqW_g[n, k]

Every dequantized value is (<= 4 significant bits) * 2^e with |e| < 150, so
every product is exact in fp64; the sum is a float64 matmul (library primitive,
accumulation error ~1e-16 relative).  bf16(Y_ref) is the RNE rounding of that.
"""
from __future__ import annotations

import numpy as np

from .formats import E3M2, E4M3
from .mx import RULE_OCP, bf16_rne, dequantize_segments, reorder_quantize


def quantize_operand(bits, perm, n, fmt6=E3M2, fmt8=E4M3, rule=RULE_OCP):
    codes, scales, _ = reorder_quantize(bits, perm, n, fmt6, fmt8, rule)
    return codes, scales


def gemm_ref(a_codes, a_scales, w_codes, w_scales, fmt6=E3M2, fmt8=E4M3,
             rows=None, cols=None) -> np.ndarray:
    """fp64 Y_ref from canonical operands; optional row / column subsets."""
    if rows is not None:
        a_codes = [c[rows] for c in a_codes]
        a_scales = [s[rows] for s in a_scales]
    if cols is not None:
        w_codes = [c[cols] for c in w_codes]
        w_scales = [s[cols] for s in w_scales]
    A = dequantize_segments(a_codes, a_scales, fmt6, fmt8)
    W = dequantize_segments(w_codes, w_scales, fmt6, fmt8)
    return A @ W.T


def mixed_linear_ref(x_bits, w_bits, perm, n, fmt6=E3M2, fmt8=E4M3, rule=RULE_OCP,
                     rows=None, cols=None):
    """End to end from BF16 X[M, K] and W[N, K]: returns (Y_ref fp64, bf16(Y_ref))."""
    x_bits = np.asarray(x_bits)
    w_bits = np.asarray(w_bits)
    if rows is not None:
        x_bits = x_bits[rows]
    if cols is not None:
        w_bits = w_bits[cols]
    ac, asf = quantize_operand(x_bits, perm, n, fmt6, fmt8, rule)
    wc, wsf = quantize_operand(w_bits, perm, n, fmt6, fmt8, rule)
    y = gemm_ref(ac, asf, wc, wsf, fmt6, fmt8)
    return y, bf16_rne(y)


def rel_fro(y, ref) -> float:
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(y - ref) / den) if den > 0 else float(np.linalg.norm(y))
