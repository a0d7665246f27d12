"""RMSNorm in front of the reorder-and-quantize -- TEST INFRASTRUCTURE ONLY.

PAPER.md §3.2 / Fig. 7 (lines 156-163): MicroMix runs ONE reorder-and-quantize
after each normalization layer, shared by the linears that follow it; the
models evaluated (Llama-3.1, Qwen2.5) use RMSNorm.  SURVEY §8(f) F2 fuses
the norm into the RQ kernel.  The paper does not define the norm's arithmetic;
DESIGN.md reading R27 fixes it so that one exact answer exists:

    ss_m  = sum_j x_mj^2                      exact, then rounded once to fp64
    r_m   = 1 / sqrt(ss_m / K + eps)          IEEE fp64 division and square root
    y_mj  = bf16_rne( (x_mj * gamma_j) * r_m ) the product x*gamma is exact in fp64
                                               (8-bit significands), the multiply
                                               by r_m rounds once in fp64, then one
                                               round-to-nearest-even to BF16

and the quantized operand is reorder_quantize(y) (oracle/mx.py).
"""
from __future__ import annotations

from fractions import Fraction

import numpy as np

from .mx import bf16_rne, bf16_rne_bits, bf16_to_f64


def exact_sumsq(x_row_bits: np.ndarray) -> float:
    """sum of squares of one BF16 row, exact (integer arithmetic), rounded once to fp64."""
    mag = (np.asarray(x_row_bits, dtype=np.uint16) & 0x7FFF).astype(np.int64)
    ef = mag >> 7
    m = (mag & 0x7F) | np.where(ef > 0, 0x80, 0)
    e = np.maximum(ef, 1) - 134                     # |x| = m * 2^e
    tot = Fraction(0)
    for ee in np.unique(e):
        s = int(np.sum((m[e == ee].astype(object)) ** 2))
        tot += Fraction(s) * (Fraction(2) ** int(2 * ee))
    return float(tot)                               # Fraction -> float is correctly rounded


def rmsnorm_bf16_bits(x_bits: np.ndarray, gamma_bits: np.ndarray, eps: float) -> np.ndarray:
    """y = RMSNorm(x) * gamma as BF16 bit patterns [rows, K] (definition above)."""
    x_bits = np.asarray(x_bits, dtype=np.uint16)
    rows, K = x_bits.shape
    x = bf16_to_f64(x_bits)
    g = bf16_to_f64(np.asarray(gamma_bits, dtype=np.uint16))
    out = np.empty_like(x_bits)
    for i in range(rows):
        ss = exact_sumsq(x_bits[i])
        r = 1.0 / np.sqrt(ss / K + eps)
        out[i] = bf16_rne_bits((x[i] * g) * r)
    return out


def rmsnorm_f64(x_bits, gamma_bits, eps):
    """The same norm without the final BF16 rounding (for tolerance pins)."""
    x = bf16_to_f64(np.asarray(x_bits, dtype=np.uint16))
    g = bf16_to_f64(np.asarray(gamma_bits, dtype=np.uint16))
    out = np.empty_like(x)
    for i in range(x.shape[0]):
        ss = exact_sumsq(np.asarray(x_bits)[i])
        out[i] = (x[i] * g) * (1.0 / np.sqrt(ss / x.shape[1] + eps))
    return out


__all__ = ["exact_sumsq", "rmsnorm_bf16_bits", "rmsnorm_f64", "bf16_rne"]
