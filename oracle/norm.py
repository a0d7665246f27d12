"""RMSNorm in front of the reorder-and-quantize -- TEST INFRASTRUCTURE ONLY.

PAPER.md §3.2 / Fig. 7 (lines 156-163): MicroMix runs ONE reorder-and-quantize
after each normalization layer, shared by the linears that follow it; the
models evaluated (Llama-3.1, Qwen2.5) use RMSNorm.  SURVEY §8(f) F2 fuses
the norm into the RQ kernel.  The paper does not define the norm's arithmetic;
DESIGN.md reading R27 fixes it so that one exact answer exists:

    ss_m  = sum_j x_mj^2                      exact, then rounded once to fp64
    r_m   = fp32( 1 / sqrt(ss_m / K + eps) )  IEEE fp64 division and square root,
                                               rounded once to fp32
    t_mj  = bf16_rne( fp32(x_mj * r_m) )      normalised activation in BF16
    y_mj  = bf16_rne( fp32(gamma_j * t_mj) )  weight applied to the BF16 value

i.e. the HF LlamaRMSNorm data flow (fp32 normalise, cast to BF16, multiply by the
BF16 weight) with the row's sum of squares taken exactly, so that the result does
not depend on a reduction order.

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


def row_scale_f32(x_row_bits, K: int, eps: float) -> np.float32:
    """r = fp32(1 / sqrt(exact_sumsq / K + eps)) (fp64 arithmetic, one fp32 rounding)."""
    return np.float32(1.0 / np.sqrt(exact_sumsq(x_row_bits) / K + eps))


def rmsnorm_bf16_bits(x_bits: np.ndarray, gamma_bits: np.ndarray, eps: float) -> np.ndarray:
    """y = RMSNorm(x) * gamma as BF16 bit patterns [rows, K] (definition above)."""
    x_bits = np.asarray(x_bits, dtype=np.uint16)
    rows, K = x_bits.shape
    x = bf16_to_f64(x_bits).astype(np.float32)                      # exact
    g = bf16_to_f64(np.asarray(gamma_bits, dtype=np.uint16)).astype(np.float32)
    out = np.empty_like(x_bits)
    for i in range(rows):
        r = row_scale_f32(x_bits[i], K, eps)
        t = bf16_rne((x[i] * r).astype(np.float64))                    # fp32 multiply, BF16 RNE
        out[i] = bf16_rne_bits((g * t.astype(np.float32)).astype(np.float64))
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


__all__ = ["exact_sumsq", "row_scale_f32", "rmsnorm_bf16_bits", "rmsnorm_f64", "bf16_rne"]
