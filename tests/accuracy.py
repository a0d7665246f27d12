"""Per-element accuracy of a BF16 GEMM output against the oracle.

Two statements per element, both against the oracle's exact Y_ref (fp64 GEMM of
the dequantized operands, Eq. 2 lines 47-51; BF16 output, line 6):

* ULP distance to bf16(Y_ref): |ord(y) - ord(bf16(Y_ref))| where ord maps BF16
  bit patterns monotonically onto the integers (adjacent BF16 values differ by 1).
* A worst-case error bound for FP32 accumulation in ANY order followed by one BF16
  rounding (readings R19/R20/R28): every product is exact, a sum of K
  terms accumulated in fp32 errs by at most gamma_K * S with gamma_K = K u/(1-K u),
  u = 2^-24, S = sum_k |a_k w_k| (Higham, Accuracy and Stability, Thm 3.1 / Eq.
  3.5), and the final RNE adds at most half a BF16 ulp of the pre-rounding value.
"""
from __future__ import annotations

import numpy as np

from oracle import gemm as ogemm
from oracle import mx as omx


def bf16_ord(bits) -> np.ndarray:
    b = np.asarray(bits, dtype=np.uint16).astype(np.int64)
    mag = b & 0x7FFF
    return np.where(b & 0x8000, -mag, mag)


def bf16_ulp(v) -> np.ndarray:
    """Spacing of BF16 values at |v| (8-bit significand, subnormal spacing 2^-133)."""
    a = np.abs(np.asarray(v, dtype=np.float64))
    _, ex = np.frexp(a)
    return np.ldexp(1.0, np.maximum(ex - 1, -126) - 7)


def ref_and_abs(x_bits, w_bits, perm, n, fmt6, fmt8, rule):
    """(Y_ref, S = |A| |W|^T) from the oracle's canonical operands."""
    ac, asf = ogemm.quantize_operand(np.asarray(x_bits), perm, n, fmt6, fmt8, rule)
    wc, wsf = ogemm.quantize_operand(np.asarray(w_bits), perm, n, fmt6, fmt8, rule)
    A = omx.dequantize_segments(ac, asf, fmt6, fmt8)
    W = omx.dequantize_segments(wc, wsf, fmt6, fmt8)
    return A @ W.T, np.abs(A) @ np.abs(W).T


def report(y_bits, yref, S, K) -> dict:
    """ULP statistics and the worst-case-bound check of one output block."""
    y = omx.bf16_to_f64(y_bits)
    want = omx.bf16_rne_bits(yref)
    d = np.abs(bf16_ord(y_bits) - bf16_ord(want))
    u = 2.0 ** -24
    gamma = K * u / (1 - K * u)
    bound = gamma * S + 0.5 * bf16_ulp(np.abs(yref) + gamma * S) * (1 + 2.0 ** -20)
    err = np.abs(y - yref)
    i = np.unravel_index(int(np.argmax(err / np.maximum(bound, 1e-300))), err.shape)
    j = np.unravel_index(int(np.argmax(d)), d.shape)
    return dict(worst_vs_bound=(float(yref[i]), float(y[i]), float(S[i])),
                worst_ulp=(float(yref[j]), float(y[j]), float(S[j])),
                # accumulation error relative to S, excluding the final rounding: the
                # effective unit roundoff the tensor core's FP32 accumulation showed
                max_accum_err_over_S=float(np.max(np.maximum(err - 0.5 * bf16_ulp(y), 0) /
                                                  np.maximum(S, 1e-300))),
                max_ulp=int(d.max()), p999_ulp=float(np.percentile(d, 99.9)),
                frac_exact=float(np.mean(d == 0)), frac_le1=float(np.mean(d <= 1)),
                bound_violations=int(np.sum(err > bound)),
                max_err_over_bound=float(np.max(err / np.maximum(bound, 1e-300))),
                rel_fro=ogemm.rel_fro(y, yref))
