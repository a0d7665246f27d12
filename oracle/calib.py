"""Threshold-based channel allocation (offline calibration) -- TEST INFRASTRUCTURE ONLY.

PAPER.md §3.1 in the paper's order:

  Q1, Definition 1, Eq. 5 (lines 97-101):
      T(n) = 2^(b+n-1) * max(|X|) / (254 * q_max)
      with b and q_max of the target format (Table 6; b is the Table-6 bias
      literally, Eq. 17 line 492 prints 2^1 for E2M1 -- DESIGN.md R11), max|X|
      the per-tensor maximum over all calibration rows (R10).  Computed as one
      correctly rounded fp64 division of two exact fp64 values.
  Eq. 6 (lines 102-106) and Eq. 17 (lines 489-496):
      P4 = channels with chmax <= T(4);  P6 = channels with T(4) < chmax <= T(6);
      P8 = the rest (channel level, R12).
  Counts rounded to multiples of 32: n8 up first, then n6 up (capped), n4 the
      remainder (R14).
  Q3, Eq. 7 (lines 120-126):
      M_k = (1/L) sum_i |X_ik|; channels sorted ascending by M (stable, lower index
      first on ties, R16): the first n4 reordered channels are MXFP4, then n6
      MXFP6, then n8 MXFP8.
      M_k is the exact mean rounded once to fp64 (R26): the sum of BF16
      magnitudes is accumulated exactly in integer arithmetic.
"""
from __future__ import annotations

import numpy as np

from .formats import E2M1, E2M3, E3M2, fmt
from .mx import bf16_to_f64

INT8_CEIL_DEN = 254  # Eq. 11: E_INT8 = max|X| / 254 (line 447)


def threshold(tmax: float, f, nbits: int) -> float:
    F = fmt(f)
    num = float(2 ** (F.bias + nbits - 1)) * float(tmax)   # exact (power of two x BF16)
    den = float(INT8_CEIL_DEN) * F.qmax                      # exact (1524, 7112, 1905)
    return num / den


def thresholds(tmax: float, fmt6=E3M2):
    return threshold(tmax, E2M1, 4), threshold(tmax, fmt6, 6)


def channel_stats(x_bits: np.ndarray):
    """(chmax fp64[K], chmean fp64[K]) of BF16 bits [L, K].

    chmax is exact.  chmean = fl64(exact_sum / L): every |x| is m * 2^(E-134)
    with m < 2^8 an integer (E = max(biased exponent, 1)), so the column sum is
    an exact integer multiple of 2^-133; Python's int/int true division is
    correctly rounded."""
    x_bits = np.asarray(x_bits, dtype=np.uint16)
    L, K = x_bits.shape
    mag = (x_bits & 0x7FFF).astype(np.int64)
    if np.any((mag >> 7) == 0xFF):
        raise ValueError("non-finite calibration input")
    chmax = bf16_to_f64(np.max(mag, axis=0).astype(np.uint16)) if L else np.zeros(K)
    ef = mag >> 7
    m = (mag & 0x7F) | np.where(ef > 0, 0x80, 0)
    eff = np.maximum(ef, 1)                      # value = m * 2^(eff - 134)
    chmean = np.zeros(K, dtype=np.float64)
    if L == 0:
        return chmax, chmean
    # exact per-(exponent, column) integer sums of m (each < 2^8 * L < 2^53)
    idx = eff * K + np.arange(K, dtype=np.int64)[None, :]
    S = np.bincount(idx.ravel(), weights=m.ravel().astype(np.float64),
                    minlength=256 * K).reshape(256, K)
    for k in range(K):
        tot = 0
        for E in np.nonzero(S[:, k])[0]:
            tot += int(S[E, k]) << int(E - 1)      # value m*2^(E-134) in units of 2^-133
        chmean[k] = tot / (L << 133)               # correctly rounded (Python int division)
    return chmax, chmean


def round_counts(c4: int, c6: int, c8: int, K: int):
    """Counts -> multiples of 32 (n8 up first, then n6 up capped, n4 remainder)."""
    n8 = -(-c8 // 32) * 32
    n6 = min(-(-c6 // 32) * 32, K - n8)
    n4 = K - n8 - n6
    return n4, n6, n8


def calibrate(x_bits: np.ndarray, fmt6=E3M2):
    """Full offline calibration: returns dict(perm, n, tmax, t4, t6, chmax, chmean, c)."""
    x_bits = np.asarray(x_bits, dtype=np.uint16)
    L, K = x_bits.shape
    if K % 32:
        raise ValueError("K must be a multiple of 32")
    chmax, chmean = channel_stats(x_bits)
    tmax = float(np.max(chmax)) if K else 0.0
    if tmax == 0.0:
        raise ValueError("degenerate calibration data: max|X| == 0")
    t4, t6 = thresholds(tmax, fmt6)
    c4 = int(np.sum(chmax <= t4))
    c6 = int(np.sum((chmax > t4) & (chmax <= t6)))
    c8 = K - c4 - c6
    n = round_counts(c4, c6, c8, K)
    perm = np.argsort(chmean, kind="stable").astype(np.int32)
    return dict(perm=perm, n=n, tmax=tmax, t4=t4, t6=t6, chmax=chmax,
                chmean=chmean, c=(c4, c6, c8))


def proportions(chmax: np.ndarray, tmax: float, fmt6=E3M2):
    t4, t6 = thresholds(tmax, fmt6)
    K = len(chmax)
    p4 = np.sum(chmax <= t4) / K
    p6 = np.sum((chmax > t4) & (chmax <= t6)) / K
    return p4, p6, 1.0 - p4 - p6


def avg_bits(n, fmt6=E3M2, fmt8=None):
    """Table 1 accounting: (4 n4 + 6 n6 + 8 n8)/K + 8/32."""
    n4, n6, n8 = n
    K = n4 + n6 + n8
    return (4 * n4 + 6 * n6 + 8 * n8) / K + 8 / 32


def eq6_violations(perm, n, chmax, t4, t6):
    """Channels whose max exceeds their group's threshold (ordering is by mean)."""
    perm = np.asarray(perm)
    n4, n6, _ = n
    g4 = chmax[perm[:n4]]
    g6 = chmax[perm[n4:n4 + n6]]
    return int(np.sum(g4 > t4)), int(np.sum(g6 > t6))


__all__ = ["threshold", "thresholds", "channel_stats", "round_counts", "calibrate",
           "proportions", "avg_bits", "eq6_violations", "E2M3"]
