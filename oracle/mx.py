"""MX block quantization and the reorder-and-quantize step -- TEST INFRASTRUCTURE ONLY.

Follows PAPER.md in the paper's order:

  Eq. 1 (§2.1, lines 40-45):  Q(X_j) = round(X_j / s),  s = 2^(floor(log2 max|X_i|) - b)
      over blocks X_i of k = 32 consecutive elements, "round" = nearest MXFP value.
      Offset reading (R1): rule "ocp" (default) subtracts
      emax = floor(log2 q_max) (E2M1 2, E3M2 4, E2M3 2, E4M3 8, E5M2 15);
      rule "paper" subtracts Table 6's bias b literally.
      Zero block -> e = -127 (R2); e clamped to [-127, 127] (R3); the exponent is
      taken from the exact binary exponent (frexp), so BF16 subnormals are exact (R7).
  §3.2 "Quantization Kernel" (line 151) + Fig. 6 caption (line 148):
      gather the channels by the calibrated indices, split the reordered row
      into the three parts P4 | P6 | P8 (§3.1 line 91), block-quantize each part
      (blocks = 32 consecutive reordered channels inside a part, R21).
  Weights (line 151, Fig. 1 caption line 20): the same permutation and the same
      three-part block quantization, blocks along K (R17).

Canonical oracle outputs (never the GPU's packed layout):
  codes[g]  uint8 [rows, n_g]      one element code per byte (sign in bit bits-1)
  scales[g] uint8 [rows, n_g/32]   E8M0 byte = e + 127
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

from .formats import E2M1, E3M2, E4M3, fmt

RULE_OCP, RULE_PAPER = 0, 1
BLOCK = 32

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def build_lib(force: bool = False) -> str:
    """Compile oracle/encode.c (plain gcc + OpenMP) next to this file."""
    so = os.path.join(_HERE, "liboracle_encode.so")
    src = os.path.join(_HERE, "encode.c")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", so, src, "-lm"])
    return so


def _lib():
    global _LIB
    if _LIB is None:
        lib = ctypes.CDLL(build_lib())
        lib.orc_encode_nearest.restype = None
        lib.orc_encode_nearest.argtypes = [
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_void_p]
        _LIB = lib
    return _LIB


# ----------------------------------------------------------------------------- BF16

def bf16_to_f64(bits) -> np.ndarray:
    """Exact value of BF16 bit patterns (BF16 = the top 16 bits of an fp32)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    with np.errstate(invalid="ignore"):
        return b.view(np.float32).astype(np.float64)


def bf16_rne(y) -> np.ndarray:
    """Round fp64 values to BF16 (8-bit significand, round-half-even), returned
    as fp64 values.  One rounding from fp64; BF16 subnormal spacing 2^-133."""
    y = np.asarray(y, dtype=np.float64)
    _, ex = np.frexp(y)                       # y = m * 2^ex, m in [0.5, 1)
    q = np.maximum(ex - 1, -126)              # exponent of y's binade (>= min normal)
    ulp_exp = q - 7
    r = np.ldexp(np.rint(np.ldexp(y, -ulp_exp)), ulp_exp)   # rint = half-to-even
    return r


def bf16_rne_bits(y) -> np.ndarray:
    r = bf16_rne(y).astype(np.float32)
    return (r.view(np.uint32) >> 16).astype(np.uint16)


# ----------------------------------------------------------------------------- Eq. 1

def scale_offset(f, rule: int) -> int:
    F = fmt(f)
    return F.emax if rule == RULE_OCP else F.bias


def block_exponent(blocks: np.ndarray, f, rule: int = RULE_OCP) -> np.ndarray:
    """Shared scale exponent e of each block (last axis = the 32 block values).

    e = floor(log2 max|X_i|) - offset, clamped to [-127, 127]; e = -127 for an
    all-zero block.  floor(log2 a) = frexp(a).exponent - 1 exactly."""
    a = np.max(np.abs(blocks), axis=-1)
    _, ex = np.frexp(a)
    e = (ex - 1) - scale_offset(f, rule)
    e = np.clip(e, -127, 127)
    e = np.where(a == 0.0, -127, e)
    return e.astype(np.int32)


def encode(v: np.ndarray, f) -> np.ndarray:
    """Nearest-code encoding of already-scaled values v = X_j / s (exact fp64)."""
    F = fmt(f)
    v = np.ascontiguousarray(v, dtype=np.float64).ravel()
    out = np.empty(v.shape[0], dtype=np.uint8)
    tab = np.ascontiguousarray(F.mag_table())
    _lib().orc_encode_nearest(v.ctypes.data, v.shape[0], tab.ctypes.data, F.n_mag,
                              F.sign_bit, out.ctypes.data)
    return out


def encode_scalar(v: float, f) -> int:
    """Pure-Python statement of the same rule for single values (test helper)."""
    F = fmt(f)
    from fractions import Fraction
    a = Fraction(abs(v))
    best, bd = None, None
    for c in range(F.n_mag):
        q = F.mag_value(c)
        if math.isnan(q):
            continue
        d = abs(a - Fraction(q))                      # exact rational distance
        if best is None or d < bd or (d == bd and c % 2 == 0 and best % 2 == 1):
            best, bd = c, d
    if math.copysign(1.0, v) < 0:
        best |= 1 << F.sign_bit
    return best


def decode(codes: np.ndarray, f) -> np.ndarray:
    F = fmt(f)
    tab = F.code_table()
    return tab[np.asarray(codes, dtype=np.int64)]


def quantize_blocks(x: np.ndarray, f, rule: int = RULE_OCP):
    """x: [..., nblk*32] fp64 values.  Returns (codes uint8 same shape, scale
    bytes uint8 [..., nblk])."""
    x = np.asarray(x, dtype=np.float64)
    shp = x.shape
    if shp[-1] % BLOCK:
        raise ValueError("last dim must be a multiple of 32")
    blocks = x.reshape(shp[:-1] + (shp[-1] // BLOCK, BLOCK))
    e = block_exponent(blocks, f, rule)
    v = np.ldexp(blocks, -e[..., None].astype(np.int64))   # exact power-of-two scaling
    codes = encode(v, f).reshape(shp)
    return codes, (e + 127).astype(np.uint8)


def dequantize_blocks(codes: np.ndarray, sbytes: np.ndarray, f) -> np.ndarray:
    codes = np.asarray(codes)
    shp = codes.shape
    vals = decode(codes, f).reshape(shp[:-1] + (shp[-1] // BLOCK, BLOCK))
    e = sbytes.astype(np.int64) - 127
    return np.ldexp(vals, e[..., None]).reshape(shp)


# ----------------------------------------------------------------------------- §3.2

def seg_bounds(n):
    n4, n6, n8 = (int(v) for v in n)
    return [(0, n4), (n4, n4 + n6), (n4 + n6, n4 + n6 + n8)]


def seg_formats(fmt6=E3M2, fmt8=E4M3):
    return (E2M1, fmt6, fmt8)


def reorder(x_bits: np.ndarray, perm: np.ndarray) -> np.ndarray:
    """x_r[m, j] = X[m, perm[j]] (BF16 bits, a pure gather)."""
    return np.asarray(x_bits)[:, np.asarray(perm, dtype=np.int64)]


def reorder_quantize(x_bits: np.ndarray, perm, n, fmt6=E3M2, fmt8=E4M3,
                     rule: int = RULE_OCP):
    """Fused reorder-and-quantize semantics (Fig. 6).

    x_bits: uint16 [rows, K] BF16; perm: int [K]; n = (n4, n6, n8).
    Returns (codes[3], scales[3], xr_bits) in canonical form."""
    x_bits = np.asarray(x_bits, dtype=np.uint16)
    if x_bits.ndim != 2 or x_bits.shape[1] != len(perm) or sum(n) != len(perm):
        raise ValueError("shape mismatch")
    xr = reorder(x_bits, perm)
    xv = bf16_to_f64(xr)
    if not np.all(np.isfinite(xv)):
        raise ValueError("non-finite input (outside the contract, DESIGN.md R8)")
    codes, scales = [], []
    for (lo, hi), f in zip(seg_bounds(n), seg_formats(fmt6, fmt8)):
        c, s = quantize_blocks(xv[:, lo:hi], f, rule)
        codes.append(c)
        scales.append(s)
    return codes, scales, xr


def dequantize_segments(codes, scales, fmt6=E3M2, fmt8=E4M3):
    """Concatenated dequantized reordered operand [rows, K] (fp64, exact)."""
    parts = [dequantize_blocks(c, s, f) for c, s, f in zip(codes, scales, seg_formats(fmt6, fmt8))]
    return np.concatenate(parts, axis=1)
