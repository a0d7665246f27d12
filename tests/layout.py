"""Test-harness decoders of the library's packed layouts (include/mm.h) into the
oracle's canonical form.  Written from the header text, independent of both the
CUDA sources and the oracle.
"""
import numpy as np


def padded(n):
    return (n + 127) // 128 * 128


def unpack_codes(buf: np.ndarray, rows: int, n: int, seg: int) -> np.ndarray:
    """buf: uint8 [rows, pitch] -> canonical uint8 codes [rows, n], plus the
    padding codes [rows, Kp - n] for the must-be-zero check."""
    kp = padded(n)
    buf = np.asarray(buf, dtype=np.uint8).reshape(rows, -1)
    if seg == 0:                        # element 2i in the low nibble of byte i
        lo = buf & 0x0F
        hi = buf >> 4
        full = np.empty((rows, 2 * buf.shape[1]), dtype=np.uint8)
        full[:, 0::2] = lo
        full[:, 1::2] = hi
    elif seg == 1:                      # LSB-first 6-bit stream
        b = buf.astype(np.uint32).reshape(rows, -1, 3)
        word = b[:, :, 0] | (b[:, :, 1] << 8) | (b[:, :, 2] << 16)
        full = np.empty((rows, word.shape[1] * 4), dtype=np.uint8)
        for i in range(4):
            full[:, i::4] = (word >> (6 * i)) & 0x3F
    else:
        full = buf.copy()
    assert full.shape[1] == kp
    return full[:, :n], full[:, n:kp]


def sf_index(r: np.ndarray, kb: np.ndarray, kp: int) -> np.ndarray:
    """Byte offset of scale (r, kb) in the 128x4-atom layout (include/mm.h)."""
    return ((r // 128) * (kp // 128) + kb // 4) * 512 + (r % 32) * 16 + ((r // 32) % 4) * 4 + kb % 4


def unpack_sf(buf: np.ndarray, rows: int, n: int):
    """-> (canonical scales [rows, n/32], padding-column bytes, padding-row bytes)."""
    kp = padded(n)
    buf = np.asarray(buf, dtype=np.uint8).ravel()
    rows_pad = (rows + 127) // 128 * 128
    r = np.arange(rows_pad)[:, None]
    kb = np.arange(kp // 32)[None, :]
    full = buf[sf_index(r, kb, kp)]
    return full[:rows, : n // 32], full[:rows, n // 32:], full[rows:, :]


def decode_operand(mx, plan_n):
    """MXTensor (torch, on GPU) -> (codes[3], scales[3]) canonical + padding arrays."""
    codes, scales, pads = [], [], []
    for g in range(3):
        n = plan_n[g]
        if n == 0:
            codes.append(np.zeros((mx.rows, 0), np.uint8))
            scales.append(np.zeros((mx.rows, 0), np.uint8))
            pads.append((np.zeros(0), np.zeros(0), np.zeros(0)))
            continue
        pitch = padded(n) * (4, 6, 8)[g] // 8
        cb = mx.codes[g][: mx.rows * pitch].cpu().numpy().reshape(mx.rows, pitch)
        c, cpad = unpack_codes(cb, mx.rows, n, g)
        s, spad_c, spad_r = unpack_sf(mx.sf[g].cpu().numpy(), mx.rows, n)
        codes.append(c)
        scales.append(s)
        pads.append((cpad, spad_c, spad_r))
    return codes, scales, pads
