"""MX element formats written out from their bit fields -- TEST INFRASTRUCTURE ONLY.

PAPER.md Appendix A, Table 6 (lines 369-403) fixes, per format, the exponent
bias b and the max normal q_max:

    E5M2  b=15  +-57344      E4M3  b=7  +-448
    E3M2  b=3   +-28         E2M3  b=1  +-7.5
    E2M1  b=1   +-6          (all: block k=32, scale E8M0, 8 scale bits)

(Table 6 prints "8" element bits for MXFP4 -- a garble, E2M1 is 4 bits; DESIGN.md
reading R23.)  The decoded value of a sign-magnitude code with exponent field
Ef and mantissa field m (E exponent bits, M mantissa bits) is the IEEE-style

    (-1)^s * (m / 2^M) * 2^(1-b)          if Ef == 0   (subnormal)
    (-1)^s * (1 + m / 2^M) * 2^(Ef-b)     otherwise

with the OCP MX v1.0 non-finite encodings excluded: E4M3 has NaN at
S.1111.111 and no infinities; E5M2 has Inf/NaN at Ef = 31; the FP6/FP4 formats
have no special values (PAPER.md line 361 defers to the OCP specification).

emax = floor(log2 q_max) is the exponent of the largest normal; it is the offset
of the OCP scale rule (reading R1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

E2M1, E3M2, E2M3, E4M3, E5M2 = 0, 1, 2, 3, 4
NAMES = {E2M1: "E2M1", E3M2: "E3M2", E2M3: "E2M3", E4M3: "E4M3", E5M2: "E5M2"}


@dataclass(frozen=True)
class Fmt:
    fid: int
    name: str
    ebits: int
    mbits: int
    bias: int          # Table 6 "Exponent Bias (b)"

    @property
    def bits(self) -> int:
        return 1 + self.ebits + self.mbits

    @property
    def sign_bit(self) -> int:
        return self.ebits + self.mbits

    @property
    def n_mag(self) -> int:
        return 1 << (self.ebits + self.mbits)

    def is_finite_mag(self, c: int) -> bool:
        ef = c >> self.mbits
        m = c & ((1 << self.mbits) - 1)
        if self.name == "E4M3":
            return not (ef == 15 and m == 7)
        if self.name == "E5M2":
            return ef != 31
        return True

    def mag_value(self, c: int) -> float:
        """Value of magnitude code c (no sign), NaN for non-finite codes."""
        if not self.is_finite_mag(c):
            return math.nan
        ef = c >> self.mbits
        m = c & ((1 << self.mbits) - 1)
        if ef == 0:
            return math.ldexp(m, 1 - self.bias - self.mbits)
        return math.ldexp((1 << self.mbits) + m, ef - self.bias - self.mbits)

    def mag_table(self) -> np.ndarray:
        return np.array([self.mag_value(c) for c in range(self.n_mag)], dtype=np.float64)

    def code_table(self) -> np.ndarray:
        """Value of every code 0 .. 2^bits-1 (sign included), NaN for non-finite."""
        mags = self.mag_table()
        vals = np.concatenate([mags, -mags])
        return vals

    @property
    def qmax(self) -> float:
        t = self.mag_table()
        return float(np.nanmax(t))

    @property
    def qmax_code(self) -> int:
        t = self.mag_table()
        return int(np.nanargmax(t))

    @property
    def emax(self) -> int:
        return math.frexp(self.qmax)[1] - 1


FORMATS = {
    E2M1: Fmt(E2M1, "E2M1", 2, 1, 1),
    E3M2: Fmt(E3M2, "E3M2", 3, 2, 3),
    E2M3: Fmt(E2M3, "E2M3", 2, 3, 1),
    E4M3: Fmt(E4M3, "E4M3", 4, 3, 7),
    E5M2: Fmt(E5M2, "E5M2", 5, 2, 15),
}


def fmt(f) -> Fmt:
    if isinstance(f, Fmt):
        return f
    if isinstance(f, str):
        for v in FORMATS.values():
            if v.name == f.upper():
                return v
        raise KeyError(f)
    return FORMATS[int(f)]
