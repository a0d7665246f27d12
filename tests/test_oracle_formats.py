"""Oracle pins: element formats and the element encoder (not gpu).

Pins used:
  * Table 6 values printed in the paper (tests/golden/table6.txt)
  * OCP MX constants, cross-checked with CUDA's cuda_fp*.hpp constants (golden/ocp_values.txt)
  * CUDA 12.9's own host conversion routines on every BF16 input (library routine)
  * torch's float8 conversions on the in-range values (library routine)
  * exhaustive enumeration: every finite code decodes and re-encodes to itself
"""
import math
import os
import shutil
import subprocess
import tempfile

import numpy as np
import pytest
import torch

from conftest import ROOT, golden
from oracle import formats, mx
from oracle.formats import E2M1, E2M3, E3M2, E4M3, E5M2, FORMATS


def test_table6_bias_and_qmax():
    rows = golden("table6.txt")
    assert len(rows) == 5
    for line in rows:
        name, bits, bias, qmax = line.split()
        F = formats.fmt(name)
        assert F.bits == int(bits)
        assert F.bias == int(bias)
        assert F.qmax == float(qmax)


def test_ocp_constants():
    const_rows = [l.split() for l in golden("ocp_values.txt")[:5]]
    for name, emax, min_sub, min_norm, max_code in const_rows:
        F = formats.fmt(name)
        tab = F.mag_table()
        fin = tab[~np.isnan(tab)]
        pos = np.sort(fin[fin > 0])
        assert F.emax == int(emax)
        assert pos[0] == float(min_sub)
        # min normal = value of code with exponent field 1, mantissa 0
        assert F.mag_value(1 << F.mbits) == float(min_norm)
        assert F.qmax_code == int(max_code, 16)


def test_e2m1_values_and_e3m2_top_binade():
    F = FORMATS[E2M1]
    assert list(F.mag_table()) == [0, 0.5, 1, 1.5, 2, 3, 4, 6]
    G = FORMATS[E3M2]
    assert list(G.mag_table()[-4:]) == [16, 20, 24, 28]


def test_every_finite_code_roundtrips():
    """Exhaustive enumeration of every FP4/FP6/FP8 code (incl. -0)."""
    for F in FORMATS.values():
        vals = F.code_table()
        codes = np.arange(1 << F.bits)
        fin = ~np.isnan(vals)
        # signed zero must keep its sign: use copysign-aware values
        v = vals[fin].copy()
        neg = codes[fin] >= (1 << F.sign_bit)
        v[neg & (v == 0)] = -0.0
        enc = mx.encode(v, F.fid)
        assert np.array_equal(enc, codes[fin].astype(np.uint8)), F.name
        # non-finite codes are exactly the OCP ones
        nonfin = codes[~fin]
        if F.name == "E4M3":
            assert set(nonfin) == {0x7F, 0xFF}
        elif F.name == "E5M2":
            assert set(nonfin) == set(range(0x7C, 0x80)) | set(range(0xFC, 0x100))
        else:
            assert len(nonfin) == 0


def _cuda_table():
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available for the host-emulation pin")
    d = tempfile.mkdtemp()
    exe = os.path.join(d, "cvt")
    src = os.path.join(ROOT, "tests", "pins", "cuda_cvt_table.cu")
    subprocess.check_call([nvcc, "-Wno-deprecated-gpu-targets", "-o", exe, src],
                          stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    out = os.path.join(d, "t.bin")
    subprocess.check_call([exe, out])
    return np.fromfile(out, dtype=np.uint8).reshape(5, 65536)


def test_encoder_matches_cuda_host_conversion_all_bf16():
    """Every finite BF16 value as the scaled input: oracle == CUDA's RNE+satfinite."""
    t = _cuda_table()
    v = mx.bf16_to_f64(np.arange(65536, dtype=np.uint16))
    fin = np.isfinite(v)
    order = [E2M1, E3M2, E2M3, E4M3, E5M2]
    for row, f in enumerate(order):
        c = mx.encode(v[fin], f)
        assert np.array_equal(c, t[row][fin]), FORMATS[f].name


def test_encoder_matches_torch_float8_in_range():
    v = mx.bf16_to_f64(np.arange(65536, dtype=np.uint16))
    fin = np.isfinite(v)
    for f, dt in ((E4M3, torch.float8_e4m3fn), (E5M2, torch.float8_e5m2)):
        q = FORMATS[f].qmax
        sel = fin & (np.abs(v) <= q)
        ref = torch.from_numpy(v[sel]).to(dt).view(torch.uint8).numpy()
        got = mx.encode(v[sel], f)
        assert np.array_equal(got, ref)


def test_encode_scalar_matches_vector_random():
    rng = np.random.default_rng(5)
    for f in FORMATS:
        q = FORMATS[f].qmax
        v = rng.uniform(-1.3 * q, 1.3 * q, size=300)
        v[:10] = 0.0
        v[10:20] = -0.0
        got = mx.encode(v, f)
        ref = [mx.encode_scalar(float(x), f) for x in v]
        assert list(got) == ref


def test_symmetry_and_monotonicity():
    v = mx.bf16_to_f64(np.arange(0, 0x7F80, dtype=np.uint16))  # all finite non-negative
    for f, F in FORMATS.items():
        pos = mx.encode(v, f)
        neg = mx.encode(-v, f)
        assert np.array_equal(neg, pos | (1 << F.sign_bit))
        dq = mx.decode(pos, f)
        assert np.all(np.diff(dq) >= 0)


def test_spec_encode_examples():
    # x/s with s = 2^1
    assert mx.decode(mx.encode(np.array([6.0 / 2]), E2M1), E2M1)[0] == 3.0
    assert mx.decode(mx.encode(np.array([2.5 / 2]), E2M1), E2M1)[0] == 1.0
    assert mx.encode(np.array([0.0]), E2M1)[0] == 0                  # SPEC.md:71 (+0 for +0.0)


def test_bf16_rne_pins():
    # SPEC.md:353-355 and torch's float32->bfloat16 (RNE) on random fp32 values
    assert mx.bf16_rne(1.0) == 1.0
    assert mx.bf16_rne(3.1415927) == 3.140625
    mid = 1.0 + 2.0 ** -8            # exact midpoint between 1 and 1+2^-7 -> even (1.0)
    assert mx.bf16_rne(mid) == 1.0
    mid2 = 1.0 + 3 * 2.0 ** -8       # midpoint between 1+2^-7 and 1+2^-6 -> even (1+2^-6)
    assert mx.bf16_rne(mid2) == 1.0 + 2.0 ** -6
    rng = np.random.default_rng(1)
    x = (rng.standard_normal(100000) * np.exp(rng.uniform(-40, 40, 100000))).astype(np.float32)
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(mx.bf16_rne(x.astype(np.float64)), ref)
