"""Oracle pins: Eq. 1 block quantization and the reorder-and-quantize semantics (not gpu).

Pins: OCP worked values (golden/ocp_values.txt), SPEC.md worked examples under
the paper-literal rule (golden/spec_examples.txt), quantize->dequantize
idempotence (OCP rule), the power-of-two scale law, sign symmetry, the
reorder special cases (identity permutation == plain MX quantization,
dequantize + inverse scatter == per-group fake quantization, empty segments),
brute force over every BF16 value x every reachable scale.
"""
import numpy as np
import pytest

from conftest import golden
from oracle import formats, mx
from oracle.formats import E2M1, E2M3, E3M2, E4M3, E5M2, FORMATS
from oracle.mx import RULE_OCP, RULE_PAPER


def _block(first, fill=0.0):
    b = np.full(32, fill, dtype=np.float64)
    b[0] = first
    return b


def test_ocp_worked_values():
    rows = [l.split() for l in golden("ocp_values.txt")[5:]]
    assert len(rows) == 13
    for name, amax, x, sbyte, code in rows:
        f = formats.fmt(name).fid
        blk = _block(float(amax))
        blk[1] = float(x)
        c, s = mx.quantize_blocks(blk[None, :], f, RULE_OCP)
        assert s[0, 0] == int(sbyte, 16), (name, amax)
        assert c[0, 1] == int(code, 16), (name, amax, x)


def test_spec_examples_paper_rule():
    # SPEC.md:61-63 (Eq. 1 literally, b = Table-6 bias)
    assert mx.block_exponent(_block(448.0)[None], E4M3, RULE_PAPER)[0] == 1
    assert mx.block_exponent(_block(6.0)[None], E2M1, RULE_PAPER)[0] == 1
    assert mx.block_exponent(np.zeros((1, 32)), E4M3, RULE_PAPER)[0] == -127
    assert mx.block_exponent(np.zeros((1, 32)), E4M3, RULE_OCP)[0] == -127
    # 32 copies of 448 -> scale 2^1, all decode to 448
    c, s = mx.quantize_blocks(np.full((1, 32), 448.0), E4M3, RULE_PAPER)
    assert s[0, 0] == 128 and np.all(mx.dequantize_blocks(c, s, E4M3) == 448.0)
    # {6, 1, 0, ...} E2M1 -> scale 2^1; 6 and 1 exact
    b = np.zeros((1, 32)); b[0, 0] = 6.0; b[0, 1] = 1.0
    c, s = mx.quantize_blocks(b, E2M1, RULE_PAPER)
    assert s[0, 0] == 128
    dq = mx.dequantize_blocks(c, s, E2M1)
    assert dq[0, 0] == 6.0 and dq[0, 1] == 1.0 and np.all(dq[0, 2:] == 0)
    # 2.5 with scale 2 -> 2.0 (tie to even), error 0.5
    b = np.zeros((1, 32)); b[0, 0] = 6.0; b[0, 1] = 2.5
    c, s = mx.quantize_blocks(b, E2M1, RULE_PAPER)
    assert mx.dequantize_blocks(c, s, E2M1)[0, 1] == 2.0


def test_subnormal_block_and_clamp():
    # BF16-subnormal block: amax 2^-130 -> e = -127 (byte 0), x*2^127 = 2^-3 in E4M3 -> code 0x20
    b = _block(2.0 ** -130)
    c, s = mx.quantize_blocks(b[None], E4M3, RULE_OCP)
    assert s[0, 0] == 0 and c[0, 0] == 0x20
    # largest BF16 -> e = 127 - emax, never 0xFF
    big = float(np.float32(3.3895313892515355e38))
    for f in FORMATS:
        e = mx.block_exponent(_block(big)[None], f, RULE_OCP)[0]
        assert e == 127 - FORMATS[f].emax
        assert e + 127 < 255


def _random_blocks(rng, n, spread=20):
    mant = rng.standard_normal((n, 32))
    scale = np.exp2(rng.integers(-spread, spread, size=(n, 1)))
    x = (mant * scale).astype(np.float32)
    # make them BF16 values
    bits = (x.view(np.uint32) + 0x7FFF + ((x.view(np.uint32) >> 16) & 1)) >> 16
    return mx.bf16_to_f64(bits.astype(np.uint16))


def test_idempotence_ocp_rule():
    """Q(DQ(Q(t))) == Q(t) blockwise (holds under the OCP offset)."""
    rng = np.random.default_rng(7)
    for f in FORMATS:
        x = _random_blocks(rng, 3000)
        c, s = mx.quantize_blocks(x, f, RULE_OCP)
        dq = mx.dequantize_blocks(c, s, f)
        c2, s2 = mx.quantize_blocks(dq, f, RULE_OCP)
        assert np.array_equal(c, c2) and np.array_equal(s, s2), FORMATS[f].name


def test_paper_rule_breaks_idempotence_as_documented():
    """DESIGN.md R1: under the literal Eq. 1 offset, RNE can round the block max
    into the next binade, e.g. E2M1 {3.9, 0.5} -> {4.0, 0.5} -> {4.0, 0.0}."""
    b = np.zeros((1, 32)); b[0, 0] = 3.9; b[0, 1] = 0.5
    b = mx.bf16_rne(b)
    c, s = mx.quantize_blocks(b, E2M1, RULE_PAPER)
    dq = mx.dequantize_blocks(c, s, E2M1)
    c2, s2 = mx.quantize_blocks(dq, E2M1, RULE_PAPER)
    assert not np.array_equal(c, c2)


def test_paper_rule_never_saturates_except_e5m2():
    """with s = 2^(floor(log2 amax) - b), max|x|/s < 2^(b+1) <= q_max."""
    rng = np.random.default_rng(9)
    for f in (E2M1, E3M2, E2M3, E4M3):
        x = _random_blocks(rng, 2000)
        e = mx.block_exponent(x.reshape(-1, 32), f, RULE_PAPER)
        v = np.ldexp(x, -e[:, None].astype(np.int64))
        assert np.max(np.abs(v)) < FORMATS[f].qmax or np.max(np.abs(v)) < 2.0 ** (FORMATS[f].bias + 1)
        assert np.max(np.abs(v)) < 2.0 ** (FORMATS[f].bias + 1) <= FORMATS[f].qmax


def test_scale_law():
    """Q(2^j t) has exponent e + j and identical codes."""
    rng = np.random.default_rng(11)
    for f in FORMATS:
        x = _random_blocks(rng, 500, spread=5)
        c, s = mx.quantize_blocks(x, f, RULE_OCP)
        for j in (-7, 3, 19):
            c2, s2 = mx.quantize_blocks(np.ldexp(x, j), f, RULE_OCP)
            assert np.array_equal(c, c2)
            assert np.array_equal(s2.astype(int), s.astype(int) + j)


def test_exhaustive_bf16_times_scales_matches_definition():
    """Brute force: every finite BF16 value x, in a block whose amax sets e, for
    several reachable e: the code equals the nearest-code rule applied to the
    exact rational x / 2^e (encode_scalar uses Fractions)."""
    vals = mx.bf16_to_f64(np.arange(0, 0x7F80, dtype=np.uint16))
    rng = np.random.default_rng(3)
    pick = rng.choice(len(vals), 400, replace=False)
    for f in FORMATS:
        F = FORMATS[f]
        for amax in (2.0 ** -130, 1.0, 3.0e5):
            sel = vals[vals <= amax]
            sub = sel[pick % len(sel)]
            blocks = np.zeros((len(sub), 32)); blocks[:, 0] = amax; blocks[:, 1] = sub
            blocks[1::2, 1] *= -1
            c, s = mx.quantize_blocks(blocks, f, RULE_OCP)
            e = int(s[0, 0]) - 127
            for i in range(len(sub)):
                x = blocks[i, 1]
                assert c[i, 1] == mx.encode_scalar(float(np.ldexp(x, -e)), f)


def test_reorder_identity_equals_plain_quantize():
    """identity permutation, single group == quantize_tensor."""
    rng = np.random.default_rng(2)
    x = mx.bf16_rne(rng.standard_normal((8, 64)) * 3)
    bits = mx.bf16_rne_bits(x)
    for g, n in enumerate([(64, 0, 0), (0, 64, 0), (0, 0, 64)]):
        codes, scales, xr = mx.reorder_quantize(bits, np.arange(64), n)
        f = (E2M1, E3M2, E4M3)[g]
        c, s = mx.quantize_blocks(x, f)
        assert np.array_equal(codes[g], c) and np.array_equal(scales[g], s)
        for h in range(3):
            if h != g:
                assert codes[h].shape == (8, 0) and scales[h].shape == (8, 0)


def test_reorder_dequant_scatter_equals_groupwise_fake_quant():
    """dequantize + inverse scatter == per-group quantize-dequantize
    of the same columns."""
    rng = np.random.default_rng(4)
    K = 256
    x = mx.bf16_rne(rng.standard_normal((6, K)) * np.exp(rng.standard_normal(K)))
    bits = mx.bf16_rne_bits(x)
    perm = rng.permutation(K)
    n = (128, 64, 64)
    codes, scales, xr = mx.reorder_quantize(bits, perm, n)
    assert np.array_equal(xr, bits[:, perm])
    dq = mx.dequantize_segments(codes, scales)
    back = np.empty_like(dq)
    back[:, perm] = dq
    for (lo, hi), f in zip(mx.seg_bounds(n), (E2M1, E3M2, E4M3)):
        cols = perm[lo:hi]
        c, s = mx.quantize_blocks(x[:, cols], f)
        assert np.array_equal(back[:, cols], mx.dequantize_blocks(c, s, f))


def test_reorder_rejects_bad_shapes():
    bits = np.zeros((2, 64), dtype=np.uint16)
    with pytest.raises(ValueError):
        mx.reorder_quantize(bits, np.arange(64), (32, 0, 0))
    with pytest.raises(ValueError):
        mx.reorder_quantize(bits, np.arange(32), (32, 0, 0))


def test_quant_error_within_half_gap():
    """|t - dq(q(t))| <= half the decoded-code gap at that magnitude
    for unsaturated elements (gap oracle from the enumerated code points)."""
    rng = np.random.default_rng(12)
    for f in FORMATS:
        F = FORMATS[f]
        x = _random_blocks(rng, 400, spread=4)
        c, s = mx.quantize_blocks(x, f)
        dq = mx.dequantize_blocks(c, s, f)
        e = (s.astype(np.int64) - 127).repeat(32, axis=1)
        v = np.abs(np.ldexp(x, -e))
        tab = np.sort(F.mag_table()[~np.isnan(F.mag_table())])
        hi = np.searchsorted(tab, v)
        ok = v <= F.qmax
        gap = np.where(hi < len(tab), tab[np.minimum(hi, len(tab) - 1)] - tab[np.maximum(hi - 1, 0)], 0)
        err = np.abs(np.ldexp(x - dq, -e))
        assert np.all(err[ok] <= gap[ok] / 2 + 0.0)
