"""Pins of the oracle's RMSNorm (oracle/norm.py, reading R27) against
things other than itself: closed forms, exact special cases, power-of-two
equivariance, and PyTorch's own fp64 RMS computation (a library routine) within
the final BF16 rounding."""
import numpy as np
import torch

from oracle import mx as omx
from oracle import norm as onorm
from synth import bf16_bits, gen_act, gen_uniform_bf16


def _bits(v):
    return omx.bf16_rne_bits(np.asarray(v, dtype=np.float64))


def test_constant_row_gives_gamma_exactly():
    # x = c (any BF16), eps = 0: ss = K c^2, r = 1/|c| exactly for c = 2^k -> y = sign(c) * gamma
    K = 64
    gamma = gen_uniform_bf16((K,), 0.5, 2.0, 3)
    for c in (1.0, -4.0, 0.125, 2.0 ** -60, 2.0 ** 40):
        x = _bits(np.full((1, K), c))
        y = onorm.rmsnorm_bf16_bits(x, bf16_bits(gamma), 0.0)
        want = bf16_bits(gamma) ^ (0x8000 if c < 0 else 0)
        assert np.array_equal(y[0], want), c


def test_power_of_two_equivariance():
    # eps = 0: scaling a row by 2^k leaves y unchanged (r scales by 2^-k exactly)
    x = bf16_bits(gen_act(4, 256, 1000, 2001))
    g = bf16_bits(gen_uniform_bf16((256,), 0.5, 1.5, 4))
    y0 = onorm.rmsnorm_bf16_bits(x, g, 0.0)
    for k in (-20, -3, 5, 30):
        xk = _bits(omx.bf16_to_f64(x) * 2.0 ** k)
        assert np.array_equal(onorm.rmsnorm_bf16_bits(xk, g, 0.0), y0), k


def test_exact_sumsq_small_integers():
    x = _bits(np.array([3.0, -4.0, 12.0, 0.0, 0.5]))
    assert onorm.exact_sumsq(x) == 9 + 16 + 144 + 0.25
    # cancellation-free but wide range: 2^100 and 1 -> correctly rounded fp64 sum
    x = _bits(np.array([2.0 ** 50, 1.0]))
    assert onorm.exact_sumsq(x) == 2.0 ** 100 + 1.0   # == 2^100 in fp64, rounded once


def test_against_torch_fp64_rms():
    x = gen_act(8, 1024, 1001, 2002)
    g = gen_uniform_bf16((1024,), 0.25, 2.0, 5)
    eps = 1e-5
    xt = x.double()
    ref = xt * torch.rsqrt(xt.pow(2).mean(-1, keepdim=True) + eps) * g.double()
    y = omx.bf16_to_f64(onorm.rmsnorm_bf16_bits(bf16_bits(x), bf16_bits(g), eps))
    rel = np.abs(y - ref.numpy()) / np.maximum(np.abs(ref.numpy()), 1e-30)
    assert rel.max() <= 2.0 * 2.0 ** -8 * 1.0001    # two BF16 roundings (t, then gamma * t)
    # and the unrounded oracle agrees with torch to fp64 accuracy
    yf = onorm.rmsnorm_f64(bf16_bits(x), bf16_bits(g), eps)
    assert np.allclose(yf, ref.numpy(), rtol=1e-12, atol=0)


def _hf_llama_rmsnorm(x_bf16, gamma_bf16, r_f32):
    """The literal HF LlamaRMSNorm forward in torch (CPU), with the row scale r
    injected instead of torch.rsqrt(variance + eps) (whose fp32 rounding is not
    what R27 fixes):  hidden = x.to(float32); hidden = hidden * r;
    return weight * hidden.to(bfloat16)."""
    hidden = x_bf16.to(torch.float32)
    hidden = hidden * r_f32[:, None]
    return gamma_bf16 * hidden.to(torch.bfloat16)


def test_rounding_order_matches_literal_hf_expression():
    """Reading R27's order of roundings -- t = bf16(fp32(x * r)) BEFORE the gamma
    multiply, then bf16(gamma * t) -- equals the literal HF expression bit for bit,
    and is distinguishable from the one-rounding alternative bf16(x * r * gamma)."""
    eps = 1e-5
    for K, seed in ((1024, 1), (4096, 2), (320, 3)):
        x = gen_act(16, K, 1000 + seed, 2100 + seed)
        g = gen_uniform_bf16((K,), 0.25, 2.0, 40 + seed)
        xb, gb = bf16_bits(x), bf16_bits(g)
        r = torch.tensor([float(onorm.row_scale_f32(xb[i], K, eps)) for i in range(x.shape[0])],
                         dtype=torch.float32)
        want = bf16_bits(_hf_llama_rmsnorm(x, g, r))
        got = onorm.rmsnorm_bf16_bits(xb, gb, eps)
        assert np.array_equal(got, want), K
        # the single-rounding alternative differs on these inputs (the pin discriminates)
        alt = bf16_bits((x.to(torch.float64) * r.double()[:, None] * g.double()).to(torch.bfloat16))
        assert not np.array_equal(alt, want), K


def test_row_scale_matches_torch_fp64():
    """r = fp32(1/sqrt(ss/K + eps)) against torch's fp64 sum of squares (a library
    reduction; equal after the fp32 rounding except on astronomically rare ties)."""
    for K, seed in ((256, 5), (4096, 6), (14336, 7)):
        x = gen_act(8, K, 1000 + seed, 2200 + seed)
        xd = x.double()
        rt = (1.0 / torch.sqrt(xd.pow(2).sum(-1) / K + 1e-6)).float()
        ro = [onorm.row_scale_f32(bf16_bits(x)[i], K, 1e-6) for i in range(8)]
        assert np.array_equal(np.array(ro, dtype=np.float32), rt.numpy()), K
