"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no block scaling, no
element encoding, no thresholds, no GEMM).  It only draws random numbers and
rounds them to the BF16 input dtype, so that both sides of every parity test
consume the very same BF16 bit patterns.

Recipe, shaped like the
LLM activations the paper calibrates on (§3.1 Q2, Fig. 2 / Fig. 4
captions: a log-normal channel body, a "warm" minority of larger channels and a
handful of outlier channels that MicroMix pushes into MXFP8):

  activations  X[L, K]:
    profile (profile_seed):  s_k = exp(N(0, 0.4^2));  30 % of channels x5;
                             n_outlier channels x40
    values  (draw_seed):     X = N(0,1) * s_k, clipped to +-0.9*spike; one random
                             row of every outlier channel set to +spike (=552),
                             which pins max|X| (so T(4), T(6) are deterministic)
  weights      W[N, K] (PyTorch Linear layout):
                             N(0,1)/sqrt(K) * exp(N(0, 0.2^2)) per output row

Everything is produced by torch's counter-based generators seeded explicitly,
either on the CPU (tests) or on a CUDA device (large bench shapes); the BF16
result is the canonical input for both sides.
"""
from __future__ import annotations

import math

import torch

SPIKE = 552.0  # exactly representable in BF16 (550 would round to 552)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def channel_profile(K: int, profile_seed: int, n_outlier: int | None = None,
                    device="cpu"):
    """Per-channel scale s_k and the outlier channel indices (profile only)."""
    if n_outlier is None:
        n_outlier = 4 if K <= 256 else 8
    g = _gen(profile_seed, "cpu")
    s = torch.exp(torch.randn(K, generator=g, dtype=torch.float64) * 0.4)
    warm = torch.randperm(K, generator=g)[: int(round(0.3 * K))]
    s[warm] *= 5.0
    outl = torch.randperm(K, generator=g)[:n_outlier]
    s[outl] *= 40.0
    return s.to(device), outl.to(device)


def gen_act(L: int, K: int, profile_seed: int = 1000, draw_seed: int = 2001,
            n_outlier: int | None = None, spike: float = SPIKE,
            device="cpu") -> torch.Tensor:
    """BF16 activations [L, K] following the recipe above."""
    s, outl = channel_profile(K, profile_seed, n_outlier, device=device)
    g = _gen(draw_seed, device)
    x = torch.randn(L, K, generator=g, device=device, dtype=torch.float32)
    x.mul_(s.to(torch.float32)[None, :])
    x.clamp_(-0.9 * spike, 0.9 * spike)
    if L > 0 and len(outl) > 0:
        rows = torch.randint(0, L, (len(outl),), generator=g, device=device)
        x[rows, outl] = spike
    return x.to(torch.bfloat16)


def gen_weight(N: int, K: int, weight_seed: int = 3000, device="cpu") -> torch.Tensor:
    """BF16 weights [N, K] (PyTorch Linear layout, K contiguous)."""
    g = _gen(weight_seed, device)
    w = torch.randn(N, K, generator=g, device=device, dtype=torch.float32)
    row = torch.exp(torch.randn(N, 1, generator=g, device=device, dtype=torch.float32) * 0.2)
    w.mul_(row / math.sqrt(K))
    return w.to(torch.bfloat16)


def gen_perm(K: int, seed: int) -> torch.Tensor:
    """A seeded random bijection on [0, K) (int32) for fixed-split plans."""
    g = _gen(seed, "cpu")
    return torch.randperm(K, generator=g).to(torch.int32)


def gen_uniform_bf16(shape, lo: float, hi: float, seed: int, device="cpu") -> torch.Tensor:
    g = _gen(seed, device)
    x = torch.rand(*shape, generator=g, device=device, dtype=torch.float32)
    return (lo + (hi - lo) * x).to(torch.bfloat16)


def bf16_bits(t: torch.Tensor):
    """BF16 tensor -> numpy uint16 bit array (host copy)."""
    return t.detach().contiguous().cpu().view(torch.int16).numpy().view("uint16")


def bits_to_bf16(a) -> torch.Tensor:
    import numpy as np
    return torch.from_numpy(np.ascontiguousarray(a).view("int16")).view(torch.bfloat16)


# Shapes of the BASELINE.json configs.
LLAMA8B = dict(hidden=4096, inter=14336, q=4096, kv=1024)
CONFIGS = {
    "cfg1": dict(M=16, K=256, N=256, split=(128, 64, 64)),
    "q_proj": dict(M=2048, K=4096, N=4096),
    "llama70b_down": dict(M=8192, K=28672, N=8192),
}
