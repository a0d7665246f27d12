"""Seeded shape fuzz of the whole path (RQ + GEMM) against the oracle: K any multiple of
32 (not only of 128 / 256: segment and box tails), segment splits with empty segments,
M from 1 to 300 (small-M cluster kernel, single-CTA and CTA-pair tiles, ragged row
tails), N any multiple of 16, both element-format variants and scale rules.  Codes and
scales bit-exact; GEMM within the per-element worst-case bound and 2e-3 Frobenius."""
import numpy as np
import pytest
import torch

import paper_2508_02343_b200 as mm
from oracle import mx as omx
from oracle.formats import E2M3, E3M2, E4M3, E5M2
from synth import bf16_bits, gen_act, gen_perm, gen_weight

from accuracy import ref_and_abs, report
from layout import decode_operand

pytestmark = pytest.mark.gpu
FMT_O = {mm.MM_E3M2: E3M2, mm.MM_E2M3: E2M3, mm.MM_E4M3: E4M3, mm.MM_E5M2: E5M2}


def _case(i):
    rng = np.random.default_rng(1000 + i)
    K = 32 * int(rng.integers(1, 80))
    b = sorted(rng.integers(0, K // 32 + 1, size=2))
    n = (32 * int(b[0]), 32 * int(b[1] - b[0]), K - 32 * int(b[1]))
    M = int(rng.choice([1, 3, 16, 31, 64, 100, 128, 129, 200, 257, 300]))
    N = 16 * int(rng.integers(1, 40))
    fmt6 = int(rng.choice([mm.MM_E3M2, mm.MM_E2M3]))
    fmt8 = int(rng.choice([mm.MM_E4M3, mm.MM_E5M2]))
    rule = int(rng.integers(0, 2))
    return K, n, M, N, fmt6, fmt8, rule


@pytest.mark.parametrize("i", range(40))
def test_fuzz_path_vs_oracle(i):
    K, n, M, N, fmt6, fmt8, rule = _case(i)
    perm = gen_perm(K, 500 + i)
    plan = mm.mm_plan_init(K, n, perm, fmt6=fmt6, fmt8=fmt8, rule=rule)
    x = gen_act(M, K, 1000 + i, 2500 + i)
    w = gen_weight(N, K, 3500 + i)
    a = mm.mm_reorder_quantize_act(x.cuda(), plan)
    wq = mm.mm_quantize_weight_offline(w.cuda(), plan)
    y = mm.mm_mixed_gemm_bf16(a, wq, plan)
    torch.cuda.synchronize()
    codes, scales, _ = decode_operand(a, plan.n)
    oc, osf, _ = omx.reorder_quantize(bf16_bits(x), perm.numpy(), n, FMT_O[fmt6], FMT_O[fmt8], rule)
    for g in range(3):
        if n[g]:
            assert np.array_equal(codes[g], oc[g]) and np.array_equal(scales[g], osf[g]), (i, g)
    yref, S = ref_and_abs(bf16_bits(x), bf16_bits(w), perm.numpy(), n, FMT_O[fmt6], FMT_O[fmt8], rule)
    r = report(bf16_bits(y.cpu()), yref, S, K)
    assert r["bound_violations"] == 0 and r["rel_fro"] <= 2e-3, (i, K, n, M, N, r)
