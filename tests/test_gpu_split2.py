"""GPU parity: the CTA-pair GEMM's balanced schedule (gemm2.cu build_sched).

When the whole 256 x 256 tiles leave a ragged last wave (T = q P + r, 0 < r < P; q_proj:
128 tiles on 74 pairs, qkv at M = 2048: 192), every pair takes q whole tiles and at most
one narrow item of 64 / 128 / 192 columns -- some starting 64 rows into a W scale atom, whose MMAs read SFB
two TMEM words in.  Every output element still sums its K products in the same order,
so the result must equal the whole-tile schedule BIT FOR BIT; it is also checked against
the oracle (Eq. 2) and on the exact-integer case (P-I(i))."""
import numpy as np
import pytest
import torch

from oracle import gemm as ogemm
from oracle import mx as omx
from oracle.formats import E3M2, E4M3
import paper_2508_02343_b200 as mm
from synth import bf16_bits, bits_to_bf16, gen_act, gen_perm, gen_weight

pytestmark = pytest.mark.gpu


def _gemm(x, w, plan, split2, monkeypatch):
    monkeypatch.setenv("MM_GEMM_SPLIT2", "1" if split2 else "0")
    a = mm.mm_reorder_quantize_act(x.cuda(), plan)
    wq = mm.mm_quantize_weight_offline(w.cuda(), plan)
    y = mm.mm_mixed_gemm_bf16(a, wq, plan)
    torch.cuda.synchronize()
    return y


# (M, N): 128 tiles on 74 pairs (192-column items), 80 tiles (64-column items, ragged M),
# 96 tiles (128-column items), ragged M and N with a partial last 64-column unit
@pytest.mark.parametrize("M,N,n", [(2048, 4096, (2272, 1152, 672)), (2500, 2048, (96, 160, 224)),
                                   (2048, 3072, (512, 256, 256)), (1800, 2992, (1024, 0, 512)),
                                   (1280, 4096, (0, 512, 0)),
                                   # q = 2 whole tiles per pair (qkv at M = 2048); q = 12 (gate_up) keeps
                                   # the whole-tile raster (balanced schedule only for q <= 3)
                                   (2048, 6144, (512, 256, 256)), (2048, 28672, (256, 128, 128))])
def test_split2_equals_whole_tiles_and_oracle(M, N, n, monkeypatch):
    K = sum(n)
    x = gen_act(M, K, 1004, 2700 + M)
    w = gen_weight(N, K, 3700 + N)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 15))
    y_s = _gemm(x, w, plan, True, monkeypatch)
    y_t = _gemm(x, w, plan, False, monkeypatch)
    assert torch.equal(y_s.view(torch.int16), y_t.view(torch.int16))
    rows = np.arange(0, M, max(1, M // 97))
    yref, _ = ogemm.mixed_linear_ref(bf16_bits(x), bf16_bits(w), plan.perm_host().numpy(), plan.n, E3M2, E4M3,
                                     plan.rule, rows=rows)
    assert ogemm.rel_fro(y_s[torch.from_numpy(rows).cuda()].double().cpu().numpy(), yref) <= 2e-3


def test_split2_exact_integer_bit_exact(monkeypatch):
    """Integer operands exact in every format (products and sums < 2^24): Y must equal
    bf16(X W^T) bit for bit under the balanced schedule at the q_proj tile count."""
    M, N, n = 2048, 4096, (512, 256, 256)
    rng = np.random.default_rng(7)
    K = sum(n)
    perm = rng.permutation(K)

    def operand(rows):
        v4 = rng.choice([-6, -4, -3, -2, -1, 0, 1, 2, 3, 4, 6], size=(rows, n[0])); v4[:, ::32] = 6
        v6 = rng.choice([-28, -12, -7, -3, 0, 1, 5, 8, 14, 24], size=(rows, n[1])); v6[:, ::32] = 28
        v8 = rng.integers(-15, 16, size=(rows, n[2])); v8[:, ::32] = 256
        r = np.concatenate([v4, v6, v8], axis=1).astype(np.float64)
        out = np.empty_like(r)
        out[:, perm] = r
        return r, out

    xr, xa = operand(M)
    wr, wa = operand(N)
    plan = mm.mm_plan_init(K, n, perm)
    y = _gemm(bits_to_bf16(omx.bf16_rne_bits(xa)), bits_to_bf16(omx.bf16_rne_bits(wa)), plan, True, monkeypatch)
    exact = xr @ wr.T
    assert np.max(np.abs(exact)) < 2 ** 24
    assert np.array_equal(bf16_bits(y.cpu()), omx.bf16_rne_bits(exact))
