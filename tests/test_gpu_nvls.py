"""Fused all-gather over NVLS / NVLink SHARP (include/mm.h): the
CTA-pair GEMM's epilogue writes each output element once with multimem.st into a
multicast object spanning every rank's Y, and a multimem.red flag barrier closes the
step.  A test box has one GPU, so the multicast object here has ONE device (the
mechanics -- create, bind, map both views, multimem stores and reductions, epochs --
are exercised; the replication across ranks runs in tests/test_gpu_multidev.py on
multi-GPU boxes).  Results must equal the 1-GPU GEMM bit for bit and the oracle within
the per-element bound."""
import numpy as np
import pytest
import torch

import paper_2508_02343_b200 as mm
from synth import bf16_bits, gen_act, gen_perm, gen_weight

from accuracy import ref_and_abs, report

pytestmark = pytest.mark.gpu


def _skip_unsupported():
    if not mm.mc_supported():
        pytest.skip("device does not support multicast objects")


@pytest.mark.parametrize("M,N,n", [(300, 512, (256, 128, 128)), (2048, 4096, (2240, 1184, 672)),
                                   (130, 272, (0, 256, 0))])
def test_nvls_world1_equals_plain_and_oracle(M, N, n):
    _skip_unsupported()
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 61))
    x, w = gen_act(M, K, 1000, 2061), gen_weight(N, K, 3061)
    a = mm.mm_reorder_quantize_act(x.cuda(), plan)
    wq = mm.mm_quantize_weight_offline(w.cuda(), plan)
    y_ref = mm.mm_mixed_gemm_bf16(a, wq, plan)
    ldy = N + 16                                     # columns past n_total must stay untouched
    win = mm.McWindow.create(M, ldy)
    try:
        win.set_timeout(20.0)
        for _ in range(2):                           # a second step re-uses the flags (next epoch)
            mm.mm_mixed_gemm_bf16_nshard_nvls(a, wq, plan, N, win, barrier=True)
        torch.cuda.synchronize()
        y = win.y().clone()
        assert not win.timed_out()
    finally:
        win.close()
    assert torch.equal(y[:, :N].view(torch.int16), y_ref.view(torch.int16))
    assert not y[:, N:].view(torch.int16).any()
    rows = np.arange(0, M, 9)
    from oracle.formats import E3M2, E4M3
    yref, S = ref_and_abs(bf16_bits(x)[rows], bf16_bits(w), plan.perm_host().numpy(), plan.n, E3M2, E4M3, plan.rule)
    r = report(bf16_bits(y[:, :N].contiguous().cpu())[rows], yref, S, K)
    assert r["bound_violations"] == 0 and r["rel_fro"] <= 2e-3, r


def test_nvls_rejects_bad_arguments():
    _skip_unsupported()
    K, n = 256, (128, 64, 64)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 62))
    a = mm.mm_reorder_quantize_act(gen_act(64, K, 1000, 2062).cuda(), plan)
    wq = mm.mm_quantize_weight_offline(gen_weight(128, K, 3062).cuda(), plan)
    win = mm.McWindow.create(64, 128)
    try:
        n0 = mm.launch_count()
        with pytest.raises(mm.MMError):
            mm.mm_mixed_gemm_bf16_nshard_nvls(a, wq, plan, 256, win)      # shard rows * world != n_total
        a2 = mm.mm_reorder_quantize_act(gen_act(80, K, 1000, 2063).cuda(), plan)
        with pytest.raises(mm.MMError):
            mm.mm_mixed_gemm_bf16_nshard_nvls(a2, wq, plan, 128, win)     # rows != window M
        assert mm.launch_count() == n0
    finally:
        win.close()
