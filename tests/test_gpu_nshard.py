"""GPU test of the N-sharded GEMM + NCCL all-gather entry point
(mm_mixed_gemm_bf16_nshard_allgather) on the one GPU a test box has:
a world-size-1 communicator exercises the library's NCCL binding, the staging
layout and the [G][M][N/G] -> [M][N] permute; the result must equal the unsharded
mm_mixed_gemm_bf16 output bit for bit (same tiles, same K order).  The world-size-2
host logic is covered on CPU by tests/test_dist_gloo.py."""
import numpy as np
import pytest
import torch

import paper_2508_02343_b200 as mm
from oracle import gemm as ogemm
from synth import bf16_bits, gen_act, gen_perm, gen_weight

from accuracy import ref_and_abs, report

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,n", [(256, 512, (256, 128, 128)), (200, 1024, (2240, 1184, 672))])
def test_nshard_world1_equals_plain(M, N, n):
    K = sum(n)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 21))
    x, wb = gen_act(M, K, 1000, 2001), gen_weight(N, K, 3000)
    a = mm.mm_reorder_quantize_act(x.cuda(), plan)
    w = mm.mm_quantize_weight_offline(wb.cuda(), plan)
    y_plain = mm.mm_mixed_gemm_bf16(a, w, plan)
    comm = mm.mm_comm_init(0, 1, mm.nccl_unique_id())
    try:
        y_shard = mm.mm_mixed_gemm_bf16_nshard_allgather(a, w, plan, N, comm)
        torch.cuda.synchronize()
    finally:
        mm.mm_comm_destroy(comm)
    assert torch.equal(y_plain.view(torch.int16), y_shard.view(torch.int16))
    # and against the oracle (sampled rows x all columns, every element inside the
    # worst-case FP32 bound of tests/accuracy.py, relative Frobenius <= 2e-3)
    rows = np.arange(0, M, 3)
    yref, S = ref_and_abs(bf16_bits(x)[rows], bf16_bits(wb), plan.perm_host().numpy(), plan.n,
                          *_fmts(plan))
    r = report(bf16_bits(y_shard.cpu())[rows], yref, S, K)
    assert r["bound_violations"] == 0 and r["rel_fro"] <= 2e-3, r


def _fmts(plan):
    from oracle.formats import E2M3, E3M2, E4M3, E5M2
    return ({mm.MM_E3M2: E3M2, mm.MM_E2M3: E2M3}[plan.fmt6], {mm.MM_E4M3: E4M3, mm.MM_E5M2: E5M2}[plan.fmt8],
            plan.rule)


def test_nshard_rejects_bad_shapes():
    K, n = 256, (128, 64, 64)
    plan = mm.mm_plan_init(K, n, gen_perm(K, 22))
    a = mm.mm_reorder_quantize_act(gen_act(32, K, 1000, 2001).cuda(), plan)
    w = mm.mm_quantize_weight_offline(gen_weight(64, K, 3000).cuda(), plan)
    comm = mm.mm_comm_init(0, 1, mm.nccl_unique_id())
    try:
        with pytest.raises(mm.MMError):
            mm.mm_mixed_gemm_bf16_nshard_allgather(a, w, plan, 128, comm)   # 64 rows x 1 rank != 128
    finally:
        mm.mm_comm_destroy(comm)
