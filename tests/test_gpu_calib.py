"""GPU parity: mm_calibrate_thresholds vs the oracle (§3.1, Eq. 5-7, 17):
channel max/mean, max|X|, T(4), T(6), counts and the permutation must all be
identical (the means are correctly rounded on both sides)."""
import numpy as np
import pytest
import torch

from oracle import calib as ocal
from oracle.formats import E2M3, E3M2
import paper_2508_02343_b200 as mm
from synth import bf16_bits, gen_act

pytestmark = pytest.mark.gpu


def _check(x, fmt6=mm.MM_E3M2):
    plan, chmax, chmean = mm.mm_calibrate_thresholds(x.cuda(), fmt6=fmt6, return_stats=True)
    ref = ocal.calibrate(bf16_bits(x), E3M2 if fmt6 == mm.MM_E3M2 else E2M3)
    assert np.array_equal(chmax.numpy(), ref["chmax"])
    assert np.array_equal(chmean.numpy(), ref["chmean"]), np.argwhere(chmean.numpy() != ref["chmean"])[:5]
    assert plan.c.tensor_max == ref["tmax"]
    assert plan.c.t4 == ref["t4"] and plan.c.t6 == ref["t6"]
    assert tuple(plan.c.c) == ref["c"]
    assert plan.n == ref["n"]
    assert np.array_equal(plan.perm_host().numpy(), ref["perm"])
    return plan


def test_cfg1_calibration_gives_fixed_split():
    plan = _check(gen_act(2048, 256, 1000, 2000))
    assert plan.n == (128, 64, 64)


@pytest.mark.parametrize("L,K", [(1, 64), (37, 96), (2048, 4096), (16384, 4096)])
def test_calibration_shapes(L, K):
    _check(gen_act(L, K, 1001, 2001))


def test_calibration_e2m3_and_wide():
    _check(gen_act(512, 14336, 1002, 2002), fmt6=mm.MM_E2M3)


def test_degenerate_raises():
    with pytest.raises(mm.MMError) as e:
        mm.mm_calibrate_thresholds(torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda"))
    assert e.value.status == 5


def test_streaming_calibration_equals_one_shot():
    """mm_calib_accumulate over three batches + mm_calib_finalize == the oracle's
    calibration of the concatenated rows (pooled statistics, R15)."""
    K = 1024
    xs = [gen_act(L, K, 1000, 2000 + i) for i, L in enumerate((700, 1500, 33))]
    st = mm.CalibState(K)
    for x in xs:
        st.accumulate(x.cuda())
    plan, chmax, chmean, rows = st.finalize(return_stats=True)
    assert rows == sum(x.shape[0] for x in xs)
    ref = ocal.calibrate(np.concatenate([bf16_bits(x) for x in xs]))
    assert plan.n == ref["n"]
    assert np.array_equal(plan.perm_host().numpy(), ref["perm"])
    assert np.array_equal(chmax.numpy(), ref["chmax"])
    assert plan.c.t4 == ref["t4"] and plan.c.t6 == ref["t6"]
    d = mm.mm_plan_diagnostics(plan, chmax)
    assert abs(d["avg_bits"] - ocal.avg_bits(plan.n)) < 1e-12
    v4, v6 = ocal.eq6_violations(ref["perm"], ref["n"], ref["chmax"], ref["t4"], ref["t6"])
    assert d["eq6_violations"] == (v4, v6)
