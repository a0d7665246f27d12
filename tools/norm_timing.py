"""Time the fused RMSNorm + reorder-quantize (F2) against RQ alone and against an
unfused torch RMSNorm followed by the RQ, q_proj activation shape."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from sweep_configs import time_loop  # noqa: E402
from synth import gen_act, gen_uniform_bf16  # noqa: E402

M, K = int(sys.argv[1]) if len(sys.argv) > 1 else 2048, int(sys.argv[2]) if len(sys.argv) > 2 else 4096
plan = mm.mm_calibrate_thresholds(gen_act(8192, K, 1000, 2000, device="cuda"))
ns = 8
xs = [gen_act(M, K, 1000, 2001 + i, device="cuda") for i in range(ns)]
g = gen_uniform_bf16((K,), 0.5, 1.5, 3, device="cuda")
aa = [mm.MXTensor(plan, M) for _ in range(ns)]
ys = [torch.empty_like(x) for x in xs]
rq = time_loop(lambda i: mm.mm_reorder_quantize_act(xs[i], plan, out=aa[i]), ns, 50)
fused = time_loop(lambda i: mm.mm_rmsnorm_reorder_quantize_act(xs[i], g, 1e-5, plan, out=aa[i]), ns, 50)


def unfused(i):
    torch.nn.functional.rms_norm(xs[i], (K,), g, 1e-5, out=ys[i]) if False else ys[i].copy_(
        torch.nn.functional.rms_norm(xs[i], (K,), g, 1e-5))
    mm.mm_reorder_quantize_act(ys[i], plan, out=aa[i])


unf = time_loop(unfused, ns, 50)
print(f"M={M} K={K}: RQ {rq:.2f} us | fused RMSNorm+RQ {fused:.2f} us | torch RMSNorm + RQ {unf:.2f} us")
