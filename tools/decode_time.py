"""Decode-shape timing (small-M kernel): q_proj / down at M = 1..128, rotating weights
> L2, CUDA events: the GEMM alone back to back, and the step (RQ of the activation +
GEMM) back to back.  python tools/decode_time.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
import sweep_configs as sc  # noqa: E402
from synth import gen_act, gen_weight  # noqa: E402

L2 = torch.cuda.get_device_properties(0).L2_cache_size
for K, N in ((4096, 4096), (14336, 4096)):
    plan = sc.calibrated_plan(K, layer=0)
    nset = max(2, min(16, -(-3 * L2 // (N * K))))
    ws = [mm.mm_quantize_weight_offline(gen_weight(N, K, 3000 + i, device="cuda"), plan) for i in range(nset)]
    res, res_step = [], []
    for M in (1, 16, 32, 64, 128):
        x = gen_act(M, K, 1000, 2001, device="cuda")
        a = mm.mm_reorder_quantize_act(x, plan)
        y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        us = sc.time_loop(lambda i: mm.mm_mixed_gemm_bf16(a, ws[i], plan, out=y), nset, 40)
        res.append(f"M={M}:{us:.2f}us")

        def step(i):
            mm.mm_reorder_quantize_act(x, plan, out=a)
            mm.mm_mixed_gemm_bf16(a, ws[i], plan, out=y)
        res_step.append(f"M={M}:{sc.time_loop(step, nset, 40):.2f}us")
    print(f"K={K} N={N} gemm " + " ".join(res), flush=True)
    print(f"K={K} N={N} step " + " ".join(res_step), flush=True)
