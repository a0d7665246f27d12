"""Time the reorder-quantize alone: python tools/rq_time.py M:K [M:K ...]
(calibrated plan per K, rotating inputs > 3x L2, CUDA events, back-to-back launches).
Env MM_RQ_ROWS / MM_RQ_STAGES pass through to the library (tuning)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
import sweep_configs as sc  # noqa: E402
from bench import rq_bytes  # noqa: E402
from synth import gen_act  # noqa: E402

L2 = torch.cuda.get_device_properties(0).L2_cache_size
hbm = sc.PK["hbm_gbs"]
plans = {}
for arg in sys.argv[1:]:
    M, K = map(int, arg.split(":"))
    if K not in plans:
        plans[K] = sc.calibrated_plan(K, layer=2)
    plan = plans[K]
    n = max(2, min(8, -(-3 * L2 // (2 * M * K))))
    xs = [gen_act(M, K, 1000, 2001 + 100 * i, device="cuda") for i in range(n)]
    outs = [mm.mm_reorder_quantize_act(x, plan) for x in xs]
    us = sc.time_loop(lambda i: mm.mm_reorder_quantize_act(xs[i], plan, out=outs[i]), n, 40)
    b = rq_bytes(M, plan.n)
    print(f"M={M} K={K} rows={os.environ.get('MM_RQ_ROWS', 'auto')} rq_us={us:.2f} GB/s={b / us / 1e3:.0f} "
          f"frac={b / us / 1e3 / hbm:.3f}")
    del xs, outs
