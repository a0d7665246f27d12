"""Standalone RQ launches for ncu: python tools/rq_prof.py M K [reps]
(calibrated Llama-3.1-8B-like plan; 3 rotating inputs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
import sweep_configs as sc  # noqa: E402
from synth import gen_act  # noqa: E402

M, K = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 6
plan = sc.calibrated_plan(K, layer=2)
xs = [gen_act(M, K, 1000, 2001 + 100 * i, device="cuda") for i in range(3)]
outs = [mm.mm_reorder_quantize_act(x, plan) for x in xs]
for i in range(reps):
    mm.mm_reorder_quantize_act(xs[i % 3], plan, out=outs[i % 3])
torch.cuda.synchronize()
print("ok", M, K)
