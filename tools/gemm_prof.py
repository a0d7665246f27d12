"""Standalone mixed-GEMM launches for ncu: python tools/gemm_prof.py M N K [reps]
(calibrated Llama-3.1-8B-like plan at K, as tools/sweep_configs.py; rotating A inputs)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
import sweep_configs as sc  # noqa: E402
from synth import gen_act, gen_weight  # noqa: E402

M, N, K = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 6
plan = sc.calibrated_plan(K, layer=2)
wq = mm.mm_quantize_weight_offline(gen_weight(N, K, 3000, device="cuda"), plan)
acts = [mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2001 + 100 * i, device="cuda"), plan) for i in range(3)]
y = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
for i in range(reps):
    mm.mm_mixed_gemm_bf16(acts[i % 3], wq, plan, out=y)
torch.cuda.synchronize()
print("ok", M, N, K)
