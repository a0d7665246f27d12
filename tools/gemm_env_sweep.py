"""GEMM tuning sweep (GPU box): time mm_mixed_gemm_bf16 over rotating operand sets (> L2)
for each env setting in ENVS ("A=1 B=2;A=3"), same process (the variables must be read
per launch by the library).  python tools/gemm_env_sweep.py M:N:K ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
import sweep_configs as sc  # noqa: E402
from bench import mix_peak_tflops, peaks  # noqa: E402
from synth import gen_act, gen_weight  # noqa: E402

L2 = torch.cuda.get_device_properties(0).L2_cache_size
pk = peaks()
variants = [v.strip() for v in os.environ.get("ENVS", "").split(";")] or [""]
for arg in sys.argv[1:]:
    M, N, K = map(int, arg.split(":"))
    plan = sc.calibrated_plan(K, layer=0)
    per = M * K + N * K + 2 * M * N
    n = max(2, min(8, -(-3 * L2 // per)))
    aa = [mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2001 + i, device="cuda"), plan) for i in range(n)]
    ws = [mm.mm_quantize_weight_offline(gen_weight(N, K, 3000 + i, device="cuda"), plan) for i in range(n)]
    ys = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    pmix = mix_peak_tflops(plan.n, pk)
    res = []
    for v in variants:
        saved = {}
        for kv in v.split():
            k, val = kv.split("=")
            saved[k] = os.environ.get(k)
            os.environ[k] = val
        us = sc.time_loop(lambda i: mm.mm_mixed_gemm_bf16(aa[i], ws[i], plan, out=ys[i]), n, int(os.environ.get("REPS", "40")))
        if os.environ.get("PAUSE"): torch.cuda.synchronize(); import time as _t; _t.sleep(float(os.environ["PAUSE"]))
        tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
        res.append(f"[{v or 'default'}] {us:.2f}us {tf / pmix:.3f}")
        for k, old in saved.items():
            if old is None:
                os.environ.pop(k)
            else:
                os.environ[k] = old
    print(f"M={M} N={N} K={K} n={plan.n} " + " | ".join(res), flush=True)
    del aa, ws, ys
    torch.cuda.empty_cache()
