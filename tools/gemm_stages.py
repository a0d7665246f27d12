import os, sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tools')
import torch
import paper_2508_02343_b200 as mm
import sweep_configs as sc
from bench import mix_peak_tflops, peaks
from synth import gen_act, gen_weight
pk = peaks()
L2 = torch.cuda.get_device_properties(0).L2_cache_size
for (M, N, K) in [(2048, 4096, 4096), (2048, 6144, 4096), (16384, 4096, 4096)]:
    plan = sc.calibrated_plan(K, layer=0)
    n = max(2, min(8, -(-3 * L2 // (M * K + N * K + 2 * M * N))))
    aa = [mm.mm_reorder_quantize_act(gen_act(M, K, 1000, 2001 + i, device="cuda"), plan) for i in range(n)]
    ws = [mm.mm_quantize_weight_offline(gen_weight(N, K, 3000 + i, device="cuda"), plan) for i in range(n)]
    ys = [torch.empty(M, N, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    res = []
    for st in (6, 5, 4, 6, 5, 4):
        mm.mm_set_gemm_config(512, st, 0)
        us = sc.time_loop(lambda i: mm.mm_mixed_gemm_bf16(aa[i], ws[i], plan, out=ys[i]), n, 40)
        res.append(f"st{st}:{us:.2f}")
    mm.mm_set_gemm_config(0, 0, 0)
    print(M, N, K, " ".join(res), flush=True)
