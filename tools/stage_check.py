import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2508_02343_b200 as mm
from synth import gen_act, gen_weight, gen_perm
K, n = 4096, (2240, 1184, 672)
plan = mm.mm_plan_init(K, n, gen_perm(K, 5))
a = mm.mm_reorder_quantize_act(gen_act(2048 + 77, K, 1000, 2001).cuda(), plan)
w = mm.mm_quantize_weight_offline(gen_weight(4096 + 256, K, 3000).cuda(), plan)
ys = {}
for st in (5, 6):
    mm.mm_set_gemm_config(512, st, 0)
    ys[st] = mm.mm_mixed_gemm_bf16(a, w, plan)
torch.cuda.synchronize()
print("6 vs 5 stages bit-identical:", torch.equal(ys[5].view(torch.int16), ys[6].view(torch.int16)))
