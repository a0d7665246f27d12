"""Timeline of one RQ + GEMM step at the bench config (q_proj 2048 x 4096 x 4096): RQ CTA
start / table ready / first tile / end (needs a build with
MM_NVCC_FLAGS=-DMM_RQ_EXPERIMENTS=1 and MM_RQ_DEBUG=32) and GEMM CTA start / setup /
first stage / tile starts / epilogue end (MM_GEMM_DEBUG=32), in us from the earliest RQ
CTA start.  Usage on the GPU box:
  MM_NVCC_FLAGS=-DMM_RQ_EXPERIMENTS=1 python -c 'from paper_2508_02343_b200.build import build; build(force=True)'
  MM_RQ_DEBUG=32 MM_GEMM_DEBUG=32 python tools/step_trace.py
(MM_NO_PDL=1 shows the step without programmatic dependent launch.)"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from synth import gen_act, gen_weight  # noqa: E402

M, K, N = 2048, 4096, 4096
dev = torch.device("cuda", 0)
if os.environ.get("STAGES"):   # GEMM ring depth (4 / 5 / 6)
    mm.mm_set_gemm_config(0, int(os.environ["STAGES"]), 0)
plan = mm.mm_calibrate_thresholds(gen_act(16384, K, 1000, 2000).to(dev))
x = gen_act(M, K, 1000, 2001, device=dev)
wq = mm.mm_quantize_weight_offline(gen_weight(N, K, 3000, device=dev), plan)
a = mm.MXTensor(plan, M, dev)
y = torch.empty(M, N, dtype=torch.bfloat16, device=dev)


def step():
    mm.mm_reorder_quantize_act(x, plan, out=a)
    mm.mm_mixed_gemm_bf16(a, wq, plan, out=y)


for _ in range(20):
    step()
torch.cuda.synchronize()
torch.cuda._sleep(int(2e-3 * 1.9e9))
step()
torch.cuda.synchronize()
rq = (ctypes.c_ulonglong * 2560)()
mm.lib().mm_debug_rq_trace(rq, 2560)
rq = np.array(rq, dtype=np.float64).reshape(160, 16)[:148]
gt = (ctypes.c_ulonglong * 3840)()
mm.lib().mm_debug_gemm_trace(gt, 3840)
gt = np.array(gt, dtype=np.float64).reshape(160, 24)[:148]
t0 = rq[:, 0][rq[:, 0] > 0].min() if (rq[:, 0] > 0).any() else gt[:, 0][gt[:, 0] > 0].min()


def us(v):
    return np.where(v > 0, (v - t0) / 1e3, np.nan)


def row(name, v):
    v = v[~np.isnan(v)]
    v = v[v > -1.0]   # slots of CTAs without that event in this launch hold older values
    if len(v):
        print(f"{name:20s} n={len(v):3d} min {v.min():7.2f} p10 {np.percentile(v, 10):7.2f} "
              f"med {np.median(v):7.2f} p90 {np.percentile(v, 90):7.2f} max {v.max():7.2f}")


print("RQ + GEMM step; times in us from the first RQ CTA start")
row("rq start", us(rq[:, 0]))
row("rq table ready", us(rq[:, 1]))
row("rq tile0 ready", us(rq[:, 2]))
row("rq last tile done", us(rq[:, 15]))
row("gemm cta start", us(gt[:, 0]))
row("gemm after dep wait", us(gt[:, 1]))
row("gemm first stage", us(gt[:, 2]))
row("gemm tile0 start", us(gt[:, 3]))
row("gemm tile0 issued", us(gt[:, 4]))
row("gemm tile1 start", us(gt[:, 5]))
row("gemm tile1 issued", us(gt[:, 6]))
row("gemm epi done", us(gt[:, 12]))
