"""Run traced reorder-quantize launches (MM_RQ_DEBUG |= 32) on a q_proj activation and
print the per-CTA timeline (us from the earliest CTA start)."""
import ctypes
import os
import sys

os.environ["MM_RQ_DEBUG"] = str(int(os.environ.get("MM_RQ_DEBUG", "0")) | 32)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from synth import gen_act  # noqa: E402

plan = mm.mm_calibrate_thresholds(gen_act(4096, 4096, 1000, 2000, device="cuda"))
xs = [gen_act(2048, 4096, 1000, 2001 + i, device="cuda") for i in range(8)]
a = mm.MXTensor(plan, 2048)
for i in range(8):
    mm.mm_reorder_quantize_act(xs[i], plan, out=a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
mm.mm_reorder_quantize_act(xs[3], plan, out=a)
e1.record()
torch.cuda.synchronize()
print(f"event time {e0.elapsed_time(e1) * 1e3:.2f} us")
buf = (ctypes.c_ulonglong * 2560)()
mm.lib().mm_debug_rq_trace(buf, 2560)
t = np.array(buf, dtype=np.float64).reshape(160, 16)[:148]
t0 = t[:, 0][t[:, 0] > 0].min()
rel = np.where(t > 0, (t - t0) / 1e3, np.nan)
names = ["start", "table", "t0 ready", "t0 done", "t1 ready", "t1 done", "t2 ready", "t2 done", "t3 ready",
         "t3 done", "t4 ready", "t4 done", "t5 ready", "t5 done", "last tma"]
for i, nm in enumerate(names):
    col = rel[:, i]
    col = col[~np.isnan(col)]
    if len(col):
        print(f"{nm:9s} n={len(col):3d} {col.min():7.2f} {np.median(col):7.2f} {col.max():7.2f}")
