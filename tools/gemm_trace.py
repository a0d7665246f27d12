"""Run one traced GEMM (MM_GEMM_DEBUG=32) and print the per-CTA timeline (us from the
earliest CTA start)."""
import ctypes
import os
import sys

os.environ["MM_GEMM_DEBUG"] = str(int(os.environ.get("MM_GEMM_DEBUG", "0")) | 32)
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_02343_b200 as mm  # noqa: E402
from gemm_timing import time_gemm  # noqa: E402

n = tuple(int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2240,1184,672").split(","))
time_gemm(2048, 4096, n, reps=3)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 2560)()
mm.lib().mm_debug_gemm_trace(buf, 2560)
a = np.array(buf, dtype=np.float64).reshape(160, 16)[:148]
t0 = a[:, 0][a[:, 0] > 0].min()
names = ["start", "setup", "first_ready", "t0_start", "t0_issued", "t1_start", "t1_issued", "t2_start", "t2_issued",
         "epi0", "epi1", "epi2", "epi_done"]
rel = np.where(a > 0, (a - t0) / 1e3, np.nan)
ok = (a[:, 13] > 0) & (a[:, 14] > a[:, 13])
if ok.any():
    f = (a[ok, 14] - a[ok, 13]) / (a[ok, 4] - a[ok, 3])
    print(f"SM clock during tile-0 mainloop: median {np.median(f):.3f} GHz (min {f.min():.3f}, max {f.max():.3f})")
rel[:, 13:] = np.nan
print("column: min / median / max over CTAs (us)")
for i, nm in enumerate(names):
    col = rel[:, i]
    col = col[~np.isnan(col)]
    if len(col):
        print(f"{nm:12s} n={len(col):3d} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}")
