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
buf = (ctypes.c_ulonglong * 3840)()
mm.lib().mm_debug_gemm_trace(buf, 3840)
a = np.array(buf, dtype=np.float64).reshape(160, 24)[:148]
t0 = a[:, 0][a[:, 0] > 0].min()
names = ["start", "setup", "first_ready", "t0_start", "t0_issued", "t1_start", "t1_issued", "t2_start", "t2_issued",
         "epi0", "epi1", "epi2", "epi_done", None, None, None, "t1_tempty_ok", "epi0_ovl_cta0", "epi0_ovl_cta1"]
rel = np.where(a > 0, (a - t0) / 1e3, np.nan)
ok = (a[:, 13] > 0) & (a[:, 14] > a[:, 13])
if ok.any():
    f = (a[ok, 14] - a[ok, 13]) / (a[ok, 4] - a[ok, 3])
    print(f"SM clock during tile-0 mainloop: median {np.median(f):.3f} GHz (min {f.min():.3f}, max {f.max():.3f})")
ok2 = (a[:, 19] > 0) & (a[:, 20] > a[:, 19])
if ok2.any():
    d = a[ok2, 20] - a[ok2, 19]
    d0 = a[ok2, 19] - a[ok2, 21]
    print(f"epilogue tile 0, CTA 0 warp 4: tfull->first ld {np.median(d0):.0f} cyc, two TMEM loads + wait {np.median(d):.0f} cyc (min {d.min():.0f}, max {d.max():.0f})")
ok3 = (a[:, 22] > a[:, 14]) & (a[:, 14] > 0)
if ok3.any():
    g = a[ok3, 22] - a[ok3, 14]
    m = a[ok3, 14] - a[ok3, 13]
    print(f"MMA warp: tile-0 issue {np.median(m):.0f} cyc, last issue of tile 0 -> tile 1 start {np.median(g):.0f} cyc (min {g.min():.0f}, max {g.max():.0f})")
rel[:, 13:16] = np.nan
rel[:, 19:] = np.nan
print("column: min / median / max over CTAs (us)")
for i, nm in enumerate(names):
    if nm is None:
        continue
    col = rel[:, i]
    col = col[~np.isnan(col)]
    if len(col):
        print(f"{nm:12s} n={len(col):3d} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}")
