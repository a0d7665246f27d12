"""Trace one small-M GEMM launch (MM_GEMM_DEBUG=32): per-CTA timeline of the swap-AB
/ split-K kernel (us from the earliest CTA start).  usage: gemm_sm_trace.py M N n4,n6,n8"""
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

M, N = int(sys.argv[1]), int(sys.argv[2])
n = tuple(int(v) for v in sys.argv[3].split(","))
time_gemm(M, N, n, reps=3)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * 10240)()
mm.lib().mm_debug_gemm_sm_trace(buf, 10240)
a = np.array(buf, dtype=np.float64).reshape(1024, 10)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
rel = np.where(a > 0, (a - t0) / 1e3, np.nan)
for i, nm in enumerate(["start", "setup", "first_full", "last_full", "mma_done", "partial_out", "end", "cluster_sync1", "reduced"]):
    col = rel[:, i]
    col = col[~np.isnan(col)]
    if len(col):
        print(f"{nm:12s} n={len(col):4d} {col.min():8.2f} {np.median(col):8.2f} {col.max():8.2f}")
