"""One cuBLASLt MXFP8 (or MXFP4) GEMM shape, a few launches (for ncu comparison)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from cublas_mx_baseline import run
M, K, N = (int(v) for v in sys.argv[1:4])
fmt = sys.argv[4] if len(sys.argv) > 4 else "fp8"
us, tf = run(fmt, M, K, N, torch.device("cuda:0"), iters=3)
print(f"{fmt} M={M} K={K} N={N}: {us:.1f} us {tf:.0f} TF/s")
