for d in 0 1 2; do MM_GEMM_DEBUG=$d timeout 120 python tools/gemm_timing.py 2048 4096; done
