for d in 0 16 20; do for n in 2240,1184,672 0,0,4096 4096,0,0; do MM_GEMM_DEBUG=$d timeout 120 python tools/gemm_timing.py 2048 4096 $n; done; done
