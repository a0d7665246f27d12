for m in 16 64 128 256; do timeout 120 python tools/gemm_timing.py $m 4096 2240,1184,672; done
