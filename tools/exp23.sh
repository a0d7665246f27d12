mkdir -p gpurun_out
{
for PF in 0 1; do for M in 1 32 128; do MM_GEMM_PREFETCH=$PF timeout 120 python tools/gemm_timing.py $M 4096 8512,3840,1984 | sed "s/^/pf=$PF /"; done; done
for PF in 0 1; do MM_GEMM_PREFETCH=$PF timeout 120 python tools/gemm_timing.py 16 4096 2240,1184,672 | sed "s/^/pf=$PF /"; done
for PF in 0 1; do MM_GEMM_PREFETCH=$PF MM_GEMM_SPLITS=1 timeout 120 python tools/gemm_timing.py 16 4096 2240,1184,672 | sed "s/^/pf=$PF sp1 /"; done
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider -k small 2>&1 | tail -2
} > gpurun_out/exp23.log 2>&1
cat gpurun_out/exp23.log
