mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -3
for M in 1 8 16 32 33 64 128; do timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672; done
for M in 1 16 32; do MM_GEMM_SPLITS=2 timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672 | sed "s/^/sp2 /"; done
for M in 16 128; do timeout 120 python tools/gemm_timing.py $M 14336 2240,1184,672; done
for M in 16; do timeout 120 python tools/gemm_timing.py $M 28672 2240,1184,672; MM_GEMM_SMALLM=0 timeout 120 python tools/gemm_timing.py $M 28672 2240,1184,672 | sed "s/^/old /"; done
} > gpurun_out/exp18.log 2>&1
cat gpurun_out/exp18.log
