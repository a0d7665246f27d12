mkdir -p gpurun_out
{
for SP in 0 1 2 4; do for M in 1 16 64 128; do MM_GEMM_SPLITS=$SP timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672 | sed "s/^/sp=$SP /"; done; done
for M in 1 16 64 128; do MM_GEMM_SMALLM=0 timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672 | sed "s/^/old /"; done
for M in 16 128; do timeout 120 python tools/gemm_timing.py $M 14336 2240,1184,672; MM_GEMM_SMALLM=0 timeout 120 python tools/gemm_timing.py $M 14336 2240,1184,672 | sed "s/^/old /"; done
timeout 120 python tools/gemm_timing.py 2048 4096 2240,1184,672
} > gpurun_out/exp17.log 2>&1
cat gpurun_out/exp17.log
