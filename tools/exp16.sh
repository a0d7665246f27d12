mkdir -p gpurun_out
{
for SP in 1 2 4 6; do for M in 1 128; do MM_GEMM_SPLITS=$SP timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672 | sed "s/^/sp=$SP /"; done; done
} > gpurun_out/exp16.log 2>&1
cat gpurun_out/exp16.log
