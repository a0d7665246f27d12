mkdir -p gpurun_out
{
for M in 16 32 64 128; do timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672; done
for M in 16 64; do BN=128 timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672; done
for M in 16 64 128; do timeout 120 python tools/gemm_timing.py $M 14336 2240,1184,672; done
} > gpurun_out/exp14.log 2>&1
cat gpurun_out/exp14.log
