mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -15
for M in 1 16 32 64 128; do timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672; done
for M in 16 128; do timeout 120 python tools/gemm_timing.py $M 14336 2240,1184,672; done
MM_GEMM_SMALLM=0 timeout 120 python tools/gemm_timing.py 16 4096 2240,1184,672
} > gpurun_out/exp15.log 2>&1
cat gpurun_out/exp15.log
