mkdir -p gpurun_out
{
MM_GEMM_STREAMK=1 timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672
MM_GEMM_STREAMK=1 MM_GEMM_DEBUG=4 timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672
MM_GEMM_STREAMK=1 timeout 300 python tools/gemm_trace.py
} > gpurun_out/exp8.log 2>&1
cat gpurun_out/exp8.log
