mkdir -p gpurun_out
{
echo "== tests"; timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_nshard.py -q -x -p no:cacheprovider 2>&1 | tail -3
MM_GEMM_STREAMK=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672
timeout 300 python tools/gemm_timing.py 16384 4096 2240,1184,672 0,0,4096 4096,0,0
MM_GEMM_DEBUG=16 timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096
MM_GEMM_DEBUG=20 timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096
MM_GEMM_DEBUG=4 timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096
timeout 300 python tools/gemm_trace.py
} > gpurun_out/exp7.log 2>&1
cat gpurun_out/exp7.log
