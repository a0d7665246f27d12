mkdir -p gpurun_out
{
echo "== tests default"; timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_nshard.py -q -x -p no:cacheprovider 2>&1 | tail -5
echo "== tests CP=2"; MM_GEMM_CP=2 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -3
echo "== tests SK"; MM_GEMM_STREAMK=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672
timeout 300 python tools/gemm_timing.py 16384 4096 2240,1184,672 0,0,4096 4096,0,0
MM_GEMM_DEBUG=2 timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096
MM_GEMM_DEBUG=8 timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096
} > gpurun_out/exp5.log 2>&1
cat gpurun_out/exp5.log
