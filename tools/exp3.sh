mkdir -p gpurun_out
{
echo "== tests CP=2 forced"; MM_GEMM_CP=2 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_nshard.py -q -x -p no:cacheprovider 2>&1 | tail -15
echo "== tests default"; timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -5
for CP in 1 2; do
 echo "== CP=$CP"
 MM_GEMM_CP=$CP timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672
 MM_GEMM_CP=$CP timeout 300 python tools/gemm_timing.py 16384 4096 2240,1184,672 0,0,4096 4096,0,0
 MM_GEMM_CP=$CP MM_GEMM_DEBUG=2 timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096
done
} > gpurun_out/exp3.log 2>&1
cat gpurun_out/exp3.log
