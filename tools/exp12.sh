mkdir -p gpurun_out
{
timeout 600 python -m pytest tests/test_gpu_peerstore.py -q -x -p no:cacheprovider 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -5
timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672
} > gpurun_out/exp12.log 2>&1
cat gpurun_out/exp12.log
