mkdir -p gpurun_out
{
echo "== tests st6"; MM_GEMM_STAGES=6 timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -3
for ST in 5 6; do
echo "== stages $ST"
MM_GEMM_STAGES=$ST timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672
MM_GEMM_STAGES=$ST timeout 300 python tools/gemm_timing.py 16384 4096 2240,1184,672 0,0,4096 4096,0,0
MM_GEMM_STAGES=$ST MM_GEMM_DEBUG=8 timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096
done
} > gpurun_out/exp6.log 2>&1
cat gpurun_out/exp6.log
