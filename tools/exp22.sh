mkdir -p gpurun_out
{
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout 900 python tools/sweep_configs.py r01e c6 2>&1 | grep "^| C6"
for M in 64 128; do MM_GEMM_SMALLM=0 timeout 120 python tools/gemm_timing.py $M 4096 8512,3840,1984 | sed "s/^/old /"; timeout 120 python tools/gemm_timing.py $M 4096 8512,3840,1984; done
} > gpurun_out/exp22.log 2>&1
bash tools/exp21.sh > /dev/null 2>&1
cat gpurun_out/exp22.log
