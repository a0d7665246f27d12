mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for M in 16 32 64; do timeout 120 python tools/gemm_timing.py $M 4096 2240,1184,672; done
timeout 120 python tools/gemm_timing.py 16 28672 2240,1184,672
} > gpurun_out/exp19.log 2>&1
cat gpurun_out/exp19.log
