mkdir -p gpurun_out
{
for D in 0 2 8 16 64; do
 echo "== dbg $D"; MM_GEMM_DEBUG=$D python tools/gemm_timing.py 16384 4096 2240,1184,672 0,0,4096 4096,0,0
done
} > gpurun_out/exp2.log 2>&1
cat gpurun_out/exp2.log
