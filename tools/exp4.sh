mkdir -p gpurun_out
{
for CP in 1 2; do
 echo "== CP=$CP"
 MM_GEMM_CP=$CP MM_GEMM_DEBUG=128 timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672 2>&1 | sort | uniq -c | head -5
 MM_GEMM_CP=$CP timeout 300 python tools/gemm_trace.py
done
} > gpurun_out/exp4.log 2>&1
cat gpurun_out/exp4.log
