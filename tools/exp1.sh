mkdir -p gpurun_out
{
echo "== DP trace"; python tools/gemm_trace.py
echo "== SK trace"; MM_GEMM_STREAMK=1 python tools/gemm_trace.py
echo "== timing DP"; python tools/gemm_timing.py 2048 4096 2240,1184,672
echo "== timing SK"; MM_GEMM_STREAMK=1 python tools/gemm_timing.py 2048 4096 2240,1184,672
echo "== timing DP 6144"; python tools/gemm_timing.py 2048 6144 2240,1184,672
echo "== cublas"; timeout 600 python tools/cublas_mx_baseline.py
} > gpurun_out/exp1.log 2>&1
tail -60 gpurun_out/exp1.log
