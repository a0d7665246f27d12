mkdir -p gpurun_out
{
for r in 1 2; do
for V in old new gs1 sc; do
 L=""; [ $V != new ] && L=paper_2508_02343_b200/variants/$V.so
 MM_LIB_PATH=$L timeout 300 python bench.py --no-cpu-baseline --steps 100 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.readline()); b=d['breakdown']; print('$V', round(d['ms_per_step']*1e3,2), round(b['rq_us'],2), round(b['gemm_us'],2), round(b['gemm_frac_mix_peak'],3), d['clocks'])"
done; done
} > gpurun_out/exp28.log 2>&1
cat gpurun_out/exp28.log
