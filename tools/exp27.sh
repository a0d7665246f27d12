mkdir -p gpurun_out
{
for r in 1 2; do
for V in old new sc rg8 scgs1; do
 L=""; [ $V != new ] && L=paper_2508_02343_b200/variants/$V.so
 MM_LIB_PATH=$L timeout 120 python tools/gemm_timing.py 2048 4096 2240,1184,672 | sed "s/^/$V /"
 MM_LIB_PATH=$L timeout 120 python tools/gemm_timing.py 16384 4096 2240,1184,672 | sed "s/^/$V /"
done; done
} > gpurun_out/exp27.log 2>&1
cat gpurun_out/exp27.log
