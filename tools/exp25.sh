mkdir -p gpurun_out
{
for r in 1 2 3; do
for V in old new; do
 L=""; [ $V = old ] && L=paper_2508_02343_b200/variants/old.so
 MM_LIB_PATH=$L timeout 120 python tools/gemm_timing.py 2048 4096 2240,1184,672 | sed "s/^/$V /"
 MM_LIB_PATH=$L timeout 120 python tools/gemm_timing.py 16384 4096 2240,1184,672 0,0,4096 | sed "s/^/$V /"
done; done
} > gpurun_out/exp25.log 2>&1
cat gpurun_out/exp25.log
