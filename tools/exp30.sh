mkdir -p gpurun_out
L=paper_2508_02343_b200/variants/cp.so
{
for n in 0,0,4096 2240,1184,672; do
MM_LIB_PATH=$L MM_GEMM_CP=1 timeout 120 python tools/gemm_timing.py 16384 4096 $n | sed "s/^/cp1 /"
MM_LIB_PATH=$L MM_GEMM_CP=1 MAXCTAS=132 timeout 120 python tools/gemm_timing.py 16384 4096 $n | sed "s/^/cp1-132 /"
MM_LIB_PATH=$L MM_GEMM_CP=2 MAXCTAS=132 timeout 120 python tools/gemm_timing.py 16384 4096 $n | sed "s/^/cp2-132 /"
MM_LIB_PATH=$L MM_GEMM_CP=2 MAXCTAS=132 MM_GEMM_DEBUG=2 timeout 120 python tools/gemm_timing.py 16384 4096 $n | sed "s/^/cp2-132-loadsonly /"
MM_LIB_PATH=$L MM_GEMM_CP=1 MAXCTAS=132 MM_GEMM_DEBUG=2 timeout 120 python tools/gemm_timing.py 16384 4096 $n | sed "s/^/cp1-132-loadsonly /"
done
} > gpurun_out/exp30.log 2>&1
cat gpurun_out/exp30.log
