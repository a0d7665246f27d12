mkdir -p gpurun_out
{
run() { echo "-- $*"; env "$@" timeout 300 python tools/gemm_timing.py 16384 4096 0,0,4096 2240,1184,672; env "$@" timeout 300 python tools/gemm_timing.py 2048 4096 2240,1184,672; }
run X=0
run MM_GEMM_NONPERSIST=1
run MM_GEMM_RASTER_G=1
run MM_GEMM_RASTER_G=2
run MM_GEMM_RASTER_G=4
run MM_GEMM_RASTER_G=16
run MM_GEMM_RASTER_G=64
run MM_GEMM_L2PROMO=0
run MM_GEMM_L2PROMO=2
run MM_GEMM_NONPERSIST=1 MM_GEMM_RASTER_G=1
} > gpurun_out/exp10.log 2>&1
cat gpurun_out/exp10.log
