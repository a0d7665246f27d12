# one full ncu capture of the RQ kernel at M K (source page + raw) -> gpurun_out/rqfull_<tag>_*
M=$1; K=$2; TAG=$3
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:rq_kernel -s 4 -c 1 \
  -o gpurun_out/rqfull_$TAG python tools/rq_prof.py $M $K > gpurun_out/rqfull_$TAG.log 2>&1
ncu -i gpurun_out/rqfull_$TAG.ncu-rep --page raw --csv > gpurun_out/rqfull_${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/rqfull_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/rqfull_${TAG}_src.csv 2>/dev/null
tail -3 gpurun_out/rqfull_$TAG.log
