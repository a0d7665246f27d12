#!/bin/bash
# GPU box: ncu --set full of the GEMM and the RQ at large shapes (b8 down / b8 o GEMM, b8 / C2 RQ).
set -u
OUT=gpurun_out/prof_large; mkdir -p $OUT
python tools/gemm_prof.py 16384 4096 14336 2 > $OUT/sanity.log 2>&1 || exit 1
python tools/rq_prof.py 16384 4096 2 >> $OUT/sanity.log 2>&1 || exit 1
for spec in "gemm_b8down:tools/gemm_prof.py 16384 4096 14336:mixgemm" "gemm_b8o:tools/gemm_prof.py 16384 4096 4096:mixgemm" \
            "rq_b8:tools/rq_prof.py 16384 4096:rq_kernel" "rq_c2:tools/rq_prof.py 2048 4096:rq_kernel"; do
  TAG=${spec%%:*}; rest=${spec#*:}; CMD=${rest%%:*}; K=${rest##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $OUT/$TAG python $CMD 6 > $OUT/$TAG.log 2>&1
  ncu -i $OUT/$TAG.ncu-rep --page raw --csv > $OUT/${TAG}_raw.csv 2>/dev/null
done
ls -la $OUT
