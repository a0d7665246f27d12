#!/bin/bash
# Run on the GPU box (via gpurun): launch list of one short bench run, then one
# `ncu --set full` capture of each hot kernel.  Outputs land in gpurun_out/; the
# summaries worth keeping are copied into profiles/ by tools/ncu_summary.py.
set -u
TAG=${1:-r01}
OUT=gpurun_out/prof_${TAG}
mkdir -p $OUT
NCU=${NCU:-ncu}
# 1) launch list (cold-cache, serialised; compare shares, not absolutes)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python bench.py --steps 4 --warmup 3 --no-cpu-baseline --large 0 \
  > $OUT/launches_bench.log 2>&1
# 2) full captures of the two hot kernels (one launch each after warm-up)
for KS in mixgemm:4 rq_kernel:10; do
  K=${KS%%:*}; SK=${KS##*:}
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:$K -s $SK -c 1 \
    -o $OUT/full_$K python bench.py --steps 2 --warmup 3 --no-cpu-baseline --large 0 \
    > $OUT/full_${K}.log 2>&1
  $NCU -i $OUT/full_$K.ncu-rep --page raw --csv > $OUT/full_${K}_raw.csv 2>/dev/null
  $NCU -i $OUT/full_$K.ncu-rep --page details --csv > $OUT/full_${K}_details.csv 2>/dev/null
done
ls -la $OUT
