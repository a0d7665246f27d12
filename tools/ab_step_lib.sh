#!/bin/bash
# Step-time A/B of library builds at the bench config, interleaved (GPU box):
#   bash tools/ab_step_lib.sh lib_base.so lib_new.so   (files in paper_2508_02343_b200/)
B="python bench.py --steps 300 --warmup 10 --large 0 --no-cpu-baseline"
for r in 1 2 3; do for L in "$@"; do echo -n "[$r] $L "; MM_LIB_PATH=$PWD/paper_2508_02343_b200/$L $B 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("step_us %.2f rq %.2f gemm %.2f" % (d["ms_per_step"]*1e3, d["breakdown"]["rq_us"], d["breakdown"]["gemm_us"]))'; done; done
