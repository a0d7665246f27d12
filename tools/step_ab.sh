#!/bin/bash
# Step-time A/B at the bench config for env switches, interleaved (ABAB...) on one box,
# e.g. CFGS="MM_GEMM_WPRE=0|MM_GEMM_WPRE=1" (W stages the pair GEMM loads before
# griddepcontrol.wait).  GPU box only.
set -u
cd "$(dirname "$0")/.."
B="python bench.py --steps 300 --warmup 10 --large 0 --no-cpu-baseline"
show() { python -c 'import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print("step_us %.2f med %.2f value %.0f rq %.2f gemm %.2f" % (d["ms_per_step"]*1e3, d["ms_per_step_stats"]["median"]*1e3, d["value"], d["breakdown"]["rq_us"], d["breakdown"]["gemm_us"]))'; }
CFGS=${CFGS:-"X=0"}
for rep in 1 2 3; do
  IFS='|'; for cfg in $CFGS; do unset IFS; echo -n "[$rep] $cfg: "; env $cfg $B 2>/dev/null | show; IFS='|'; done; unset IFS
done
