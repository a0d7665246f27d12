#!/bin/bash
# Step time vs K, with and without the untimed lead-in after the pre-queue sleep
# (BENCH_LEAD).  GPU box.
for r in 1 2; do
  for lead in 0 64; do
    for a in "--steps 20 --warmup 3" "--steps 50 --warmup 5" "--steps 300 --warmup 10"; do
      echo -n "[$r] lead=$lead $a: "; BENCH_LEAD=$lead python bench.py $a --large 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); s=d["ms_per_step_stats"]; print("step_us %.2f med %.2f p10 %.2f p90 %.2f rq %.2f gemm %.2f host %.1f launches %d mhz %s" % (d["ms_per_step"]*1e3, s["median"]*1e3, s["p10"]*1e3, s["p90"]*1e3, d["breakdown"]["rq_us"], d["breakdown"]["gemm_us"], d["host_enqueue_us_per_step"], d["gpu_launches"], d["clocks"]["sm_mhz"]))'
    done
  done
done
