# shared-memory wavefronts / conflicts / duration of the RQ at one shape for each row count (GPU box)
M=l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
for R in ${ROWS:-2 4}; do
  echo "== rows $R"
  MM_RQ_ROWS=$R timeout 300 ncu --metrics $M --clock-control none -k regex:rq_kernel -s 10 -c 1 --csv python tools/rq_time.py ${SHAPE:-16384:4096} 2>/dev/null | grep -E "rq_kernel" | awk -F'","' '{print $(NF-2), $(NF)}'
done
