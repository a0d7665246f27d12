# DRAM / L2 traffic of the RQ at one shape under debug switches (GPU box)
M=${M:-dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,lts__t_requests_op_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write_lookup_miss.sum,lts__average_t_sector_hit_rate_realtime.pct}
for D in ${DBGS:-0 64 128}; do
  echo "== MM_RQ_DEBUG=$D"
  MM_RQ_DEBUG=$D MM_LIB_PATH=$PWD/paper_2508_02343_b200/lib_exp.so timeout 300 ncu --metrics $M --clock-control none -k regex:rq_kernel -s 10 -c 1 --csv python tools/rq_time.py ${SHAPE:-16384:4096} 2>/dev/null | grep -E "rq_kernel" | awk -F'","' '{print $(NF-2), $(NF)}'
done
