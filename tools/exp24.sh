mkdir -p gpurun_out
{
timeout 400 python bench.py
timeout 200 python bench.py --config cfg1 --steps 20 --no-cpu-baseline
timeout 300 python bench.py --config llama70b_down --comm peer --steps 10 --warmup 3 --no-cpu-baseline
timeout 300 python bench.py --impl reference --steps 2 --warmup 1
} > gpurun_out/exp24.log 2>&1
bash tools/profile.sh r01e > gpurun_out/prof_e.log 2>&1
MET=gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_requests_srcunit_tex.sum,dram__bytes_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum
timeout 600 ncu --metrics $MET --clock-control none --csv -k regex:cutlass -c 2 python tools/cublas_one.py 16384 4096 4096 fp8 > gpurun_out/cublas_lts.csv 2>&1
cut -c1-400 gpurun_out/exp24.log
