mkdir -p gpurun_out/exp21
MET=gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_lookup_hit.sum,lts__t_sectors_srcunit_tex_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_srcnode_gpc.sum,lts__t_sectors.sum,lts__t_requests_srcunit_tex.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex.sum
timeout 600 ncu --metrics $MET --clock-control none --csv -c 3 python tools/cublas_one.py 16384 4096 4096 fp8 > gpurun_out/exp21/cublas.csv 2>&1
timeout 600 ncu --metrics $MET --clock-control none --csv -k regex:mixgemm -c 3 python tools/gemm_timing.py 16384 4096 0,0,4096 > gpurun_out/exp21/ours.csv 2>&1
ls -la gpurun_out/exp21
