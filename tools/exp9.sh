mkdir -p gpurun_out/exp9
MET=gpu__time_duration.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,launch__shared_mem_per_block_dynamic,lts__t_bytes.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,smsp__cycles_active.avg
timeout 600 ncu --metrics $MET --clock-control none --csv python tools/cublas_one.py 16384 4096 4096 fp8 > gpurun_out/exp9/cublas_fp8.csv 2>&1
timeout 600 ncu --metrics $MET --clock-control none --csv -k regex:mixgemm python tools/gemm_timing.py 16384 4096 0,0,4096 > gpurun_out/exp9/ours_fp8.csv 2>&1
timeout 600 ncu --metrics $MET --clock-control none --csv python tools/cublas_one.py 2048 4096 4096 fp8 > gpurun_out/exp9/cublas_fp8_q.csv 2>&1
ls -la gpurun_out/exp9
