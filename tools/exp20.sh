mkdir -p gpurun_out
timeout 1500 python tools/sweep_configs.py r01d > gpurun_out/sweep_r01d.log 2>&1
tail -50 gpurun_out/sweep_r01d.log
