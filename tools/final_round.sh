mkdir -p gpurun_out
bash tools/profile.sh r01i > gpurun_out/prof_i.log 2>&1
timeout 400 python bench.py > gpurun_out/bench_final2.log 2>&1
timeout 1500 python tools/sweep_configs.py r01i c2,c3,c4,c5 > gpurun_out/sweep_r01i.log 2>&1
tail -1 gpurun_out/bench_final2.log | cut -c1-200
