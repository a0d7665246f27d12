mkdir -p gpurun_out/rqb8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rq_kernel -s 5 -c 1 -o gpurun_out/rqb8/rq python tools/rq_time.py 16384:4096 > gpurun_out/rqb8/log 2>&1
ncu -i gpurun_out/rqb8/rq.ncu-rep --page raw --csv > gpurun_out/rqb8/raw.csv 2>/dev/null
ncu -i gpurun_out/rqb8/rq.ncu-rep --page source --csv --print-source sass > gpurun_out/rqb8/src.csv 2>/dev/null
ls -la gpurun_out/rqb8
