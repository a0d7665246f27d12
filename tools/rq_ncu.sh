ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"rq_kernel" -s 14 -c 1 --csv python bench.py --no-cpu-baseline --steps 3 2>/dev/null | grep -E "rq_kernel" | python -c "
import sys,csv
for r in csv.reader(sys.stdin):
    print('rq', r[4][:24], r[7], r[-3], r[-1])
"
timeout 200 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown']; print('step_us', round(d['ms_per_step']*1e3,1), 'gemm_us', round(b['gemm_us'],1), 'rq_us', round(b['rq_us'],2))"
timeout 300 python -m pytest tests/test_gpu_rq.py -q -p no:cacheprovider -o timeout=120 2>&1 | tail -2
timeout 200 python tools/norm_timing.py 2048 4096
