for dbg in 12 28 2 3; do
MM_RQ_DEBUG=$dbg ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:"rq_kernel" -s 14 -c 1 --csv python bench.py --no-cpu-baseline --steps 3 2>/dev/null | grep -E "rq_kernel" | python -c "
import sys,csv
for r in csv.reader(sys.stdin):
    print('rq dbg=$dbg', r[-3], r[-1])
"
done
