mkdir -p gpurun_out
{
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 300 python bench.py --config llama70b_down --comm peer --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
timeout 300 python bench.py --config llama70b_down --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -2
} > gpurun_out/exp13.log 2>&1
cat gpurun_out/exp13.log
