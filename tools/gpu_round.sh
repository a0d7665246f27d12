#!/bin/bash
# GPU box: full GPU test suite, smoke, one bench line.  Logs -> gpurun_out/.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -o timeout=300 > gpurun_out/gpu_tests.log 2>&1
echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 400 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
tail -30 gpurun_out/gpu_tests.log; tail -5 gpurun_out/smoke.log; tail -5 gpurun_out/bench.log
