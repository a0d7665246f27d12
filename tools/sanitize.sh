#!/bin/bash
# GPU box: compute-sanitizer tier T3 over tools/sanitize_cases.py (logs -> gpurun_out/san/).
# The library is rebuilt with a long mbarrier watchdog (kernels run 10-1000x slower
# under the tools).
set -u
mkdir -p gpurun_out/san
MM_NVCC_FLAGS="-DMM_WATCHDOG_NS=900000000000ull" python -c "from paper_2508_02343_b200.build import build; build(force=True)"
for T in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $T --error-exitcode 99 --print-limit 50 \
    python tools/sanitize_cases.py > gpurun_out/san/$T.log 2>&1
  echo "$T rc=$?" >> gpurun_out/san/$T.log
  tail -3 gpurun_out/san/$T.log
done
