mkdir -p gpurun_out
{
MM_NVCC_FLAGS=-DMM_RQ_EXPERIMENTS=1 python -m paper_2508_02343_b200.build --force > /dev/null 2>&1
timeout 300 python tools/rq_trace.py
MM_NO_PDL=1 timeout 300 python tools/rq_trace.py
python -m paper_2508_02343_b200.build --force > /dev/null 2>&1
} > gpurun_out/exp11.log 2>&1
cat gpurun_out/exp11.log
