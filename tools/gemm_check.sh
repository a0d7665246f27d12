timeout 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider -o timeout=120 -x 2>&1 | tail -15
timeout 120 python tools/gemm_timing.py 2048 4096
timeout 200 python bench.py --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); b=d['breakdown']; print('step_us', round(d['ms_per_step']*1e3,1), 'gemm_us', round(b['gemm_us'],1), 'TF', round(b['gemm_tflops']), 'frac', round(b['gemm_frac_mix_peak'],3), 'rq_us', round(b['rq_us'],2), 'e2e', round(d['e2e']['value']))"
