# RQ change check: GPU RQ tests + the RQ columns of the config sweep (C2, C3, C4)
timeout 300 python -m pytest tests/test_gpu_rq.py tests/test_gpu_gemm.py -q -p no:cacheprovider -o timeout=120 2>&1 | tail -2
timeout 1200 python tools/sweep_configs.py rqcheck c2,c3,c4 2>&1 | grep "^| C" | cut -d'|' -f2,6,7,8
