# RQ change check: GPU RQ tests + the RQ columns of the config sweep (C2, C3, C4)
timeout 300 python -m pytest tests/test_gpu_rq.py tests/test_gpu_gemm.py -q -p no:cacheprovider -o timeout=120 2>&1 | tail -2
timeout 1200 python tools/sweep_configs.py rqcheck ${1:-c2,c3,c4} 2>&1 | grep "^| C" | cut -d'|' -f2,6,7,8
if [ -n "$2" ]; then echo "MM_RQ_ROWS=$2"; MM_RQ_ROWS=$2 timeout 1200 python tools/sweep_configs.py rqcheck2 ${1:-c2,c3,c4} 2>&1 | grep "^| C" | cut -d'|' -f2,6,7,8; fi
