timeout 300 python -m pytest tests/test_gpu_gemm.py -q -p no:cacheprovider -o timeout=120 2>&1 | tail -2
timeout 900 python -c "
import sys; sys.argv=['x','r01b','c2,c3']
sys.path.insert(0,'tools')
import sweep_configs as s
s.main()
" 2>&1 | grep "^|"
