timeout 300 python -m pytest tests/test_gpu_rq.py -q -p no:cacheprovider -o timeout=120 2>&1 | tail -2
timeout 900 python -c "
import sys; sys.argv=['x','r01c','c4']
sys.path.insert(0,'tools')
import sweep_configs as s
s.main()
" 2>&1 | grep "^| C"
timeout 900 python -c "
import sys
sys.path.insert(0,'tools')
import sweep_configs as s, torch
s.L2 = torch.cuda.get_device_properties(0).L2_cache_size
p = s.calibrated_plan(14336, layer=2)
s.measure_layer('C3 b8 down', 16384, 14336, 4096, p, reps=5, sets=2)
" 2>&1 | grep rq_us | cut -c1-220
