# RQ cost breakdown (GPU box, experiments build lib_exp.so): full / no stores (16) /
# no gather+quantize (1) / no transpose either (2) / no loads (4)
for D in ${DBGS:-0 16 1 2 4}; do
  echo "== MM_RQ_DEBUG=$D"
  MM_RQ_DEBUG=$D MM_LIB_PATH=$PWD/paper_2508_02343_b200/lib_exp.so GWS=0 timeout 300 python tools/rq_sweep.py ${SHAPES:-2048:4096 16384:4096 16384:14336} 2>&1 | grep "^M="
done
