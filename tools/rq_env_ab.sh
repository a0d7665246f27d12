# RQ env A/B (GPU box): ENVS="A=1 B=2" pairs separated by ';'  e.g. ENVS="MM_RQ_BLOCKED=0;MM_RQ_BLOCKED=1"
IFS=';' read -ra VARIANTS <<< "${ENVS}"
for V in "${VARIANTS[@]}"; do
  echo "== $V"; env $V MM_LIB_PATH=$PWD/paper_2508_02343_b200/${LIBNAME:-libmicromix_b200.so} GWS=0 timeout 300 python tools/rq_sweep.py ${SHAPES:-2048:4096 16384:4096 16384:14336 8192:28672} 2>&1 | grep "^M="
done
