# A/B of RQ library variants (GPU box): bash tools/ab_rq.sh lib1.so lib2.so ...
for L in "$@"; do
  echo "== $L"; MM_LIB_PATH=$PWD/paper_2508_02343_b200/$L GWS=${GWS:-0} timeout 300 python tools/rq_sweep.py ${SHAPES:-2048:4096 16384:4096 16384:14336 8192:28672} 2>&1 | grep "^M="
done
