# RQ ring-lookahead / table-mode grid (GPU box): MM_RQ_LOOKAHEAD x MM_RQ_TABMODE over the
# main shapes, one process per setting (both knobs are read once per process).
for tm in 1 2; do for la in 1 2 3; do
  echo -n "tab=$tm look=$la: "; MM_RQ_LOOKAHEAD=$la MM_RQ_TABMODE=$tm GWS=0 python tools/rq_sweep.py ${SHAPES:-2048:4096 16384:4096 65536:4096 16384:14336 8192:28672} | tr '\n' ' ' | sed 's/rows=auto //g; s/gw=auto://g'; echo
done; done
