# RQ config grid at one shape (GPU box): table mode x lookahead x group count, one
# process per setting (the knobs are read once per process).  SHAPE=M:K
S=${SHAPE:-8192:5120}
for tm in ${TMS:-1 2}; do for la in ${LAS:-1 2 3}; do for g in ${GS:-0}; do
  if [ "$g" = 0 ]; then unset MM_RQ_GROUPS; else export MM_RQ_GROUPS=$g; fi
  echo -n "tab=$tm look=$la groups=$g: "
  MM_RQ_TABMODE=$tm MM_RQ_LOOKAHEAD=$la GWS=0 python tools/rq_sweep.py $S 2>&1 | grep "^M=" | sed 's/rows=auto //; s/gw=auto://'
done; done; done
