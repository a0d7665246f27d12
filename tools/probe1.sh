mkdir -p gpurun_out
P=gpurun_out/probe1.log
: > $P
for sc in "0,0,256 128 256 0 0 onehot" "0,256,0 128 256 0 0 onehot" "256,0,0 128 256 0 0 onehot" "0,0,256 128 128 128 0 onehot" "128,64,64 128 256" ; do
  echo "=== $sc" >> $P
  timeout 60 python tools/gemm_probe.py $sc >> $P 2>&1; echo "rc=$?" >> $P
done
echo "=== RQ tests" >> $P
timeout 400 python -m pytest tests/test_gpu_rq.py -x -q -p no:cacheprovider -o timeout=120 >> $P 2>&1; echo "rc=$?" >> $P
cat $P | tail -80
