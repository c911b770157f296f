set -u
OUT=gpurun_out/bal1; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for w in 2 3 4; do for m in balanced balanced_cloud; do
  timeout 300 $TR --nproc-per-node $w --master-port $((29530+w)) tests/mgpu_check.py --side 20 --mode $m > $OUT/${m}_$w.log 2>&1; echo "$m $w rc=$?" >> $OUT/summary.txt
done; done
timeout 600 python -m pytest tests/test_mgpu.py -q -k "not balanced" > $OUT/mgpu_old.log 2>&1; echo "old rc=$?" >> $OUT/summary.txt
timeout 600 python -m pytest tests -m gpu -q -x --ignore=tests/test_mgpu.py > $OUT/gpu.log 2>&1; echo "gpu rc=$?" >> $OUT/summary.txt
