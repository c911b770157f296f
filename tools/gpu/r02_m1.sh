cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_m1; mkdir -p $O
nvidia-smi -L > $O/gpus.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -s -k "not c4 and not c3" > $O/gpu_parity.log 2>&1; echo "rc=$?" >> $O/gpu_parity.log
for m in tiled refined orb orb_cloud step; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tests/mgpu_check.py --side 16 --mode $m > $O/mgpu_$m.log 2>&1; echo "rc=$?" >> $O/mgpu_$m.log
done
