cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_m5; mkdir -p $O
timeout 1500 python -m pytest tests/test_mgpu.py -q -s > $O/mgpu_tests.log 2>&1; echo "rc=$?" >> $O/mgpu_tests.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $R --nproc-per-node 2 --master-port 29600 bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e > $O/n2.json 2> $O/n2.err
timeout 300 $R --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e > $O/n4.json 2> $O/n4.err
