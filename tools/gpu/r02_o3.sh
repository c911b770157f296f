cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_o3; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $R --nproc-per-node 3 --master-port 29606 bench.py --gpus 3 --side 128 --mode strong --partition orb --steps 3 --warmup 3 --no-e2e > $O/o3t.json 2> $O/o3t.err
timeout 400 $R --nproc-per-node 3 --master-port 29605 bench.py --gpus 3 --side 512 --mode strong --partition orb --steps 5 --warmup 3 --no-e2e > $O/o3.json 2> $O/o3.err
timeout 400 $R --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --side 512 --mode strong --partition orb --steps 5 --warmup 3 --no-e2e > $O/o4.json 2> $O/o4.err
timeout 1500 python -m pytest tests/test_mgpu.py -q -s > $O/mgpu_tests.log 2>&1; echo "rc=$?" >> $O/mgpu_tests.log
