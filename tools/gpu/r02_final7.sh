cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_final7; mkdir -p $O
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 300 $R --nproc-per-node 2 --master-port 29600 bench.py --gpus 2 --steps 10 --warmup 3 > $O/n2.json 2> $O/n2.err
timeout 300 $R --nproc-per-node 4 --master-port 29601 bench.py --gpus 4 --steps 10 --warmup 3 > $O/n4.json 2> $O/n4.err
timeout 400 python bench.py --side 512 --mode strong --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/s1.json 2> $O/s1.err
timeout 400 $R --nproc-per-node 2 --master-port 29602 bench.py --gpus 2 --side 512 --mode strong --steps 5 --warmup 3 --no-e2e > $O/s2.json 2> $O/s2.err
timeout 400 $R --nproc-per-node 4 --master-port 29603 bench.py --gpus 4 --side 512 --mode strong --steps 5 --warmup 3 --no-e2e > $O/s4.json 2> $O/s4.err
timeout 400 $R --nproc-per-node 3 --master-port 29605 bench.py --gpus 3 --side 512 --mode strong --partition orb --steps 5 --warmup 3 --no-e2e > $O/o3.json 2> $O/o3.err
timeout 400 $R --nproc-per-node 4 --master-port 29604 bench.py --gpus 4 --side 512 --mode strong --partition orb --steps 5 --warmup 3 --no-e2e > $O/o4.json 2> $O/o4.err
