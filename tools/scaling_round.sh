#!/bin/bash
# Development tool (GPU box, 4 GPUs): bench lines at N = 1, 2, 4 (C5 weak, tiled)
# and C4 strong scaling (512^3 split by Morton octants), plus the multi-GPU
# parity tests, under gpurun_out/$TAG/.   usage: tools/scaling_round.sh TAG
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29517"
timeout 900 python -m pytest tests/test_mgpu.py -q > $OUT/mgpu_tests.log 2>&1
timeout 600 python bench.py > $OUT/n1.json 2> $OUT/n1.err
timeout 600 $TR --nproc-per-node 2 bench.py --gpus 2 > $OUT/n2.json 2> $OUT/n2.err
timeout 600 $TR --nproc-per-node 4 bench.py --gpus 4 > $OUT/n4.json 2> $OUT/n4.err
timeout 900 python bench.py --mode strong --side 512 --steps 3 --warmup 3 --no-cpu-baseline > $OUT/s1.json 2> $OUT/s1.err
timeout 900 $TR --nproc-per-node 2 bench.py --gpus 2 --mode strong --side 512 --steps 3 --warmup 3 > $OUT/s2.json 2> $OUT/s2.err
timeout 900 $TR --nproc-per-node 4 bench.py --gpus 4 --mode strong --side 512 --steps 3 --warmup 3 > $OUT/s4.json 2> $OUT/s4.err
echo done
