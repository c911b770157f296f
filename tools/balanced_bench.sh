#!/bin/bash
# Development tool (GPU box, 4 GPUs): C4 strong scaling with the balanced
# partition (every rank passes a random 1/N subset, redistributed every step).
set -u
OUT=gpurun_out/$1; mkdir -p $OUT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29541"
for w in 2 4; do
  timeout 900 $TR --nproc-per-node $w bench.py --gpus $w --mode strong --side 512 --steps 3 --warmup 3 --partition balanced > $OUT/b$w.json 2> $OUT/b$w.err
done
echo done
