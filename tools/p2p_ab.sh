#!/bin/bash
# Development tool (GPU box, 1 GPU): A/B of the default library against
# variants built by tools/build_variant.py (P2P phase time at C3, alternated
# twice, and whether each variant's (u, d) is identical to the default's;
# the 400 MB arrays stay in /tmp on the box, only the logs come back).
set -u
OUT=gpurun_out/ab; mkdir -p $OUT
for r in 1 2; do
  timeout 600 python tools/p2p_sweep.py --reps 5 --save /tmp/ab_base.npy > $OUT/base_$r.log 2>&1
  for V in "$@"; do
    FMM_LIB=paper_1106_5273_b200/build/variants/$V/libfmm_b200.so timeout 600 python tools/p2p_sweep.py --reps 5 --save /tmp/ab_$V.npy > $OUT/${V}_$r.log 2>&1
  done
done
for V in "$@"; do
python -c "
import numpy as np; a=np.load('/tmp/ab_base.npy'); b=np.load('/tmp/ab_$V.npy')
print('$V max abs diff', float(np.abs(a-b).max()), 'identical', bool((a==b).all()))" >> $OUT/diff.log 2>&1
done
tail -n 2 $OUT/*.log
