#!/bin/bash
# Development tool (runs on the GPU box): the measurement set of one round step,
# written under gpurun_out/$TAG/ --
#   flops.csv      ncu per-instruction FP32 counters of one k_p2p launch (C3 bench command)
#   p2p.ncu-rep    ncu --set full capture of one k_p2p launch (+ p2p_raw.csv)
#   latest_p2p.json  profiles/latest_p2p.json updated from the two (bench.py's roofline input)
#   bench.json     the default bench line (N = 1, C3), run after the update
#   launches.csv   ncu launch list (gpu__time_duration) of one bench step
# usage: tools/profile_round.sh TAG "commit note" [light]   (light: skip the all-kernel and M2L captures)
set -u
TAG=$1; NOTE=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
M=gpu__time_duration.sum
for op in fadd fmul ffma fadd2 fmul2 ffma2; do M=$M,sm__sass_thread_inst_executed_op_${op}_pred_on.sum; done
timeout 600 ncu --clock-control none --metrics $M -k regex:k_p2p -c 1 --csv --log-file $OUT/flops.csv $B > $OUT/flops_bench.json 2> $OUT/flops.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_p2p -c 1 -o $OUT/p2p $B > $OUT/full.log 2>&1
ncu -i $OUT/p2p.ncu-rep --page raw --csv > $OUT/p2p_raw.csv
python tools/ncu_flops.py $OUT/flops.csv $OUT/flops_bench.json > $OUT/flops.txt 2>&1
python tools/p2p_raw_json.py $OUT/p2p_raw.csv "$NOTE" >> $OUT/flops.txt 2>&1
cp profiles/latest_p2p.json $OUT/latest_p2p.json
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > /dev/null 2>&1
python tools/ncu_summary.py $OUT/launches.csv > $OUT/launches_summary.json 2>&1
[ "${3:-}" = "light" ] && { echo done; exit 0; }
# every kernel of one step with DRAM bytes, FMA / issue / tensor utilisation (HBM GB/s of keys, sort, tree)
K="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"
K=$K,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed
timeout 900 ncu --metrics $K --clock-control none --csv --log-file $OUT/all_kernels.csv $B > /dev/null 2>&1
python tools/ncu_summary.py $OUT/all_kernels.csv $OUT/all_kernels.json > $OUT/all_kernels.txt 2>&1
# the tensor-core M2L, full set
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_m2l_tc -c 1 -o $OUT/m2l_tc $B > /dev/null 2>&1
ncu -i $OUT/m2l_tc.ncu-rep --page raw --csv > $OUT/m2l_tc_raw.csv 2>/dev/null
echo done
