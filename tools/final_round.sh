#!/bin/bash
# Development tool (GPU box, 1 GPU): GPU tests + smoke, the default bench line,
# the launch list and the all-kernel DRAM/utilisation table, and a full ncu
# capture of the tensor-core M2L, under gpurun_out/$TAG/.
set -u
TAG=$1; OUT=gpurun_out/$TAG; mkdir -p $OUT
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/ref.json 2> $OUT/ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $B > /dev/null 2>&1
python tools/ncu_summary.py $OUT/launches.csv > $OUT/launches_summary.txt 2>&1
K="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"
K=$K,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --metrics $K --clock-control none --csv --log-file $OUT/all_kernels.csv $B > /dev/null 2>&1
python tools/ncu_summary.py $OUT/all_kernels.csv $OUT/all_kernels.json > $OUT/all_kernels.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_m2l_tc -c 1 -o $OUT/m2l_tc $B > /dev/null 2>&1
ncu -i $OUT/m2l_tc.ncu-rep --page raw --csv > $OUT/m2l_tc_raw.csv 2>/dev/null
echo done
