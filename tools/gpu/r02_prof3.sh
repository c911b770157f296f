cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_prof3; mkdir -p $O
B="python bench.py --workload jitter --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
timeout 600 $B > $O/plain.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_m2l_reg -c 1 -o $O/m2l_reg $B > $O/ncu.log 2>&1
ncu -i $O/m2l_reg.ncu-rep --page raw --csv > $O/m2l_reg_raw.csv 2>/dev/null
