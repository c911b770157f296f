cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_v5; mkdir -p $O
for nc in 80 96 128; do
timeout 600 python bench.py --workload advected --ncrit $nc --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/adv_$nc.json 2> $O/adv_$nc.err
timeout 600 python bench.py --workload jitter --ncrit $nc --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/jit_$nc.json 2> $O/jit_$nc.err
done
timeout 600 python bench.py --ncrit 96 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/lat_96.json 2> $O/lat_96.err
