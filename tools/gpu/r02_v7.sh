cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_v7; mkdir -p $O
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload advected --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/adv.json 2> $O/adv.err
timeout 300 python tools/tc_levels.py > $O/levels.log 2>&1
