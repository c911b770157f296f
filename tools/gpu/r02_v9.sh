cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_v9; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -s -k "not mgpu and not c4" > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload advected --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/adv.json 2> $O/adv.err
timeout 600 python bench.py --workload jitter --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/jit.json 2> $O/jit.err
