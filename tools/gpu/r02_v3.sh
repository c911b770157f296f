cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_v3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -s > $O/gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > $O/bench.json 2> $O/bench.err
timeout 600 python bench.py --workload advected --no-cpu-baseline --no-e2e > $O/bench_advected.json 2> $O/bench_advected.err
timeout 600 python bench.py --workload jitter --no-cpu-baseline --no-e2e > $O/bench_jitter.json 2> $O/bench_jitter.err
