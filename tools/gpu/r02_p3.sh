cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_p3; mkdir -p $O
timeout 900 python -m pytest tests/ -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > $O/b.json 2> $O/b.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --workload jitter > $O/b_jit.json 2> $O/b_jit.err
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --workload advected > $O/b_adv.json 2> $O/b_adv.err
