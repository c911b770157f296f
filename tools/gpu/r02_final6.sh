cd $GRAFT_REPO_ROOT
bash tools/profile_round.sh r02_final6 "r02 final 6: P2P unrolls 6 (singular) / 3 (regularised)"
O=gpurun_out/r02_final6
timeout 1200 python -m pytest tests -m gpu -q -s > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 600 python bench.py --workload advected --no-cpu-baseline --no-e2e > $O/adv.json 2> $O/adv.err
timeout 600 python bench.py --workload jitter --no-cpu-baseline --no-e2e > $O/jit.json 2> $O/jit.err
