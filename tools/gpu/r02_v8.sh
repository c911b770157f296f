cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_v8; mkdir -p $O
for m in 0 1 2; do
FMM_CONCURRENT=$m timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_$m.json 2> $O/bench_$m.err
done
FMM_CONCURRENT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not c4 and not c3" > $O/tests_1.log 2>&1; echo "rc=$?" >> $O/tests_1.log
FMM_CONCURRENT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "not c4 and not c3" > $O/tests_2.log 2>&1; echo "rc=$?" >> $O/tests_2.log
