cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_at; mkdir -p $O
V=paper_1106_5273_b200/build/variants
timeout 600 python -m pytest tests/test_gpu_m2l_tc.py -x -q > $O/tc_tests.log 2>&1; echo "rc=$?" >> $O/tc_tests.log
if grep -q "rc=0" $O/tc_tests.log; then
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_at.json 2> $O/b_at.err
  for v in at0 ats2 atpf5 atc48; do
    FMM_LIB=$V/$v/libfmm_b200.so timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_$v.json 2> $O/b_$v.err
  done
  timeout 900 python -m pytest tests/ -x -q -m gpu > $O/gpu_tests.log 2>&1; echo "rc=$?" >> $O/gpu_tests.log
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_m2l_tc -c 1 -o $O/m2l_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
fi
