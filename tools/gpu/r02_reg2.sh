cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_reg2; mkdir -p $O
V=paper_1106_5273_b200/build/variants
timeout 900 python -m pytest tests/test_gpu_m2l_tc.py tests/test_gpu_parity.py tests/test_gpu_edge.py -x -q > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
FMM_LIB=$V/lb6/libfmm_b200.so timeout 900 python -m pytest tests/test_gpu_m2l_tc.py -x -q > $O/tests_lb6.log 2>&1; echo "rc=$?" >> $O/tests_lb6.log
for v in default split0 lb6; do
  if [ $v = default ]; then L=""; else L="FMM_LIB=$V/$v/libfmm_b200.so"; fi
  env $L timeout 300 python bench.py --workload jitter --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/jit_$v.json 2> $O/jit_$v.err
  env $L timeout 300 python bench.py --workload advected --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/adv_$v.json 2> $O/adv_$v.err
done
