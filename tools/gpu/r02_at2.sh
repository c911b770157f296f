cd $GRAFT_REPO_ROOT
O=gpurun_out/r02_at2; mkdir -p $O
V=paper_1106_5273_b200/build/variants
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_m2l_tc.py -x -q > $O/tests_default.log 2>&1; echo "rc=$?" >> $O/tests_default.log
FMM_LIB=$V/atr128/libfmm_b200.so timeout 600 python -m pytest tests/test_gpu_m2l_tc.py -x -q > $O/tests_r128.log 2>&1; echo "rc=$?" >> $O/tests_r128.log
for v in default at0 atr128 atr128s3 atr128pf4 pre0; do
  if [ $v = default ]; then L=""; else L="FMM_LIB=$V/$v/libfmm_b200.so"; fi
  env $L timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > $O/b_$v.json 2> $O/b_$v.err
done
FMM_LIB=$V/atr128/libfmm_b200.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_m2l_tc -c 1 -o $O/m2l_tc_r128 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
